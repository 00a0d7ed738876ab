"""LM cost parity: the cost after each LM iteration within `bar` (1e-4) relative of
the oracle's, with no relaxation.  PCG stops at a relative residual of 1e-2 (reading C11); where the
GPU's FP32 solve stops at a different iteration count than the oracle's FP64 solve (the tolerance
edge), §8c re-runs the iteration with the oracle's count fixed: the GPU state and LM schedule from
before the iteration are restored through the C ABI (rba_set_state, rba_set_lm) and the iteration
is replayed with rba_set_pcg_limits(0, n_oracle), which runs exactly that many PCG iterations."""


def lm_parity(s, o, iters, bar=1e-4, pcg_tol=1e-2, pcg_max=500, allow_indefinite=False):
    """Run `iters` LM iterations on the GPU solver `s` and the oracle `o` from their current states;
    returns the list of (gpu_report, oracle_report, replayed)."""
    out = []
    for i in range(iters):
        cams, pts = s.state()
        lam, nu, _ = s.get_lm()
        rg = s.lm_step()
        ro = o.lm_step(pcg_tol, pcg_max)
        replayed = False
        if rg["pcg_iters"] != ro["pcg_iters"]:
            s.set_state(cams, pts)
            s.set_lm(lam, nu)
            s.set_pcg_limits(0.0, ro["pcg_iters"])
            rg = s.lm_step()
            s.set_pcg_limits(pcg_tol, pcg_max)
            replayed = True
            assert rg["pcg_iters"] == ro["pcg_iters"] or rg["pcg_reason"] == 2, (i, rg, ro)
        if not allow_indefinite:
            assert rg["pcg_reason"] != 2 and ro["pcg_reason"] != 2, (i, rg, ro)  # never indefinite
        assert abs(rg["cost_after"] - ro["cost_after"]) <= bar * ro["cost_after"], (i, replayed, rg, ro)
        out.append((rg, ro, replayed))
    return out
