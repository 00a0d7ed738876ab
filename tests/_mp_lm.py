"""Worker of tests/test_gpu_multirank.py (launched by torch.distributed.run, one process per GPU):
the landmark-sharded LM on config 2 with the NCCL all-reduces, against the oracle
(every rank runs its own copy; each iteration at the oracle's PCG count, the §8c replay rule), and
the lockstep assertion: the all-reduced camera-space vectors are bit-identical on every rank."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2103_01843_b200 import rba, synth  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [rba.rba_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    p = synth.make_problem(int(os.environ.get("MP_CFG", "2")))
    s = rba.Solver(p, device=local, world=world, rank=rank, nccl_id=obj[0])
    o = oracle.Oracle(p)
    info = s.info()
    assert info["nccl"] == 1, info
    for i in range(4):
        ro = o.lm_step()
        s.set_pcg_limits(0.0, ro["pcg_iters"])
        rg = s.lm_step()
        err = abs(rg["cost_after"] - ro["cost_after"]) / ro["cost_after"]
        assert rg["pcg_iters"] == ro["pcg_iters"] and err <= 1e-4, (rank, i, rg, ro)
        cs = torch.tensor(np.array(s.checksums(), dtype=np.uint64).view(np.int64), device="cuda")
        allcs = [torch.zeros_like(cs) for _ in range(world)]
        dist.all_gather(allcs, cs)
        for r in range(world):
            assert torch.equal(allcs[r], allcs[0]), (rank, i, [a.tolist() for a in allcs])
        print(f"rank {rank} iter {i} cost {rg['cost_after']:.6f} oracle {ro['cost_after']:.6f} rel {err:.2e} "
              f"landmarks {info['n_landmarks']} graph {s.info()['lm_graph']}", flush=True)
    cams, pts = s.state()
    co, po = o.state()
    assert np.abs(cams - co).max() <= 1e-3 * max(1.0, np.abs(co).max())
    dist.barrier()
    s.close()
    dist.destroy_process_group()
    print(f"MP_OK rank {rank}", flush=True)


if __name__ == "__main__":
    main()
