"""Host check of bench.py's evidence lookup (no GPU): the newest committed `ncu --set full` summary
of each benched config is found and parsed whatever refresh suffix its name carries (r2, r2c, ...),
so that a new capture under profiles/ cannot break the bench's `roofline.traffic`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def test_round_key_orders_refreshes():
    names = ["x/profiles/r1_cfg4_ncu_full.json", "x/profiles/r2c_cfg4_ncu_full.json",
             "x/profiles/r2_cfg4_ncu_full.json", "x/profiles/r10_cfg4_ncu_full.json"]
    assert [os.path.basename(f)[:3] for f in sorted(names, key=bench._round_key)] == ["r1_", "r2_", "r2c", "r10"]


def test_ncu_traffic_found_for_benched_configs():
    for cfg in (3, 4):
        mv, mg, src = bench.ncu_traffic(cfg)
        assert src is not None and mv > 0 and mg > 0, (cfg, src)
