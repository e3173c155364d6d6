"""bench.py helpers that do not need a GPU: the WADG flop model, the committed
ncu traffic table, and the reference arm's JSON contract on a tiny sample."""
import importlib.util
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_wadg_flop_model_matches_hand_count():
    b = load_bench()
    # N = 5: nt = 21, nq = 6, nc = 49 (DESIGN.md 3.3 / bench.py)
    nt, nq, nc = 21, 6, 49
    want = 2 * nt * nc * nt + 8 * nt * nt * nq + 8 * nt * nq * nq + 12 * nt * nq * nq + 8 * nt * nt * nq
    assert b.wadg_flops_per_wedge_stage(5) == want


def test_traffic_table_is_committed_and_close_to_algorithmic():
    b = load_bench()
    tab = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    for n in range(1, 8):
        nq, nt = n + 1, (n + 1) * (n + 2) // 2
        later = 8 * (16 * nq * nt + nt * nt + 3 * nt * nq + 34 + 2 * nq) + 48  # non-first stage, per wedge
        got = b.load_traffic("exact", n)
        assert got is not None
        assert 0.95 * later * 1e6 <= got <= 1.15 * later * 1e6, (n, got, later * 1e6)
