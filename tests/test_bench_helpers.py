"""bench.py helpers that do not need a GPU: the WADG flop model, the committed
ncu traffic table, and the reference arm's JSON contract on a tiny sample."""
import importlib.util
import json
import os

import numpy as np

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


def test_reference_arm_never_loads_the_product(tmp_path):
    """bench.py --impl reference builds its mesh / discretization inside
    liboracle.so and times the oracle: libprismdg_b200.so must not be mapped."""
    import subprocess
    import sys
    probe = tmp_path / "probe.py"
    probe.write_text(
        "import sys, runpy, io, contextlib\n"
        f"sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '3', '--degree', '1']\n"
        "buf = io.StringIO()\n"
        "with contextlib.redirect_stdout(buf):\n"
        "    try:\n"
        f"        runpy.run_path({os.path.join(ROOT, 'bench.py')!r}, run_name='__main__')\n"
        "    except SystemExit:\n"
        "        pass\n"
        "maps = open('/proc/self/maps').read()\n"
        "print(buf.getvalue().strip().splitlines()[-1])\n"
        "print('PRODUCT_MAPPED' if 'libprismdg_b200' in maps else 'PRODUCT_NOT_MAPPED')\n"
        "print('ORACLE_MAPPED' if 'liboracle.so' in maps else 'ORACLE_NOT_MAPPED')\n")
    env = dict(os.environ, OMP_NUM_THREADS="2")
    out = subprocess.run([sys.executable, str(probe)], capture_output=True, text=True, env=env, timeout=600)
    lines = out.stdout.strip().splitlines()
    assert lines[-2] == "PRODUCT_NOT_MAPPED" and lines[-1] == "ORACLE_MAPPED", out.stdout + out.stderr
    line = json.loads(lines[-3])
    assert line["impl"] == "reference" and line["value"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["faithful_serial_update"] > 0 and cb["cpu"]
    assert line["variants"]["parallel_update"] == line["value"]
    assert line["config"]["same_config"] is False


def test_multi_gpu_bench_refuses_missing_gpus():
    """--gpus N outside torchrun relaunches N ranks, and refuses (non-zero exit,
    clear message) when fewer than N GPUs are visible instead of timing one GPU."""
    import subprocess
    import sys
    import torch
    if torch.cuda.device_count() >= 2:
        import pytest
        pytest.skip("this host has 2 GPUs")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode != 0
    assert "needs 2 visible GPUs" in out.stderr
    assert out.stdout.strip() == ""


def test_strong_partition_covers_the_single_domain_mesh():
    """config 5 strong: the sublayers of one fixed mesh split over the ranks,
    every element owned once, contiguous z ranges, one ghost sublayer each way."""
    from paper_1607_03399_b200 import partition as P
    for world in (1, 2, 3, 8):
        layers = P.layered_strong_layers([-1.0, -0.4, 0.2, 1.0], [15, 15, 20], [(1, 1), (1, 4), (1, 2.25)], world)
        owners = [lay[3] for lay in layers]
        assert len(layers) == 50 and owners == sorted(owners) and set(owners) == set(range(world))
        counts = [owners.count(r) for r in range(world)]
        assert max(counts) - min(counts) <= 1
    parts = [P.layered_strong(3, [-1.0, 0.0, 1.0], [2, 3], [(1, 1), (1, 4)], 2, r) for r in range(2)]
    assert sum(p.n_owned for p in parts) == 5 * 18
    for p in parts:
        for q, ids in p.send.items():
            assert np.array_equal(p.local_to_global[ids], parts[q].local_to_global[parts[q].recv[p.rank]])


def test_multi_gpu_bench_spawns_one_rank_per_gpu():
    """--gpus 2 outside torchrun re-launches bench.py under torch.distributed.run
    with two ranks (127.0.0.1 rendezvous); --launch-check makes each rank report
    itself instead of touching a GPU."""
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launch-check"],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert sorted(l["rank"] for l in lines) == [0, 1]
    assert all(l["world_size"] == 2 and l["master"] == "127.0.0.1" for l in lines)
