"""bench.py's reference arm runs on CPU; its JSON line follows the contract
(the driver launches it as `bench.py --impl reference`)."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], capture_output=True, text=True,
                         timeout=600, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0", "--traces", "16", "--no-python")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["metric"] == "scheduler decisions/sec" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_pool_and_audit_lines():
    c = _run("--impl", "reference", "--workload", "C", "--steps", "1", "--warmup", "0", "--traces", "20000",
             "--pool-steps", "200")
    assert c["impl"] == "reference" and c["value"] > 0
    a = _run("--impl", "reference", "--workload", "audit", "--steps", "1", "--warmup", "0", "--traces", "8")
    assert a["impl"] == "reference" and a["unit"] == "pairs/s" and a["value"] > 0


def test_reference_arm_config_a_with_python_reference():
    """Config A: the C port and the unmodified Python Simulator (baseline/_ref)
    on the medical trace; the arm never loads the product's CUDA library."""
    d = _run("--impl", "reference", "--workload", "A", "--steps", "1", "--warmup", "0")
    assert d["config"]["name"] == "A" and d["decisions_per_step"] > 20000
    assert not any("libsemsched_b200" in x for x in d["native_so_loaded"])
    py = d["python_reference"]
    if os.path.isdir(os.path.join(REPO, "baseline", "_ref", "semsched")):
        assert py["kind"] == "reference" and py["value"] > 0 and py["cores"] == 1
    else:
        assert "unavailable" in py


def test_bench_config_is_the_same_in_both_arms():
    sys.path.insert(0, REPO)
    import bench

    for name in ("A", "B", "D", "E"):
        wl = bench.WORKLOADS[name]
        for world in (1, 2, 8):
            seeds, per, total = bench.job_layout(wl, world, 0)
            if name == "E":
                assert total == 65536 and per * world == total and len(seeds) == per
            elif name in ("B", "D"):
                assert per == 4096 and total == 4096 * world
