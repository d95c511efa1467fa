"""bench.py's reference arm (the CPU oracle timed on the host, `--impl
reference`) runs without a GPU: one JSON line with the contract's keys, the
same metric / unit / config as the GPU arm, e2e with zero transfer bytes."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["dtype"] == "f64" and d["higher_is_better"] is True
    assert d["unit"] == "cell-updates/s" and d["value"] > 0
    assert d["config"]["workload"].startswith("cfg4")
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_work_model_reproduces_survey_rows():
    # the fp64 work model reproduces SURVEY 8(d)'s literal
    # telescoped 16^3 step (1498, by construction) and its per-stage row
    # (1033) to 1 %; the borrowed ring on cfg4's 16^3-block brick is 1065
    sys.path.insert(0, ROOT)
    import bench
    assert abs(bench.step_fp64_model([(20, 20, 20)] * 8) - 1498.0) < 1e-9
    assert abs(bench.step_fp64_model([(16, 16, 16)] * 8) / 1033.0 - 1) < 0.01
    regions = bench.borrowed_ring_regions((16, 16, 16))
    assert len(regions) == 4096
    assert sum(r[0] == 18 for r in regions) == 16 ** 3 - 16 * 14 * 14          # an x or y brick face
    assert sum(r == (16, 16, 18) for r in regions) == 2 * 14 * 14              # z faces only
    assert abs(bench.step_fp64_model(regions) - 1065.3) < 0.1
    # a brick one block wide in x: both x sides self, the 20 x 20 box
    assert all(r[0] == 20 for r in bench.borrowed_ring_regions((1, 4, 4)))
    # one block, every side self: the literal box
    assert abs(bench.step_fp64_model(bench.borrowed_ring_regions((1, 1, 1))) - 1498.0) < 1e-9
