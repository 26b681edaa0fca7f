"""The reference arm of bench.py (tier framing: the oracle, timed on the host cores) keeps the
JSON-line contract: one line on stdout with the metric / unit / config of the GPU arm plus
impl, cpu_baseline and a zero-byte e2e object."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--order", "1500",
           "--steps", "1", "--warmup", "0", "--ref-seconds", "1.0"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_projected_oracle_time_and_recorded_cases():
    """the projected oracle time to solution is (8 N^2 matvecs + iterations x
    (8 N^2 n_e + 40 N n_e^2)) / the oracle's rate, labelled "projected"; the recorded config-4
    runs are read from the committed profiles."""
    sys.path.insert(0, ROOT)
    import bench
    case = {"config": "x", "N": 1000, "nev": 40, "nex": 10, "matvecs": 5000, "iterations": 3}
    out = bench.projected_oracle_tts(2.0, [case])[0]
    flops = 8.0 * 1000 ** 2 * 5000 + 3 * (8.0 * 1000 ** 2 * 50 + 40.0 * 1000 * 50 ** 2)
    assert out["label"] == "projected"
    assert abs(out["projected_oracle_s"] - flops / 2e12) <= 1e-12 * flops
    cases = bench._recorded_tts()
    assert any(c["config"].startswith("config4") for c in cases)
    for c in cases:
        assert c["matvecs"] > 0 and c["iterations"] > 0 and c["N"] == 115000


def test_config1_oracle_solve_times():
    """cpu_baseline.config1_full_solve on the host: the oracle's config-1 solve, 1 thread and all
    threads (GPU part skipped here)."""
    sys.path.insert(0, ROOT)
    import bench
    import paper_2205_02491_b200 as pkg
    out = bench.config1_compare(pkg, gpu=False, runs=1)
    assert out["oracle_all_threads_s"] > 0 and out["oracle_1_thread_s"] > 0
    assert out["oracle_eig_err_rel"] <= 1e-10
