"""bench.py's JSON contract on the CPU: the reference arm (the oracle on the host, this tier's
reference implementation) prints one line with the keys the driver reads, and the GPU arm's
helpers (algorithmic bytes of SURVEY §8(d), peaks, ncu traffic lookup) are consistent."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_prints_the_contract_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "3", "--edge", "12", "--ref-iters", "3"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["metric"] == json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]


def test_algorithmic_bytes_are_survey_8d():
    import bench
    nb = bench.algorithmic_bytes(8_000_000, 23_880_000)
    assert nb["A"] == 24 * 8_000_000 + 16 * 23_880_000  # Amul + dot: 24 B/cell + 16 B/face
    assert nb["B"] == 56 * 8_000_000 and nb["C"] == 32 * 8_000_000
    assert nb["iter"] == nb["A"] + nb["B"] + nb["C"] == 1_278_080_000
    peak, kind = bench.peaks()
    assert peak > 1000 and isinstance(kind, str)


def test_loop_bytes_count_the_on_chip_residual_once():
    """The persistent loop's bytes per iteration: 100 B/cell on a K = 3 lattice with
    rA fully on chip (C 36 = rD + pA_prev + pA + half of the psi pair's 24; A 48; B 16 = wA + rD);
    every pair of rA left in HBM adds its 24 B (read + write in the update, read in the direction)."""
    import bench
    N = 8_000_000
    full = bench.loop_bytes(N, 3, 1.0)
    assert full["C"] == 36 * N and full["A"] == 48 * N and full["B"] == 16 * N and full["iter"] == 100 * N
    assert full["per_launch_fixed"] == 16 * N  # rA loaded once and written back once per launch
    none = bench.loop_bytes(N, 3, 0.0)
    assert none["iter"] == 124 * N  # = the graph batches' 124 B/cell with the psi pairs in the direction
    half = bench.loop_bytes(N, 3, 0.5)
    assert half["iter"] == 112 * N


def test_traffic_lookup_names_the_kernel():
    import bench
    w = "C3 cube 200^3 per GPU (weak), gamma=1, tol 1e-6"
    t = bench.load_traffic(w, "k_pcg_loop")
    assert t is None or t > 1e11  # one launch = the whole solve
    assert bench.load_traffic("another workload", "k_pcg_loop") is None
