"""bench.py keeps the driver's contract: one JSON line with the required keys
(reference arm on CPU; our arm on the GPU, short run)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches"}


def _run(args, timeout):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "1"], 600)
    assert d["impl"] == "reference" and BASE_KEYS <= set(d)
    assert d["unit"] == "matrices/s" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"] == "llama3-8b"            # the north-star set is the default
    # the reference arm reports what it timed: one pass per step
    assert len(d["cpu_baseline"]["step_ms"]) == d["steps"]
    assert abs(d["ms_per_step"] - sum(d["cpu_baseline"]["step_ms"]) / d["steps"]) <= 1e-3 * d["ms_per_step"] + 1e-3


@pytest.mark.gpu
def test_our_arm_line():
    d = _run(["--workload", "gpt2-small", "--steps", "2", "--warmup", "3", "--extra", "", "--no-cpu-baseline"], 900)
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["steps"] == 2 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    assert d["gpu_launches"] > 0 and d["dtype"] == "bf16"
    assert d["roofline"]["bound"] == "tensor" and 0 < d["roofline"]["frac"] < 1
    assert d["clocks"]["sm_max_mhz"] and d["e2e"]["h2d_bytes_per_step"] > 0
    assert len(d["ms_per_step_stats"]["all_ms"]) == 2


def test_kernel_accounting_helpers():
    """bench.py's algorithmic counts: symmetric-aware GEMM flops
    per launch, norm bytes, copy-pass bytes only for rows that are not 16-byte
    multiples; every launched kind against its own roofline."""
    sys.path.insert(0, ROOT)
    import bench
    shapes = [(768, 3072), (3072, 768), (100, 90)]
    fl, by = bench.kind_work(shapes, 5)
    m, n = 768, 3072
    assert fl["gram"] == 2 * m * (m + 1) * n + 90 * 91 * 100
    assert fl["poly"] == 2 * m * m * (m + 1) + 90 * 90 * 91
    assert fl["update"] == 2 * (2.0 * m * m * n) + 2.0 * 90 * 90 * 100
    assert by["norm"] == 2 * (2.0 * m * n) + 2.0 * 90 * 100
    assert by["scale"] == 4.0 * 90 * 100 and by["transpose_back"] == 4.0 * 90 * 100   # only the unaligned one
    peaks = {"bf16_tflops": 1000.0, "bf16_tflops_sustained": 800.0, "hbm_gbs": 5000.0}
    prof = {"norm": (0.2, 2), "gram": (3.0, 10), "poly": (0.0, 0), "update": (5.0, 10)}
    t = bench.kernel_table(prof, shapes, 5, 10.0, peaks)
    assert set(t) == {"norm", "gram", "update"}
    assert t["gram"]["bound"] == "tensor" and t["gram"]["peak"] == 1000.0       # short step: burst peak
    assert abs(t["gram"]["achieved"] - fl["gram"] / 0.3e-3 / 1e12) < 0.01
    assert t["norm"]["bound"] == "hbm" and abs(t["norm"]["achieved"] - by["norm"] / 0.1e-3 / 1e9) < 0.1
    assert bench.kernel_table(prof, shapes, 5, 100.0, peaks)["update"]["peak"] == 800.0   # long step: sustained
