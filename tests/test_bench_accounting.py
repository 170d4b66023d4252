"""bench.py's roofline accounting (SURVEY.md §8(d) byte formulas, Appendix A) on CPU: the
algorithmic bytes per call and the step roofline the JSON line reports."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from synth import model_layers  # noqa: E402


def test_k_from_kchunk_floor():
    # 10 % of 14336 channels -> 1433 (floor); k_chunk 21 of 4096 -> 84
    assert bench.k_of(102.4, 14336) == 1433
    assert bench.k_of(21, 4096) == 84 and bench.k_of(21, 14336) == 294 and bench.k_of(0, 4096) == 0


def test_bytes_per_call():
    # gu 4096 x 28672, 3-bit: codes d_in*d_out*3/8 + (fp16 s + u8 z) per 128-group + x + y
    assert bench.bytes_hbm(4096, 28672, 3) == 4096 * 28672 * 3 // 8 + 3 * 28672 * 32 + 2 * 4096 + 2 * 28672 == 46858240
    # PCIe: k rows of d_out/2 bytes (4-bit residual) + all d_out fp16 scales
    assert bench.bytes_pcie(84, 28672) == 84 * 14336 + 2 * 28672 == 1261568
    assert bench.bytes_pcie(0, 28672) == 0


def test_step_roofline_llama3_8b():
    # 3-bit linear stack at k_chunk 0 ~ 430.8 µs at 6455 GB/s
    t = sum(bench.bytes_hbm(d_in, d_out, 3) / 6455e3 for _, d_in, d_out in model_layers("llama3_8b", fused=True)) * 32
    assert abs(t - 430.8) < 1.0
