"""DecDEC CPU oracle -- TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct float64 NumPy statement of what
the DecDEC decode hot path computes (arXiv 2412.20185, /root/reference/PAPER.md;
SURVEY.md §8(c) rows O1-O6).  It exists to prove the CUDA path right.

Rules:
  * Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
    ``cpu_baseline`` / ``--impl reference`` legs may import it.
  * It shares no code with ``paper_2412_20185_b200`` (the CUDA path) and never
    imports it; the only shared module is ``synth`` (seeded inputs, no method
    arithmetic).
  * Parity status per function is listed in ``oracle.decdec_ref.__doc__``.
"""

from .decdec_ref import (  # noqa: F401
    fp16_rne,
    round_half_away,
    quantize_base,
    residual,
    quantize_residual,
    dequantize_residual_rows,
    topk_ref,
    k_from_kchunk,
    dequantize_base,
    decdec_linear_ref,
    decdec_linear_ref_cols,
    pack_w4k_ref,
    pack_w3k_ref,
    pack_rq_ref,
    unpack_w4k_ref,
    unpack_w3k_ref,
    unpack_rq_ref,
    tolerance_ok,
    rel_err_unfloored,
    quantize_base_lut,
    dequantize_lut,
)
