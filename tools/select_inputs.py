"""Write synth decode activations for csrc/probe/probe_select.cu (gpurun_out/x{n}.bin)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from synth import gen_activations  # noqa: E402

os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
for n, kind in ((4096, "qkv"), (14336, "d")):
    gen_activations(n, 1, seed=3, kind=kind)[0].tofile(os.path.join(ROOT, "gpurun_out", f"x{n}.bin"))
