"""Small workload for compute-sanitizer: config 1 (1024x1024, 3-bit, k=16,
r4 and r16), one Llama-3-8B shape (o 4096x4096 at k_chunk 21), the standalone selector, a
3-layer stack replay and a LUT layer.  Outputs checked against the oracle so a run that
"passes" the tool also computed the right thing.
usage: compute-sanitizer --tool memcheck --kernel-name kns=decdec python tools/sanitize_run.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2412_20185_b200 as dd  # noqa: E402
from synth import gen_activations, gen_perf_layer, gen_weight_fp16, layer_seed  # noqa: E402


def check(y, ref, what):
    ok, err, _ = oracle.tolerance_ok(y.cpu().numpy(), ref["y64"], ref["A"])
    assert ok.all(), what
    print("ok", what, flush=True)


W = gen_weight_fp16(1024, 1024, layer_seed("san", "W"))
q, s, z = oracle.quantize_base(W, 3)
R = oracle.residual(W, oracle.dequantize_base(q, s, z))
rc, rS = oracle.quantize_residual(R, 4)
r16 = oracle.quantize_residual(R, 16)
x = gen_activations(1024, 1, seed=1)[0]
xd = torch.from_numpy(x).cuda()
ws = dd.Workspace(1024, 4096)
lin = dd.QuantLinear.from_codes(q, s, z, 3, rc=rc, rS=rS)
sel = torch.empty(16, dtype=torch.int32, device="cuda")
check(lin(xd, 16, sel=sel, workspace=ws), oracle.decdec_linear_ref(q, s, z, x, 16, rc=rc, rS=rS), "config1 r4 k16")
check(lin(xd, 0, workspace=ws), oracle.decdec_linear_ref(q, s, z, x, 0), "config1 k0")
lin16 = dd.QuantLinear.from_codes(q, s, z, 3, r16=r16)
check(lin16(xd, 16, workspace=ws), oracle.decdec_linear_ref(q, s, z, x, 16, r16=r16), "config1 r16 k16")
idx, xs = dd.select(xd, 100)
assert np.array_equal(idx.cpu().numpy(), oracle.topk_ref(x, 100)[0])
print("ok select", flush=True)
L = gen_perf_layer(4096, 4096, 3, seed=layer_seed("san", "o"))
lo = dd.QuantLinear.from_codes(L["q"], L["s"], L["z"], 3, rc=L["rc"], rS=L["rS"])
xo = gen_activations(4096, 1, seed=2)[0]
check(lo(torch.from_numpy(xo).cuda(), 84, workspace=ws), oracle.decdec_linear_ref(L["q"], L["s"], L["z"], xo, 84, rc=L["rc"], rS=L["rS"]),
      "llama o k_chunk 21")
ys = [torch.empty(d, dtype=torch.float16, device="cuda") for d in (1024, 4096, 1024)]
xs3 = [xd, torch.from_numpy(xo).cuda(), xd]
st = dd.Stack([lin, lo, lin], [16, 84, 0], xs3, ys, ws)
st.launch()
torch.cuda.synchronize()
check(ys[1], oracle.decdec_linear_ref(L["q"], L["s"], L["z"], xo, 84, rc=L["rc"], rS=L["rS"]), "stack layer 1")
st.close()
ql, lut = oracle.quantize_base_lut(W[:, :256], 3)
ll = dd.QuantLinear.from_lut_codes(ql, lut, 3)
check(ll(xd, 0), oracle.decdec_linear_ref(ql, None, None, x, 0, lut=lut), "lut k0")
