"""Launch decdec_select a few times for one d_in (for ncu)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2412_20185_b200 as dd  # noqa: E402
from synth import gen_activations  # noqa: E402

d_in = int(sys.argv[1]) if len(sys.argv) > 1 else 14336
kc = int(sys.argv[2]) if len(sys.argv) > 2 else 21
k = kc * d_in // 1024
x = torch.from_numpy(gen_activations(d_in, 1, seed=1)[0]).cuda()
idx = torch.empty(k, dtype=torch.int32, device="cuda")
xs = torch.empty(k, dtype=torch.float16, device="cuda")
for _ in range(6):
    dd.decdec_select(x.data_ptr(), d_in, k, 0, idx.data_ptr(), xs.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
