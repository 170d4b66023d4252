"""Time decdec_select alone (CUDA events, back-to-back launches) for several d_in / k."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_20185_b200 as dd  # noqa: E402
from synth import gen_activations  # noqa: E402

for d_in in (1024, 4096, 14336, 28672):
    X = [torch.from_numpy(gen_activations(d_in, 1, seed=s)[0]).cuda() for s in range(64)]
    for kc in (4, 21, 82):
        k = kc * d_in // 1024
        idx = torch.empty(k, dtype=torch.int32, device="cuda")
        xs = torch.empty(k, dtype=torch.float16, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        for x in X[:8]:
            dd.decdec_select(x.data_ptr(), d_in, k, 0, idx.data_ptr(), xs.data_ptr(), st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for x in X:
            dd.decdec_select(x.data_ptr(), d_in, k, 0, idx.data_ptr(), xs.data_ptr(), st)
        e1.record()
        e1.synchronize()
        # graph of 64 selects
        g = torch.cuda.CUDAGraph()
        s2 = torch.cuda.Stream()
        with torch.cuda.stream(s2):
            with torch.cuda.graph(g, stream=s2):
                for x in X:
                    dd.decdec_select(x.data_ptr(), d_in, k, 0, idx.data_ptr(), xs.data_ptr(), s2.cuda_stream)
        g.replay(); torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        for _ in range(5):
            g.replay()
        f1.record()
        f1.synchronize()
        print(f"d_in {d_in:6d} k {k:5d}  eager {e0.elapsed_time(e1) * 1e3 / 64:7.2f} us   graph {f0.elapsed_time(f1) * 1e3 / 320:7.2f} us")

# internal timeline of one select (decdec_debug_trace)
NB = 2 + 1024 * 20
buf = torch.zeros(NB, dtype=torch.int64, device="cuda")
for d_in in (1024, 4096, 14336):
    x = torch.from_numpy(gen_activations(d_in, 1, seed=1)[0]).cuda()
    k = 21 * d_in // 1024
    idx = torch.empty(k, dtype=torch.int32, device="cuda")
    xs = torch.empty(k, dtype=torch.float16, device="cuda")
    dd.decdec_debug_trace(buf.data_ptr(), NB * 8)
    for _ in range(3):
        dd.decdec_select(x.data_ptr(), d_in, k, 0, idx.data_ptr(), xs.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    dd.decdec_debug_trace(0, 0)
    t = buf.cpu().numpy()
    t0 = t[0]
    cyc = t[2 + 1024 * 20 - 1] - t[2 + 1024 * 20 - 2]
    c0 = t[2 + 1024 * 20 - 2]
    ph = [int(t[2 + 1024 * 20 - 16 + i] - c0) for i in range(6)]
    print(d_in, "select us (start->end):", round((t[1] - t0) / 1e3, 2), "cycles", cyc, "=> MHz", round(cyc / ((t[1] - t0) / 1e3)),
          "phase cycles zeroed/hist/T/scan:", ph[:4])
