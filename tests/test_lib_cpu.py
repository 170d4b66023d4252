"""libdecdec on the CPU host: it loads, exports every symbol include/decdec.h declares, and
its C++ packers match the oracle's independent layout implementation byte for byte.
No CUDA compute calls (no GPU here)."""

import os
import re

import numpy as np
import pytest

import oracle
from synth import gen_perf_layer

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dd():
    import paper_2412_20185_b200 as m
    return m


def header_functions():
    src = open(os.path.join(ROOT, "include", "decdec.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(decdec_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_header_symbol(dd):
    import ctypes
    names = header_functions()
    assert len(names) >= 15
    lib = ctypes.CDLL(dd.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(dd.EXPORTED)


def test_version_and_status(dd):
    assert "sm_100a" in dd.decdec_version()
    assert dd.decdec_status_string(-3).startswith("residual pointer")


@pytest.mark.parametrize("bits", [3, 4])
@pytest.mark.parametrize("shape", [(256, 64), (1024, 96), (512, 32)])
def test_pack_weights_matches_oracle(dd, bits, shape):
    L = gen_perf_layer(*shape, bits, seed=shape[0] + bits, with_residual=False)
    mine = dd.pack_weights(L["q"], bits)
    ref = oracle.pack_w3k_ref(L["q"]) if bits == 3 else oracle.pack_w4k_ref(L["q"])
    assert mine.dtype == np.uint32 and np.array_equal(mine, ref)


def test_pack_residual_matches_oracle(dd):
    L = gen_perf_layer(256, 128, 3, seed=4)
    out = np.zeros((256, 16), np.uint32)
    dd.pack_residual_into(L["rc"], out)
    assert np.array_equal(out, oracle.pack_rq_ref(L["rc"]))


def test_pack_golden_words_c(dd, golden):
    for ln in golden("pack_words.txt"):
        kind, rest = ln.split(None, 1)
        lhs, rhs = (p.strip() for p in rest.split(";"))
        exp = [int(w, 16) for w in rhs.split()]
        if kind == "w4k":
            q = np.zeros((32, 1), np.uint8)
            q[:8, 0] = [int(v) for v in lhs.split()]
            assert int(dd.pack_weights(q, 4)[0, 0]) == exp[0]
        elif kind == "w3k":
            q = np.zeros((32, 1), np.uint8)
            for tok in lhs.split():
                c, v = tok.split(":")
                q[int(c), 0] = int(v)
            assert [int(w) for w in dd.pack_weights(q, 3)[0]] == exp
        elif kind == "rq":
            c = np.zeros((1, 8), np.int8)
            c[0] = [int(v) for v in lhs.split()]
            out = np.zeros((1, 1), np.uint32)
            dd.pack_residual_into(c, out)
            assert int(out[0, 0]) == exp[0]


def test_packer_rejects_bad_codes(dd):
    with pytest.raises(dd.DecdecError):
        dd.pack_weights(np.full((32, 1), 8, np.uint8), 3)
    out = np.zeros((1, 1), np.uint32)
    with pytest.raises(dd.DecdecError):
        dd.pack_residual_into(np.full((1, 8), -8, np.int8), out)


def test_num_selected_and_workspace(dd):
    assert dd.decdec_num_selected(4096, 128, 0) == 128
    assert dd.decdec_num_selected(4096, 32, 1024) == 128            # P:255 example
    assert dd.decdec_num_selected(17920, 600, 1024) == 17 * 600 + 512  # short last chunk
    assert dd.decdec_num_selected(4096, 4097, 0) == -1
    assert dd.decdec_num_selected(4096, 2000, 1024) == -1
    # the paper's k x (4+2) B buffer is part of the workspace
    assert dd.decdec_workspace_bytes(1433, 4096) >= 1433 * 6


def test_peer_offsets_symmetric_layout():
    """Fused P2P all-gather: y_full buffers of a stack in the peer user area (tp.peer_offsets)
    are 256-B aligned, disjoint and in layer order -- the same offsets on every rank."""
    from paper_2412_20185_b200.tp import peer_offsets

    d_outs = [768, 512, 3584, 512]
    for world in (1, 2, 8):
        offs, total = peer_offsets(d_outs, world)
        ends = [o + world * d * 2 for o, d in zip(offs, d_outs)]
        assert all(o % 256 == 0 for o in offs)
        assert all(e <= o2 for e, o2 in zip(ends, offs[1:]))
        assert total >= ends[-1] and total % 256 == 0
