"""C-ABI boundary on the CPU: the library loads, exports every declared symbol,
validates arguments, and its planner tables equal the oracle's bit for bit."""
import ctypes
import os
import re

import pytest

from oracle import counts
from oracle.nested import plan_tables
from paper_2102_13272_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "nw.h")).read()
    declared = set(re.findall(r"NW_API [\w\s\*]*?\b(nw_\w+)\(", hdr))
    assert declared, "no declarations parsed"
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.EXPORTS)


def test_status_strings_and_errors():
    lib = _lib.load()
    h = ctypes.c_void_p()
    assert lib.nw_plan(9, 3, 3, 3, 4, 4, ctypes.byref(h)) == _lib.NW_ERR_UNSUPPORTED
    assert lib.nw_plan(9, 1, 0, 3, 4, 4, ctypes.byref(h)) == _lib.NW_ERR_INVALID
    assert lib.nw_plan(9, 1, 7, 3, 4, 4, ctypes.byref(h)) == _lib.NW_ERR_INVALID
    assert lib.nw_plan(10, 1, 3, 3, 4, 4, ctypes.byref(h)) == _lib.NW_ERR_UNSUPPORTED
    assert lib.nw_plan(9, 1, 3, 3, 4, 4, None) == _lib.NW_ERR_INVALID
    assert lib.nw_plan(9, 1, 3, 3, 0, 4, ctypes.byref(h)) == _lib.NW_ERR_INVALID
    assert _lib.status_str(_lib.NW_ERR_WORKSPACE) == "workspace too small"
    p = _lib.Plan(5, 1, 3, 3, 4, 4)
    with pytest.raises(_lib.NWError) as e:
        lib2 = _lib.load()
        st = lib2.nw_plan_set(p.handle, _lib.ATTR_MATH, 0)
        _lib._chk(st, "late set")
    assert e.value.status == _lib.NW_ERR_STATE
    with pytest.raises(_lib.NWError):
        _lib.Plan(5, 1, 3, 3, 4, 4, transposed=True)          # transposed needs stride 2


CASES = [
    # K, stride, m_o, m_i, Cin, Cout, transposed, pad, outer_taps
    (5, 1, 2, 2, 16, 16, False, 2, 3),     # configs[0]
    (5, 1, 3, 3, 64, 64, False, 2, 3),
    (7, 1, 3, 3, 64, 64, False, 3, 3),
    (9, 1, 3, 3, 64, 64, False, 4, 3),     # configs[1]
    (9, 1, 3, 3, 256, 256, False, 4, 3),   # configs[2]
    (7, 2, 3, 3, 3, 64, False, 3, 3),      # configs[3]
    (9, 2, 3, 3, 64, 64, False, 4, 3),
    (9, 2, 3, 3, 32, 1, True, 4, 3),       # configs[4] deconv
    (3, 2, 3, 3, 4, 4, True, 1, 3),
    (5, 1, 3, 3, 8, 8, False, 2, 0),       # mixed outer kernel F(3,2)
    (4, 1, 2, 3, 8, 8, False, 1, 3),
    (8, 1, 4, 3, 8, 8, False, 3, 3),
    (6, 1, 6, 6, 8, 8, False, 3, 3),
    (3, 1, 1, 1, 8, 8, False, 1, 3),
]


@pytest.mark.parametrize("K,stride,m_o,m_i,Cin,Cout,tr,pad,ot", CASES)
def test_tables_bit_exact_vs_oracle(K, stride, m_o, m_i, Cin, Cout, tr, pad, ot):
    plan = _lib.Plan(K, stride, m_o, m_i, Cin, Cout, transposed=tr, pad=pad, outer_taps=ot,
                     output_padding=1 if tr else 0)
    ref = plan_tables(K, stride, m_o, m_i, Cin, Cout, transposed=tr, pad=pad, outer_taps=ot)
    for which in range(8):
        assert plan.tables(which) == ref[which], f"table {which}"


@pytest.mark.parametrize("K,stride,m_o,m_i,Cin,Cout,tr,pad,ot", CASES[:9])
def test_count_mults_vs_closed_form(K, stride, m_o, m_i, Cin, Cout, tr, pad, ot):
    plan = _lib.Plan(K, stride, m_o, m_i, Cin, Cout, transposed=tr, pad=pad, outer_taps=ot,
                     output_padding=1 if tr else 0)
    N, H, W = 2, 37, 29
    Ho, Wo = plan.output_size(H, W)
    inf = plan.info()
    if tr:
        Hq, Wq = (Ho + 1) // 2, (Wo + 1) // 2
    else:
        Hq, Wq = Ho, Wo
    ref = counts.layer_ewmm_nested(N, Hq, Wq, inf["cin_e"], inf["cout_e"], m_o, inf["r_outer"], m_i)
    assert plan.count_mults(N, H, W) == ref


def test_output_sizes():
    assert _lib.Plan(9, 2, 3, 3, 32, 1, transposed=True, pad=4, output_padding=1).output_size(540, 960) == (1080, 1920)
    assert _lib.Plan(7, 2, 3, 3, 3, 64, pad=3).output_size(224, 224) == (112, 112)
    assert _lib.Plan(9, 2, 3, 3, 64, 64, pad=4).output_size(112, 112) == (56, 56)
    assert _lib.Plan(9, 1, 3, 3, 256, 256, pad=4).output_size(64, 64) == (64, 64)


def _r256(b):
    return (b + 255) // 256 * 256


@pytest.mark.parametrize("K,pad", [(5, 2), (7, 3), (9, 4)])
def test_comparison_workspace_geometry(K, pad):
    # OLA (Eq. 2.3): ceil(K/3)^2 blocks of F(3,3) over a 3x3-output tile grid extended by nb-1;
    # direct (Eq. 2.1): K^2 taps over the pixel grid extended by K-1.  Sizes = U + V + M, 4 B/elt.
    N, C, H = 2, 64, 40
    plan = _lib.Plan(K, 1, 3, 3, C, C, pad=pad)
    nb = -(-K // 3)
    tiles = -(-H // 3) + nb - 1
    T = N * tiles * tiles
    Tp = -(-T // 128) * 128
    ola = _r256(25 * C * nb * nb * C * 4) + 2 * _r256(25 * Tp * C * 4)
    assert plan.workspace_size(N, H, H, "ola") == ola
    px = H + K - 1
    T = N * px * px
    Tp = -(-T // 128) * 128
    direct = _r256(C * K * K * C * 4) + 2 * _r256(Tp * C * 4)
    assert plan.workspace_size(N, H, H, "direct") == direct


def test_m_rows_reports_fused_inner_output_level():
    # the contraction writes M (P_a^2 rows per slice) or, with the inner output level of A^T_hat
    # fused into its epilogue along w, P_a * l_o * m_i rows, along both axes (l_o * m_i)^2 rows
    # (A^T_hat = A_o^T (x) A_i^T)
    for K, m_o, C in ((9, 4, 64), (9, 3, 64), (9, 4, 256), (5, 3, 16)):
        inf = _lib.Plan(K, 1, m_o, 3, C, C).info()
        l_o = m_o + 2
        assert inf["m_rows"] in (inf["points"], inf["points_axis"] * l_o * 3, (l_o * 3) ** 2)
    assert _lib.Plan(9, 1, 4, 3, 64, 64, math=_lib.MATH_FP32_SIMT).info()["m_rows"] == 900


def test_single_kernel_for_one_input_channel():
    # Cin = 1 (stride 1, m_i = 3): the contraction over input channels (Eq. 2.1) is one product per
    # point, so the layer runs as one on-chip kernel and writes no transform-domain rows
    for K, m_o, r_o in ((5, 4, 0), (9, 4, 3), (7, 3, 3)):
        inf = _lib.Plan(K, 1, m_o, 3, 1, 32, outer_taps=r_o).info()
        assert inf["single_kernel"] == 1 and inf["m_rows"] == 0
    assert _lib.Plan(9, 1, 5, 3, 1, 32).info()["single_kernel"] == 0      # V of 32 slices exceeds smem
    assert _lib.Plan(5, 2, 4, 3, 1, 32).info()["single_kernel"] == 0      # stride 2: 4 phase channels
    assert _lib.Plan(5, 1, 2, 2, 1, 32).info()["single_kernel"] == 0      # coverage phases (m_i = 2)
    assert _lib.Plan(5, 1, 4, 3, 2, 32).info()["single_kernel"] == 0


def test_single_kernel_for_four_or_fewer_outputs():
    # Cout_e <= 4 (C5's deconvolution: 4 output phases of 1 channel; SRCNN 5x5 1 <- 32): the
    # channel sum runs in registers, one kernel, no transform-domain rows in HBM
    dec = _lib.Plan(9, 2, 4, 3, 32, 1, transposed=True, output_padding=1, outer_taps=0, pad=4).info()
    assert dec["cout_e"] == 4 and dec["single_kernel"] == 1
    assert _lib.Plan(5, 1, 4, 3, 32, 1, outer_taps=0).info()["single_kernel"] == 1
    assert _lib.Plan(9, 1, 4, 3, 48, 3).info()["single_kernel"] == 1             # P_a 30
    assert _lib.Plan(9, 1, 4, 3, 48, 5).info()["single_kernel"] == 0             # five outputs
    assert _lib.Plan(9, 2, 4, 3, 8, 2, outer_taps=0).info()["single_kernel"] == 0  # stride-2 input phases


def test_forward_argument_errors_without_touching_memory():
    # argument validation happens before any CUDA call: fake (never dereferenced) pointers suffice
    lib = _lib.load()
    p = _lib.Plan(9, 1, 3, 3, 16, 16)
    FAKE = 1 << 20          # 16-byte aligned, never dereferenced
    ws_need = p.workspace_size(2, 20, 20)
    fwd = lib.nw_conv_forward
    assert fwd(p.handle, FAKE, FAKE, FAKE, 0, 20, 20, FAKE, ws_need, None) == _lib.NW_ERR_INVALID   # empty batch
    assert fwd(p.handle, FAKE, FAKE, FAKE, 2, 0, 20, FAKE, ws_need, None) == _lib.NW_ERR_INVALID   # empty image
    assert fwd(p.handle, 0, FAKE, FAKE, 2, 20, 20, FAKE, ws_need, None) == _lib.NW_ERR_INVALID     # null x
    assert fwd(p.handle, FAKE + 4, FAKE, FAKE, 2, 20, 20, FAKE, ws_need, None) == _lib.NW_ERR_INVALID  # misaligned
    assert fwd(p.handle, FAKE, FAKE, FAKE, 2, 20, 20, FAKE, ws_need - 1, None) == _lib.NW_ERR_WORKSPACE
    assert fwd(p.handle, FAKE, FAKE, FAKE, 2, 20, 20, 0, ws_need, None) == _lib.NW_ERR_WORKSPACE
    q = _lib.Plan(9, 1, 3, 3, 16, 16, pad=0)
    # 9x9 filter, no padding, 5x5 image: no output
    assert lib.nw_conv_forward(q.handle, FAKE, FAKE, FAKE, 1, 5, 5, FAKE, 1 << 30, None) == _lib.NW_ERR_INVALID
    # an outer kernel with no compiled transform (F(6,3) (x) F(3,3)) is refused, not emulated
    r = _lib.Plan(9, 1, 6, 3, 16, 16)
    need = r.workspace_size(1, 30, 30)
    assert lib.nw_conv_forward(r.handle, FAKE, FAKE, FAKE, 1, 30, 30, FAKE, need, None) == _lib.NW_ERR_UNSUPPORTED
    # comparison paths validate the same way
    assert lib.nw_conv_ola(p.handle, FAKE, FAKE, FAKE, 0, 20, 20, FAKE, 1 << 30, None) == _lib.NW_ERR_INVALID
    assert lib.nw_conv_direct(p.handle, FAKE, FAKE, FAKE, 2, 20, 20, FAKE, 16, None) == _lib.NW_ERR_WORKSPACE


def test_decompose_matches_oracle_planner():
    # the library's section IV.B planner (csrc/decompose.cu) vs the oracle's (oracle/planner.py):
    # same token stream and output length over the Fig. 7 kernels, strides 1-3 and R up to 30
    from oracle import planner
    kernels = [(2, 2), (3, 3), (4, 4), (6, 3), (4, 3), (3, 2), (5, 3), (4, 2)]
    for (m, r) in kernels:
        for S in (1, 2, 3):
            for R in list(range(1, 19)) + [25, 27, 30]:
                p = planner.plan(R, S, m, r)
                assert _lib.decompose(R, S, m, r) == (planner.rpn_text(p), p.M), (R, S, m, r)


def test_decompose_errors():
    import pytest
    with pytest.raises(_lib.NWError):
        _lib.decompose(0, 1, 3, 3)
    with pytest.raises(_lib.NWError):
        _lib.decompose(5, 1, 2, 3)      # m < r nesting leaves holes
    assert _lib.decompose(3, 1, 2, 3) == ("K2,3", 2)   # no nesting needed: fine


def test_depthwise_plan_info_and_errors():
    # depthwise (Table I PNASNet row): U holds one fp32 filter per channel; EWMM count has no
    # channel product; Cin != Cout and stride 2 are refused
    p = _lib.Plan(7, 1, 4, 3, 54, 54, depthwise=True)
    inf = p.info()
    assert inf["filter_bytes"] == 900 * 64 * 4 and inf["single_kernel"] == 0 and inf["m_rows"] == 900
    assert p.count_mults(8, 83, 83) == 8 * 7 * 7 * 900 * 54
    import pytest
    with pytest.raises(_lib.NWError):
        _lib.Plan(7, 1, 4, 3, 54, 32, depthwise=True)
    with pytest.raises(_lib.NWError):
        _lib.Plan(7, 2, 4, 3, 54, 54, depthwise=True)
