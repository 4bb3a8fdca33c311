"""CPU-side checks of the C ABI boundary: the library loads and exports every symbol that
include/masq.h declares; the binding mirrors the header; workspace arithmetic; argument
validation paths that return before any CUDA call."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "masq.h")
SO = os.path.join(ROOT, "paper_2603_04800_b200", "libmasq.so")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(masq_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def so():
    if not os.path.exists(SO):
        import __graft_entry__
        __graft_entry__.build()
    return ctypes.CDLL(SO)


def test_header_declares_the_five_operations():
    fns = header_functions()
    for f in ("masq_calibrate_stats", "masq_init_factors", "masq_quantize_weight", "masq_linear_forward",
              "masq_calib_loss"):
        assert f in fns


def test_library_exports_every_header_symbol(so):
    for f in header_functions():
        assert hasattr(so, f), f


def test_binding_mirrors_header():
    from paper_2603_04800_b200._lib import SIGNATURES
    assert sorted(SIGNATURES) == header_functions()


def test_status_strings_and_version(so):
    from paper_2603_04800_b200._lib import lib
    L = lib()
    assert L.masq_version().decode().endswith("sm_100a")
    for st in range(10):
        assert L.masq_status_string(st)


def test_workspace_sizes(so):
    from paper_2603_04800_b200._lib import lib
    L = lib()
    T, d, n, M = 16384, 3584, 18944, 2
    fwd0 = L.masq_workspace_size(4, T, d, n, M, 0)
    fwd64 = L.masq_workspace_size(4, T, d, n, M, 64)
    assert fwd0 >= T * d + 4 * T
    assert fwd64 - fwd0 >= 2 * T * 2 * 64 * (M - 1)   # Z hi/lo
    loss = L.masq_workspace_size(5, T, d, n, M, 0)
    assert loss >= M * n * d                          # one Q(S_m W) per modality
    assert L.masq_workspace_size(0, T, d, 0, M, 0) == 256


def test_argument_errors_return_before_launch(so):
    """Synchronous validation (no device needed): NULL, shape, bits, workspace."""
    from paper_2603_04800_b200._lib import lib
    L = lib()
    ws = ctypes.create_string_buffer(4096)
    p = ctypes.c_void_p(ctypes.addressof(ws))
    # n_mod out of range -> SHAPE
    assert L.masq_calibrate_stats(None, 1, 64, None, 10, 64, 9, p, p, 1, p, 4096, None) == 2
    # d not multiple of 16 -> SHAPE
    assert L.masq_calibrate_stats(None, 1, 64, None, 10, 60, 2, p, p, 1, p, 4096, None) == 2
    # R NULL -> NULL
    assert L.masq_calibrate_stats(None, 1, 64, None, 10, 64, 2, None, p, 1, p, 4096, None) == 1
    # wbits 16 -> UNSUPPORTED, wbits 1 -> BITS
    assert L.masq_quantize_weight(p, 1, p, 64, 128, 16, p, p, p, 4096, None) == 8
    assert L.masq_quantize_weight(p, 1, p, 64, 128, 1, p, p, p, 4096, None) == 3
    # r not multiple of 16 -> SHAPE
    assert L.masq_linear_forward(p, 1, 64, p, 10, 64, 128, 2, p, p, p, 8, 8, p, p, 128, 8, p, 128, p, 4096,
                                 None, None) == 2
    # workspace too small -> WORKSPACE
    assert L.masq_quantize_weight(p, 1, p, 64, 128, 8, p, p, p, 16, None) == 5


def test_every_workspace_op_has_a_layout(so):
    """Every MASQ_OP_* the header declares has its own workspace layout (a switch case lost in an
    edit would silently hand the op a 256-byte layout and overlapping buffers)."""
    from paper_2603_04800_b200._lib import lib
    L = lib()
    src = open(HEADER).read()
    ops = {k: int(v, 0) for k, v in re.findall(r"\b(MASQ_OP_[A-Z_]+)\s*=\s*(0x[0-9a-fA-F]+|\d+)", src)}
    flag = ops.pop("MASQ_OP_SELF_REF")
    assert len(ops) >= 14
    T, d, n, M, r = 4096, 1024, 2048, 2, 64
    stateless = {"MASQ_OP_STATS", "MASQ_OP_INIT", "MASQ_OP_REFERENCE"}   # only the status word (at d < 4096)
    cpu_only_unknown = {"MASQ_OP_CMC", "MASQ_OP_CMC_FACTORS"}   # need the eigensolver's query (GPU)
    for name, op in ops.items():
        size = L.masq_workspace_size(op, T, d, n, M, r)
        if name in stateless:
            assert size == 256, name
        elif name in cpu_only_unknown:
            assert size >= 256, name
        else:
            assert size > 4096, (name, size)
    # deep K: the GEMM's stream-K scratch (partial tiles + flags) joins the layouts that run it
    assert L.masq_workspace_size(ops["MASQ_OP_REFERENCE"], T, 4096, n, 1, 0) > (1 << 20)
    assert L.masq_workspace_size(ops["MASQ_OP_FORWARD"], T, 8192, n, M, r) > \
        L.masq_workspace_size(ops["MASQ_OP_FORWARD"], T, 8192 - 128, n, M, r) + (1 << 20)
    # the self-reference flag appends the loss target X W (f32 [T x n]) to the loss layouts
    for name in ("MASQ_OP_LOSS", "MASQ_OP_LOSS_GRAD"):
        base = L.masq_workspace_size(ops[name], T, d, n, M, 0)
        assert L.masq_workspace_size(ops[name] | flag, T, d, n, M, 0) >= base + 4 * T * n
