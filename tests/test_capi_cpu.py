"""CPU-side checks of the boundary: the C-ABI library builds for sm_100a,
loads, and exports every symbol include/qpb200.h declares; argument
validation runs without a GPU; the oracle stays out of the product path."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "qpb200.h")


def declared_symbols():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w]+\*?\s+\*?(qp_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2605_17913_b200 import _build
    _build.build()
    from paper_2605_17913_b200 import capi
    return capi.load()


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("qp_create", "qp_solve_batched", "qp_backward_batched", "qp_destroy", "qp_error_string",
              "qp_config_default", "qp_get_info", "qp_set_stream", "qp_max_kkt_dim"):
        assert s in syms, s


def test_library_exports_every_declared_symbol(lib):
    from paper_2605_17913_b200 import _build
    out = subprocess.run(["nm", "-D", "--defined-only", _build.LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (qp_\w+)", out))
    for s in declared_symbols():
        assert s in exported, s
        assert hasattr(lib, s)


def test_sass_is_sm100a(lib):
    from paper_2605_17913_b200 import _build
    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_validation_without_gpu(lib):
    from paper_2605_17913_b200 import capi
    cfg = capi.default_config()
    assert abs(cfg.tol - 1e-5) < 1e-9 and cfg.max_iter == 100 and abs(cfg.sigma - 0.1) < 1e-7
    h = C.c_void_p()
    bad = capi.QpDims(0, 5, 0, 3, 25, 5, 0, 0, 15, 3)
    assert lib.qp_create(C.byref(h), C.byref(bad), C.byref(cfg), 0, None) == -2  # QP_ERR_SHAPE
    good = capi.QpDims(4, 5, 0, 3, 25, 5, 0, 0, 15, 3)
    cfg.sigma = 1.5
    assert lib.qp_create(C.byref(h), C.byref(good), C.byref(cfg), 0, None) == -1  # invalid config
    cfg = capi.default_config()
    # config 5 (n = 1024, p = 2048) is supported; p = 8192 needs more than the
    # 227 KB of shared memory for the per-constraint vectors alone
    big = capi.QpDims(4, 1024, 0, 8192, 1024 * 1024, 1024, 0, 0, 8192 * 1024, 8192)
    assert lib.qp_create(C.byref(h), C.byref(big), C.byref(cfg), 0, None) == -2
    # mem_kind: QP_MEM_DEVICE / QP_MEM_HOST / QP_MEM_HOST_ASYNC pass validation
    # (then fail on the missing device), anything else is an invalid config
    for mk, want in ((capi.QP_MEM_HOST_ASYNC, -4), (3, -1)):
        cfg.mem_kind = mk
        assert lib.qp_create(C.byref(h), C.byref(good), C.byref(cfg), 0, None) == want, mk
    # padded batch strides (bstride > per-problem size): device mode only;
    # the host modes stage contiguous copies and reject them
    padded = capi.QpDims(4, 5, 0, 3, 32, 8, 0, 0, 16, 4)
    for mk, want in ((capi.QP_MEM_DEVICE, -4), (capi.QP_MEM_HOST, -2), (capi.QP_MEM_HOST_ASYNC, -2)):
        cfg.mem_kind = mk
        assert lib.qp_create(C.byref(h), C.byref(padded), C.byref(cfg), 0, None) == want, mk
    cfg = capi.default_config()
    assert lib.qp_error_string(-4) == b"CUDA error"
    assert lib.qp_solve_batched(*([None] * 13)) == -1
    assert lib.qp_backward_batched(*([None] * 10)) == -1


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2605_17913_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "qp_oracle" not in txt, f


def test_empty_batch_binding_cpu():
    """Degenerate case B = 0 (host buffers, no GPU needed): the binding returns
    empty outputs without creating a ctx (the C ABI itself takes B >= 1 and
    answers QP_ERR_SHAPE, checked above); gradients of shared fields are sums
    over no problems, i.e. zero."""
    import torch
    from paper_2605_17913_b200.solver import QPSolver
    n, m, p = 5, 2, 3
    s = QPSolver(0, n, m, p, shared=("G", "h"), mem="host")
    f = lambda *sh: torch.zeros(*sh, dtype=torch.float32)
    out = s.solve(f(0, n, n), f(0, n), f(0, m, n), f(0, m), f(p, n), f(p))
    assert out["x"].shape == (0, n) and out["z"].shape == (0, p) and out["iters"].shape == (0,)
    g = s.backward(f(0, n))
    assert g["dQ"].shape == (0, n, n) and g["dG"].shape == (p, n) and g["dh"].shape == (p,)
    assert float(g["dG"].abs().sum()) == 0.0 and float(g["dh"].abs().sum()) == 0.0
    assert s.info() == {} and s.last_flops() == (0.0, 0.0)
    with pytest.raises(RuntimeError):
        QPSolver(0, n, m, p, mem="host").backward(f(0, n))
