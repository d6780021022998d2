"""C-ABI boundary checks that need no GPU: the library builds, loads, exports every symbol
include/crvpinn.h declares, validates arguments before touching a device, and fails loudly
(CRVPINN_ECUDA, never a CPU fallback) when no sm_100 device is present."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2604_20731_b200 as crv
from paper_2604_20731_b200 import build as crvbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "crvpinn.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(crvpinn_[a-z_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    crvbuild.build()
    return crv.load()


def test_header_declares_the_north_star_calls():
    decl = _declared()
    for name in ["crvpinn_create", "crvpinn_pretrain", "crvpinn_step", "crvpinn_eval"]:
        assert name in decl
    assert decl == sorted(crv.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", crv.LIB_PATH]).decode()
    exported = set(re.findall(r" T (crvpinn_\w+)", out))
    missing = [s for s in _declared() if s not in exported]
    assert not missing, missing
    for s in _declared():
        assert hasattr(lib, s)


def test_library_is_sm100a_only(lib):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", crv.LIB_PATH]).decode()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def test_default_opts(lib):
    o = crv.default_opts()
    assert o.lr == 1e-3 and o.beta1 == 0.9 and o.beta2 == 0.999 and o.eps == 1e-8
    assert abs(o.mobility_ratio - 25.35 / 3.95) < 1e-15
    assert o.precision == crv.PREC_TENSOR


@pytest.mark.parametrize("N,widths,msg", [
    (30, (2, 32, 1), "power of two"),
    (8, (2, 32, 1), "power of two"),
    (32, (3, 32, 1), "widths"),
    (32, (2, 32, 2), "widths"),
    (32, (2, 48, 1), "multiples of 32"),
    (32, (2, 512, 1), "multiples of 32"),
])
def test_invalid_arguments_rejected_before_device(lib, N, widths, msg):
    nn = (N + 1) ** 2
    z = np.zeros(nn, np.float32)
    with pytest.raises(crv.CrvpinnError) as ei:
        crv.Crvpinn(N, widths, np.ones(nn), z, z, precision=crv.PREC_FP32)
    assert ei.value.code == crv.CRVPINN_EINVAL and msg in str(ei.value)


def test_domain_errors(lib):
    N = 16
    nn = (N + 1) ** 2
    z = np.zeros(nn, np.float32)
    K = np.ones(nn, np.float32)
    K[5] = 0.0
    with pytest.raises(crv.CrvpinnError) as ei:
        crv.Crvpinn(N, (2, 32, 1), K, z, z, precision=crv.PREC_FP32)
    assert ei.value.code == crv.CRVPINN_EDOMAIN
    f = z.copy()
    f[3] = np.nan
    with pytest.raises(crv.CrvpinnError) as ei:
        crv.Crvpinn(N, (2, 32, 1), np.ones(nn), z, f, precision=crv.PREC_FP32)
    assert ei.value.code == crv.CRVPINN_EDOMAIN


def test_no_cpu_fallback_without_gpu(lib):
    """Without a B200 the library must refuse (ECUDA), not compute on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    N = 16
    nn = (N + 1) ** 2
    with pytest.raises(crv.CrvpinnError) as ei:
        crv.Crvpinn(N, (2, 32, 1), np.ones(nn), np.zeros(nn), np.zeros(nn), precision=crv.PREC_FP32)
    assert ei.value.code == crv.CRVPINN_ECUDA


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2604_20731_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, fn)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", text).lower().replace("oracle/", ""), fn


def test_context_code_has_no_legacy_stream_fills_or_uploads():
    """crvpinn.cu works on a non-blocking context stream, which does not wait for the legacy stream:
    a bare cudaMemset / host-to-device cudaMemcpy there can land after later context-stream work
    (round 2: the fp32 path's reduction-job table was zeroed after its copy). Zero fills and uploads
    in the context code must be stream-ordered (…Async on ctx->stream)."""
    text = open(os.path.join(ROOT, "paper_2604_20731_b200", "csrc", "crvpinn.cu")).read()
    code = re.sub(r"//.*", "", text)
    assert not re.search(r"\bcudaMemset\s*\(", code)
    for m in re.finditer(r"\bcudaMemcpy\s*\(([^;]*);", code):
        assert "cudaMemcpyDeviceToHost" in m.group(1), m.group(0)
