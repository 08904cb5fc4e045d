"""CPU: the C-ABI library loads, exports every entry point include/qft_b200.h
declares, validates arguments in the reference's order, and -- on a host with
no GPU -- refuses compute calls instead of falling back to the CPU."""
import ctypes as C
import os
import re
import subprocess

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qft_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qftc_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_path():
    names = declared_functions()
    for must in ("qftc_quantize_state", "qftc_dequantize", "qftc_outlier_thresholds",
                 "qftc_decompose_dense_sparse", "qftc_reconstruct", "qftc_reconstruct_bf16",
                 "qftc_plan_create", "qftc_plan_step", "qftc_lion_step", "qftc_lion_apply"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2310_07147_b200 import _native as N
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (qftc_\w+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, f"declared but not exported: {missing}"
    # and the ctypes binding covers exactly the declared surface
    assert set(N.EXPORTS) == set(declared_functions())


def test_library_is_sm100a():
    from paper_2310_07147_b200 import _native as N
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_validation_precedes_device_check():
    from paper_2310_07147_b200 import _native as N
    assert N.lib.qftc_quantize_state(None, 2, 2, 9, None, None, None, 0, None) == N.QFTC_EINVAL
    assert "bit width" in N.last_error()
    assert N.lib.qftc_outlier_thresholds(None, 2, 2, 0.5, 0, None, None, None) == N.QFTC_EINVAL
    assert "fraction" in N.last_error()
    assert N.lib.qftc_dequantize(None, 0, 4, None, None, 1, None, None) == N.QFTC_EINVAL
    with pytest.raises(ValueError):
        N.check(N.QFTC_EINVAL)
    with pytest.raises(IndexError):
        N.check(N.QFTC_ERANGE)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    from paper_2310_07147_b200 import _native as N
    rc = N.lib.qftc_synth(None, 16, 1, 1.0, 0.0, None)
    assert rc == N.QFTC_ECUDA and "no CPU fallback" in N.last_error()
    rc = N.lib.qftc_quantize_state(None, 2, 2, 8, None, None, None, 0, None)
    assert rc == N.QFTC_ECUDA


def test_gradient_stack_semantics():
    # gradflow.hpp:15-47: FILO, pop on empty -> std::out_of_range (IndexError)
    from paper_2310_07147_b200 import GradientStack
    s = GradientStack()
    with pytest.raises(IndexError):
        s.pop()
    s.push(2, "g2")
    s.push(1, "g1")
    assert s.pop().layer_index == 1 and s.pop().layer_index == 2 and s.empty()


def test_no_contracted_packed_fma_in_sass():
    """ptxas 12.9 fuses mul.rn.f32x2 + add.rn.f32x2 into FFMA2 despite .rn, so every Lion
    SUM of products is a scalar FADD.  The only FFMA2 forms allowed are the deliberate
    ones: pair * scalar + scalar (the sign factor of the saturating update,
    magic-number rounding), pair * scalar + pair where the pair addend is the weight
    itself (w' = fma(s, lr, w), s in {-1,0,1}: exact product, one rounding) and
    pair * scalar - pair (the quantizer's tie distance x*inv - rint, whose proof holds
    for the exact or the rounded product).  A contracted sum shows up as
    pair * pair-or-scalar + pair on a product register; the parity tests are the
    authoritative check, this one catches the pattern early: every FFMA2 with a
    non-negated pair addend must multiply by the lr register of the sign update."""
    import re
    from paper_2310_07147_b200 import _native as N
    out = subprocess.run(["cuobjdump", "-sass", N.LIB_PATH], capture_output=True, text=True)
    assert out.returncode == 0 and "FMUL2" in out.stdout
    bad = []
    sign_regs = set()   # pair registers holding s = fma(a, -2, 1) (the -sign factor)
    for line in out.stdout.splitlines():
        if "Function :" in line:
            sign_regs = set()
            continue
        m = re.search(r"\b(FFMA2|FMUL2|FADD2|[A-Z][A-Z0-9.]*)\s+(R\d+)\s*,(.*);", line)
        if not m:
            continue
        op, dst, rest = m.group(1), m.group(2), m.group(3)
        ops = [o.strip() for o in rest.split(",")]
        if op == "FFMA2":
            addend = ops[-1]
            if ops[1] == "-2":      # s = fma(a, -2, 1)
                sign_regs.add(dst)
                continue
            src = ops[0].split(".")[0]
            if ".F32x2" in addend and not addend.startswith("-") and src not in sign_regs:
                bad.append(line.strip())
        sign_regs.discard(dst) if op != "FFMA2" else None
    assert not bad, f"contracted packed FMA: {bad[:4]}"


def test_gemm_entry_points_validate_before_the_device():
    """The GEMM entry points reject bad shapes / null pointers before touching the device
    (no GPU needed), and the forward and dx index workspaces have the same size."""
    from paper_2310_07147_b200 import _native as N
    p = C.c_void_p(16)  # a dummy (16-byte aligned) pointer: never dereferenced here
    assert N.lib.qftc_dequant_gemm_index(p, None, p, 8, 100, p, None) == N.QFTC_EINVAL
    assert N.lib.qftc_dequant_gemm_index(None, None, p, 8, 128, p, None) == N.QFTC_EINVAL
    assert N.lib.qftc_dequant_gemm_prebuilt(p, 4, 100, p, 8, p, p, p, p, p, p, None) == N.QFTC_ENOTSUP
    assert N.lib.qftc_dequant_gemm_prebuilt(p, 4, 128, p, 8, p, p, p, p, None, p, None) == N.QFTC_EINVAL
    assert N.lib.qftc_dequant_gemm_t_prebuilt(p, 4, 96, p, 128, p, p, p, p, p, p, None) == N.QFTC_ENOTSUP
    assert N.lib.qftc_dequant_gemm(p, 4, 128, p, 8, p, p, p, None, p, p, p, None, None) == N.QFTC_EINVAL
    for r, c in ((4096, 4096), (11008, 4096), (4096, 11008), (192, 320)):
        assert (N.lib.qftc_dequant_gemm_workspace_bytes(r, c) ==
                N.lib.qftc_dequant_gemm_t_workspace_bytes(r, c) == r * (c // 32 + 1) * 4)
