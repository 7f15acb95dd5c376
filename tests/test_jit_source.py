"""K1c source (jit.cpp) without a GPU: the CUDA C++ the library generates
for a program and run shape compiles with NVRTC for sm_100a in every mode
(write records into the bucket regions or into the record planes,
fuel-checked, direct commit, every read logged), for the workload
kernels, the opcode corpus and random kernels.  Semantics are checked on the
GPU (tests/test_gpu_parity.py runs every parity test under K1 and K1c)."""
import ctypes
import os

import numpy as np
import pytest

from workloads import kernels as K

NVRTC = None
for name in ("libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12"):
    try:
        NVRTC = ctypes.CDLL(name)
        break
    except OSError:
        pass


@pytest.fixture(scope="module")
def rc():
    import paper_1308_3203_b200 as pkg
    pkg.lib()
    return pkg


def nvrtc_compile(src: str) -> tuple[int, str, int]:
    prog = ctypes.c_void_p()
    assert NVRTC.nvrtcCreateProgram(ctypes.byref(prog), src.encode(), b"k1c.cu", 0, None, None) == 0
    opts = [b"--gpu-architecture=sm_100a", b"--std=c++17", b"-w"]
    arr = (ctypes.c_char_p * len(opts))(*opts)
    r = NVRTC.nvrtcCompileProgram(prog, len(opts), arr)
    n = ctypes.c_size_t()
    NVRTC.nvrtcGetProgramLogSize(prog, ctypes.byref(n))
    log = ctypes.create_string_buffer(n.value + 1)
    NVRTC.nvrtcGetProgramLog(prog, log)
    nb = ctypes.c_size_t(0)
    if r == 0:
        NVRTC.nvrtcGetCUBINSize(prog, ctypes.byref(nb))
    NVRTC.nvrtcDestroyProgram(ctypes.byref(prog))
    return r, log.value.decode(errors="replace"), nb.value


def programs():
    out = [("stencil", K.program(K.STENCIL), 1 << 20, [(1 << 20) + 2] * 2),
           ("tree", K.program(K.TREE), 1024, [1024]),
           ("fig1", K.program(K.FIG1), 8, None),
           ("cfg4", K.random_stencil_kernel(0), 65536, None),
           ("cfg4_full", K.random_stencil_kernel(3, isa="full"), 4096, None)]
    for name, src in list(K.BENIGN.items())[:3]:
        out.append((name, K.program(src), 32, None))
    rng = np.random.default_rng(7)
    for i in range(3):
        out.append((f"tiny{i}", K.random_tiny_kernel(rng), 4, None))
    return out


@pytest.mark.skipif(NVRTC is None, reason="libnvrtc not found")
@pytest.mark.parametrize("name,p,n,sizes", programs(), ids=[x[0] for x in programs()])
def test_k1c_source_compiles(rc, name, p, n, sizes):
    prog = rc.rc_load_program(p.bytecode)
    sizes = sizes or [n + 16] * prog.n_arrays
    modes = [dict(wbucket=True, narrow=True), dict(), dict(fuel=True), dict(direct=True, narrow=True),
             dict(ro_skip=False, wbucket=True)]
    for m in modes[: 5 if name in ("stencil", "tree", "tiny0") else 2]:
        src = prog.jit_source(n, sizes, **m)
        assert 'extern "C" __global__' in src and "rc_k1c" in src
        r, log, nb = nvrtc_compile(src)
        assert r == 0 and nb > 0, f"{name} {m}: {log[:2000]}"


def test_k1c_source_shape_constants(rc):
    """Operands and array geometry are immediates: the stencil's B array
    starts at cell size(A) and its bounds check is against size(B)."""
    prog = rc.rc_load_program(K.program(K.STENCIL).bytecode)
    src = prog.jit_source(1000, [1002, 1002])
    assert "cb + 1002u + (u32)idx" in src and ">= 1002u" in src
    assert "switch (pc)" in src and "case 0u:" in src
    # the first loads of an interval search no overlay (nothing stored yet)
    first_ld = src.index("pc 4\n")
    assert "oc0 == cell" not in src[first_ld:src.index("pc 5\n")]


def test_k1c_rematerialised_registers(rc):
    """The affine-register analysis on the stencil (hand-derived: c = tid+1,
    the index registers r0 = tid, r1 = tid + 1, r3 = tid + 2 at both barrier
    entries; r7, the loop counter, is not a function of tid): r0 / r1 / r3 are
    recomputed at the entries and never loaded or stored, r7 is carried."""
    prog = rc.rc_load_program(K.program(K.STENCIL).bytecode)
    src = prog.jit_source(1 << 10, [(1 << 10) + 2] * 2, wbucket=True)
    for e in (11, 14):
        case = next(l for l in src.splitlines() if l.strip().startswith(f"case {e}u:"))
        assert "r0 = (i32)(1u * tid + 0u)" in case and "r1 = (i32)(1u * tid + 1u)" in case
        assert "r3 = (i32)(1u * tid + 2u)" in case and "r7 =" not in case
    loads = [l for l in src.splitlines() if "p.regs_in[" in l]
    stores = [l for l in src.splitlines() if "p.regs_out[" in l and "rc_k1c_fix" not in l]
    assert loads and all("(u64)7 *" in l for l in loads)
    assert any("(u64)7 *" in l for l in stores)
    # the fix kernel writes exactly the rematerialised ones for K1
    fix = src[src.index("rc_k1c_fix"):]
    assert "(u64)0 * p.reg_stride" in fix and "(u64)3 * p.reg_stride" in fix and "(u64)7 * p.reg_stride" not in fix


def test_k1c_no_aligned_barrier_after_body(rc):
    """After the goto-structured body a warp's lanes need not have
    reconverged: the generated kernel has no block barrier past its start."""
    for src_text in (K.STENCIL, K.TREE):
        prog = rc.rc_load_program(K.program(src_text).bytecode)
        src = prog.jit_source(1024, [1100] * prog.n_arrays, wbucket=True)
        body = src[src.index("switch (pc)"):src.index("rc_k1c_fix")]
        assert "__syncthreads" not in body
