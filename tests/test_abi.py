"""C ABI checks that need no GPU: librc.so loads, exports every symbol that
include/rc.h declares, and rc_load_program validates bytecode (host only)."""
import ctypes
import os
import re
import struct

import pytest

from workloads import kernels as K
from workloads.asm import OPCODES, assemble, encode

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rc():
    from paper_1308_3203_b200 import _build
    _build.build()
    import paper_1308_3203_b200 as pkg
    return pkg


def header_symbols():
    src = open(os.path.join(ROOT, "include", "rc.h")).read()
    return sorted(set(re.findall(r"RC_API\s+[\w\s\*]+?\b(rc_\w+)\s*\(", src)))


def test_exports_every_header_symbol(rc):
    syms = header_symbols()
    assert len(syms) >= 7
    L = ctypes.CDLL(rc.rc.LIB_PATH)
    for s in syms:
        assert hasattr(L, s), f"librc.so does not export {s}"
    assert rc.lib().rc_abi_version() == 1


def test_struct_sizes_match_header(rc):
    from paper_1308_3203_b200 import rc as b
    assert ctypes.sizeof(b.rc_report) == 32
    assert ctypes.sizeof(b.rc_stats) == 13 * 8
    assert ctypes.sizeof(b.rc_array) == 16


def test_opcodes_match_header():
    src = open(os.path.join(ROOT, "include", "rc.h")).read()
    hdr = {m.group(1).lower(): int(m.group(2)) for m in re.finditer(r"RC_OP_(\w+)\s*=\s*(\d+)", src)}
    assert hdr == OPCODES


@pytest.mark.parametrize("src", [K.FIG1, K.FIG1_GUARDED, K.FIG2, K.TREE, K.TREE_OFF_BY_ONE, K.STENCIL]
                         + list(K.BENIGN.values()))
def test_valid_programs_load(rc, src):
    p = assemble(src)
    prog = rc.rc_load_program(p.bytecode)
    assert (prog.n_regs, prog.n_arrays, prog.n_instr) == (p.n_regs, len(p.arrays), p.n_instr)


def test_random_stencil_kernels_load(rc):
    for seed in range(8):
        rc.rc_load_program(K.random_stencil_kernel(seed).bytecode)


EXIT = (26, 0, 0, 0, 0)


@pytest.mark.parametrize("blob,msg", [
    (b"", "shorter"),
    (encode(1, 0, [EXIT], magic=0x12345678), "magic"),
    (encode(1, 0, [EXIT], version=2), "version"),
    (encode(1, 0, [EXIT], flags=1), "flags"),
    (encode(0, 0, [EXIT]), "n_regs"),
    (encode(1, 300, [EXIT]), "n_arrays"),
    (encode(1, 0, []), "n_instr"),
    (encode(1, 0, [EXIT])[:-1], "size mismatch"),
    (encode(1, 0, [(99, 0, 0, 0, 0), EXIT]), "unknown opcode"),
    (encode(2, 0, [(5, 0, 1, 2, 0), EXIT]), "register r2"),
    (encode(2, 1, [(19, 0, 1, 0, 0), EXIT]), "array 1"),
    (encode(2, 1, [(20, 3, 0, 0, 0), EXIT]), "array 3"),
    (encode(1, 0, [(25, 0, 0, 0, 7), EXIT]), "target 7"),
    (encode(1, 0, [(24, 0, 0, 0, 9), EXIT]), "true target 9"),
    (encode(1, 0, [(24, 0, 5, 0, 0), EXIT]), "false target 5"),
    (encode(1, 0, [(1, 0, 0, 0, 3)]), "falls off the end"),
    (encode(1, 0, [(25, 0, 0, 0, 0), EXIT]), "no EXIT"),
])
def test_validator_rejects(rc, blob, msg):
    with pytest.raises(rc.RCError) as ei:
        rc.rc_load_program(blob)
    assert ei.value.code == 1  # RC_EINVAL
    assert msg in str(ei.value)


def test_unreachable_fallthrough_is_fine(rc):
    # the dead CONST at the end is never executed
    rc.rc_load_program(encode(1, 0, [EXIT, (1, 0, 0, 0, 3)]))


def test_run_without_gpu_fails_loudly(rc):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    prog = rc.rc_load_program(assemble(".arrays A\n exit").bytecode)
    import numpy as np
    with pytest.raises(rc.RCError) as ei:
        rc.rc_run(prog, 4, [np.zeros((1, 4), np.int32)])
    assert ei.value.code in (3, 1)  # RC_ECUDA (no device)


def test_explore_result_layout(rc):
    from paper_1308_3203_b200 import rc as b
    assert ctypes.sizeof(b.rc_explore_result) == 6 * 8
    src = open(os.path.join(ROOT, "include", "rc.h")).read()
    assert re.search(r"#define RC_EXPLORE_REDUCED 1u", src) and b.RC_EXPLORE_REDUCED == 1


def test_explore_argument_errors_without_gpu(rc):
    """rc_explore validates its arguments before any CUDA call: each bad
    argument gives RC_EINVAL / RC_ELIMIT with a message (include/rc.h)."""
    from paper_1308_3203_b200 import rc as b
    L = rc.lib()
    p = rc.rc_load_program(assemble(K.BENIGN["K_inc"]).bytecode)  # 2 arrays
    sizes = (ctypes.c_uint32 * 2)(1, 4)
    buf = (ctypes.c_int32 * 4096)()
    ptr = ctypes.cast(buf, ctypes.c_void_p)
    out = b.rc_explore_result()

    def call(prog=p._h, n=4, sz=sizes, heap=ptr, regs=ptr, pc=ptr, st=ptr, begin=0, end=16, flags=1,
             term=None, cap=0, ws=None, max_len=0):
        return L.rc_explore(prog, n, sz, heap, regs, pc, st, 0, begin, end, flags, term, cap, ws, max_len, None,
                            ctypes.byref(out))

    EINVAL, ELIMIT = 1, 5
    assert call(prog=None) == EINVAL
    assert call(n=0) == EINVAL and "work_group_size" in rc.rc_last_error()
    assert call(n=33) == EINVAL
    assert call(sz=None) == EINVAL and "sizes" in rc.rc_last_error()
    assert call(pc=None) == EINVAL and "lane state" in rc.rc_last_error()
    assert call(begin=5, end=4) == EINVAL
    assert call(flags=2) == EINVAL and "flags" in rc.rc_last_error()
    assert call(cap=8) == EINVAL and "terminals" in rc.rc_last_error()
    assert call(max_len=8) == EINVAL and "witness_sched" in rc.rc_last_error()
    big = (ctypes.c_uint32 * 2)(4000, 100)
    assert call(sz=big) == ELIMIT and "state row" in rc.rc_last_error()
    assert out.n_schedules == 0 and out.complete == 0  # `out` is cleared on every call


def test_host_arrays_must_be_int32(rc):
    """The host-buffer path rejects non-int32 arrays exactly like the device
    path (no silent wrap of int64 or truncation of floats); the check runs
    before any CUDA call."""
    import numpy as np
    prog = rc.rc_load_program(assemble(K.BENIGN["K_c"]).bytecode)
    for bad in (np.zeros((2, 1), np.int64), np.zeros((2, 1), np.float32)):
        with pytest.raises(TypeError):
            rc.rc_run(prog, 4, [bad, np.zeros((2, 4), np.int32)])
