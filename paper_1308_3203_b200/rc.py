"""Thin Python binding of librc.so (include/rc.h): argument marshalling only.

Every step of the race-checking path runs in the CUDA kernels behind
rc_run; this module converts Python / torch arguments into the C ABI's plain
pointers and sizes and the results back.  There is no fallback: if librc.so
is missing or no CUDA device is present, rc_run raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librc.so")

RC_OK, RC_EINVAL, RC_ENOMEM, RC_ECUDA, RC_ETRUNC, RC_ELIMIT = range(6)
STATUS_NAMES = {0: "RC_OK", 1: "RC_EINVAL", 2: "RC_ENOMEM", 3: "RC_ECUDA", 4: "RC_ETRUNC", 5: "RC_ELIMIT"}
KINDS = {1: "RW", 2: "WW_BENIGN", 3: "WW_NONBENIGN", 4: "OOB", 5: "ASSERT", 6: "DIV0", 7: "FUEL",
         8: "BARRIER_DIVERGENCE", 9: "IG_RW", 10: "IG_WW_BENIGN", 11: "IG_WW_NONBENIGN"}
RC_OPT_HOST_IO = 1
RC_OPT_KEEP_ALL_READS = 2
RC_OPT_CLASSIFY_RW = 4
RC_OPT_PREPASS = 8
PROF_CLASSES = ["interp", "hist", "sort", "detect", "boundary", "finalize", "copy", "filter"]

REPORT_DTYPE = np.dtype([("instance", "<u4"), ("interval", "<u4"), ("array", "<i4"), ("index", "<i4"),
                         ("tid1", "<u4"), ("tid2", "<u4"), ("kind", "<u2"), ("flags", "<u2"),
                         ("reserved", "<u4")])


class rc_report(C.Structure):
    _fields_ = [("instance", C.c_uint32), ("interval", C.c_uint32), ("array", C.c_int32), ("index", C.c_int32),
                ("tid1", C.c_uint32), ("tid2", C.c_uint32), ("kind", C.c_uint16), ("flags", C.c_uint16),
                ("reserved", C.c_uint32)]


class rc_stats(C.Structure):
    _fields_ = [("checked_accesses", C.c_uint64), ("loads", C.c_uint64), ("stores", C.c_uint64),
                ("instructions", C.c_uint64), ("intervals_max", C.c_uint64), ("lanes_final", C.c_uint64 * 8)]


class rc_profile(C.Structure):
    _fields_ = [("launches", C.c_uint64 * 8), ("ms", C.c_double * 8), ("alg_bytes", C.c_uint64 * 8),
                ("items", C.c_uint64 * 8), ("total_ms", C.c_double), ("kernel_launches", C.c_uint64),
                ("sample_every", C.c_uint32), ("flags", C.c_uint32)]


class rc_array(C.Structure):
    _fields_ = [("data", C.c_void_p), ("size", C.c_uint32)]


class rc_options(C.Structure):
    _fields_ = [("instance_offset", C.c_uint32), ("max_intervals", C.c_uint32), ("fuel_per_interval", C.c_uint64),
                ("device", C.c_int32), ("flags", C.c_uint32), ("cuda_stream", C.c_void_p),
                ("max_batch_instances", C.c_uint32), ("n_groups", C.c_uint32),
                ("profile", C.POINTER(rc_profile))]


assert C.sizeof(rc_report) == 32

class rc_explore_result(C.Structure):
    _fields_ = [("n_schedules", C.c_uint64), ("n_differ", C.c_uint64), ("witness", C.c_uint64),
                ("max_product", C.c_uint64), ("n_terminal", C.c_uint64), ("witness_len", C.c_uint32),
                ("complete", C.c_uint32)]


RC_EXPLORE_REDUCED = 1


class rc_prove_result(C.Structure):
    _fields_ = [("verdict", C.c_uint32), ("reason", C.c_uint32), ("pc", C.c_uint32), ("intervals", C.c_uint32),
                ("terms", C.c_uint64), ("work", C.c_uint64)]


PROVE_VERDICTS = {0: "UNKNOWN", 1: "NO_CONFLICT", 2: "NORACE"}
PROVE_REASONS = {0: None, 1: "RW", 2: "WW", 3: "OOB", 4: "DATA_INDEX", 5: "ASSERT", 6: "DIV0", 7: "DIVERGENCE",
                 8: "OWN_ALIAS", 9: "FUEL", 10: "BUDGET", 11: "UNSUPPORTED"}
_lib = None


class RCError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


def lib():
    """Load librc.so (raises if it was not built: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        L.rc_load_program.argtypes = [C.c_void_p, C.c_size_t, P(C.c_void_p)]
        L.rc_load_program.restype = C.c_int
        L.rc_free_program.argtypes = [C.c_void_p]
        L.rc_free_program.restype = None
        L.rc_program_info.argtypes = [C.c_void_p, P(C.c_uint32), P(C.c_uint32), P(C.c_uint32)]
        L.rc_program_info.restype = C.c_int
        L.rc_run.argtypes = [C.c_void_p, C.c_uint32, P(rc_array), C.c_uint32, C.c_uint32, P(rc_options),
                             P(rc_report), C.c_uint64, P(C.c_uint64), P(rc_stats), P(C.c_void_p)]
        L.rc_run.restype = C.c_int
        L.rc_last_error.argtypes = []
        L.rc_last_error.restype = C.c_char_p
        L.rc_abi_version.restype = C.c_int
        L.rc_release_workspace.argtypes = [C.c_void_p]
        L.rc_release_workspace.restype = C.c_int
        L.rc_explore.argtypes = [C.c_void_p, C.c_uint32, P(C.c_uint32), C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, C.c_void_p,
                                 C.c_uint64, C.c_void_p, C.c_uint32, C.c_void_p, P(rc_explore_result)]
        L.rc_explore.restype = C.c_int
        L.rc_prove.argtypes = [C.c_void_p, C.c_uint32, P(C.c_uint32), C.c_uint32, C.c_uint64, C.c_uint64,
                               P(rc_prove_result)]
        L.rc_prove.restype = C.c_int
        # test hooks (jit.cpp; not part of include/rc.h)
        L.rc_debug_jit_kernels.argtypes = [C.c_void_p]
        L.rc_debug_jit_kernels.restype = C.c_int
        L.rc_debug_jit_source.argtypes = [C.c_void_p, C.c_uint32, P(C.c_uint32), C.c_uint32, C.c_uint32,
                                          C.c_char_p, C.c_size_t]
        L.rc_debug_jit_source.restype = C.c_size_t
        _lib = L
    return _lib


def rc_last_error() -> str:
    return lib().rc_last_error().decode()


class Program:
    """An rc_program loaded from RCB1 bytecode (library-owned)."""

    def __init__(self, handle: int, bytecode: bytes):
        self._h = C.c_void_p(handle)
        self.bytecode = bytecode
        nr, na, ni = C.c_uint32(), C.c_uint32(), C.c_uint32()
        lib().rc_program_info(self._h, C.byref(nr), C.byref(na), C.byref(ni))
        self.n_regs, self.n_arrays, self.n_instr = nr.value, na.value, ni.value

    def release_workspace(self):
        lib().rc_release_workspace(self._h)

    def jit_kernels(self) -> int:
        """Test hook: K1c kernels compiled for this program so far (jit.cpp)."""
        return int(lib().rc_debug_jit_kernels(self._h))

    def jit_source(self, work_group_size: int, sizes: list, *, direct=False, fuel=False, ro_skip=True,
                   wbucket=False, narrow=False) -> str:
        """Test hook: the K1c CUDA source for this program and shape (no GPU needed)."""
        arr = (C.c_uint32 * max(1, len(sizes)))(*sizes)
        flags = (1 if direct else 0) | (2 if fuel else 0) | (4 if ro_skip else 0) | (8 if wbucket else 0) | (16 if narrow else 0)
        f = lib().rc_debug_jit_source
        nb = f(self._h, work_group_size, arr, len(sizes), flags, None, 0)
        buf = C.create_string_buffer(nb + 1)
        f(self._h, work_group_size, arr, len(sizes), flags, buf, nb + 1)
        return buf.value.decode()

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value and _lib is not None:
            _lib.rc_free_program(self._h)
            self._h = C.c_void_p(0)


def rc_load_program(bytecode: bytes) -> Program:
    h = C.c_void_p()
    buf = C.create_string_buffer(bytes(bytecode), len(bytecode))
    st = lib().rc_load_program(buf, len(bytecode), C.byref(h))
    if st != RC_OK:
        raise RCError(st, rc_last_error())
    return Program(h.value, bytes(bytecode))


@dataclass
class RunResult:
    reports: np.ndarray                 # REPORT_DTYPE, canonical order
    n_reports_total: int
    stats: dict
    final: list = field(default_factory=list)   # per array [n_instances, size] (torch or numpy)
    profile: dict | None = None

    def report_tuples(self):
        return [tuple(int(r[f]) for f in ("instance", "interval", "array", "index", "kind", "tid1", "tid2", "flags"))
                for r in self.reports]


def _stats_dict(s: rc_stats) -> dict:
    return {"checked_accesses": s.checked_accesses, "loads": s.loads, "stores": s.stores,
            "instructions": s.instructions, "intervals_max": s.intervals_max,
            "lanes_final": [int(x) for x in s.lanes_final]}


def _profile_dict(p: rc_profile) -> dict:
    return {"total_ms": p.total_ms, "kernel_launches": int(p.kernel_launches), "sample_every": int(p.sample_every),
            "k1c": bool(p.flags & 1),
            **{c: {"launches": int(p.launches[i]), "ms": float(p.ms[i]), "alg_bytes": int(p.alg_bytes[i]),
                   "items": int(p.items[i])} for i, c in enumerate(PROF_CLASSES)}}


def rc_run(prog: Program, work_group_size: int, arrays: list, *, n_instances: int | None = None,
           instance_offset: int = 0, fuel_per_interval: int = 0, max_intervals: int = 0, device: int | None = None,
           stream=None, capacity: int = 1 << 20, want_final: bool = True, final_out: list | None = None,
           profile: bool = False, max_batch_instances: int = 0, allow_truncate: bool = False,
           keep_all_reads: bool = False, classify_rw: bool = False, n_groups: int = 1,
           prepass: bool = False) -> RunResult:
    """Run `prog` on the arrays (n_groups work-groups of work_group_size
    work-items per instance, include/rc.h rc_options.n_groups).

    arrays: per shared array either a CUDA int32 torch tensor [n_instances, size]
    (device path), or a host numpy / CPU torch int32 array (RC_OPT_HOST_IO: the
    library copies host<->device itself).  Mixed residency is rejected.
    """
    import torch  # plumbing only: device memory and streams

    if len(arrays) != prog.n_arrays:
        raise ValueError(f"program has {prog.n_arrays} arrays, got {len(arrays)}")
    on_dev = [isinstance(a, torch.Tensor) and a.is_cuda for a in arrays]
    host_io = not all(on_dev) if arrays else False
    if arrays and any(on_dev) and not all(on_dev):
        raise ValueError("arrays must be all on the GPU or all on the host")
    keep = []
    arr = (rc_array * max(1, len(arrays)))()
    if n_instances is None:
        n_instances = int(arrays[0].shape[0]) if arrays else 1
    for i, a in enumerate(arrays):
        if host_io:
            a = a.numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
            if a.dtype != np.int32:  # as on the device path: no silent wrap or truncation
                raise TypeError(f"array {i}: arrays must be int32, got {a.dtype}")
            a = np.ascontiguousarray(a)
            if a.ndim == 1:
                a = a[None, :]
            keep.append(a)
            arr[i].data = a.ctypes.data
            arr[i].size = a.shape[1]
        else:
            if a.dtype != torch.int32:
                raise TypeError("arrays must be int32")
            a = a.contiguous()
            if a.dim() == 1:
                a = a[None, :]
            keep.append(a)
            arr[i].data = a.data_ptr()
            arr[i].size = a.shape[1]
        if a.shape[0] != n_instances:
            raise ValueError(f"array {i}: {a.shape[0]} instances, expected {n_instances}")
    if device is None:
        device = keep[0].device.index if (keep and not host_io) else (torch.cuda.current_device() if torch.cuda.is_available() else 0)
    if stream is None and torch.cuda.is_available():
        stream = torch.cuda.current_stream(device)
    opt = rc_options()
    opt.instance_offset = instance_offset
    opt.max_intervals = max_intervals
    opt.fuel_per_interval = fuel_per_interval
    opt.device = device
    opt.flags = (RC_OPT_HOST_IO if host_io else 0) | (RC_OPT_KEEP_ALL_READS if keep_all_reads else 0) | \
        (RC_OPT_CLASSIFY_RW if classify_rw else 0) | (RC_OPT_PREPASS if prepass else 0)
    opt.cuda_stream = C.c_void_p(stream.cuda_stream if stream is not None else 0)
    opt.max_batch_instances = max_batch_instances
    opt.n_groups = n_groups
    prof = rc_profile()
    if profile:
        opt.profile = C.pointer(prof)
    # final heaps
    fin_ptrs = None
    finals = []
    if want_final and arrays:
        if final_out is not None:
            finals = final_out
        elif host_io:
            finals = [np.empty_like(a) for a in keep]
        else:
            finals = [torch.empty_like(a) for a in keep]
        fin_ptrs = (C.c_void_p * len(arrays))(*[(f.ctypes.data if isinstance(f, np.ndarray) else f.data_ptr())
                                                 for f in finals])
    # report buffer: uninitialised (the library writes the first min(capacity,
    # total) records; zero-filling a large ctypes array costs milliseconds)
    out = np.empty(max(1, capacity), dtype=REPORT_DTYPE)
    total = C.c_uint64()
    st = rc_stats()
    code = lib().rc_run(prog._h, work_group_size, arr, len(arrays), n_instances, C.byref(opt),
                        out.ctypes.data_as(C.POINTER(rc_report)), capacity, C.byref(total), C.byref(st), fin_ptrs)
    if code not in (RC_OK, RC_ETRUNC) or (code == RC_ETRUNC and not allow_truncate):
        raise RCError(code, rc_last_error())
    n = min(total.value, capacity)
    reps = out[:n].copy()
    return RunResult(reps, int(total.value), _stats_dict(st), finals, _profile_dict(prof) if profile else None)


@dataclass
class ExploreResult:
    n_schedules: int
    n_differ: int
    witness: int | None          # schedule index whose end heap differs from schedule 0's
    witness_sched: list          # its choices (tids), up to max_len
    max_product: int
    complete: bool
    terminals: object            # CUDA int32 tensor [n_terminal, row_words] or None


def rc_explore(prog: Program, work_group_size: int, heap, *, regs=None, pc=None, status=None, sizes=None,
               fuel: int = 0, index_end: int = 1 << 20, index_begin: int = 0, reduced: bool = True,
               cap: int = 0, max_len: int = 256, stream=None) -> ExploreResult:
    """Every interleaving of one barrier interval (include/rc.h rc_explore).

    heap: CUDA int32 tensor of all arrays concatenated; `sizes` their element
    counts (default: one array holding the whole heap when the program has
    one).  regs [n, n_regs] / pc [n] / status [n] CUDA tensors (default:
    zeros = the kernel's start state, reading L18).
    """
    import torch  # plumbing only: device memory and streams

    n = work_group_size
    dev = heap.device
    if sizes is None:
        if prog.n_arrays != 1:
            raise ValueError("sizes is required for programs with more than one array")
        sizes = [heap.numel()]
    sz = (C.c_uint32 * max(1, len(sizes)))(*sizes)
    heap = heap.to(torch.int32).contiguous()
    regs = torch.zeros((n, prog.n_regs), dtype=torch.int32, device=dev) if regs is None else regs.to(torch.int32).contiguous()
    pc = torch.zeros(n, dtype=torch.int32, device=dev) if pc is None else pc.to(torch.int32).contiguous()
    status = torch.zeros(n, dtype=torch.uint8, device=dev) if status is None else status.to(torch.uint8).contiguous()
    row_words = int(sum(sizes)) + n * (4 + prog.n_regs)
    terms = torch.empty((max(1, cap), row_words), dtype=torch.int32, device=dev)
    wsched = torch.empty(max(1, max_len), dtype=torch.int32, device=dev)
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    out = rc_explore_result()
    with torch.cuda.device(dev):  # the C side launches on the current device (the tensors' GPU)
        code = lib().rc_explore(prog._h, n, sz, heap.data_ptr(), regs.data_ptr(), pc.data_ptr(), status.data_ptr(),
                                fuel, index_begin, index_end, RC_EXPLORE_REDUCED if reduced else 0, terms.data_ptr(),
                                cap, wsched.data_ptr(), max_len, C.c_void_p(stream.cuda_stream), C.byref(out))
    if code != RC_OK:
        raise RCError(code, rc_last_error())
    wl = min(out.witness_len, max_len)
    return ExploreResult(int(out.n_schedules), int(out.n_differ),
                         None if out.witness == (1 << 64) - 1 else int(out.witness),
                         wsched[:wl].cpu().tolist() if out.witness != (1 << 64) - 1 else [],
                         int(out.max_product), bool(out.complete), terms[:out.n_terminal] if cap else None)


@dataclass
class ProveResult:
    verdict: str          # "NO_CONFLICT" | "NORACE" | "UNKNOWN"
    reason: str | None    # why UNKNOWN (RC_PROVE_R_*)
    pc: int
    intervals: int
    terms: int
    work: int


def rc_prove(prog: Program, work_group_size: int, sizes: list, *, fuel_per_interval: int = 0,
             budget: int = 0) -> ProveResult:
    """The symbolic NoRace pre-pass (include/rc.h rc_prove): host only."""
    sz = (C.c_uint32 * max(1, len(sizes)))(*[int(x) for x in sizes])
    out = rc_prove_result()
    code = lib().rc_prove(prog._h, work_group_size, sz, len(sizes), fuel_per_interval, budget, C.byref(out))
    if code != RC_OK:
        raise RCError(code, rc_last_error())
    return ProveResult(PROVE_VERDICTS[out.verdict], PROVE_REASONS.get(out.reason, str(out.reason)), int(out.pc),
                       int(out.intervals), int(out.terms), int(out.work))
