"""ctypes front-end of the C oracle (TEST INFRASTRUCTURE ONLY).

Argument marshalling only; every step of the oracle's arithmetic is in
oracle.c.  Builds liboracle.so with gcc on first use if it is missing.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

# report record, same field order as DESIGN.md §2 (own definition)
REPORT_DTYPE = np.dtype([("instance", "<u4"), ("interval", "<u4"), ("array", "<i4"), ("index", "<i4"),
                         ("tid1", "<u4"), ("tid2", "<u4"), ("kind", "<u2"), ("flags", "<u2"),
                         ("reserved", "<u4")])
IG_INTERVAL = 0xFFFFFFFF  # interval field of the inter-group reports (kinds 9-11, reading L20)
STATUS = {"RUNNING": 0, "WAITING": 1, "EXITED": 2, "PRUNED": 3, "OOB": 4, "ASSERT": 5, "DIV0": 6, "FUEL": 7}
STAT_NAMES = ["checked_accesses", "loads", "stores", "instructions", "intervals_max"] + \
    [f"lanes_final{i}" for i in range(8)]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-Wall", "-shared", "-fPIC", "-o", _LIB, _SRC,
                               "-lpthread"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(_LIB)
        P = C.POINTER
        lib.oracle_run.argtypes = [C.c_char_p, C.c_size_t, C.c_uint32, P(C.c_uint32), P(P(C.c_int32)),
                                   C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_int,
                                   P(C.c_void_p), P(C.c_uint64), P(P(C.c_int32)), P(C.c_uint64), C.c_int,
                                   C.c_uint32]
        lib.oracle_run.restype = C.c_int
        lib.oracle_free.argtypes = [C.c_void_p]
        lib.oracle_state_at.argtypes = [C.c_char_p, C.c_size_t, C.c_uint32, P(C.c_uint32), P(P(C.c_int32)),
                                        C.c_uint64, C.c_uint32, P(C.c_int32), P(C.c_int32), P(C.c_uint32),
                                        P(C.c_uint8)]
        lib.oracle_state_at.restype = C.c_int
        lib.oracle_enumerate.argtypes = [C.c_char_p, C.c_size_t, C.c_uint32, P(C.c_uint32), P(C.c_int32),
                                         P(C.c_int32), P(C.c_uint32), P(C.c_uint8), C.c_uint64, C.c_int,
                                         C.c_uint64, P(C.c_uint64), P(C.c_void_p), P(C.c_uint64),
                                         P(C.c_uint64)]
        lib.oracle_enumerate.restype = C.c_int
        _lib = lib
    return _lib


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t))


def _header(bytecode: bytes) -> tuple[int, int]:
    n_regs = int.from_bytes(bytecode[8:10], "little")
    n_arrays = int.from_bytes(bytecode[10:12], "little")
    return n_regs, n_arrays


@dataclass
class Result:
    reports: np.ndarray          # structured REPORT_DTYPE, canonical order
    final: list[np.ndarray]      # per array [n_instances, size]
    stats: dict

    def report_tuples(self):
        return [tuple(int(r[f]) for f in ("instance", "interval", "array", "index", "kind", "tid1", "tid2", "flags"))
                for r in self.reports]


DEFAULT_FUEL = 1 << 20
DEFAULT_MAX_INTERVALS = 65536


def run(bytecode: bytes, n: int, inputs: list[np.ndarray], *, instance_offset: int = 0,
        fuel: int = DEFAULT_FUEL, max_intervals: int = DEFAULT_MAX_INTERVALS, threads: int | None = None,
        want_final: bool = True, classify_rw: bool = False, n_groups: int = 1) -> Result:
    """Run the canonical algorithm.  inputs[a] has shape [n_instances, size(a)].
    classify_rw: RW value classification flags (bit 4 / bit 5) on the RW reports.
    n_groups: work-groups per instance, each of n work-items (reading L20)."""
    lib = _load()
    _, n_arrays = _header(bytecode)
    assert len(inputs) == n_arrays, (len(inputs), n_arrays)
    ins = [np.ascontiguousarray(x, dtype=np.int32) for x in inputs]
    n_inst = ins[0].shape[0] if ins else 0
    sizes = np.array([x.shape[1] for x in ins] or [0], dtype=np.uint32)
    in_ptrs = (C.POINTER(C.c_int32) * max(n_arrays, 1))(*[_ptr(x, C.c_int32) for x in ins])
    finals = [np.zeros_like(x) for x in ins] if want_final else []
    fin_ptrs = (C.POINTER(C.c_int32) * max(n_arrays, 1))(*[_ptr(x, C.c_int32) for x in finals]) if want_final else None
    rep_p = C.c_void_p()
    n_rep = C.c_uint64()
    stats = np.zeros(13 + 32, dtype=np.uint64)
    if threads is None:
        threads = max(1, min(len(os.sched_getaffinity(0)), n_inst))
    rc = lib.oracle_run(bytecode, len(bytecode), n, _ptr(sizes, C.c_uint32), in_ptrs, n_inst, instance_offset,
                        fuel, max_intervals, threads, C.byref(rep_p), C.byref(n_rep), fin_ptrs,
                        _ptr(stats, C.c_uint64), 1 if classify_rw else 0, n_groups)
    if rc != 0:
        raise ValueError("oracle: bytecode decode failed")
    nr = n_rep.value
    if nr:
        buf = (C.c_char * (nr * 32)).from_address(rep_p.value)
        reps = np.frombuffer(bytes(buf), dtype=REPORT_DTYPE).copy()
    else:
        reps = np.zeros(0, dtype=REPORT_DTYPE)
    lib.oracle_free(rep_p)
    st = dict(zip(STAT_NAMES, (int(x) for x in stats)))
    st["lanes_final"] = [int(x) for x in stats[5:13]]
    st["op_counts"] = [int(x) for x in stats[13:45]]  # executed instructions per opcode (coverage)
    return Result(reps, finals, st)


def state_at(bytecode: bytes, n: int, inputs: list[np.ndarray], k: int, fuel: int = DEFAULT_FUEL):
    """Canonical state at the start of interval k of one instance.
    Returns (reached, heap(concatenated), regs[n, n_regs], pc[n], status[n])."""
    lib = _load()
    n_regs, n_arrays = _header(bytecode)
    ins = [np.ascontiguousarray(x.reshape(-1), dtype=np.int32) for x in inputs]
    sizes = np.array([x.shape[0] for x in ins] or [0], dtype=np.uint32)
    in_ptrs = (C.POINTER(C.c_int32) * max(n_arrays, 1))(*[_ptr(x, C.c_int32) for x in ins])
    heap = np.zeros(max(int(sizes[:n_arrays].sum()), 1), dtype=np.int32)
    regs = np.zeros((max(n, 1), n_regs), dtype=np.int32)
    pc = np.zeros(max(n, 1), dtype=np.uint32)
    status = np.zeros(max(n, 1), dtype=np.uint8)
    r = lib.oracle_state_at(bytecode, len(bytecode), n, _ptr(sizes, C.c_uint32), in_ptrs, fuel, k,
                            _ptr(heap, C.c_int32), _ptr(regs, C.c_int32), _ptr(pc, C.c_uint32),
                            _ptr(status, C.c_uint8))
    if r < 0:
        raise ValueError("oracle: bytecode decode failed")
    cells = int(sizes[:n_arrays].sum())
    return bool(r), heap[:cells], regs[:n], pc[:n], status[:n]


@dataclass
class Enumeration:
    n_schedules: int
    heaps: list[tuple]           # distinct terminal heaps (concatenated arrays)
    lanes: list[tuple]           # distinct terminal (heap, lane-state) rows
    complete: bool


def enumerate_interval(bytecode: bytes, n: int, sizes: list[int], heap: np.ndarray, regs: np.ndarray,
                       pc: np.ndarray, status: np.ndarray, *, fuel: int = DEFAULT_FUEL, memo: bool = True,
                       budget: int = 5_000_000, reduced: bool = False) -> Enumeration:
    """All interleavings of one barrier interval from the given state under the
    paper's immediate-visibility global semantics.
    reduced: only LD / ST are scheduling points (private steps commute with
    every other thread's steps): the same terminal states, fewer schedules."""
    lib = _load()
    n_regs, _ = _header(bytecode)
    sz = np.array(sizes or [0], dtype=np.uint32)
    heap = np.ascontiguousarray(heap, dtype=np.int32)
    regs = np.ascontiguousarray(regs, dtype=np.int32).reshape(-1)
    pc = np.ascontiguousarray(pc, dtype=np.uint32)
    status = np.ascontiguousarray(status, dtype=np.uint8)
    nsch = C.c_uint64(); terms = C.c_void_p(); nterm = C.c_uint64(); roww = C.c_uint64()
    rc = lib.oracle_enumerate(bytecode, len(bytecode), n, _ptr(sz, C.c_uint32), _ptr(heap, C.c_int32),
                              _ptr(regs, C.c_int32), _ptr(pc, C.c_uint32), _ptr(status, C.c_uint8), fuel,
                              (1 if memo else 0) | (2 if reduced else 0), budget, C.byref(nsch), C.byref(terms), C.byref(nterm),
                              C.byref(roww))
    if rc < 0:
        raise ValueError("oracle: bytecode decode failed")
    rows = []
    if nterm.value:
        buf = (C.c_int32 * (nterm.value * roww.value)).from_address(terms.value)
        arr = np.frombuffer(buf, dtype=np.int32).reshape(nterm.value, roww.value).copy()
        rows = [tuple(int(x) for x in row) for row in arr]
    lib.oracle_free(terms)
    cells = int(sum(sizes))
    heaps = sorted(set(r[:cells] for r in rows))
    return Enumeration(int(nsch.value), heaps, sorted(rows), rc == 0)
