"""Pins of the CPU oracle against what the paper and mathematics fix.

Each test names the passage it follows.  Expected values are the paper's
worked examples (tests/golden/*.json, hand-derived in SURVEY.md App. A),
closed forms (sums, numpy recurrences) or textbook arithmetic — never the
oracle's own output and never the CUDA path.
"""
import json
import os

import numpy as np
import pytest

from workloads import inputs as I
from workloads import kernels as K
from workloads.asm import assemble

GOLD = os.path.join(os.path.dirname(__file__), "golden")
KIND = {"RW": 1, "WW_BENIGN": 2, "WW_NONBENIGN": 3, "OOB": 4, "ASSERT": 5, "DIV0": 6, "FUEL": 7,
        "BARRIER_DIVERGENCE": 8}
NOTID = 0xFFFFFFFF


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def exp_tuple(r, arrays, instance=0):
    arr = arrays.index(r["array"]) if isinstance(r["array"], str) else r["array"]
    return (instance, r["interval"], arr, r["index"], KIND[r["kind"]], r["tid1"], r.get("tid2", NOTID),
            r.get("flags", 0))


# --------------------------------------------------------------- Figure 1
def test_fig1_verbatim(oracle_lib):
    """PAPER.md:62-74; App. A.1: 2 OOB in interval 0, RW on R[2..6] in interval 1."""
    g = gold("fig1.json")
    p = K.program(K.FIG1)
    r = oracle_lib.run(p.bytecode, 8, I.cfg1_inputs())
    assert r.report_tuples() == [exp_tuple(x, p.arrays) for x in g["reports_verbatim"]]
    assert r.final[2][0].tolist() == g["final_R"]
    assert r.final[0][0].tolist() == g["inputs"]["A"] and r.final[1][0].tolist() == g["inputs"]["B"]
    assert r.stats["checked_accesses"] == g["checked_accesses_verbatim"]
    assert r.stats["loads"] == g["loads_verbatim"] and r.stats["stores"] == g["stores_verbatim"]
    assert r.stats["intervals_max"] == 2
    assert r.stats["lanes_final"][:3] == [6, 0, 2]  # 6 exited, 2 halted by OOB


def test_fig1_interval0_heap(oracle_lib):
    """App. A.1: after interval 0, R[t] = 11t+20 for t=1..6 (A[t-1]+B[t+1])."""
    g = gold("fig1.json")
    p = K.program(K.FIG1)
    ins = [x[0] for x in I.cfg1_inputs()]
    reached, heap, regs, pc, st = oracle_lib.state_at(p.bytecode, 8, ins, 1)
    assert reached
    assert heap[16:24].tolist() == g["after_interval0_R"]
    assert heap[16:24].tolist() == [100] + [11 * t + 20 for t in range(1, 7)] + [107]


def test_fig1_guarded(oracle_lib):
    """SPEC S:500/S:517 guarded variant: same 5 RW, no OOB, same final R."""
    g = gold("fig1.json")
    p = K.program(K.FIG1_GUARDED)
    r = oracle_lib.run(p.bytecode, 8, I.cfg1_inputs())
    exp = [exp_tuple(x, p.arrays) for x in g["reports_verbatim"] if x["kind"] == "RW"]
    assert r.report_tuples() == exp
    assert r.final[2][0].tolist() == g["final_R"]
    assert r.stats["checked_accesses"] == g["checked_accesses_guarded"]
    assert r.stats["lanes_final"][:2] == [6, 2]  # tids 0 and 7 pruned by assume


# --------------------------------------------------------------- Figure 2
@pytest.mark.parametrize("case", [0, 1])
def test_fig2(oracle_lib, case):
    """PAPER.md:453-468, App. A.2."""
    g = gold("fig2.json")
    c = g["cases"][case]
    p = K.program(K.FIG2)
    A = np.array([[7, 9, c["A2"]]], dtype=np.int32)
    G = np.array([[42]], dtype=np.int32)
    r = oracle_lib.run(p.bytecode, 2, [A, G])
    assert r.report_tuples() == [exp_tuple(x, p.arrays) for x in c["reports"]]
    assert r.final[0][0].tolist() == c["final_A"] and r.final[1][0].tolist() == c["final_G"]
    assert r.stats["intervals_max"] == 3  # two barriers + the implicit final one


def test_fig2_size2(oracle_lib):
    g = gold("fig2.json")["size2"]
    p = K.program(K.FIG2)
    r = oracle_lib.run(p.bytecode, 2, [np.array([[3, 4]], np.int32), np.array([[0]], np.int32)])
    got = [t for t in r.report_tuples() if t[1] == 1]
    exp = [exp_tuple(dict(x, interval=1), p.arrays) for x in g["reports_interval1"]]
    assert got == exp


# --------------------------------------------------------------- benign suite (config 2)
def _benign_expect(name, A0, B, n):
    """App. A.3 closed forms."""
    if name == "K_c":
        return [(0, 0, 0, 2, 0, 1, 0b1010)], 7
    if name == "K_tid":
        return [(0, 0, 0, 3, 0, 1, 0b1010)], n - 1
    if name == "K_B0":
        return [(0, 0, 0, 2, 0, 1, 0b1010)], int(B[0])
    if name == "K_Btid":
        diff = [t for t in range(n) if B[t] != B[0]]
        if diff:
            return [(0, 0, 0, 3, 0, diff[0], 0b1010)], int(B[n - 1])
        return [(0, 0, 0, 2, 0, 1, 0b1010)], int(B[n - 1])
    if name == "K_last":
        return [(0, 0, 0, 2, 0, 1, 0b1010)], 7
    if name == "K_inc":  # RW (kind 1) sorts before WW (kind 2) in one cell
        v = int(np.int32(np.int64(A0) + 1)) if A0 != 2**31 - 1 else -2**31
        return [(0, 0, 0, 1, 0, 1, 0xF), (0, 0, 0, 2, 0, 1, 0xF)], v
    raise KeyError(name)


@pytest.mark.parametrize("name", list(K.BENIGN))
def test_benign_suite(oracle_lib, name):
    """Config 2 at n=256 over 64 seeded instances (even: constant B, odd: bits)."""
    n = 256
    A, B = I.cfg2_inputs(0, 64, n)
    p = K.program(K.BENIGN[name])
    r = oracle_lib.run(p.bytecode, n, [A, B], threads=4)
    got = {}
    for t in r.report_tuples():
        got.setdefault(t[0], []).append(t[1:])
    for i in range(64):
        exp, final = _benign_expect(name, int(A[i, 0]), B[i], n)
        assert got.get(i, []) == exp, (name, i)
        assert int(r.final[0][i, 0]) == final
    per = {"K_c": 256, "K_tid": 256}.get(name, 512)
    assert r.stats["checked_accesses"] == per * 64


def test_spec_examples(oracle_lib):
    """A[0]:=5 by 2 threads -> only benign; A[0]:=tid -> non-benign."""
    p5 = assemble(".arrays A\n const r0, 0\n const r1, 5\n st A, r0, r1\n exit")
    r = oracle_lib.run(p5.bytecode, 2, [np.zeros((1, 1), np.int32)])
    assert [t[4] for t in r.report_tuples()] == [2]
    pt = K.program(K.BENIGN["K_tid"])
    r = oracle_lib.run(pt.bytecode, 2, [np.zeros((1, 1), np.int32), np.zeros((1, 1), np.int32)])
    assert [t[4] for t in r.report_tuples()] == [3]


def test_private_only_race_free(oracle_lib):
    """a kernel touching only private variables is race-free for all n."""
    p = K.program(K.PRIVATE_ONLY)
    for n in (1, 2, 7, 64):
        r = oracle_lib.run(p.bytecode, n, [np.zeros((1, 4), np.int32)])
        assert len(r.reports) == 0 and r.stats["checked_accesses"] == 0


def test_disjoint_writes_clean(oracle_lib):
    """A[tid] := tid has no report, final A[t] = t."""
    p = assemble(".arrays A\n tid r0\n st A, r0, r0\n exit")
    r = oracle_lib.run(p.bytecode, 100, [np.full((3, 100), -1, np.int32)])
    assert len(r.reports) == 0
    assert (r.final[0] == np.arange(100)).all()


# --------------------------------------------------------------- tree reduction (config 3)
def _tree_numpy(A, off_by_one):
    """App. A.4 recurrence: per interval with s = n/2, n/4, ..., 1 every live t
    (t < s, or t <= s) sets A[t] <- A[t] + A[t+s] from interval-start values
    (int32 wrap).  Off-by-one: tid n/2 faults in interval 0 (A[n] is OOB)."""
    A = A.astype(np.int64).copy()
    n = A.shape[0]
    s = n // 2
    while s > 0:
        hi = s + 1 if off_by_one else s
        t = np.arange(hi)
        ok = t + s < n
        t = t[ok]
        new = (A[t] + A[t + s]) & 0xFFFFFFFF
        A[t] = new
        s //= 2
    return ((A + 2**31) % 2**32 - 2**31).astype(np.int32)


@pytest.mark.parametrize("n", [16, 1024])
def test_tree_reduction_race_free(oracle_lib, n):
    A = I.cfg3_inputs(0, 6, n)[0]
    p = K.program(K.TREE)
    r = oracle_lib.run(p.bytecode, n, [A])
    assert len(r.reports) == 0
    for i in range(A.shape[0]):
        total = int(A[i].astype(np.int64).sum()) % 2**32
        assert int(np.uint32(r.final[0][i, 0].view(np.uint32))) == total  # A[0] = Σ mod 2^32
        assert (r.final[0][i] == _tree_numpy(A[i], False)).all()
    log = n.bit_length() - 1
    assert r.stats["checked_accesses"] == 3 * (n - 1) * A.shape[0]
    assert r.stats["intervals_max"] == log + 1


def test_tree_reduction_off_by_one(oracle_lib):
    """App. A.4: 1 OOB (A, n, tid n/2) + RW(A, s, (0, s), 0xD) for s = n/4 .. 1."""
    n = 1024
    A = I.cfg3_inputs(0, 4, n)[0]
    p = K.program(K.TREE_OFF_BY_ONE)
    r = oracle_lib.run(p.bytecode, n, [A])
    for i in range(A.shape[0]):
        got = [t for t in r.report_tuples() if t[0] == i]
        exp = [(i, 0, 0, n, 4, n // 2, NOTID, 0)]
        s, k = n // 4, 1
        while s >= 1:
            exp.append((i, k, 0, s, 1, 0, s, 0xD))
            s //= 2
            k += 1
        assert got == exp
        assert (r.final[0][i] == _tree_numpy(A[i], True)).all()
    assert r.stats["checked_accesses"] == 3097 * A.shape[0]


# --------------------------------------------------------------- stencil (config 5)
def _stencil_numpy(A, steps=4):
    """App. A.5: A'[c] = A[c-1]+A[c]+A[c+1] for c in [1,n], halos fixed (int32 wrap)."""
    A = A.astype(np.int64).copy()
    B = np.zeros_like(A)
    for _ in range(steps):
        B[1:-1] = (A[:-2] + A[1:-1] + A[2:]) & 0xFFFFFFFF
        A[1:-1] = B[1:-1]
    w = lambda x: ((x + 2**31) % 2**32 - 2**31).astype(np.int32)
    return w(A), w(B)


def test_stencil(oracle_lib):
    n = 300
    A, B = I.cfg5_inputs(0, 3, n)
    p = K.program(K.STENCIL)
    r = oracle_lib.run(p.bytecode, n, [A, B])
    assert len(r.reports) == 0
    for i in range(3):
        eA, eB = _stencil_numpy(A[i])
        assert (r.final[0][i] == eA).all() and (r.final[1][i][1:-1] == eB[1:-1]).all()
    assert r.stats["checked_accesses"] == 24 * n * 3
    assert r.stats["intervals_max"] == 9  # 8 barriers + the final (EXIT) interval


# --------------------------------------------------------------- arithmetic (reading L7)
def test_int32_arithmetic(oracle_lib):
    """Reading L7: int32 wrap, C99 truncating DIV/MOD, INT_MIN/-1 = INT_MIN, INT_MIN%-1 = 0."""
    rng = np.random.default_rng(7)
    vals = [0, 1, -1, 2, -2, 7, -7, 2**31 - 1, -2**31, 3, -3] + [int(x) for x in rng.integers(-2**31, 2**31, 20)]
    pairs = [(a, b) for a in vals for b in vals if b != 0]
    ops = ["add", "sub", "mul", "div", "mod", "min", "max", "and", "or", "xor", "lt", "eq", "land"]

    def ref(op, a, b):
        w = lambda x: (x + 2**31) % 2**32 - 2**31
        if op == "add": return w(a + b)
        if op == "sub": return w(a - b)
        if op == "mul": return w(a * b)
        if op == "div":
            q = abs(a) // abs(b)
            return w(q if (a >= 0) == (b >= 0) else -q)
        if op == "mod":
            q = abs(a) // abs(b)
            q = q if (a >= 0) == (b >= 0) else -q
            return w(a - b * q)
        if op == "min": return min(a, b)
        if op == "max": return max(a, b)
        if op == "and": return w(a & b)
        if op == "or": return w(a | b)
        if op == "xor": return w(a ^ b)
        if op == "lt": return int(a < b)
        if op == "eq": return int(a == b)
        if op == "land": return int(a != 0 and b != 0)

    # unary forms: v := v' (mov) and ¬b (lnot) of the first operand
    unary = {"mov": lambda a: a, "lnot": lambda a: int(a == 0)}
    cols = ops + list(unary)
    src = [".arrays X Y O", " tid r0", " ld r1, X, r0", " ld r2, Y, r0"]
    for j, op in enumerate(cols):
        operands = "r1" if op in unary else "r1, r2"
        src += [f" {op} r3, {operands}", f" const r4, {len(cols)}", " mul r5, r0, r4", f" addi r5, r5, {j}",
                " st O, r5, r3"]
    src += [" exit"]
    p = assemble("\n".join(src))
    n = len(pairs)
    X = np.array([[a for a, _ in pairs]], np.int32)
    Y = np.array([[b for _, b in pairs]], np.int32)
    O = np.zeros((1, n * len(cols)), np.int32)
    r = oracle_lib.run(p.bytecode, n, [X, Y, O])
    assert len(r.reports) == 0  # every work-item writes its own row of O
    out = r.final[2][0].reshape(n, len(cols))
    for t, (a, b) in enumerate(pairs):
        for j, op in enumerate(cols):
            want = unary[op](a) if op in unary else ref(op, a, b)
            assert int(out[t, j]) == want, (op, a, b)


def test_mov_operand_order(oracle_lib):
    """MOV rd, rs (`v := v'`, rc.h RC_OP_MOV: r[a] := r[b]),
    hand-derived.  Per work-item t: r1 := t; r2 := 100; mov r2, r1 (r2 = t);
    addi r1, r1, 5 (r1 = t + 5, r2 must keep t: a copy, not an alias);
    mov r3, r3 (self-copy keeps the zero-initialised r3, reading L18);
    A[t] := r2 + 1000 r3 = t; B[t] := r1 = t + 5.  A transposed MOV
    (r[b] := r[a]) would give r1 = 100, so A[t] = 100 and B[t] = 105; a
    MOV that aliases the registers would give A[t] = t + 5."""
    src = """
.arrays A B
    tid   r1
    const r2, 100
    mov   r2, r1
    addi  r1, r1, 5
    mov   r3, r3
    const r4, 1000
    mul   r4, r4, r3
    add   r5, r2, r4
    tid   r6
    st    A, r6, r5
    st    B, r6, r1
    exit
"""
    n = 6
    p = assemble(src)
    r = oracle_lib.run(p.bytecode, n, [np.zeros((1, n), np.int32), np.zeros((1, n), np.int32)])
    assert len(r.reports) == 0
    assert r.final[0][0].tolist() == [0, 1, 2, 3, 4, 5]
    assert r.final[1][0].tolist() == [5, 6, 7, 8, 9, 10]
    assert r.stats["op_counts"][2] == 2 * n  # both MOVs executed by every work-item


# --------------------------------------------------------------- ⊥ / ⊤ policy
def test_error_reports(oracle_lib):
    """PAPER.md:156, 188-197; readings L5/L6/L17."""
    src = """
.arrays A
    tid r0
    const r1, 0
    const r2, 1
    eq r3, r0, r1        ; tid == 0
    br r3, div0, n1
div0:
    div r4, r2, r1       ; tid 0: DIV0 at pc 5
n1:
    eq r3, r0, r2        ; tid == 1
    lnot r3, r3
    assert r3            ; tid 1: ASSERT at pc 8
    const r5, 2
    eq r3, r0, r5
    lnot r3, r3
    assume r3            ; tid 2: pruned silently
    const r5, 3
    eq r3, r0, r5
    br r3, spin, done
spin:
    jmp spin             ; tid 3: FUEL
done:
    st A, r0, r0         ; tids >= 4
    exit
"""
    p = assemble(src)
    r = oracle_lib.run(p.bytecode, 6, [np.zeros((1, 6), np.int32)], fuel=1000)
    got = r.report_tuples()
    assert got == [(0, 0, -1, 5, 6, 0, NOTID, 0), (0, 0, -1, 8, 5, 1, NOTID, 0),
                   (0, 0, -1, p.labels["spin"], 7, 3, NOTID, 0)]
    assert r.stats["lanes_final"] == [2, 1, 0, 1, 1, 1, 0, 0]
    # DIV0 lane did not fall through to n1 (its pc stayed at the div)
    assert r.final[0][0].tolist() == [0, 0, 0, 0, 4, 5]


def test_fuel_counts_instructions(oracle_lib):
    """Reading L17: every executed instruction costs 1; the refused one is not counted."""
    p = assemble(".arrays A\nspin:\n jmp spin")
    r = oracle_lib.run(p.bytecode, 3, [np.zeros((1, 1), np.int32)], fuel=50)
    assert r.stats["instructions"] == 150
    assert [t[4] for t in r.report_tuples()] == [7, 7, 7]


def test_max_intervals(oracle_lib):
    """Instance-level FUEL when barriers never stop (reading L17)."""
    p = assemble(".arrays A\nloop:\n bar\n jmp loop")
    r = oracle_lib.run(p.bytecode, 4, [np.zeros((2, 1), np.int32)], max_intervals=5)
    assert r.report_tuples() == [(0, 5, -1, -1, 7, NOTID, NOTID, 0), (1, 5, -1, -1, 7, NOTID, NOTID, 0)]
    assert r.stats["intervals_max"] == 5
    assert r.stats["lanes_final"][6] == 8


def test_barrier_divergence(oracle_lib):
    """P:97 'reached the same instruction barrier'; reading L9."""
    src = """
.arrays A
    tid r0
    const r1, 2
    lt r2, r0, r1
    br r2, b1, b2
b1:
    bar              ; tids 0,1 at pc 4
    exit
b2:
    const r3, 3
    eq r3, r0, r3
    br r3, ex, b3
b3:
    bar              ; tids 2,4 at pc 9
    exit
ex:
    exit             ; tid 3 exits in interval 0
"""
    p = assemble(src)
    r = oracle_lib.run(p.bytecode, 5, [np.zeros((1, 1), np.int32)])
    assert r.report_tuples() == [(0, 0, -1, 4, 8, 0, 2, 0)]
    # only one arrival node in interval 1 (all exit) -> no report there
    assert r.stats["intervals_max"] == 2


def test_rw_pair_rule(oracle_lib):
    """Reading L4: lex-min (t1<t2) with one reading and the other writing;
    non-benign pair = (min W, min{w: val_w != val_minW})."""
    # cell A[0]: tids 2,3 read; tid 1 writes 5; tid 0 writes 5; tid 4 writes 9
    src = """
.arrays A
    tid r0
    const r1, 0
    const r2, 2
    lt r3, r0, r2         ; tid < 2 -> write 5
    br r3, w5, r
w5:
    const r4, 5
    st A, r1, r4
    exit
r:
    const r2, 4
    eq r3, r0, r2
    br r3, w9, rd
w9:
    const r4, 9
    st A, r1, r4
    exit
rd:
    ld r4, A, r1
    exit
"""
    p = assemble(src)
    r = oracle_lib.run(p.bytecode, 5, [np.zeros((1, 1), np.int32)])
    # RW: candidates (0,2): 0 in W, 2 in R -> lex-min.  flags: tid0 wrote (2), tid2 read (4)
    # WW: W = {0:5, 1:5, 4:9} -> non-benign (0, 4), flags both wrote
    assert r.report_tuples() == [(0, 0, 0, 0, 1, 0, 2, 0b0110), (0, 0, 0, 0, 3, 0, 4, 0b1010)]
    assert int(r.final[0][0, 0]) == 9  # max-tid writer (tid 4) wins


def test_own_write_visible(oracle_lib):
    """Delayed visibility (reading L2): a work-item reads its own earlier write,
    others' writes only after the barrier."""
    src = """
.arrays A O
    tid r0
    const r1, 10
    add r2, r0, r1
    st A, r0, r2          ; A[tid] := tid+10
    ld r3, A, r0          ; own write
    addi r4, r0, 1
    const r5, 4
    mod r4, r4, r5
    ld r6, A, r4          ; neighbour: interval-start value
    st O, r0, r3
    addi r7, r0, 4
    st O, r7, r6
    exit
"""
    p = assemble(src)
    A0 = np.array([[100, 101, 102, 103]], np.int32)
    r = oracle_lib.run(p.bytecode, 4, [A0, np.zeros((1, 8), np.int32)])
    assert r.final[1][0].tolist() == [10, 11, 12, 13, 101, 102, 103, 100]
    kinds = [t[4] for t in r.report_tuples()]
    assert kinds == [1, 1, 1, 1]  # each A[c] written by c, read by c-1


def test_many_writes_per_interval(oracle_lib):
    """the store rule bounds nothing, so a work-item may
    write any number of distinct cells in one interval (workloads
    many_writes_kernel, hand-derived).  Work-item t writes A[64t + j] :=
    1000t + j, j = 0..69; cells 64(t+1) + j, j < 6, are also written by t+1
    with 1000(t+1) + j: WW_NONBENIGN (t, t+1); t also reads 64(t+1) + 2, so
    that cell has RW (t, t+1) with flags 0xB (t read + wrote, t+1 wrote) and
    its WW flags are 0xB too; t+1 reads its own 64(t+1) + 3, which t wrote:
    RW (t, t+1) with flags 0xE (t wrote, t+1 read + wrote), WW flags 0xE.
    B[t] = A[64t+3] + A[64t+40] + A[64t+66] read from t's own writes:
    (1000t + 3) + (1000t + 40) + (1000t + 66).  Final A: the max-tid writer."""
    n = 5
    p = K.many_writes_kernel()
    A = np.zeros((1, 64 * n + 6), np.int32)
    B = np.zeros((1, n), np.int32)
    r = oracle_lib.run(p.bytecode, n, [A, B])
    want = []
    for t in range(n - 1):
        for j in range(6):
            c = 64 * (t + 1) + j
            fl = {2: 0xB, 3: 0xE}.get(j, 0xA)
            if j in (2, 3):
                want.append((0, 0, 0, c, 1, t, t + 1, fl))
            want.append((0, 0, 0, c, 3, t, t + 1, fl))
    assert r.report_tuples() == want
    assert r.final[1][0].tolist() == [3000 * t + 109 for t in range(n)]
    fin = r.final[0][0]
    for t in range(n):  # a cell written by t and t+1 keeps t+1's value
        for j in range(70):
            c = 64 * t + j
            if j >= 64 and t + 1 < n:
                assert fin[c] == 1000 * (t + 1) + (j - 64)
            else:
                assert fin[c] == 1000 * t + j, (t, j)


def test_many_writes_loop(oracle_lib):
    """The loop variant (no static bound on the stores of an interval):
    work-item t writes A[64t + j] := j - t for j < 40 + 30 (t mod 3); when
    the count exceeds 64 (t mod 3 = 1, 2) its last cells are t+1's first:
    WW_NONBENIGN (t, t+1) there; after the barrier each reads A[64t + 39]
    (no writer in that interval: clean)."""
    n = 7
    p = K.program(K.MANY_WRITES_LOOP)
    A = np.full((1, 64 * n + 64), -7, np.int32)
    r = oracle_lib.run(p.bytecode, n, [A])
    want = []
    for t in range(n - 1):
        cnt = 40 + 30 * (t % 3)
        for j in range(64, cnt):
            want.append((0, 0, 0, 64 * t + j, 3, t, t + 1, 0xA))
    assert r.report_tuples() == want
    fin = r.final[0][0]
    for t in range(n):
        cnt = 40 + 30 * (t % 3)
        for j in range(cnt):
            c = 64 * t + j
            if j >= 64 and t + 1 < n:
                assert fin[c] == (j - 64) - (t + 1)
            else:
                assert fin[c] == j - t


# --------------------------------------------------------------- work-groups (reading L20)
IG = 0xFFFFFFFF  # interval field of the inter-group reports


def test_groups_write_write(oracle_lib):
    """PAPER.md:55-56 (work-groups with ids and a size), reading L20: G
    work-groups of n work-items run one after another; no barrier orders
    two groups.  A[lid] := gid: every cell c < n is written by work-item c of
    every group and by nobody else in that group: no intra-group report; per
    cell one IG_WW_NONBENIGN with the smallest cross-group writer pair
    (c, n + c) (the groups' last values 0, 1, 2 differ); the last group's
    value stays.  A[lid] := 7 instead: IG_WW_BENIGN."""
    n, G = 4, 3
    for val, kind, final in (("gid r1", 11, 2), ("const r1, 7", 10, 7)):
        src = f".arrays A\n lid r0\n {val}\n st A, r0, r1\n exit\n"
        p = assemble(src)
        r = oracle_lib.run(p.bytecode, n, [np.zeros((1, n), np.int32)], n_groups=G)
        assert r.report_tuples() == [(0, IG, 0, c, kind, c, n + c, 0) for c in range(n)]
        assert r.final[0][0].tolist() == [final] * n
        assert r.stats["lanes_final"][0] == n * G and r.stats["intervals_max"] == 1
        assert r.stats["checked_accesses"] == n * G


def test_groups_ids_and_partial_sums(oracle_lib):
    """Per-group tree reduction over the group's own slice of A (tid = gid*n +
    lid, LSIZE = n, barriers inside each group), then work-item 0 of every
    group adds its partial sum into S[0] and reads the next group's partial
    P[(gid+1) mod G].  Hand-derived: the slices are disjoint, so the
    reduction is race-free; S[0] is read and written by lid 0 of every group:
    IG_RW (0, n) and IG_WW_NONBENIGN (0, n) at S[0] (last values differ:
    running sums); P[g] is written by group g (lid 0) and read by group g-1's
    lid 0: IG_RW at P[g] with pair (lid 0 of group g-1, lid 0 of group g) for
    g >= 1 and (0, (G-1) n) at P[0].  Final S[0] = sum of all A; P[g] = the
    sum of group g's slice."""
    n, G = 8, 3
    src = """
.arrays A P S
    lid   r0
    gid   r1
    lsize r2
    tid   r3               ; = gid * n + lid
    const r4, 2
    div   r5, r2, r4       ; s := n/2
loop:
    const r6, 0
    lt    r7, r6, r5
    br    r7, body, done
body:
    lt    r7, r0, r5
    br    r7, work, sync
work:
    ld    r8, A, r3
    add   r9, r3, r5
    ld    r10, A, r9
    add   r8, r8, r10
    st    A, r3, r8
sync:
    bar
    div   r5, r5, r4
    jmp   loop
done:
    const r6, 0
    eq    r7, r0, r6
    br    r7, lead, end
lead:
    ld    r8, A, r3        ; the group's sum
    st    P, r1, r8
    ld    r9, S, r6
    add   r9, r9, r8
    st    S, r6, r9        ; S[0] += partial
    addi  r11, r1, 1
    const r12, 3
    mod   r11, r11, r12
    ld    r13, P, r11      ; the next group's partial
end:
    exit
"""
    p = assemble(src)
    A = np.arange(1, n * G + 1, dtype=np.int32)[None, :]
    r = oracle_lib.run(p.bytecode, n, [A, np.zeros((1, G), np.int32), np.zeros((1, 1), np.int32)], n_groups=G)
    want = [(0, IG, 1, 0, 9, 0, (G - 1) * n, 0)]  # P[0]: written by group 0, read by group G-1
    want += [(0, IG, 1, g, 9, (g - 1) * n, g * n, 0) for g in range(1, G)]
    want += [(0, IG, 2, 0, 9, 0, n, 0), (0, IG, 2, 0, 11, 0, n, 0)]
    assert r.report_tuples() == want
    sums = [int(A[0, g * n:(g + 1) * n].sum()) for g in range(G)]
    assert r.final[1][0].tolist() == sums and r.final[2][0].tolist() == [sum(sums)]
    assert r.stats["intervals_max"] == 4  # log2(8) = 3 barriers per group


def test_one_group_is_the_plain_run(oracle_lib):
    """n_groups = 1 is exactly the single-work-group semantics; and G groups
    on disjoint slices (index = tid) report each group's intra-group races
    with global tids, the same as G separate instances would (tids offset)."""
    p = K.program(K.TREE_OFF_BY_ONE)
    ins = I.cfg3_inputs(0, 3, 16)
    a = oracle_lib.run(p.bytecode, 16, ins)
    b = oracle_lib.run(p.bytecode, 16, ins, n_groups=1)
    assert a.report_tuples() == b.report_tuples() and a.stats == b.stats
    # every group works on its own slice R[gid*n .. gid*n + n-1] (Fig. 1's
    # second interval with the neighbour taken mod n): the groups' reports are
    # the single-group run's on each slice, cells and tids shifted by gid*n;
    # no inter-group report (the slices are disjoint); heaps concatenate
    src = """
.arrays R
    lid   r0
    lsize r1
    gid   r2
    mul   r3, r2, r1       ; gid * n
    add   r4, r3, r0       ; my cell
    st    R, r4, r0        ; R[me] := lid
    bar
    addi  r5, r0, 1
    mod   r5, r5, r1
    add   r5, r5, r3
    ld    r6, R, r5        ; R[gid*n + (lid+1) mod n]
    add   r6, r6, r6
    st    R, r4, r6
    exit
"""
    pg = assemble(src)
    n, G = 6, 4
    X = np.arange(n * G, dtype=np.int32)[None, :] * 5
    g = oracle_lib.run(pg.bytecode, n, [X], n_groups=G)
    want, fin = [], []
    for j in range(G):
        sr = oracle_lib.run(pg.bytecode, n, [X[:, j * n:(j + 1) * n]])
        want += [(i, iv, a, idx + j * n, k, t1 + j * n, t2 + j * n, fl)
                 for i, iv, a, idx, k, t1, t2, fl in sr.report_tuples()]
        fin += sr.final[0][0].tolist()
    assert len(want) == G * n and g.report_tuples() == sorted(want)
    assert g.final[0][0].tolist() == fin
