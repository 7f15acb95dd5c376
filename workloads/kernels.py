"""The paper-shaped kernels of SURVEY.md App. A, as RCB1 programs.

Each kernel cites the passage it encodes.  Lowering of the §3 grammar
 to three-address bytecode follows DESIGN.md reading L10:
expression indices are computed into registers first.
"""
from __future__ import annotations

import numpy as np

from .asm import Program, assemble

# --- Figure 1: R[tid]=A[tid-1]+B[tid+1]; barrier; R[tid]=2*R[tid+1]
FIG1 = """
.arrays A B R
    tid   r0
    const r1, 1
    sub   r2, r0, r1
    ld    r3, A, r2        ; A[tid-1]
    add   r4, r0, r1
    ld    r5, B, r4        ; B[tid+1]
    add   r6, r3, r5
    st    R, r0, r6        ; R[tid] := A[tid-1] + B[tid+1]
    bar
    add   r7, r0, r1
    ld    r8, R, r7        ; R[tid+1]
    const r9, 2
    mul   r10, r9, r8
    st    R, r0, r10       ; R[tid] := 2 * R[tid+1]
    exit
"""

# Figure 1 guarded by assume(¬(tid<1) ∧ tid<size(A)−1)
FIG1_GUARDED = """
.arrays A B R
    tid   r0
    const r1, 1
    lt    r11, r0, r1
    lnot  r11, r11         ; ¬(tid < 1)
    size  r12, A
    sub   r12, r12, r1
    lt    r13, r0, r12     ; tid < size(A)-1
    land  r11, r11, r13
    assume r11
    sub   r2, r0, r1
    ld    r3, A, r2
    add   r4, r0, r1
    ld    r5, B, r4
    add   r6, r3, r5
    st    R, r0, r6
    bar
    add   r7, r0, r1
    ld    r8, R, r7
    const r9, 2
    mul   r10, r9, r8
    st    R, r0, r10
    exit
"""

# --- Figure 2: g=0; A[tid]=0; barrier; A[tid]=1;
#     if A[tid+1]=0 then g=1; barrier.   Shared scalar g = 1-element array G (L12).
FIG2 = """
.arrays A G
    const r0, 0
    st    G, r0, r0        ; g := 0
    tid   r1
    st    A, r1, r0        ; A[tid] := 0
    bar
    const r2, 1
    st    A, r1, r2        ; A[tid] := 1
    addi  r3, r1, 1
    ld    r4, A, r3        ; r := A[tid+1]
    eq    r5, r4, r0
    br    r5, then, end    ; if r = 0
then:
    st    G, r0, r2        ; g := 1
end:
    bar
    exit
"""

# --- Benign suite (config 2) ---------
BENIGN = {
    "K_c": """
.arrays A B
    const r0, 0
    const r1, 7
    st    A, r0, r1        ; A[0] := 7
    exit
""",
    "K_tid": """
.arrays A B
    const r0, 0
    tid   r1
    st    A, r0, r1        ; A[0] := tid
    exit
""",
    "K_B0": """
.arrays A B
    const r0, 0
    ld    r1, B, r0        ; r := B[0]
    st    A, r0, r1        ; A[0] := r
    exit
""",
    "K_Btid": """
.arrays A B
    const r0, 0
    tid   r2
    ld    r1, B, r2        ; r := B[tid]
    st    A, r0, r1        ; A[0] := r
    exit
""",
    "K_last": """
.arrays A B
    const r0, 0
    tid   r1
    st    A, r0, r1        ; A[0] := tid
    const r2, 7
    st    A, r0, r2        ; A[0] := 7
    exit
""",
    "K_inc": """
.arrays A B
    const r0, 0
    ld    r1, A, r0        ; r := A[0]
    addi  r1, r1, 1
    st    A, r0, r1        ; A[0] := r + 1
    exit
""",
}

# --- Tree reduction (config 3):  s:=size(A)/2; while 0<s { if tid<s {x:=A[tid];
#     y:=A[tid+s]; A[tid]:=x+y}; barrier; s:=s/2 }      (off-by-one: tid<=s)
_TREE = """
.arrays A
    tid   r0
    size  r1, A
    const r2, 2
    div   r1, r1, r2       ; s := size(A)/2
    const r3, 0
loop:
    lt    r4, r3, r1       ; 0 < s
    br    r4, body, done
body:
{guard}
    br    r5, work, sync
work:
    ld    r6, A, r0        ; x := A[tid]
    add   r7, r0, r1
    ld    r8, A, r7        ; y := A[tid+s]
    add   r6, r6, r8
    st    A, r0, r6        ; A[tid] := x + y
sync:
    bar
    div   r1, r1, r2       ; s := s/2
    jmp   loop
done:
    exit
"""
TREE = _TREE.format(guard="    lt    r5, r0, r1       ; tid < s")
TREE_OFF_BY_ONE = _TREE.format(guard="    lt    r5, r1, r0\n    lnot  r5, r5           ; tid <= s")

# --- 3-point stencil (config 5): c = tid+1;
#     4 x (B[c] := A[c-1]+A[c]+A[c+1]; barrier; A[c] := B[c]; barrier)
STENCIL = """
.arrays A B
    tid   r0
    addi  r1, r0, 1        ; c
    addi  r3, r0, 2        ; c+1
    const r7, 4
loop:
    ld    r4, A, r0        ; A[c-1]
    ld    r5, A, r1        ; A[c]
    ld    r6, A, r3        ; A[c+1]
    add   r4, r4, r5
    add   r4, r4, r6
    st    B, r1, r4        ; B[c] := A[c-1]+A[c]+A[c+1]
    bar
    ld    r4, B, r1
    st    A, r1, r4        ; A[c] := B[c]
    bar
    addi  r7, r7, -1
    br    r7, loop, done
done:
    exit
"""

# Private-only kernel (race-free for all n)
PRIVATE_ONLY = """
.arrays A
    tid   r0
    addi  r1, r0, 3
    mul   r2, r1, r1
    bar
    xor   r3, r2, r0
    exit
"""


def program(src: str) -> Program:
    return assemble(src)


# --- Config 4: random straight-line stencil kernels ----------------------------
HALO = 4


def random_stencil_kernel(seed: int, n_commands: int = 64, isa: str = "cfg4") -> Program:
    """Config 4 generator: 64 commands over 4 arrays X0..X3.

    Mix per command: 30% stencil load pair (ri := tid+K+k, k in [-4,4]; load
    from X_j, j != w), 30% ALU (ADD/SUB/MUL/XOR/MIN/MAX on data registers),
    20% home store Xw[tid+K], 4% indirect store Xw[X3[tid+K]], 4% indirect
    load Xw[X3[tid+K]], 8% barrier (w := (w+1) mod 3).  Then EXIT.
    Registers: r0 = tid, r1 = tid+K, r2..r9 data, r10 index temp.

    isa="full" (parity corpus, not config 4): the ALU draws from every
    register-to-register opcode of the §3 grammar: add sub
    mul div mod min max and or xor lt eq land, and the unary mov / lnot; a
    div / mod divisor is sometimes a 0/1 comparison result, so DIV0 (⊥)
    occurs.  Same memory-command mix.
    """
    rng = np.random.default_rng(np.random.SeedSequence([0x13083203, 4, seed]))
    lines = [".arrays X0 X1 X2 X3", ".regs 11", "    tid r0", f"    addi r1, r0, {HALO}"]
    w = 0
    alu = ["add", "sub", "mul", "xor", "min", "max"]
    if isa == "full":
        alu = alu + ["div", "mod", "and", "or", "lt", "eq", "land", "mov", "lnot"]
    elif isa != "cfg4":
        raise ValueError(isa)
    for _ in range(n_commands):
        u = rng.random()
        d = int(rng.integers(2, 10))
        if u < 0.30:
            k = int(rng.integers(-4, 5))
            j = int(rng.choice([x for x in range(3) if x != w]))
            lines += [f"    addi r10, r0, {HALO + k}", f"    ld r{d}, X{j}, r10"]
        elif u < 0.60:
            op = alu[int(rng.integers(0, len(alu)))]
            a, b = int(rng.integers(2, 10)), int(rng.integers(2, 10))
            if op in ("mov", "lnot"):
                lines.append(f"    {op} r{d}, r{a}")
            elif op in ("div", "mod") and rng.random() < 0.5:
                # divisor from a comparison (0 or 1): DIV0 on some work-items
                lines += [f"    lt r10, r{a}, r{b}", f"    {op} r{d}, r{a}, r10"]
            else:
                lines.append(f"    {op} r{d}, r{a}, r{b}")
        elif u < 0.80:
            lines.append(f"    st X{w}, r1, r{d}")
        elif u < 0.84:
            lines += ["    ld r10, X3, r1", f"    st X{w}, r10, r{d}"]
        elif u < 0.88:
            lines += ["    ld r10, X3, r1", f"    ld r{d}, X{w}, r10"]
        else:
            lines.append("    bar")
            w = (w + 1) % 3
    lines.append("    exit")
    return assemble("\n".join(lines))


def random_tiny_kernel(rng: np.random.Generator, n_arrays: int = 2, n_regs: int = 4,
                       n_commands: int = 6, size: int = 3, allow_bar: bool = True,
                       allow_branch: bool = True, groups: bool = False) -> Program:
    """Tiny random kernels for the brute-force interleaving checks (n <= 4).

    Indices are drawn as (tid*m + c) mod size so most accesses are in bounds
    and threads collide often; values come from tid, constants and loads.
    The ALU draws from every register-to-register opcode of the grammar
    (PAPER.md:87-88), mov and lnot included; div / mod by a zero register
    halts the work-item with DIV0.
    """
    lines = [".arrays " + " ".join(f"A{i}" for i in range(n_arrays)), f".regs {n_regs + (5 if groups else 3)}",
             "    tid r0", f"    const r1, {size}"]
    t = n_regs  # temp registers: r{n_regs}, r{n_regs+1}, r{n_regs+2}
    ids = ["r0"]
    if groups:  # work-group ids as index bases too (reading L20): r{n_regs+3} = lid, r{n_regs+4} = gid
        lines += [f"    lid r{n_regs + 3}", f"    gid r{n_regs + 4}"]
        ids = ["r0", f"r{n_regs + 3}", f"r{n_regs + 4}"]
    body = []
    for ci in range(n_commands):
        u = rng.random()
        if u < 0.30:  # store
            m, c = int(rng.integers(0, 3)), int(rng.integers(0, size))
            v = int(rng.integers(0, n_regs))
            base = ids[int(rng.integers(0, len(ids)))] if groups else "r0"
            body += [f"    const r{t}, {m}", f"    mul r{t}, {base}, r{t}", f"    addi r{t}, r{t}, {c}",
                     f"    mod r{t}, r{t}, r1", f"    st A{int(rng.integers(0, n_arrays))}, r{t}, r{v}"]
        elif u < 0.60:  # load
            m, c = int(rng.integers(0, 3)), int(rng.integers(0, size))
            d = int(rng.integers(2, n_regs)) if n_regs > 2 else 2
            base = ids[int(rng.integers(0, len(ids)))] if groups else "r0"
            body += [f"    const r{t}, {m}", f"    mul r{t}, {base}, r{t}", f"    addi r{t}, r{t}, {c}",
                     f"    mod r{t}, r{t}, r1", f"    ld r{d}, A{int(rng.integers(0, n_arrays))}, r{t}"]
        elif u < 0.80:  # alu
            d = int(rng.integers(2, n_regs)) if n_regs > 2 else 2
            ops = ["add", "sub", "mul", "xor", "min", "max", "eq", "lt", "and", "or", "land", "div", "mod",
                   "mov", "lnot"]
            op = ops[int(rng.integers(0, len(ops)))]
            x, y = int(rng.integers(0, n_regs)), int(rng.integers(0, n_regs))
            if op in ("mov", "lnot"):  # unary (v := v', ¬b)
                body.append(f"    {op} r{d}, r{x}")
            else:  # div / mod by a zero register halts the work-item (DIV0, reading L7)
                body.append(f"    {op} r{d}, r{x}, r{y}")
        elif u < 0.88 and allow_bar:
            body.append("    bar")
        elif u < 0.96 and allow_branch:
            # if (r_x < r_y) skip next command block: forward branch only (terminates)
            lab = f"L{ci}"
            d = int(rng.integers(2, n_regs)) if n_regs > 2 else 2
            body += [f"    lt r{t + 1}, r{int(rng.integers(0, n_regs))}, r{int(rng.integers(0, n_regs))}",
                     f"    br r{t + 1}, {lab}, {lab}_n",
                     f"{lab}_n:", f"    addi r{d}, r{d}, 1", f"{lab}:"]
        else:
            body.append(f"    addi r{int(rng.integers(2, n_regs)) if n_regs > 2 else 2}, r0, {int(rng.integers(-2, 3))}")
    lines += body + ["    exit"]
    return assemble("\n".join(lines))


# --- Many distinct writes per work-item per interval (PAPER.md:176-179 puts no
#     bound on them; the own-write overlay's capacity must not be semantic):
#     work-item t writes A[64t + j] := 1000 t + j for j = 0..69 (its last 6
#     cells are the first 6 of t+1), then reads back A[64t+3], A[64t+40] and
#     A[64t+66] (its own writes) and stores B[t] := their sum.
def many_writes_kernel(per_item: int = 64, extra: int = 6) -> Program:
    lines = [".arrays A B", "    tid r0", f"    const r1, {per_item}", "    mul r2, r0, r1",
             "    const r3, 1000", "    mul r3, r0, r3"]
    for j in range(per_item + extra):
        lines += [f"    addi r4, r2, {j}", f"    addi r5, r3, {j}", "    st A, r4, r5"]
    lines += ["    addi r4, r2, 3", "    ld r6, A, r4", "    addi r4, r2, 40", "    ld r7, A, r4",
              f"    addi r4, r2, {per_item + 2}", "    ld r8, A, r4", "    add r6, r6, r7", "    add r6, r6, r8",
              "    st B, r0, r6", "    exit"]
    return assemble("\n".join(lines))


# the same with a loop (no static bound on the stores of an interval):
# work-item t writes A[t*stride + j] := j - t for j = 0 .. count-1, count =
# 40 + 30 (t mod 3); then a barrier and a read of A[t*stride + 39]
MANY_WRITES_LOOP = """
.arrays A
    tid   r0
    const r1, 3
    mod   r2, r0, r1
    const r1, 30
    mul   r2, r2, r1
    addi  r2, r2, 40       ; count
    const r1, 64
    mul   r3, r0, r1       ; base
    const r4, 0            ; j
loop:
    add   r5, r3, r4
    sub   r6, r4, r0
    st    A, r5, r6        ; A[base + j] := j - t
    addi  r4, r4, 1
    lt    r7, r4, r2
    br    r7, loop, done
done:
    bar
    addi  r5, r3, 39
    ld    r6, A, r5
    exit
"""
