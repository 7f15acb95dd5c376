"""Text assembler for RCB1 bytecode (test / bench tooling, no semantics).

Encodes the §3 kernel language in the three-address CFG
form described in include/rc.h.  This module only ENCODES: it holds none of
the method's arithmetic, so both the oracle (oracle/) and the CUDA path
(paper_1308_3203_b200/) may be fed from it without sharing code.

Syntax (one instruction per line, ';' or '#' starts a comment):

    .arrays A B R          # shared arrays, ids in declaration order
    .regs 16               # optional; default = highest register used + 1
    label:
        tid   r0
        const r1, 1
        sub   r2, r0, r1
        ld    r3, A, r2     # r3 := A[r2]
        st    R, r0, r3     # R[r0] := r3
        br    r4, then, else
        jmp   label
        bar | exit | assume r5 | assert r5
"""
from __future__ import annotations

import re
import struct

MAGIC = 0x31424352  # 'RCB1' little-endian
VERSION = 1

OPCODES = {
    "const": 1, "mov": 2, "tid": 3, "size": 4,
    "add": 5, "sub": 6, "mul": 7, "div": 8, "mod": 9, "min": 10, "max": 11,
    "and": 12, "or": 13, "xor": 14, "lt": 15, "eq": 16, "land": 17, "lnot": 18,
    "ld": 19, "st": 20, "bar": 21, "assume": 22, "assert": 23, "br": 24,
    "jmp": 25, "exit": 26, "addi": 27,
    "gid": 28, "lid": 29, "lsize": 30,  # work-group id / local id / work-group size (reading L20)
}
_ALU3 = {"add", "sub", "mul", "div", "mod", "min", "max", "and", "or", "xor",
         "lt", "eq", "land"}


class AsmError(ValueError):
    pass


def encode(n_regs: int, n_arrays: int, instrs: list[tuple[int, int, int, int, int]],
           *, magic: int = MAGIC, version: int = VERSION, flags: int = 0) -> bytes:
    """Raw encoder: instrs = [(op, a, b, c, imm), ...]."""
    out = bytearray(struct.pack("<IHHHHI", magic, version, flags, n_regs, n_arrays, len(instrs)))
    for op, a, b, c, imm in instrs:
        out += struct.pack("<BBBBi", op & 0xFF, a & 0xFF, b & 0xFF, c & 0xFF, imm)
    return bytes(out)


def decode(blob: bytes) -> tuple[int, int, list[tuple[int, int, int, int, int]]]:
    magic, version, flags, n_regs, n_arrays, n_instr = struct.unpack_from("<IHHHHI", blob, 0)
    ins = [struct.unpack_from("<BBBBi", blob, 16 + 8 * i) for i in range(n_instr)]
    return n_regs, n_arrays, ins


class Program:
    """An assembled kernel: bytecode plus the symbol names used to build it."""

    def __init__(self, bytecode: bytes, arrays: list[str], n_regs: int, n_instr: int,
                 labels: dict[str, int], source: str = ""):
        self.bytecode = bytecode
        self.arrays = arrays
        self.n_regs = n_regs
        self.n_instr = n_instr
        self.labels = labels
        self.source = source

    def array_id(self, name: str) -> int:
        return self.arrays.index(name)

    def __repr__(self):
        return f"Program(arrays={self.arrays}, n_regs={self.n_regs}, n_instr={self.n_instr})"


def _reg(tok: str) -> int:
    m = re.fullmatch(r"r(\d+)", tok)
    if not m:
        raise AsmError(f"expected register, got {tok!r}")
    v = int(m.group(1))
    if v > 255:
        raise AsmError(f"register {tok} > r255")
    return v


def _imm(tok: str) -> int:
    v = int(tok, 0)
    if not -(2 ** 31) <= v < 2 ** 31:
        raise AsmError(f"immediate {tok} does not fit int32")
    return v


def assemble(text: str) -> Program:
    arrays: list[str] = []
    n_regs_decl = None
    lines = []
    for raw in text.splitlines():
        line = re.split(r"[;#]", raw, maxsplit=1)[0].strip()
        if not line:
            continue
        if line.startswith(".arrays"):
            arrays += line.split()[1:]
            continue
        if line.startswith(".regs"):
            n_regs_decl = int(line.split()[1])
            continue
        while True:  # allow "label: instr" on one line
            m = re.match(r"^([A-Za-z_]\w*):\s*(.*)$", line)
            if not m:
                break
            lines.append(("label", m.group(1)))
            line = m.group(2).strip()
        if line:
            lines.append(("ins", line))

    labels: dict[str, int] = {}
    pc = 0
    for kind, val in lines:
        if kind == "label":
            if val in labels:
                raise AsmError(f"duplicate label {val}")
            labels[val] = pc
        else:
            pc += 1

    def arr(tok: str) -> int:
        if tok not in arrays:
            raise AsmError(f"unknown array {tok!r}")
        return arrays.index(tok)

    def target(tok: str) -> int:
        if tok in labels:
            return labels[tok]
        return int(tok, 0)

    instrs = []
    max_reg = -1
    for kind, val in lines:
        if kind != "ins":
            continue
        parts = val.replace(",", " ").split()
        mn, args = parts[0].lower(), parts[1:]
        if mn not in OPCODES:
            raise AsmError(f"unknown mnemonic {mn!r}")
        op = OPCODES[mn]
        a = b = c = imm = 0
        regs = []
        try:
            if mn == "const":
                a, imm = _reg(args[0]), _imm(args[1]); regs = [a]
            elif mn == "mov" or mn == "lnot":
                a, b = _reg(args[0]), _reg(args[1]); regs = [a, b]
            elif mn in ("tid", "gid", "lid", "lsize"):
                a = _reg(args[0]); regs = [a]
            elif mn == "size":
                a, b = _reg(args[0]), arr(args[1]); regs = [a]
            elif mn in _ALU3:
                a, b, c = _reg(args[0]), _reg(args[1]), _reg(args[2]); regs = [a, b, c]
            elif mn == "addi":
                a, b, imm = _reg(args[0]), _reg(args[1]), _imm(args[2]); regs = [a, b]
            elif mn == "ld":
                a, b, c = _reg(args[0]), arr(args[1]), _reg(args[2]); regs = [a, c]
            elif mn == "st":
                a, b, c = arr(args[0]), _reg(args[1]), _reg(args[2]); regs = [b, c]
            elif mn in ("assume", "assert"):
                a = _reg(args[0]); regs = [a]
            elif mn == "br":
                a = _reg(args[0]); regs = [a]
                imm = target(args[1])
                f = target(args[2])
                b, c = f & 0xFF, (f >> 8) & 0xFF
            elif mn == "jmp":
                imm = target(args[0])
            elif mn in ("bar", "exit"):
                pass
        except IndexError:
            raise AsmError(f"missing operand in {val!r}") from None
        if regs:
            max_reg = max(max_reg, *regs)
        instrs.append((op, a, b, c, imm))
    n_regs = n_regs_decl if n_regs_decl is not None else max(max_reg + 1, 1)
    bc = encode(n_regs, len(arrays), instrs)
    return Program(bc, arrays, n_regs, len(instrs), labels, text)
