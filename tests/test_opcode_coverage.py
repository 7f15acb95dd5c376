"""The GPU parity corpus executes every RCB1 opcode (include/rc.h, the §3
grammar of PAPER.md:85-107 lowered): checked here on the oracle's per-opcode
execution counts, so an opcode no parity kernel reaches (a wrong MOV, say)
cannot pass unnoticed.  The GPU test runs the same corpus through the C ABI."""
import oracle
from parity_corpus import FUEL, all_opcodes, corpus


def test_corpus_executes_every_opcode(oracle_lib):
    counts = [0] * 32
    for name, p, n, ins, kw in corpus():
        r = oracle.run(p.bytecode, n, ins, fuel=FUEL, **kw)
        counts = [a + b for a, b in zip(counts, r.stats["op_counts"])]
    missing = [op for op in all_opcodes() if counts[op] == 0]
    assert not missing, f"opcodes never executed by the parity corpus: {missing}"
