"""GPU (librc.so, sm_100a) vs CPU oracle: bit-exact parity.

Every comparison is element by element on the same seeded inputs: the full
canonical report list (all fields incl. flags), every final heap cell and the
exact rc_stats counters.  Small configurations are compared in full; the
BASELINE.json sizes are run in the launch configuration bench.py times and
compared on sampled instances the oracle computes one by one (instances are
independent, PAPER.md:56 / DESIGN.md §4).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from workloads import inputs as I  # noqa: E402
from workloads import kernels as K  # noqa: E402
from workloads.asm import assemble  # noqa: E402

STAT_KEYS = ("checked_accesses", "loads", "stores", "instructions", "intervals_max", "lanes_final")


@pytest.fixture(scope="module", params=["k1", "k1c"])
def rc(request):
    """The library, once per interval kernel: K1 (the bytecode interpreter,
    RC_JIT=0) and K1c (the kernel compiled per program with NVRTC, RC_JIT=1
    forces it at every size; programs it declines run K1)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import os
    import paper_1308_3203_b200 as pkg
    pkg.lib()
    old = os.environ.get("RC_JIT")
    os.environ["RC_JIT"] = "1" if request.param == "k1c" else "0"
    yield pkg
    if old is None:
        os.environ.pop("RC_JIT", None)
    else:
        os.environ["RC_JIT"] = old


def run_both(rc, src_or_prog, n, ins, *, fuel=0, max_intervals=0, host=False, **kw):
    p = assemble(src_or_prog) if isinstance(src_or_prog, str) else src_or_prog
    prog = rc.rc_load_program(p.bytecode)
    arrays = ins if host else [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in ins]
    g = rc.rc_run(prog, n, arrays, fuel_per_interval=fuel, max_intervals=max_intervals, **kw)
    o = oracle.run(p.bytecode, n, ins, fuel=fuel or oracle.oracle.DEFAULT_FUEL,
                   max_intervals=max_intervals or oracle.oracle.DEFAULT_MAX_INTERVALS,
                   instance_offset=kw.get("instance_offset", 0), classify_rw=kw.get("classify_rw", False),
                   n_groups=kw.get("n_groups", 1))
    return p, g, o


def assert_parity(g, o, ins):
    gt, ot = g.report_tuples(), o.report_tuples()
    if gt != ot:
        sg, so = set(gt), set(ot)
        raise AssertionError(f"reports differ: {len(gt)} vs {len(ot)}; gpu-only {sorted(sg - so)[:5]}, "
                             f"oracle-only {sorted(so - sg)[:5]}")
    assert g.n_reports_total == len(ot)
    for a in range(len(ins)):
        fin = g.final[a].cpu().numpy() if hasattr(g.final[a], "cpu") else g.final[a]
        if not np.array_equal(fin, o.final[a]):
            bad = np.argwhere(fin != o.final[a])[:5]
            raise AssertionError(f"final heap of array {a} differs at {bad.tolist()}")
    for k in STAT_KEYS:
        assert g.stats[k] == o.stats[k], (k, g.stats[k], o.stats[k])


# ------------------------------------------------------------------ config 1
@pytest.mark.parametrize("src", [K.FIG1, K.FIG1_GUARDED])
def test_config1_fig1(rc, src):
    p, g, o = run_both(rc, src, 8, I.cfg1_inputs())
    assert_parity(g, o, I.cfg1_inputs())
    assert len(o.reports) >= 5


@pytest.mark.parametrize("a2,size", [(0, 3), (5, 3), (5, 2)])
def test_fig2(rc, a2, size):
    ins = [np.array([[7, 9, a2][:size]], np.int32), np.array([[42]], np.int32)]
    p, g, o = run_both(rc, K.FIG2, 2, ins)
    assert_parity(g, o, ins)


# ------------------------------------------------------------------ config 2
@pytest.mark.parametrize("name", list(K.BENIGN))
def test_config2_benign_suite(rc, name):
    ins = I.cfg2_inputs(0, 1024, 256)
    p, g, o = run_both(rc, K.BENIGN[name], 256, ins)
    assert_parity(g, o, ins)


# ------------------------------------------------------------------ config 3
@pytest.mark.parametrize("src", [K.TREE, K.TREE_OFF_BY_ONE])
def test_config3_tree_full(rc, src):
    ins = I.cfg3_inputs(0, 16384, 1024)
    p, g, o = run_both(rc, src, 1024, ins)
    assert_parity(g, o, ins)


# ------------------------------------------------------------------ config 4
@pytest.mark.parametrize("isa", ["cfg4", "full"])
@pytest.mark.parametrize("seed", range(8))
def test_config4_small(rc, seed, isa):
    """Config 4's generator (isa="cfg4") and its full-ALU variant (every
    register op incl. mov / lnot / div / mod, DIV0 on some work-items)."""
    n = 200  # ragged: not a multiple of 32; several sort tiles
    ins = I.cfg4_inputs(0, 6, n)
    # denser index perturbation than the 2^-12 of the full config so races occur
    rng = np.random.default_rng(seed)
    x3 = ins[3]
    hit = rng.random(x3.shape) < 0.05
    x3[hit] = np.clip(x3[hit] + rng.choice([-1, 1], size=hit.sum()), 0, n + 7)
    p, g, o = run_both(rc, K.random_stencil_kernel(seed, isa=isa), n, ins)
    assert_parity(g, o, ins)
    assert len(o.reports) > 0


def _stencil_closed_form(A, steps=4):
    """App. A.5 (numpy, batched over instances): A'[c] = A[c-1]+A[c]+A[c+1]
    for c in [1, n] with fixed halos, int32 wrap; B holds the last step."""
    A = A.astype(np.int64)
    B = np.zeros_like(A)
    for _ in range(steps):
        B[:, 1:-1] = (A[:, :-2] + A[:, 1:-1] + A[:, 2:]) & 0xFFFFFFFF
        A[:, 1:-1] = B[:, 1:-1]
    return A.astype(np.uint32).view(np.int32), B.astype(np.uint32).view(np.int32)


def _host_final(g, a):
    return g.final[a].cpu().numpy()


@pytest.mark.slow
@pytest.mark.parametrize("seed", range(8))
def test_config4_full_size(rc, seed):
    """BASELINE config 4 per-GPU shard at full size (n = 65536, 512
    instances, X3 perturbed with p = 2^-12), every one of the 8 generator
    seeds, in bench.py's launch configuration: the complete report list,
    every final heap cell of all 512 instances and the counters against
    the oracle run over all instances."""
    n, n_inst = 65536, 512
    ins = I.cfg4_inputs(0, n_inst, n)
    p = K.random_stencil_kernel(seed)
    prog = rc.rc_load_program(p.bytecode)
    g = rc.rc_run(prog, n, [torch.from_numpy(x).cuda() for x in ins])
    o = oracle.run(p.bytecode, n, ins)
    assert_parity(g, o, ins)
    assert g.stats["checked_accesses"] > 10**9


@pytest.mark.slow
def test_config5_full_size(rc):
    """BASELINE config 5 at full size (2^20 work-items x 512 instances, 8
    barriers), the launch configuration bench.py times: all 512 instances'
    final A and B against the App. A.5 numpy closed form, no report, the
    exact access / interval counts; and 32 instances spread over every
    instance batch compared with the oracle run one by one (reports, heaps)."""
    n, n_inst = 1 << 20, 512
    ins = I.cfg5_inputs(0, n_inst, n)
    p = K.program(K.STENCIL)
    prog = rc.rc_load_program(p.bytecode)
    g = rc.rc_run(prog, n, [torch.from_numpy(x).cuda() for x in ins])
    assert g.n_reports_total == 0
    assert g.stats["checked_accesses"] == 24 * n * n_inst
    assert g.stats["intervals_max"] == 9
    assert g.stats["lanes_final"][0] == n * n_inst  # every work-item exited
    for i0 in range(0, n_inst, 32):
        eA, eB = _stencil_closed_form(ins[0][i0:i0 + 32])
        gA = g.final[0][i0:i0 + 32].cpu().numpy()
        gB = g.final[1][i0:i0 + 32].cpu().numpy()
        assert np.array_equal(gA, eA), f"A of instances {i0}..{i0 + 31}"
        assert np.array_equal(gB[:, 1:-1], eB[:, 1:-1]) and not gB[:, [0, -1]].any(), f"B of {i0}..{i0 + 31}"
    sample = list(range(0, n_inst, 16))  # 32 instances, one every 16 (batches of 7: every batch phase)
    sub = [x[sample] for x in ins]
    o = oracle.run(p.bytecode, n, sub)
    assert len(o.reports) == 0
    for a in range(2):
        assert np.array_equal(g.final[a][sample].cpu().numpy(), o.final[a]), a


# ------------------------------------------------------------------ opcode coverage
def test_opcode_corpus(rc):
    """tests/parity_corpus.py through the C ABI, element by element against
    the oracle; the oracle's per-opcode counts show every RCB1 opcode
    executed (so every K1 dispatch case ran under a parity check)."""
    from parity_corpus import FUEL, all_opcodes, corpus
    counts = [0] * 32
    for name, p, n, ins, kw in corpus():
        _, g, o = run_both(rc, p, n, ins, fuel=FUEL, **kw)
        try:
            assert_parity(g, o, ins)
        except AssertionError as ex:
            raise AssertionError(f"{name}: {ex}") from None
        counts = [a + b for a, b in zip(counts, o.stats["op_counts"])]
    assert [op for op in all_opcodes() if counts[op] == 0] == []


# ------------------------------------------------------------------ config 5 (small)
def test_config5_small(rc):
    ins = I.cfg5_inputs(0, 5, 1000)
    p, g, o = run_both(rc, K.STENCIL, 1000, ins)
    assert_parity(g, o, ins)


# ------------------------------------------------------------------ edge cases
def test_error_kinds_and_divergence(rc):
    src = """
.arrays A
    tid r0
    const r1, 0
    const r2, 1
    eq r3, r0, r1
    br r3, div0, n1
div0:
    div r4, r2, r1
n1:
    eq r3, r0, r2
    lnot r3, r3
    assert r3
    const r5, 2
    eq r3, r0, r5
    lnot r3, r3
    assume r3
    const r5, 3
    eq r3, r0, r5
    br r3, spin, more
spin:
    jmp spin
more:
    const r5, 5
    lt r3, r0, r5
    br r3, b1, b2
b1:
    bar
    st A, r0, r0
    exit
b2:
    bar
    exit
"""
    ins = [np.zeros((3, 40), np.int32)]
    p, g, o = run_both(rc, src, 40, ins, fuel=300)
    assert_parity(g, o, ins)
    kinds = {t[4] for t in o.report_tuples()}
    assert {5, 6, 7, 8} <= kinds


@pytest.mark.parametrize("fuel", [1, 5, 8, 9, 10, 40])
def test_fuel_around_static_bound(rc, fuel):
    """Straight-line intervals (FIG1: the longest barrier-free path is
    9 instructions, BAR / EXIT included): K1 drops the per-instruction fuel check
    when that bound fits in the fuel (reading L17); FUEL reports must appear
    exactly as the oracle's on both sides of the bound."""
    ins = I.cfg1_inputs()
    p, g, o = run_both(rc, K.FIG1, 8, ins, fuel=fuel)
    assert_parity(g, o, ins)
    has_fuel = any(t[4] == 7 for t in o.report_tuples())
    assert has_fuel == (fuel < 9)


def test_max_intervals(rc):
    src = (".arrays A\n tid r0\n addi r2, r0, 1\nloop:\n bar\n ld r1, A, r0\n addi r1, r1, 1\n st A, r0, r1\n"
           " br r2, loop, end\nend:\n exit")
    ins = [np.arange(6 * 50, dtype=np.int32).reshape(6, 50)]
    p, g, o = run_both(rc, src, 50, ins, max_intervals=7)
    assert_parity(g, o, ins)


def test_int32_semantics(rc):
    rng = np.random.default_rng(3)
    vals = np.concatenate([[0, 1, -1, 2**31 - 1, -2**31, 7, -7], rng.integers(-2**31, 2**31, 200)]).astype(np.int32)
    X = np.repeat(vals, len(vals))[None, :]
    Y = np.tile(vals, len(vals))[None, :]
    Y[Y == 0] = 3
    n = X.shape[1]
    ops = ["add", "sub", "mul", "div", "mod", "min", "max", "and", "or", "xor", "lt", "eq", "land"]
    src = [".arrays X Y O", " tid r0", " ld r1, X, r0", " ld r2, Y, r0", f" const r4, {len(ops) + 2}",
           " mul r5, r0, r4"]
    for op in ops:
        src += [f" {op} r3, r1, r2", " st O, r5, r3", " addi r5, r5, 1"]
    src += [" lnot r3, r1", " st O, r5, r3", " addi r5, r5, 1", " mov r3, r2", " st O, r5, r3", " exit"]
    ins = [X, Y, np.zeros((1, n * (len(ops) + 2)), np.int32)]
    p, g, o = run_both(rc, "\n".join(src), n, ins)
    assert_parity(g, o, ins)


@pytest.mark.parametrize("n,n_inst", [(1, 1), (1, 37), (31, 3), (33, 5), (1000, 1), (4097, 2)])
def test_ragged_shapes(rc, n, n_inst):
    ins = I.cfg5_inputs(0, n_inst, n)
    p, g, o = run_both(rc, K.STENCIL, n, ins)
    assert_parity(g, o, ins)


def test_empty_inputs(rc):
    prog_src = K.STENCIL
    # zero instances
    p = assemble(prog_src)
    prog = rc.rc_load_program(p.bytecode)
    g = rc.rc_run(prog, 16, [torch.zeros((0, 18), dtype=torch.int32, device="cuda")] * 2, n_instances=0)
    assert g.n_reports_total == 0 and g.stats["intervals_max"] == 0
    # zero work-items
    ins = [np.ones((3, 4), np.int32), np.ones((3, 4), np.int32)]
    p, g, o = run_both(rc, prog_src, 0, ins)
    assert_parity(g, o, ins)
    # zero-size arrays: every access is out of bounds
    ins = [np.zeros((2, 0), np.int32), np.zeros((2, 0), np.int32)]
    p, g, o = run_both(rc, prog_src, 5, ins)
    assert_parity(g, o, ins)


def test_host_io_matches_device(rc):
    ins = I.cfg3_inputs(0, 64, 256)
    p, g, o = run_both(rc, K.TREE_OFF_BY_ONE, 256, ins, host=True)
    assert_parity(g, o, ins)


def test_instance_offset_and_batches(rc):
    ins = I.cfg3_inputs(0, 40, 128)
    p = K.program(K.TREE_OFF_BY_ONE)
    prog = rc.rc_load_program(p.bytecode)
    dev = [torch.from_numpy(ins[0]).cuda()]
    o = oracle.run(p.bytecode, 128, ins, instance_offset=1000)
    for mb in (0, 1, 7, 40):
        g = rc.rc_run(prog, 128, dev, instance_offset=1000, max_batch_instances=mb)
        assert_parity(g, o, ins)


def test_batches_host_io_shapes_and_workspace(rc):
    """Several batches through host buffers (A2 double-buffered copy stream,
    final heaps copied back per batch), with and without RW classification;
    the same program re-run with other shapes (batch plan cache) and after
    its device workspace was released."""
    p = K.program(K.TREE_OFF_BY_ONE)
    prog = rc.rc_load_program(p.bytecode)
    for n, n_inst, mb in ((128, 37, 5), (256, 9, 2), (64, 50, 0), (128, 37, 4)):
        ins = I.cfg3_inputs(0, n_inst, n)
        for classify in (False, True):
            g = rc.rc_run(prog, n, ins, max_batch_instances=mb, classify_rw=classify)
            o = oracle.run(p.bytecode, n, ins, classify_rw=classify)
            assert_parity(g, o, ins)
        prog.release_workspace()
    ins = I.cfg5_inputs(0, 5, 300)
    p5 = K.program(K.STENCIL)
    prog5 = rc.rc_load_program(p5.bytecode)
    for mb in (1, 2, 0):
        g = rc.rc_run(prog5, 300, ins, max_batch_instances=mb)
        assert_parity(g, oracle.run(p5.bytecode, 300, ins), ins)


def test_truncation(rc):
    ins = I.cfg3_inputs(0, 50, 64)
    p = K.program(K.TREE_OFF_BY_ONE)
    prog = rc.rc_load_program(p.bytecode)
    o = oracle.run(p.bytecode, 64, ins)
    g = rc.rc_run(prog, 64, [torch.from_numpy(ins[0]).cuda()], capacity=17, allow_truncate=True)
    assert g.n_reports_total == len(o.reports)
    assert g.report_tuples() == o.report_tuples()[:17]
    with pytest.raises(rc.RCError) as ei:
        rc.rc_run(prog, 64, [torch.from_numpy(ins[0]).cuda()], capacity=17)
    assert ei.value.code == 4


@pytest.mark.parametrize("classify", [False, True])
def test_many_writes_spill(rc, monkeypatch, classify):
    """The own-write overlay holds 15 cells per work-item in shared memory and
    spills the rest to HBM (its capacity is not semantic):
    70 distinct cells per work-item in one interval (reads hitting both the
    shared-memory part and the spill list, WW / RW on spilled cells), and a
    loop with no static bound writing up to 100; ragged n, several batches,
    the spill lists grown by re-running the interval (and with
    RC_DEBUG_SMALL_BUFFERS every other buffer too)."""
    for small in (False, True):
        if small:
            monkeypatch.setenv("RC_DEBUG_SMALL_BUFFERS", "1")
        for n, n_inst, mb in ((5, 1, 0), (97, 3, 0), (300, 4, 2)):
            p = K.many_writes_kernel()
            ins = [np.arange(n_inst * (64 * n + 6), dtype=np.int32).reshape(n_inst, -1), np.zeros((n_inst, n), np.int32)]
            _, g, o = run_both(rc, p, n, ins, classify_rw=classify, max_batch_instances=mb)
            assert_parity(g, o, ins)
            ins = [np.full((n_inst, 64 * n + 64), -7, np.int32)]
            _, g, o = run_both(rc, K.program(K.MANY_WRITES_LOOP), n, ins, classify_rw=classify, max_batch_instances=mb)
            assert_parity(g, o, ins)


def test_random_tiny_kernels(rc):
    rng = np.random.default_rng(99)
    for it in range(300):
        n = int(rng.integers(1, 70))
        pr = K.random_tiny_kernel(rng, n_arrays=2, n_regs=5, n_commands=int(rng.integers(3, 12)), size=5)
        ins = [rng.integers(-3, 4, size=(int(rng.integers(1, 4)), 5)).astype(np.int32)]
        ins.append(rng.integers(-3, 4, size=(ins[0].shape[0], 5)).astype(np.int32))
        p, g, o = run_both(rc, pr, n, ins, fuel=500)
        assert_parity(g, o, ins)


def test_static_write_set_elision_after_divergence(rc):
    """K1 skips the read records of arrays an interval region never stores to
    (program.cpp analyze() (5)) only when every running work-item of the
    instance starts the interval at the same entry.  Here the work-items split
    over two barriers; in the next interval the ones after b1 read X[0] (their
    region stores no X) while the ones after b2 write it: the RW race must be
    reported, and the instance without the split (n = 2) must stay clean."""
    src = """
.arrays X Y
    tid r0
    const r1, 2
    lt r2, r0, r1
    br r2, left, right
left:
    bar
    const r5, 0
    ld r3, X, r5
    exit
right:
    bar
    const r5, 0
    st X, r5, r0
    exit
"""
    for n in (2, 5, 300):
        ins = [np.arange(4, dtype=np.int32).reshape(2, 2), np.zeros((2, 3), np.int32)]
        p, g, o = run_both(rc, src, n, ins)
        assert_parity(g, o, ins)
        kinds = {t[4] for t in o.report_tuples()}
        assert (1 in kinds) == (n > 2) and (8 in kinds) == (n > 2)


def test_rw_classification(rc):
    """SURVEY §8(f) row 1 (reading L19): with RC_OPT_CLASSIFY_RW every RW
    report carries bit 4 or 5 exactly as the oracle's re-run decides; all
    other results are unchanged."""
    cases = [(K.BENIGN["K_inc"], 64, I.cfg2_inputs(0, 6, 64)),
             (".arrays A\n const r0, 0\n ld r1, A, r0\n const r2, 5\n st A, r0, r2\n exit\n", 40,
              [np.array([[9], [5], [1]], np.int32)]),
             (".arrays A B\n tid r0\n addi r1, r0, 1\n ld r2, A, r1\n st A, r0, r0\n st B, r0, r2\n exit\n", 50,
              [np.arange(3 * 51, dtype=np.int32).reshape(3, 51), np.zeros((3, 50), np.int32)]),
             (K.FIG1, 8, I.cfg1_inputs()),
             (K.TREE_OFF_BY_ONE, 256, I.cfg3_inputs(0, 5, 256)),
             (K.STENCIL, 100, I.cfg5_inputs(0, 2, 100))]
    for src, n, ins in cases:
        p, g, o = run_both(rc, src, n, ins, classify_rw=True)
        assert_parity(g, o, ins)
        assert all(t[7] & 0x30 in (0x10, 0x20) for t in g.report_tuples() if t[4] == 1)
    rng = np.random.default_rng(17)
    for it in range(150):
        n = int(rng.integers(1, 40))
        pr = K.random_tiny_kernel(rng, n_arrays=2, n_regs=5, n_commands=int(rng.integers(3, 12)), size=5)
        ins = [rng.integers(-3, 4, size=(int(rng.integers(1, 4)), 5)).astype(np.int32)]
        ins.append(rng.integers(-3, 4, size=(ins[0].shape[0], 5)).astype(np.int32))
        p, g, o = run_both(rc, pr, n, ins, fuel=500, classify_rw=True)
        assert_parity(g, o, ins)
    ins = I.cfg4_inputs(0, 2, 400)
    ins[3][:, 50:90] += 1
    p, g, o = run_both(rc, K.random_stencil_kernel(3), 400, ins, classify_rw=True)
    assert_parity(g, o, ins)


def test_sort_64bit_lookback_words(rc, monkeypatch):
    """The onesweep look-back uses 32-bit status words for sorts of < 2^26
    records and 64-bit words otherwise; RC_DEBUG_SORT_W64 forces the 64-bit
    format on small sorts (the format switch clears the words)."""
    monkeypatch.setenv("RC_DEBUG_SORT_W64", "1")
    for src, n, ins in [(K.TREE_OFF_BY_ONE, 1024, I.cfg3_inputs(0, 6, 1024)),
                        (K.BENIGN["K_Btid"], 256, I.cfg2_inputs(0, 9, 256)),
                        (K.STENCIL, 3000, I.cfg5_inputs(0, 3, 3000))]:
        p, g, o = run_both(rc, src, n, ins)
        assert_parity(g, o, ins)
        p, g, o = run_both(rc, src, n, ins, keep_all_reads=True)
        assert_parity(g, o, ins)


@pytest.mark.parametrize("h", ["1", "2"])
def test_interp_lanes_per_thread(rc, monkeypatch, h):
    """K1 runs one or two work-items per thread (two only for large batches
    by default); RC_DEBUG_INTERP_H forces either so both are checked on small
    cases: ragged tiles, every report kind, divergence, overlay hits, loops."""
    monkeypatch.setenv("RC_DEBUG_INTERP_H", h)
    rng = np.random.default_rng(7 + int(h))
    for it in range(120):
        n = int(rng.integers(1, 600))
        pr = K.random_tiny_kernel(rng, n_arrays=2, n_regs=5, n_commands=int(rng.integers(3, 12)), size=5)
        ins = [rng.integers(-3, 4, size=(int(rng.integers(1, 4)), 5)).astype(np.int32)]
        ins.append(rng.integers(-3, 4, size=(ins[0].shape[0], 5)).astype(np.int32))
        p, g, o = run_both(rc, pr, n, ins, fuel=500)
        assert_parity(g, o, ins)
    for src, n, ins in [(K.TREE_OFF_BY_ONE, 1024, I.cfg3_inputs(0, 5, 1024)),
                        (K.BENIGN["K_last"], 256, I.cfg2_inputs(0, 9, 256)),
                        (K.STENCIL, 1000, I.cfg5_inputs(0, 3, 1000)),
                        (K.FIG1, 8, I.cfg1_inputs())]:
        p, g, o = run_both(rc, src, n, ins)
        assert_parity(g, o, ins)
    ins = I.cfg4_inputs(0, 2, 700)
    ins[3][:, 100:140] += 1
    p, g, o = run_both(rc, K.random_stencil_kernel(5), 700, ins)
    assert_parity(g, o, ins)


def test_deterministic_repeats(rc):
    """repeated runs are byte-identical."""
    ins = I.cfg4_inputs(0, 4, 300)
    ins[3][:, 50:60] += 1
    p = K.random_stencil_kernel(3)
    prog = rc.rc_load_program(p.bytecode)
    dev = [torch.from_numpy(x).cuda() for x in ins]
    a = rc.rc_run(prog, 300, dev)
    b = rc.rc_run(prog, 300, dev)
    assert a.reports.tobytes() == b.reports.tobytes()
    for x, y in zip(a.final, b.final):
        assert torch.equal(x, y)


@pytest.mark.parametrize("src,n,gen", [
    (K.FIG1, 8, lambda: I.cfg1_inputs()),
    (K.TREE_OFF_BY_ONE, 256, lambda: I.cfg3_inputs(0, 16, 256)),
    (K.BENIGN["K_inc"], 64, lambda: I.cfg2_inputs(0, 8, 64)),
    (K.STENCIL, 500, lambda: I.cfg5_inputs(0, 3, 500)),
])
def test_keep_all_reads_same_results(rc, src, n, gen):
    """RC_OPT_KEEP_ALL_READS (no write-set pruning before the sort) gives the
    same reports, heaps and counters as the default path and the oracle."""
    ins = gen()
    p, g, o = run_both(rc, src, n, ins, keep_all_reads=True)
    assert_parity(g, o, ins)


def test_random_tiny_kernels_keep_all_reads(rc):
    rng = np.random.default_rng(7)
    for it in range(100):
        n = int(rng.integers(1, 70))
        pr = K.random_tiny_kernel(rng, n_arrays=2, n_regs=5, n_commands=int(rng.integers(3, 12)), size=5)
        ins = [rng.integers(-3, 4, size=(2, 5)).astype(np.int32) for _ in range(2)]
        p, g, o = run_both(rc, pr, n, ins, fuel=500, keep_all_reads=True)
        assert_parity(g, o, ins)


def test_grow_and_retry_paths(rc, monkeypatch):
    """With RC_DEBUG_SMALL_BUFFERS the log and report buffers start tiny, so
    every interval overflows first and is re-run after growing (K1 retry from
    the saved lane state, detect re-run); results must be unchanged."""
    monkeypatch.setenv("RC_DEBUG_SMALL_BUFFERS", "1")
    cases = [(K.TREE_OFF_BY_ONE, 256, I.cfg3_inputs(0, 40, 256)),
             (K.BENIGN["K_inc"], 128, I.cfg2_inputs(0, 16, 128)),
             (K.FIG1, 8, I.cfg1_inputs())]
    for src, n, ins in cases:
        p, g, o = run_both(rc, src, n, ins)
        assert_parity(g, o, ins)
    ins = I.cfg4_inputs(0, 3, 300)
    ins[3][:, 20:60] += 1
    p, g, o = run_both(rc, K.random_stencil_kernel(2), 300, ins)
    assert_parity(g, o, ins)


# ------------------------------------------------------------------ work-groups (§8(f) row 3, reading L20)
def _groups_cases():
    lead = """
.arrays A P S
    lid   r0
    gid   r1
    lsize r2
    tid   r3
    const r4, 2
    div   r5, r2, r4
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
    ld    r8, A, r3
    st    P, r1, r8
    ld    r9, S, r6
    add   r9, r9, r8
    st    S, r6, r9
    addi  r11, r1, 1
    const r12, 3
    mod   r11, r11, r12
    ld    r13, P, r11
end:
    exit
"""
    return [(".arrays A\n lid r0\n gid r1\n st A, r0, r1\n exit\n", 4, 3,
             [np.zeros((2, 4), np.int32)]),
            (lead, 8, 3, [np.arange(1, 3 * 24 + 1, dtype=np.int32).reshape(3, 24), np.zeros((3, 3), np.int32),
                          np.zeros((3, 1), np.int32)]),
            (lead, 256, 3, [I.cfg3_inputs(0, 4, 768)[0], np.zeros((4, 3), np.int32), np.zeros((4, 1), np.int32)]),
            (K.TREE_OFF_BY_ONE, 64, 4, I.cfg3_inputs(0, 5, 64)),
            (K.FIG1, 8, 2, I.cfg1_inputs()),
            (K.many_writes_kernel(), 12, 3, [np.zeros((2, 64 * 12 + 6), np.int32), np.zeros((2, 12), np.int32)])]


@pytest.mark.parametrize("classify", [False, True])
def test_work_groups(rc, classify):
    """n_groups > 1 (groups one after another, inter-group races over the
    whole kernel) through the C ABI against the oracle: the hand-pinned
    kernels of test_oracle_pins, shared-array kernels with every report kind,
    random tiny kernels indexing by tid / lid / gid."""
    for src, n, G, ins in _groups_cases():
        _, g, o = run_both(rc, src, n, ins, n_groups=G, classify_rw=classify)
        assert_parity(g, o, ins)
        if "lsize" in (src if isinstance(src, str) else ""):  # the shared-partial kernel races across groups
            assert any(t[1] == 0xFFFFFFFF for t in o.report_tuples())
    rng = np.random.default_rng(404)
    for it in range(120):
        n = int(rng.integers(1, 40))
        G = int(rng.integers(2, 6))
        pr = K.random_tiny_kernel(rng, n_arrays=2, n_regs=5, n_commands=int(rng.integers(3, 12)), size=7,
                                  groups=True)
        ins = [rng.integers(-3, 4, size=(int(rng.integers(1, 4)), 7)).astype(np.int32)]
        ins.append(rng.integers(-3, 4, size=(ins[0].shape[0], 7)).astype(np.int32))
        _, g, o = run_both(rc, pr, n, ins, fuel=500, n_groups=G, classify_rw=classify)
        assert_parity(g, o, ins)


# ------------------------------------------------- grouping paths
def _grouping_cases(rng):
    """Cases that hit every branch of the log grouping: single-record cells
    only (stencil), multi-record cells (tree, benign suite, random kernels),
    report buffers that overflow (detect-only re-run), ragged bucket
    boundaries (cells per instance not a multiple of 4096)."""
    yield K.TREE_OFF_BY_ONE, 1024, I.cfg3_inputs(0, 24, 1024)
    yield K.BENIGN["K_inc"], 256, I.cfg2_inputs(0, 40, 256)
    yield K.BENIGN["K_Btid"], 256, I.cfg2_inputs(1, 33, 256)
    yield K.STENCIL, 5000, I.cfg5_inputs(0, 5, 5000)
    ins = I.cfg4_inputs(0, 6, 3000)
    ins[3][:, 100:180] += 1
    yield K.random_stencil_kernel(2), 3000, ins
    for it in range(40):
        n = int(rng.integers(1, 300))
        pr = K.random_tiny_kernel(rng, n_arrays=2, n_regs=5, n_commands=int(rng.integers(3, 12)), size=5)
        ins = [rng.integers(-3, 4, size=(int(rng.integers(1, 60)), 5)).astype(np.int32)]
        ins.append(rng.integers(-3, 4, size=(ins[0].shape[0], 5)).astype(np.int32))
        yield pr, n, ins


@pytest.mark.parametrize("path", ["bucket", "count", "lsd"])
def test_grouping_paths(rc, monkeypatch, path):
    """The bucket path (MSD scatter + per-bucket counting sort and detection,
    the default: fixed bucket regions, no count pass), its count mode
    (RC_BUCKET_COUNT=1; also taken after a bucket outgrew its region) and the
    onesweep LSD path (RC_SORT_LSD=1; also taken when one instance has more
    cells than the buckets cover) give the oracle's results, also when every
    buffer starts tiny (grow-and-retry, detect-only re-runs)."""
    if path == "lsd":
        monkeypatch.setenv("RC_SORT_LSD", "1")
    if path == "count":
        monkeypatch.setenv("RC_BUCKET_COUNT", "1")
    for small in (False, True):
        if small:
            monkeypatch.setenv("RC_DEBUG_SMALL_BUFFERS", "1")
        rng = np.random.default_rng(11)
        for src, n, ins in _grouping_cases(rng):
            p, g, o = run_both(rc, src, n, ins, fuel=500 if not isinstance(src, str) else 0)
            assert_parity(g, o, ins)


@pytest.mark.parametrize("n", [8193, 20000])
def test_oversized_bucket(rc, n):
    """A bucket with more records than its region (8192 slots) makes the host
    regroup the interval with the bucket counts, and one with more than the
    shared-memory capacity (8192) is counting-sorted in global scratch: every
    work-item reads and writes A[0] (K_inc: 2n records in one cell) and writes
    its own B cell."""
    src = """
.arrays A B
    tid   r0
    const r1, 0
    ld    r2, A, r1
    add   r3, r2, r0
    st    A, r1, r3
    st    B, r0, r3
    bar
    ld    r4, B, r0
    add   r5, r0, r1
    st    B, r5, r4
    exit
"""
    ins = [np.array([[5], [7]], np.int32), np.zeros((2, n), np.int32)]
    p, g, o = run_both(rc, src, n, ins)
    assert_parity(g, o, ins)
    for src2, ins2 in [(K.BENIGN["K_inc"], I.cfg2_inputs(0, 3, n)), (K.BENIGN["K_tid"], I.cfg2_inputs(0, 2, n))]:
        p, g, o = run_both(rc, src2, n, ins2)
        assert_parity(g, o, ins2)


def test_lsd_for_huge_instances(rc):
    """One instance with more cells than the buckets cover (> 2^25) takes the
    LSD path automatically; results as the oracle's."""
    n = 3000
    ins = I.cfg5_inputs(0, 1, n)
    big = [np.zeros((1, (1 << 24) + 7), np.int32) for _ in ins]
    for a, b in zip(ins, big):
        b[:, :a.shape[1]] = a
    p, g, o = run_both(rc, K.STENCIL, n, big)
    assert_parity(g, o, big)


def test_prepass_direct_commit(rc):
    """RC_OPT_PREPASS: runs the symbolic pre-pass proves
    conflict-free are interpreted in direct-commit mode with no grouping or
    detect kernels — same (no) reports, final heaps and stats as the oracle;
    runs it cannot prove take the normal path with the same results."""
    proved = [(K.STENCIL, 3000, I.cfg5_inputs(0, 6, 3000)), (K.TREE, 1024, I.cfg3_inputs(0, 20, 1024)),
              (K.PRIVATE_ONLY, 100, [np.arange(12, dtype=np.int32).reshape(3, 4)])]
    for src, n, ins in proved:
        p, g, o = run_both(rc, src, n, ins, prepass=True, profile=True)
        assert_parity(g, o, ins)
        assert g.profile["sort"]["launches"] == 0 and g.profile["hist"]["launches"] == 0, "direct mode not taken"
        assert g.profile["interp"]["launches"] > 0
    unproved = [(K.TREE_OFF_BY_ONE, 1024, I.cfg3_inputs(0, 10, 1024)), (K.BENIGN["K_c"], 256, I.cfg2_inputs(0, 8, 256)),
                (K.BENIGN["K_inc"], 64, I.cfg2_inputs(0, 8, 64)), (K.FIG1, 8, I.cfg1_inputs())]
    for src, n, ins in unproved:
        p, g, o = run_both(rc, src, n, ins, prepass=True)
        assert_parity(g, o, ins)
    rng = np.random.default_rng(5)
    for it in range(150):
        n = int(rng.integers(1, 300))
        pr = K.random_tiny_kernel(rng, n_arrays=2, n_regs=4, n_commands=int(rng.integers(2, 9)), size=5)
        ins = [rng.integers(-3, 4, size=(int(rng.integers(1, 5)), 5)).astype(np.int32)]
        ins.append(rng.integers(-3, 4, size=(ins[0].shape[0], 5)).astype(np.int32))
        p, g, o = run_both(rc, pr, n, ins, fuel=500, prepass=True)
        assert_parity(g, o, ins)
