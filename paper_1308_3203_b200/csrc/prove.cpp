// prove.cpp — rc_prove: the symbolic NoRace pre-pass (
// PAPER.md:318-447, Table 1 at P:345-368, NoRace at P:415-431).  Host only.
//
// The paper's symbolic execution runs ONE generic thread whose `tid` is a
// universally quantified variable, over sets of symbolic heaps
// (P:380-382); at a barrier it instantiates the parametric state for two
// distinct tids i != j (`rename`) and asks a prover (left
// unspecified) whether every pair of shared locations that cannot
// be proved disjoint holds provably equal values (NoRace).
//
// Here, for one concrete run shape (work-group size n, array sizes):
//  * symbolic values are hash-consed terms: affine forms k0 + k1*tid (mod
//    2^32: the int32 wrap of reading L7 is exact on them), loads of the
//    interval-start heap `load(k, a, e)` (the heap of interval k is opaque:
//    any input), and other operations over those;
//  * a symbolic state = (pc, registers, path condition = atoms `t != 0` /
//    `t == 0` from BR / ASSUME), one generic thread (Table 1: assign, load,
//    store into the own-write overlay with the last-value rule L3, assume,
//    assert, and the out-of-bounds rule `C(a[e]) -> ⊥`); BR forks (the
//    assume(b) / assume(¬b) pair); at a barrier the states with equal
//    live registers are merged keeping their common atoms (an
//    over-approximation, as the paper's sets of symbolic heaps);
//  * the prover is a decision procedure over the concrete range: an atom or
//    an index is evaluated for every tid in [0, n) (unknown when it depends on
//    a load: then "possibly true"); two accesses of an interval conflict when
//    some tids i != j that may follow their paths hit the same cell
//    (`disjoint` fails); the values of two writes are provably equal
//    (`compare`) when their terms instantiated at i and j coincide.
// Verdict (include/rc.h): RC_PROVE_NO_CONFLICT — no access conflict, no ⊥, no
// divergence in any interval for ANY input, so rc_run would report nothing;
// RC_PROVE_NORACE — additionally write-write conflicts are possible but every
// one is provably benign (the paper's NoRace: the shared state at every
// barrier is deterministic); RC_PROVE_UNKNOWN — nothing proved (run the
// checker), with the reason.  The prover is sound, not complete: any
// construct it does not model (data-dependent indices or loops, aliasing in a
// work-item's own writes, budgets) yields UNKNOWN.
#include <algorithm>
#include <cstring>
#include <unordered_map>

#include "rc_internal.h"

namespace rc {
int fail(int code, const char* fmt, ...);

namespace {
using u32 = uint32_t;
using u64 = uint64_t;

enum TermKind : uint8_t { T_AFF = 0, T_LOAD = 1, T_OP = 2 };
struct Term {
  uint8_t kind, op;
  u32 k0, k1;      // T_AFF: k0 + k1 * tid (mod 2^32)
  int region, arr; // T_LOAD
  int x, y;        // T_LOAD: x = index term; T_OP: operands (y = -1 for unary)
  bool tid_free;   // the DAG holds no affine form with k1 != 0
  bool evaluable;  // the DAG holds no load
};

struct Key {  // (no padding: compared and hashed byte-wise)
  u32 kind_op, k0, k1;
  int region, arr, x, y;
  bool operator==(const Key& o) const { return memcmp(this, &o, sizeof(Key)) == 0; }
};
static_assert(sizeof(Key) == 28, "Key has no padding");
struct KeyHash {
  size_t operator()(const Key& k) const {
    uint64_t h = 1469598103934665603ull;
    const unsigned char* p = reinterpret_cast<const unsigned char*>(&k);
    for (size_t i = 0; i < sizeof(Key); i++) h = (h ^ p[i]) * 1099511628211ull;
    return (size_t)h;
  }
};

struct Unknown {  // thrown: the prover gives up with a reason
  uint32_t reason;
  uint32_t pc;
};

int32_t alu(uint8_t op, int32_t x, int32_t y) {  // reading L7 (y != 0 for DIV / MOD)
  const uint32_t ux = (uint32_t)x, uy = (uint32_t)y;
  switch (op) {
    case RC_OP_ADD: return (int32_t)(ux + uy);
    case RC_OP_SUB: return (int32_t)(ux - uy);
    case RC_OP_MUL: return (int32_t)(ux * uy);
    case RC_OP_DIV: return y == -1 ? (int32_t)(0u - ux) : x / y;
    case RC_OP_MOD: return y == -1 ? 0 : x % y;
    case RC_OP_MIN: return x < y ? x : y;
    case RC_OP_MAX: return x > y ? x : y;
    case RC_OP_AND: return x & y;
    case RC_OP_OR: return x | y;
    case RC_OP_XOR: return x ^ y;
    case RC_OP_LT: return x < y;
    case RC_OP_EQ: return x == y;
    case RC_OP_LAND: return x != 0 && y != 0;
    case RC_OP_LNOT: return x == 0;
    default: return 0;
  }
}

struct Prover {
  const rc_program* P;
  u32 n;
  std::vector<u32> size;
  u64 fuel, max_intervals, budget;
  u64 work = 0;
  int depth = 0;  // forks explored recursively (bounded)
  std::vector<Term> T;
  std::unordered_map<Key, int, KeyHash> index;
  std::vector<uint8_t> live;  // registers live across some barrier

  int intern(const Key& k, const Term& t) {
    auto it = index.find(k);
    if (it != index.end()) return it->second;
    T.push_back(t);
    index.emplace(k, (int)T.size() - 1);
    return (int)T.size() - 1;
  }
  int aff(u32 k0, u32 k1) {
    Key k{T_AFF, k0, k1, 0, 0, 0, 0};
    Term t{T_AFF, 0, k0, k1, 0, 0, -1, -1, k1 == 0, true};
    return intern(k, t);
  }
  int load(int region, int arr, int idx) {
    Key k{T_LOAD, 0, 0, region, arr, idx, -1};
    Term t{T_LOAD, 0, 0, 0, region, arr, idx, -1, T[idx].tid_free, false};
    return intern(k, t);
  }
  bool is_const(int x, int32_t* v) const {
    if (T[x].kind != T_AFF || T[x].k1 != 0) return false;
    *v = (int32_t)T[x].k0;
    return true;
  }
  // op(x, y): affine forms stay affine under +, -, * by a constant; constants fold
  int op2(uint8_t op, int x, int y, u32 pc) {
    int32_t cx, cy;
    const bool kx = is_const(x, &cx), ky = is_const(y, &cy);
    if (kx && ky) {
      if ((op == RC_OP_DIV || op == RC_OP_MOD) && cy == 0) throw Unknown{RC_PROVE_R_DIV0, pc};
      return aff((u32)alu(op, cx, cy), 0);
    }
    const Term &a = T[x], &b = T[y];
    if (a.kind == T_AFF && b.kind == T_AFF) {
      if (op == RC_OP_ADD) return aff(a.k0 + b.k0, a.k1 + b.k1);
      if (op == RC_OP_SUB) return aff(a.k0 - b.k0, a.k1 - b.k1);
      if (op == RC_OP_MUL && b.k1 == 0) return aff(a.k0 * b.k0, a.k1 * b.k0);
      if (op == RC_OP_MUL && a.k1 == 0) return aff(a.k0 * b.k0, b.k1 * a.k0);
    }
    Key k{T_OP | (u32)op << 8, 0, 0, 0, 0, x, y};
    Term t{T_OP, op, 0, 0, 0, 0, x, y, a.tid_free && (y < 0 || b.tid_free), a.evaluable && (y < 0 || b.evaluable)};
    return intern(k, t);
  }
  int op1(uint8_t op, int x) {  // LNOT
    int32_t c;
    if (is_const(x, &c)) return aff((u32)alu(op, c, 0), 0);
    Key k{T_OP | (u32)op << 8, 0, 0, 0, 0, x, -1};
    Term t{T_OP, op, 0, 0, 0, 0, x, -1, T[x].tid_free, T[x].evaluable};
    return intern(k, t);
  }
  // the value of term x for thread i (false: it depends on a load, or divides by 0)
  bool eval(int x, u32 i, int32_t* out) const {
    const Term& t = T[x];
    if (t.kind == T_AFF) {
      *out = (int32_t)(t.k0 + t.k1 * i);
      return true;
    }
    if (!t.evaluable) return false;
    int32_t a = 0, b = 0;
    if (!eval(t.x, i, &a)) return false;
    if (t.y >= 0 && !eval(t.y, i, &b)) return false;
    if ((t.op == RC_OP_DIV || t.op == RC_OP_MOD) && b == 0) return false;
    *out = alu(t.op, a, b);
    return true;
  }
  // compare: x at thread i and y at thread j denote the same value for every input
  bool same(int x, u32 i, int y, u32 j) const {
    if (x == y && T[x].tid_free) return true;
    const Term &a = T[x], &b = T[y];
    if (a.evaluable && b.evaluable) {
      int32_t va, vb;
      if (eval(x, i, &va) && eval(y, j, &vb)) return va == vb;
    }
    if (a.kind != b.kind || a.op != b.op) return false;
    if (a.kind == T_LOAD) return a.region == b.region && a.arr == b.arr && same(a.x, i, b.x, j);
    if (a.kind == T_OP) return same(a.x, i, b.x, j) && (a.y < 0 || same(a.y, i, b.y, j));
    return false;
  }

  struct Atom {
    int t;
    bool truth;  // (t != 0) == truth
  };
  struct Access {
    bool write;
    int arr, idx, val;
  };
  struct Own {
    int arr, idx, val;
  };
  struct State {
    u32 pc = 0;
    std::vector<int> regs;
    std::vector<Atom> path;
    std::vector<Access> acc;  // this interval: reads as performed, writes at the end (final values)
    std::vector<Own> own;
    u64 steps = 0;
    int end = 0;  // 0 running, 1 at a barrier (pc = after it), 2 exit, 3 pruned
  };

  // may thread i follow a state's path? (an atom over a load: possibly)
  bool possible(const std::vector<Atom>& path, u32 i) const {
    for (const Atom& a : path) {
      int32_t v;
      if (eval(a.t, i, &v) && ((v != 0) != a.truth)) return false;
    }
    return true;
  }
  void charge(u64 w, u32 pc) {
    work += w;
    if (work > budget) throw Unknown{RC_PROVE_R_BUDGET, pc};
  }
  bool satisfiable(const std::vector<Atom>& path, u32 pc) {
    charge(n, pc);
    for (u32 i = 0; i < n; i++)
      if (possible(path, i)) return true;
    return false;
  }
  // every thread that may follow the path satisfies pred(value of x)
  template <class F>
  void require_all(const State& s, int x, F pred, uint32_t reason, u32 pc) {
    int32_t c;
    if (is_const(x, &c)) {
      if (!pred(c) && satisfiable(s.path, pc)) throw Unknown{reason, pc};
      return;
    }
    charge(n, pc);
    for (u32 i = 0; i < n; i++) {
      if (!possible(s.path, i)) continue;
      int32_t v;
      if (!eval(x, i, &v)) throw Unknown{reason == RC_PROVE_R_OOB ? RC_PROVE_R_DATA_INDEX : reason, pc};
      if (!pred(v)) throw Unknown{reason, pc};
    }
  }
  // might x and y (a work-item's own two indices) denote one cell for some thread of the path?
  bool may_alias(const State& s, int x, int y, u32 pc) {
    if (x == y) return true;
    charge(n, pc);
    for (u32 i = 0; i < n; i++) {
      if (!possible(s.path, i)) continue;
      int32_t a, b;
      if (!eval(x, i, &a) || !eval(y, i, &b) || a == b) return true;
    }
    return false;
  }
  int own_lookup(State& s, int arr, int idx, u32 pc) {  // -1: not written by this work-item
    int hit = -1;
    for (size_t k = 0; k < s.own.size(); k++) {
      if (s.own[k].arr != arr) continue;
      if (s.own[k].idx == idx) hit = (int)k;
      else if (may_alias(s, s.own[k].idx, idx, pc)) throw Unknown{RC_PROVE_R_OWN_ALIAS, pc};
    }
    return hit;
  }

  // run one state to the end of its interval; forks are appended to `out`
  void run(State s, int region, std::vector<State>& out) {
    const std::vector<Ins>& code = P->code;
    for (;;) {
      const u32 pc = s.pc;
      const Ins& I = code[pc];
      if (++s.steps > fuel) throw Unknown{RC_PROVE_R_FUEL, pc};
      charge(1, pc);
      auto R = [&](uint8_t r) { return s.regs[r]; };
      switch (I.op) {
        case RC_OP_CONST: s.regs[I.a] = aff((u32)I.imm, 0); s.pc++; break;
        case RC_OP_MOV: s.regs[I.a] = R(I.b); s.pc++; break;
        case RC_OP_TID: s.regs[I.a] = aff(0, 1); s.pc++; break;
        case RC_OP_LID: s.regs[I.a] = aff(0, 1); s.pc++; break;
        case RC_OP_GID: s.regs[I.a] = aff(0, 0); s.pc++; break;
        case RC_OP_LSIZE: s.regs[I.a] = aff(n, 0); s.pc++; break;
        case RC_OP_SIZE: s.regs[I.a] = aff(size[I.b], 0); s.pc++; break;
        case RC_OP_ADDI: s.regs[I.a] = op2(RC_OP_ADD, R(I.b), aff((u32)I.imm, 0), pc); s.pc++; break;
        case RC_OP_LNOT: s.regs[I.a] = op1(RC_OP_LNOT, R(I.b)); s.pc++; break;
        case RC_OP_DIV: case RC_OP_MOD:
          require_all(s, R(I.c), [](int32_t v) { return v != 0; }, RC_PROVE_R_DIV0, pc);
          s.regs[I.a] = op2(I.op, R(I.b), R(I.c), pc);
          s.pc++;
          break;
        case RC_OP_ADD: case RC_OP_SUB: case RC_OP_MUL: case RC_OP_MIN: case RC_OP_MAX: case RC_OP_AND:
        case RC_OP_OR: case RC_OP_XOR: case RC_OP_LT: case RC_OP_EQ: case RC_OP_LAND:
          s.regs[I.a] = op2(I.op, R(I.b), R(I.c), pc);
          s.pc++;
          break;
        case RC_OP_LD: {  // v := a[e] (reading L11): own write, else the interval-start heap
          const int idx = R(I.c);
          const u32 sz = size[I.b];
          require_all(s, idx, [sz](int32_t v) { return (uint32_t)v < sz; }, RC_PROVE_R_OOB, pc);
          const int k = own_lookup(s, I.b, idx, pc);
          s.regs[I.a] = k >= 0 ? s.own[k].val : load(region, I.b, idx);
          s.acc.push_back({false, I.b, idx, -1});
          s.pc++;
          break;
        }
        case RC_OP_ST: {  // a[e] := e': the own-write overlay, last value (L3)
          const int idx = R(I.b);
          const u32 sz = size[I.a];
          require_all(s, idx, [sz](int32_t v) { return (uint32_t)v < sz; }, RC_PROVE_R_OOB, pc);
          const int k = own_lookup(s, I.a, idx, pc);
          if (k >= 0) s.own[k].val = R(I.c);
          else s.own.push_back({I.a, idx, R(I.c)});
          s.pc++;
          break;
        }
        case RC_OP_ASSUME: {  // false: the work-item stops silently (⊤, reading L6)
          int32_t c;
          if (is_const(R(I.a), &c)) {
            if (!c) { s.end = 3; out.push_back(std::move(s)); return; }
          } else {
            s.path.push_back({R(I.a), true});
            if (!satisfiable(s.path, pc)) { s.end = 3; out.push_back(std::move(s)); return; }
          }
          s.pc++;
          break;
        }
        case RC_OP_ASSERT:
          require_all(s, R(I.a), [](int32_t v) { return v != 0; }, RC_PROVE_R_ASSERT, pc);
          s.pc++;
          break;
        case RC_OP_BR: {  // the assume(b) / assume(¬b) pair: fork unless b is decided
          const u32 tt = (u32)I.imm, ff = I.b + 256u * I.c;
          int32_t c;
          if (is_const(R(I.a), &c)) { s.pc = c ? tt : ff; break; }
          State f = s;
          f.path.push_back({R(I.a), false});
          f.pc = ff;
          s.path.push_back({R(I.a), true});
          s.pc = tt;
          const bool ok_f = satisfiable(f.path, pc), ok_t = satisfiable(s.path, pc);
          if (ok_f && ok_t) {
            if (out.size() + 2 > 4096 || depth >= 256) throw Unknown{RC_PROVE_R_BUDGET, pc};
            depth++;
            run(std::move(f), region, out);  // (depth-first; the taken side continues here)
            depth--;
          } else if (ok_f) {
            s = std::move(f);
          } else if (!ok_t) {
            s.end = 3;
            out.push_back(std::move(s));
            return;
          }
          break;
        }
        case RC_OP_JMP: s.pc = (u32)I.imm; break;
        case RC_OP_BAR: s.end = 1; s.pc++; finish(s); out.push_back(std::move(s)); return;
        case RC_OP_EXIT: s.end = 2; finish(s); out.push_back(std::move(s)); return;
        default: throw Unknown{RC_PROVE_R_UNSUPPORTED, pc};
      }
    }
  }
  static void finish(State& s) {  // one write per distinct cell, its final value (L3)
    for (const Own& o : s.own) s.acc.push_back({true, o.arr, o.idx, o.val});
    s.own.clear();
  }

  // NoRace over the interval's states, and the access conflicts
  // the concrete checker reports: returns true when a write-write
  // conflict is possible (all of them provably benign)
  bool check_interval(const std::vector<State>& st, u32* reason_pc) {
    // barrier divergence (reading L9): the satisfiable states must end at one node
    int node = -2;
    for (const State& s : st) {
      if (s.end == 3) continue;
      const int nd = s.end == 2 ? -1 : (int)s.pc - 1;
      if (node == -2) node = nd;
      else if (nd != node) throw Unknown{RC_PROVE_R_DIVERGENCE, (u32)std::max(nd, node)};
    }
    struct Hit {
      u32 cell, tid;
      int s, a;  // state, access
    };
    std::vector<Hit> hits;
    bool ww = false;
    for (u32 arr = 0; arr < P->n_arrays; arr++) {
      hits.clear();
      for (size_t si = 0; si < st.size(); si++) {
        const State& s = st[si];
        if (s.end == 3) continue;
        for (size_t ai = 0; ai < s.acc.size(); ai++) {
          const Access& A = s.acc[ai];
          if ((u32)A.arr != arr) continue;
          charge(n, 0);
          for (u32 i = 0; i < n; i++) {
            if (!possible(s.path, i)) continue;
            int32_t c;
            if (!eval(A.idx, i, &c)) throw Unknown{RC_PROVE_R_DATA_INDEX, 0};
            hits.push_back({(u32)c, i, (int)si, (int)ai});
          }
        }
      }
      std::sort(hits.begin(), hits.end(), [](const Hit& x, const Hit& y) {
        return x.cell != y.cell ? x.cell < y.cell : x.tid < y.tid;
      });
      for (size_t b = 0; b < hits.size();) {
        size_t e = b;
        while (e < hits.size() && hits[e].cell == hits[b].cell) e++;
        // readers / writers of this cell (a tid may appear in several states: its path is undecided)
        const Hit* w0 = nullptr;
        u32 rmin = 0xFFFFFFFFu, rmax = 0;
        bool has_r = false;
        for (size_t k = b; k < e; k++) {
          const Access& A = st[hits[k].s].acc[hits[k].a];
          if (!A.write) {
            has_r = true;
            rmin = std::min(rmin, hits[k].tid);
            rmax = std::max(rmax, hits[k].tid);
          } else if (!w0) {
            w0 = &hits[k];
          }
        }
        for (size_t k = b; k < e && w0; k++) {
          const Access& A = st[hits[k].s].acc[hits[k].a];
          if (!A.write) continue;
          const u32 t = hits[k].tid;
          // RW: a reader other than this writer
          if (has_r && (rmin != t || rmax != t)) { *reason_pc = 0; throw Unknown{RC_PROVE_R_RW, 0}; }
          // WW: two writers must write provably equal values (benign)
          if (t != w0->tid) {
            const Access& W0 = st[w0->s].acc[w0->a];
            if (!same(W0.val, w0->tid, A.val, t)) throw Unknown{RC_PROVE_R_WW, 0};
            ww = true;
          }
        }
        b = e;
      }
    }
    return ww;
  }

  // merge the states waiting at one barrier whose live registers are equal
  // (their path: the atoms they share — a superset of their threads)
  void merge(std::vector<State>& st) {
    std::vector<State> m;
    for (State& s : st) {
      if (s.end != 1) continue;
      for (size_t r = 0; r < s.regs.size(); r++)
        if (!live[r]) s.regs[r] = -1;
      s.acc.clear();
      bool done = false;
      for (State& o : m) {
        if (o.pc != s.pc || o.regs != s.regs) continue;
        std::vector<Atom> common;
        for (const Atom& a : o.path)
          for (const Atom& b : s.path)
            if (a.t == b.t && a.truth == b.truth) { common.push_back(a); break; }
        o.path = std::move(common);
        done = true;
        break;
      }
      if (!done) m.push_back(std::move(s));
    }
    st = std::move(m);
  }

  void prove(rc_prove_result* out) {
    live.assign(P->n_regs, 0);
    for (uint8_t r : P->live_regs) live[r] = 1;
    State s0;
    s0.regs.assign(P->n_regs, aff(0, 0));  // registers start at 0 (reading L18)
    std::vector<State> cur{s0};
    bool ww = false;
    u32 region = 0;
    while (!cur.empty()) {
      if (region >= max_intervals) throw Unknown{RC_PROVE_R_FUEL, 0};
      std::vector<State> ended;
      for (State& s : cur) {
        s.steps = 0;
        run(std::move(s), (int)region, ended);
      }
      u32 rpc = 0;
      ww |= check_interval(ended, &rpc);
      merge(ended);  // the states waiting at the barrier continue
      cur = std::move(ended);
      region++;
      out->intervals = region;
    }
    out->verdict = ww ? RC_PROVE_NORACE : RC_PROVE_NO_CONFLICT;
  }
};

}  // namespace
}  // namespace rc

extern "C" int rc_prove(const rc_program* prog, uint32_t work_group_size, const uint32_t* sizes, uint32_t n_arrays,
                        uint64_t fuel_per_interval, uint64_t budget, rc_prove_result* out) {
  if (!out) return rc::fail(RC_EINVAL, "out is NULL");
  memset(out, 0, sizeof *out);
  if (!prog) return rc::fail(RC_EINVAL, "program is NULL");
  if (n_arrays != prog->n_arrays) return rc::fail(RC_EINVAL, "n_arrays %u != program's %u", n_arrays, prog->n_arrays);
  if (n_arrays && !sizes) return rc::fail(RC_EINVAL, "sizes is NULL");
  if (work_group_size == 0 || work_group_size > rc::MAX_WG)
    return rc::fail(RC_EINVAL, "work_group_size %u outside 1..2^27", work_group_size);
  rc::Prover pv;
  pv.P = prog;
  pv.n = work_group_size;
  pv.size.assign(sizes, sizes + n_arrays);
  pv.fuel = fuel_per_interval ? fuel_per_interval : (1ull << 20);
  pv.max_intervals = 65536;
  pv.budget = budget ? budget : (1ull << 32);
  try {
    pv.prove(out);
  } catch (const rc::Unknown& u) {
    out->verdict = RC_PROVE_UNKNOWN;
    out->reason = u.reason;
    out->pc = u.pc;
  } catch (const std::bad_alloc&) {
    out->verdict = RC_PROVE_UNKNOWN;
    out->reason = RC_PROVE_R_BUDGET;
  }
  out->terms = pv.T.size();
  out->work = pv.work;
  return RC_OK;
}
