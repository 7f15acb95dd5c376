// program.cpp — rc_load_program: RCB1 decode + CFG validation (host only).
//
// The bytecode encodes a kernel K(Args) = (tid, C, ->, Locals)
// as a control-flow graph: instruction nodes, successors given by fall-through,
// BR (the assume(b)/assume(¬b) successor pair) and JMP, a unique start (pc 0)
// and the exit node (every EXIT instruction).  Validation guarantees the
// interpreter never reads outside the program, registers or array table.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>

#include "rc_internal.h"

namespace rc {
thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

void analyze(rc_program* P);

static uint32_t rd32(const uint8_t* p) { uint32_t v; memcpy(&v, p, 4); return v; }
static uint16_t rd16(const uint8_t* p) { uint16_t v; memcpy(&v, p, 2); return v; }

static const char* op_name(int op) {
  static const char* names[] = {"?", "CONST", "MOV", "TID", "SIZE", "ADD", "SUB", "MUL", "DIV", "MOD", "MIN",
                                "MAX", "AND", "OR", "XOR", "LT", "EQ", "LAND", "LNOT", "LD", "ST", "BAR",
                                "ASSUME", "ASSERT", "BR", "JMP", "EXIT", "ADDI", "GID", "LID", "LSIZE"};
  return (op >= 1 && op <= RC_OP_LSIZE) ? names[op] : "?";
}

// register / array operands of each opcode: 'r' register, 'a' array, '-' unused
static const char* operand_kinds(int op) {
  switch (op) {
    case RC_OP_CONST: case RC_OP_TID: case RC_OP_GID: case RC_OP_LID: case RC_OP_LSIZE: return "r--";
    case RC_OP_MOV: case RC_OP_LNOT: case RC_OP_ADDI: return "rr-";
    case RC_OP_SIZE: return "ra-";
    case RC_OP_ADD: case RC_OP_SUB: case RC_OP_MUL: case RC_OP_DIV: case RC_OP_MOD: case RC_OP_MIN:
    case RC_OP_MAX: case RC_OP_AND: case RC_OP_OR: case RC_OP_XOR: case RC_OP_LT: case RC_OP_EQ:
    case RC_OP_LAND: return "rrr";
    case RC_OP_LD: return "rar";
    case RC_OP_ST: return "arr";
    case RC_OP_ASSUME: case RC_OP_ASSERT: case RC_OP_BR: return "r--";
    case RC_OP_BAR: case RC_OP_JMP: case RC_OP_EXIT: return "---";
    default: return nullptr;
  }
}

int validate(const uint8_t* bc, size_t nbytes, rc_program* P) {
  if (!bc) return fail(RC_EINVAL, "bytecode pointer is NULL");
  if (nbytes < 16) return fail(RC_EINVAL, "bytecode shorter than the 16-byte header (%zu bytes)", nbytes);
  if (rd32(bc) != RC_MAGIC) return fail(RC_EINVAL, "bad magic 0x%08x (expected 'RCB1')", rd32(bc));
  if (rd16(bc + 4) != 1) return fail(RC_EINVAL, "unsupported version %u", rd16(bc + 4));
  if (rd16(bc + 6) != 0) return fail(RC_EINVAL, "header flags must be 0 (got %u)", rd16(bc + 6));
  uint32_t n_regs = rd16(bc + 8), n_arrays = rd16(bc + 10), n_instr = rd32(bc + 12);
  if (n_regs < 1 || n_regs > 256) return fail(RC_EINVAL, "n_regs %u outside 1..256", n_regs);
  if (n_arrays > 256) return fail(RC_EINVAL, "n_arrays %u > 256", n_arrays);
  if (n_instr < 1 || n_instr > 65536) return fail(RC_EINVAL, "n_instr %u outside 1..65536", n_instr);
  if (nbytes != 16 + 8 * (size_t)n_instr)
    return fail(RC_EINVAL, "size mismatch: %zu bytes for %u instructions (expected %zu)", nbytes, n_instr,
                16 + 8 * (size_t)n_instr);
  std::vector<Ins> code(n_instr);
  memcpy(code.data(), bc + 16, 8 * (size_t)n_instr);
  for (uint32_t pc = 0; pc < n_instr; pc++) {
    const Ins& I = code[pc];
    const char* k = operand_kinds(I.op);
    if (!k) return fail(RC_EINVAL, "pc %u: unknown opcode %u", pc, I.op);
    const uint8_t f[3] = {I.a, I.b, I.c};
    for (int j = 0; j < 3; j++) {
      if (k[j] == 'r' && f[j] >= n_regs)
        return fail(RC_EINVAL, "pc %u (%s): register r%u >= n_regs %u", pc, op_name(I.op), f[j], n_regs);
      if (k[j] == 'a' && f[j] >= n_arrays)
        return fail(RC_EINVAL, "pc %u (%s): array %u >= n_arrays %u", pc, op_name(I.op), f[j], n_arrays);
    }
    if (I.op == RC_OP_BR) {
      uint32_t t = (uint32_t)I.imm, e = (uint32_t)I.b + 256u * I.c;
      if (I.imm < 0 || t >= n_instr) return fail(RC_EINVAL, "pc %u (BR): true target %d >= n_instr %u", pc, I.imm, n_instr);
      if (e >= n_instr) return fail(RC_EINVAL, "pc %u (BR): false target %u >= n_instr %u", pc, e, n_instr);
    }
    if (I.op == RC_OP_JMP && (I.imm < 0 || (uint32_t)I.imm >= n_instr))
      return fail(RC_EINVAL, "pc %u (JMP): target %d >= n_instr %u", pc, I.imm, n_instr);
  }
  // reachability from start (pc 0): no fall-through off the end, some EXIT reachable
  std::vector<uint8_t> seen(n_instr, 0);
  std::vector<uint32_t> stack{0};
  bool exit_reachable = false;
  seen[0] = 1;
  while (!stack.empty()) {
    uint32_t pc = stack.back();
    stack.pop_back();
    const Ins& I = code[pc];
    uint32_t succ[2];
    int ns = 0;
    if (I.op == RC_OP_EXIT) { exit_reachable = true; continue; }
    if (I.op == RC_OP_BR) { succ[ns++] = (uint32_t)I.imm; succ[ns++] = (uint32_t)I.b + 256u * I.c; }
    else if (I.op == RC_OP_JMP) succ[ns++] = (uint32_t)I.imm;
    else {
      if (pc + 1 >= n_instr)
        return fail(RC_EINVAL, "pc %u (%s): execution falls off the end of the program", pc, op_name(I.op));
      succ[ns++] = pc + 1;
    }
    for (int j = 0; j < ns; j++)
      if (!seen[succ[j]]) { seen[succ[j]] = 1; stack.push_back(succ[j]); }
  }
  if (!exit_reachable) return fail(RC_EINVAL, "no EXIT instruction is reachable from pc 0");
  P->n_regs = n_regs;
  P->n_arrays = n_arrays;
  P->n_instr = n_instr;
  P->code = std::move(code);
  analyze(P);
  return RC_OK;
}

// ---- static analysis used to size the interpreter (no semantic effect) ------
//
// (1) Registers live across a barrier: a work-item suspended at BAR b resumes
//     at b+1 in the next interval (a new kernel launch), so only registers in
//     live_in(b+1) — possibly read before redefined — must be saved / reloaded;
//     interval 0 starts at pc 0 with all registers 0 (reading L18), so
//     live_in(0) is loaded too (from the zeroed buffer).
// (2) Bound on distinct cells one work-item writes in one interval: the max
//     number of ST executions on a barrier-free path (unbounded if a
//     barrier-free cycle contains a ST).  Sizes the own-write overlay.
// (3) Bound on log records per work-item per interval (LD executions + (2)),
//     sizing the per-warp staging buffer (overflow is handled either way),
//     and on executed instructions per work-item per interval (every node of a
//     barrier-free path, its final BAR / EXIT included): when it is <= the
//     fuel no work-item can exhaust its fuel, so K1 skips the per-instruction
//     check (the FUEL report cannot occur).
// (4) K1 issues every heap LD as an asynchronous copy (cp.async) straight into
//     the destination register and waits for its outstanding copies only
//     before an instruction that may read or write a register some pending
//     load targets: a forward may-analysis of pending load targets; an
//     instruction flagged OP_WAIT empties the set, BAR / EXIT end the interval
//     (the lane waits for everything there).  The flag travels in the device
//     copy of the program (dev_code).
// (5) Per interval entry, the arrays no instruction of its barrier-free region
//     stores to (entry_ro; see the comment at the computation).
static void successors(const Ins& I, uint32_t pc, uint32_t n_instr, uint32_t* s, int* ns) {
  *ns = 0;
  if (I.op == RC_OP_EXIT) return;
  if (I.op == RC_OP_BR) { s[(*ns)++] = (uint32_t)I.imm; s[(*ns)++] = (uint32_t)I.b + 256u * I.c; return; }
  if (I.op == RC_OP_JMP) { s[(*ns)++] = (uint32_t)I.imm; return; }
  if (pc + 1 < n_instr) s[(*ns)++] = pc + 1;
}

static void uses_defs(const Ins& I, int* use, int* nu, int* def) {
  *nu = 0;
  *def = -1;
  const char* k = operand_kinds(I.op);
  switch (I.op) {
    case RC_OP_ST: use[(*nu)++] = I.b; use[(*nu)++] = I.c; return;
    case RC_OP_LD: use[(*nu)++] = I.c; *def = I.a; return;
    case RC_OP_ASSUME: case RC_OP_ASSERT: case RC_OP_BR: use[(*nu)++] = I.a; return;
    case RC_OP_BAR: case RC_OP_JMP: case RC_OP_EXIT: return;
    default: break;
  }
  *def = I.a;  // every remaining opcode writes register a
  if (k[1] == 'r') use[(*nu)++] = I.b;
  if (k[2] == 'r') use[(*nu)++] = I.c;
}

// Longest barrier-free path weight from any interval entry (pc 0 or BAR+1);
// -1 = unbounded.  Tarjan SCCs of the barrier-free CFG (edges out of BAR and
// EXIT removed): a cyclic SCC with positive weight is unbounded, otherwise DP
// over the condensation (Tarjan emits SCCs in reverse topological order).
// from >= 0: the longest path from that entry only.
static int64_t max_path_weight(const rc_program* P, const std::vector<int>& w, int64_t from = -1) {
  const uint32_t N = P->n_instr;
  auto succ = [&](uint32_t pc, uint32_t* s, int* ns) {
    successors(P->code[pc], pc, N, s, ns);
    if (P->code[pc].op == RC_OP_BAR) *ns = 0;
  };
  std::vector<int64_t> index(N, -1), low(N, 0), comp(N, -1);
  std::vector<uint8_t> on(N, 0);
  std::vector<uint32_t> stk;
  std::vector<int64_t> comp_best;
  int64_t idx = 0;
  bool unbounded = false;
  for (uint32_t root = 0; root < N; root++) {
    if (index[root] >= 0) continue;
    std::vector<std::pair<uint32_t, int>> call{{root, 0}};
    index[root] = low[root] = idx++;
    stk.push_back(root);
    on[root] = 1;
    while (!call.empty()) {
      uint32_t pc = call.back().first;
      int& i = call.back().second;
      uint32_t s[2];
      int ns;
      succ(pc, s, &ns);
      if (i < ns) {
        uint32_t q = s[i++];
        if (index[q] < 0) {
          index[q] = low[q] = idx++;
          stk.push_back(q);
          on[q] = 1;
          call.push_back({q, 0});
        } else if (on[q]) {
          low[pc] = std::min(low[pc], index[q]);
        }
        continue;
      }
      if (low[pc] == index[pc]) {  // pc roots an SCC; successors' SCCs are complete
        const int64_t c = (int64_t)comp_best.size();
        std::vector<uint32_t> members;
        uint32_t x;
        do {
          x = stk.back();
          stk.pop_back();
          on[x] = 0;
          comp[x] = c;
          members.push_back(x);
        } while (x != pc);
        int64_t weight = 0, out = 0;
        bool cyclic = members.size() > 1;
        for (uint32_t m : members) {
          weight += w[m];
          uint32_t s2[2];
          int n2;
          succ(m, s2, &n2);
          for (int j = 0; j < n2; j++) {
            if (s2[j] == m) cyclic = true;
            if (comp[s2[j]] != c && comp[s2[j]] >= 0) out = std::max(out, comp_best[comp[s2[j]]]);
          }
        }
        if (cyclic && weight > 0) unbounded = true;
        comp_best.push_back(weight + out);
      }
      call.pop_back();
      if (!call.empty()) low[call.back().first] = std::min(low[call.back().first], low[pc]);
    }
  }
  if (unbounded) return -1;
  if (from >= 0) return comp_best[comp[from]];
  int64_t m = comp_best[comp[0]];
  for (uint32_t pc = 0; pc + 1 < N; pc++)
    if (P->code[pc].op == RC_OP_BAR) m = std::max(m, comp_best[comp[pc + 1]]);
  return m;
}

void analyze(rc_program* P) {
  const uint32_t N = P->n_instr, R = P->n_regs;
  // (1) liveness: live_in[pc] as bitsets over registers
  const uint32_t words = (R + 63) / 64;
  std::vector<uint64_t> live(N * (size_t)words, 0);
  bool changed = true;
  while (changed) {
    changed = false;
    for (int64_t pc = N - 1; pc >= 0; pc--) {
      const Ins& I = P->code[pc];
      uint32_t s[2];
      int ns;
      successors(I, (uint32_t)pc, N, s, &ns);
      std::vector<uint64_t> v(words, 0);
      for (int j = 0; j < ns; j++)
        for (uint32_t k = 0; k < words; k++) v[k] |= live[s[j] * (size_t)words + k];
      int use[3], nu, def;
      uses_defs(I, use, &nu, &def);
      if (def >= 0) v[def / 64] &= ~(1ull << (def % 64));
      for (int j = 0; j < nu; j++) v[use[j] / 64] |= 1ull << (use[j] % 64);
      for (uint32_t k = 0; k < words; k++)
        if (v[k] != live[pc * (size_t)words + k]) { live[pc * (size_t)words + k] = v[k]; changed = true; }
    }
  }
  std::vector<uint64_t> keep(words, 0);
  for (uint32_t k = 0; k < words; k++) keep[k] = live[k];  // live_in(0)
  P->live_at_entry.clear();
  for (uint32_t r = 0; r < R; r++)
    if (live[r / 64] >> (r % 64) & 1) P->live_at_entry.push_back((uint8_t)r);
  for (uint32_t pc = 0; pc + 1 < N; pc++)
    if (P->code[pc].op == RC_OP_BAR)
      for (uint32_t k = 0; k < words; k++) keep[k] |= live[(pc + 1) * (size_t)words + k];
  P->live_regs.clear();
  for (uint32_t r = 0; r < R; r++)
    if (keep[r / 64] >> (r % 64) & 1) P->live_regs.push_back((uint8_t)r);
  // (2)/(3) per-interval bounds
  std::vector<int> wst(N, 0), wrec(N, 0);
  for (uint32_t pc = 0; pc < N; pc++) {
    wst[pc] = P->code[pc].op == RC_OP_ST;
    wrec[pc] = P->code[pc].op == RC_OP_ST || P->code[pc].op == RC_OP_LD;
  }
  const int64_t st = max_path_weight(P, wst);
  const int64_t rec = max_path_weight(P, wrec);
  P->ovl_cap = (st < 0 || st > OVL_CAP) ? OVL_CAP : (int)std::max<int64_t>(st, 1);
  P->may_spill = st < 0 || st > OVL_CAP;  // more distinct written cells than the smem overlay holds
  P->rec_bound = (rec < 0 || rec > 1024) ? -1 : (int)rec;
  const int64_t ins = max_path_weight(P, std::vector<int>(N, 1));
  P->instr_bound = (ins < 0 || ins >= (1ll << 31)) ? -1 : ins;
  // (4) asynchronous loads: pend[pc] = registers that may still be the target
  //     of an LD issued (and not yet waited on) when pc is reached.
  //     Outer loop: pend is the least fixpoint for the current wait flags; a
  //     flag is added wherever the instruction touches a pending register,
  //     until no flag changes (flags only grow, so this terminates).
  std::vector<uint64_t> pend(N * (size_t)words, 0);
  std::vector<uint8_t> wait(N, 0);
  auto touches_pending = [&](uint32_t pc) {
    int use[3], nu, def;
    uses_defs(P->code[pc], use, &nu, &def);
    const uint64_t* in = &pend[pc * (size_t)words];
    bool w = def >= 0 && (in[def / 64] >> (def % 64) & 1);
    for (int j = 0; j < nu; j++) w = w || (in[use[j] / 64] >> (use[j] % 64) & 1);
    return w;
  };
  for (bool grew = true; grew;) {
    std::fill(pend.begin(), pend.end(), 0ull);
    for (changed = true; changed;) {
      changed = false;
      for (uint32_t pc = 0; pc < N; pc++) {
        const Ins& I = P->code[pc];
        if (I.op == RC_OP_BAR || I.op == RC_OP_EXIT) continue;  // the lane waits at the end of its interval
        std::vector<uint64_t> out(words, 0);
        if (!wait[pc])
          for (uint32_t k = 0; k < words; k++) out[k] = pend[pc * (size_t)words + k];
        if (I.op == RC_OP_LD) out[I.a / 64] |= 1ull << (I.a % 64);
        uint32_t s[2];
        int ns;
        successors(I, pc, N, s, &ns);
        for (int j = 0; j < ns; j++)
          for (uint32_t k = 0; k < words; k++) {
            uint64_t& d = pend[s[j] * (size_t)words + k];
            if ((d | out[k]) != d) { d |= out[k]; changed = true; }
          }
      }
    }
    grew = false;
    for (uint32_t pc = 0; pc < N; pc++)
      if (!wait[pc] && touches_pending(pc)) { wait[pc] = 1; grew = true; }
  }
  P->dev_code = P->code;
  for (uint32_t pc = 0; pc < N; pc++)
    if (wait[pc]) P->dev_code[pc].op |= OP_WAIT;
  // (5) arrays no instruction of an interval region stores to: for every
  //     interval entry e (pc 0, BAR + 1), the instructions reachable from e
  //     without crossing a BAR; entry_ro[e] bit a (a < 31) = no ST to array a
  //     there.  When every running work-item of an instance starts interval k
  //     at the same entry e (interval 0, or interval k - 1 had no barrier
  //     divergence), no work-item writes array a in interval k, so a read of a
  //     can take part in no RW / WW report and no commit and
  //     K1 need not log it — the static half of the write-set filter.
  P->entry_ro.assign(N, 0u);
  if ((uint64_t)N * 64 <= (1ull << 26)) {  // (bounded work: skip for huge programs)
    std::vector<uint32_t> mark(N, 0xFFFFFFFFu), stack;
    for (uint32_t e = 0; e < N; e++) {
      if (!(e == 0 || P->code[e - 1].op == RC_OP_BAR)) continue;
      uint32_t stored = 0, loaded = 0;
      bool big_load = false;  // a load of an array >= 31 (outside the mask): always logged
      stack.assign(1, e);
      mark[e] = e;
      while (!stack.empty()) {
        const uint32_t pc = stack.back();
        stack.pop_back();
        const Ins& I = P->code[pc];
        if (I.op == RC_OP_ST && I.a < 31) stored |= 1u << I.a;
        if (I.op == RC_OP_LD) {
          if (I.b < 31) loaded |= 1u << I.b;
          else big_load = true;
        }
        if (I.op == RC_OP_BAR) continue;  // the region ends at the barrier
        uint32_t sc[2];
        int ns;
        successors(I, pc, N, sc, &ns);
        for (int j = 0; j < ns; j++)
          if (mark[sc[j]] != e) { mark[sc[j]] = e; stack.push_back(sc[j]); }
      }
      const uint32_t ro = ~stored & (P->n_arrays >= 31 ? 0x7FFFFFFFu : ((1u << P->n_arrays) - 1));
      // bit 31: no read of the region is logged (every load reads an array of
      // the mask) — then no filter consults the write-set map for this
      // instance's cells, and K1 need not mark it
      P->entry_ro[e] = ro | ((!big_load && (loaded & ~ro) == 0) ? 0x80000000u : 0u);
    }
  }
  // (6) records per work-item per interval with (5) applied: per entry e, the
  //     longest barrier-free path from e counting every ST and every LD of an
  //     array e's region stores to.  Sizes K1c's record planes (jit.cpp); a
  //     lane of a divergent instance (which logs every read) that exceeds it
  //     makes K1c hand the interval back to the interpreter.
  //     The same for the read records alone (K1c writes its write records
  //     straight into the bucket regions): read_bound_ro, and read_bound
  //     when every read is logged.
  auto bound = [&](bool with_st, bool elide) -> int {
    int64_t b = 0;
    std::vector<int> w(N, 0);
    for (uint32_t e = 0; e < N && b >= 0; e++) {
      if (!(e == 0 || P->code[e - 1].op == RC_OP_BAR)) continue;
      const uint32_t ro = elide ? P->entry_ro[e] & 0x7FFFFFFFu : 0u;
      for (uint32_t pc = 0; pc < N; pc++) {
        const Ins& I = P->code[pc];
        w[pc] = (with_st && I.op == RC_OP_ST) || (I.op == RC_OP_LD && (I.b >= 31 || !((ro >> I.b) & 1u)));
      }
      const int64_t x = max_path_weight(P, w, e);
      b = x < 0 ? -1 : std::max(b, x);
    }
    return (b < 0 || b > 1024) ? -1 : (int)b;
  };
  P->rec_bound_ro = P->rec_bound >= 0 ? bound(true, true) : -1;
  P->read_bound = P->rec_bound >= 0 ? bound(false, false) : -1;
  P->read_bound_ro = P->rec_bound >= 0 ? bound(false, true) : -1;
}

}  // namespace rc

extern "C" {

int rc_load_program(const void* bytecode, size_t nbytes, rc_program** out) {
  if (!out) return rc::fail(RC_EINVAL, "out pointer is NULL");
  *out = nullptr;
  rc_program* P = new (std::nothrow) rc_program();
  if (!P) return rc::fail(RC_ENOMEM, "host allocation failed");
  int st = rc::validate(static_cast<const uint8_t*>(bytecode), nbytes, P);
  if (st != RC_OK) { delete P; return st; }
  *out = P;
  return RC_OK;
}

int rc_program_info(const rc_program* P, uint32_t* n_regs, uint32_t* n_arrays, uint32_t* n_instr) {
  if (!P) return rc::fail(RC_EINVAL, "program is NULL");
  if (n_regs) *n_regs = P->n_regs;
  if (n_arrays) *n_arrays = P->n_arrays;
  if (n_instr) *n_instr = P->n_instr;
  return RC_OK;
}

const char* rc_last_error(void) { return rc::g_last_error.c_str(); }
int rc_abi_version(void) { return RC_ABI_VERSION; }

}  // extern "C"
