// jit.cpp — K1c: the interval interpreter (K1, interp.cu) specialised to one
// program and run shape.  The bytecode is translated into CUDA C++ — one
// basic block of straight-line code per instruction run, a `goto` per branch,
// one `switch` on the work-item's resume pc (the interval entries: pc 0 and
// every BAR + 1) — compiled by NVRTC for sm_100a at the program's first large
// run, loaded through the driver API and cached on the program object.
//
// The same §4 thread-local semantics as K1 (the readings in
// DESIGN.md §3), with what the interpreter pays per executed instruction gone:
// no fetch / decode / dispatch, no warp vote on the minimum pc (a warp runs
// its lanes' own control flow; divergent lanes are the hardware's business —
// a lane's result never depends on the order, delayed visibility, reading
// L2), work-item registers (Locals) in machine registers, operands and
// array bases / sizes as immediates, the own-write overlay as named registers
// whose occupancy is known statically at every instruction (so the first
// loads of an interval search nothing).  One thread runs one work-item; a
// warp walks 32 consecutive lanes of the batch, persistent grid.
//
// Layout contract with the rest of the path (unchanged consumers):
//  * lane state in / out: the same SoA rows as K1 (status, pc, the live
//    registers — program.cpp analyze() (1));
//  * records: the same u64 records (rc_internal.h), but at fixed slots: record
//    k of lane g goes to stage[k * lane_pad + g] for k < planes, and the
//    unused slots of a lane hold the sentinel — no atomics, no staging scan,
//    no block barrier.  `planes` = the static bound on records per work-item
//    per interval (analyze() (6): with the static write-set elision applied,
//    or (3) when every read is logged).  A lane that would exceed it (a
//    divergent instance logs every read) sets `jit_bail` + `log_overflow`:
//    nothing downstream commits and the host re-runs the interval with K1;
//  * wval[slot][lane], the write-set map, A4's per-instance arrival-node
//    range, the report buffer and the counters exactly as K1 writes them.
// Not compiled (K1 runs instead): programs whose overlay may spill
// (may_spill), record bounds above 32 planes, the RW-classification re-run.
#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include <cuda.h>
#include <nvrtc.h>

#include "rc_internal.h"

namespace rc {

namespace {

constexpr int JIT_MAX_PLANES = 32;
constexpr uint32_t JIT_MAX_INSTR = 4096;
constexpr int JIT_THREADS = 256;
// resident blocks per SM the register allocation must allow (RC_JIT_MINB, A/B knob)
int jit_min_blocks() {
  const char* e = getenv("RC_JIT_MINB");
  return e ? std::max(1, atoi(e)) : 5;
}

// ---- NVRTC (dlopen: librc.so loads without it) and the driver API (entry
//      points through the runtime: no -lcuda) -------------------------------
struct Api {
  bool ok = false;
  std::string why;
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) get_log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) get_cubin = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  decltype(&cuModuleLoadData) load = nullptr;
  decltype(&cuModuleGetFunction) get_fn = nullptr;
  decltype(&cuModuleUnload) unload = nullptr;
  decltype(&cuLaunchKernel) launch = nullptr;
  decltype(&cuOccupancyMaxActiveBlocksPerMultiprocessor) occupancy = nullptr;
};

Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    for (const char* name : {"libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so"})
      if ((h = dlopen(name, RTLD_NOW | RTLD_LOCAL)) != nullptr) break;
    if (!h) {
      a.why = "libnvrtc.so.12 not found";
      return;
    }
#define SYM(field, name)                                                   \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name));           \
  if (!a.field) {                                                          \
    a.why = std::string("nvrtc symbol missing: ") + name;                  \
    return;                                                                \
  }
    SYM(create, "nvrtcCreateProgram")
    SYM(compile, "nvrtcCompileProgram")
    SYM(log_size, "nvrtcGetProgramLogSize")
    SYM(get_log, "nvrtcGetProgramLog")
    SYM(cubin_size, "nvrtcGetCUBINSize")
    SYM(get_cubin, "nvrtcGetCUBIN")
    SYM(destroy, "nvrtcDestroyProgram")
#undef SYM
#define DRV(field, name)                                                                                 \
  {                                                                                                      \
    void* f = nullptr;                                                                                   \
    cudaDriverEntryPointQueryResult q;                                                                   \
    if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess || !f) {                 \
      a.why = std::string("driver entry point missing: ") + name;                                        \
      return;                                                                                            \
    }                                                                                                    \
    a.field = reinterpret_cast<decltype(a.field)>(f);                                                    \
  }
    DRV(load, "cuModuleLoadData")
    DRV(get_fn, "cuModuleGetFunction")
    DRV(unload, "cuModuleUnload")
    DRV(launch, "cuLaunchKernel")
    DRV(occupancy, "cuOccupancyMaxActiveBlocksPerMultiprocessor")
#undef DRV
    a.ok = true;
  });
  return a;
}

}  // namespace
struct JitEntry {
  int device = -1;
  std::string key;
  CUmodule mod = nullptr;
  JitKernel k;
  bool ok = false;
  std::string why;
};
struct JitCache {
  std::vector<std::unique_ptr<JitEntry>> v;
};
namespace {

std::string shape_key(const JitShape& S) {
  std::ostringstream o;
  o << S.n << ':' << S.gid << ':' << S.cpi << ':' << S.direct << S.fuel << S.ro_skip << S.wbucket << S.narrow;
  for (size_t a = 0; a < S.off.size(); a++) o << ':' << S.off[a] << '/' << S.size[a];
  return o.str();
}

// static facts the generator uses: interval entries, branch targets, and the
// most own-write overlay entries a work-item can hold when it reaches pc
struct Facts {
  std::vector<uint8_t> entry, target;
  std::vector<int> own_in;  // max distinct ST executions since the interval entry, over barrier-free paths
  std::vector<uint8_t> stored;  // per array: some ST of the program writes it
};

Facts facts(const rc_program* P) {
  const uint32_t N = P->n_instr;
  Facts F;
  F.entry.assign(N, 0);
  F.target.assign(N, 0);
  F.own_in.assign(N, -1);
  F.stored.assign(std::max<uint32_t>(P->n_arrays, 1), 0);
  F.entry[0] = 1;
  for (uint32_t pc = 0; pc < N; pc++) {
    const Ins& I = P->code[pc];
    if (I.op == RC_OP_BAR && pc + 1 < N) F.entry[pc + 1] = 1;
    if (I.op == RC_OP_BR) {
      F.target[(uint32_t)I.imm] = 1;
      F.target[(uint32_t)I.b + 256u * I.c] = 1;
    }
    if (I.op == RC_OP_JMP) F.target[(uint32_t)I.imm] = 1;
    if (I.op == RC_OP_ST) F.stored[I.a] = 1;
  }
  // forward max-dataflow; bounded by the static overlay bound (no barrier-free
  // cycle holds a ST when the program does not spill), so it terminates
  for (uint32_t pc = 0; pc < N; pc++)
    if (F.entry[pc]) F.own_in[pc] = 0;
  for (bool changed = true; changed;) {
    changed = false;
    for (uint32_t pc = 0; pc < N; pc++) {
      if (F.own_in[pc] < 0) continue;
      const Ins& I = P->code[pc];
      if (I.op == RC_OP_BAR || I.op == RC_OP_EXIT) continue;
      const int out = F.own_in[pc] + (I.op == RC_OP_ST ? 1 : 0);
      uint32_t s[2];
      int ns = 0;
      if (I.op == RC_OP_BR) { s[ns++] = (uint32_t)I.imm; s[ns++] = (uint32_t)I.b + 256u * I.c; }
      else if (I.op == RC_OP_JMP) s[ns++] = (uint32_t)I.imm;
      else s[ns++] = pc + 1;
      for (int j = 0; j < ns; j++)
        if (s[j] < N && F.own_in[s[j]] < out) { F.own_in[s[j]] = std::min(out, OVL_CAP); changed = true; }
    }
  }
  return F;
}

// Registers live on entry to each pc (backward dataflow; BAR -> pc + 1 is an
// edge: registers persist across barriers).
std::vector<std::vector<uint8_t>> live_in(const rc_program* P) {
  const uint32_t N = P->n_instr, R = P->n_regs;
  std::vector<std::vector<uint8_t>> L(N, std::vector<uint8_t>(R, 0));
  for (bool changed = true; changed;) {
    changed = false;
    for (int64_t pc = (int64_t)N - 1; pc >= 0; pc--) {
      const Ins& I = P->code[pc];
      std::vector<uint8_t> v(R, 0);
      uint32_t s[2];
      int ns = 0;
      if (I.op == RC_OP_BR) { s[ns++] = (uint32_t)I.imm; s[ns++] = (uint32_t)I.b + 256u * I.c; }
      else if (I.op == RC_OP_JMP) s[ns++] = (uint32_t)I.imm;
      else if (I.op != RC_OP_EXIT && pc + 1 < N) s[ns++] = (uint32_t)pc + 1;
      for (int j = 0; j < ns; j++)
        for (uint32_t r = 0; r < R; r++) v[r] |= L[s[j]][r];
      int def = -1, use[2] = {-1, -1};
      switch (I.op) {
        case RC_OP_ST: use[0] = I.b; use[1] = I.c; break;
        case RC_OP_LD: use[0] = I.c; def = I.a; break;
        case RC_OP_ASSUME: case RC_OP_ASSERT: case RC_OP_BR: use[0] = I.a; break;
        case RC_OP_BAR: case RC_OP_JMP: case RC_OP_EXIT: break;
        case RC_OP_CONST: case RC_OP_TID: case RC_OP_GID: case RC_OP_LID: case RC_OP_LSIZE: case RC_OP_SIZE:
          def = I.a; break;
        case RC_OP_MOV: case RC_OP_LNOT: case RC_OP_ADDI: def = I.a; use[0] = I.b; break;
        default: def = I.a; use[0] = I.b; use[1] = I.c; break;
      }
      if (def >= 0) v[def] = 0;
      for (int u : use)
        if (u >= 0) v[u] = 1;
      if (v != L[pc]) { L[pc] = v; changed = true; }
    }
  }
  return L;
}

// Register values that are the same affine function a*lid + b (mod 2^32) of
// the work-item's local id on every path into pc — over the whole program,
// barriers included (registers start at 0, reading L18).  K1c rematerialises
// such a register at an interval entry instead of carrying it through HBM.
struct Aff {
  uint8_t k = 0;  // 0 unreached, 1 known, 2 unknown
  uint32_t a = 0, b = 0;
  bool operator==(const Aff& o) const { return k == o.k && (k != 1 || (a == o.a && b == o.b)); }
};
std::vector<std::vector<Aff>> affine_in(const rc_program* P, const JitShape& S) {
  const uint32_t N = P->n_instr, R = P->n_regs;
  std::vector<std::vector<Aff>> A(N, std::vector<Aff>(R));
  for (uint32_t r = 0; r < R; r++) A[0][r] = Aff{1, 0, 0};
  auto known = [](uint32_t a, uint32_t b) { return Aff{1, a, b}; };
  const Aff top{2, 0, 0};
  auto join = [](Aff& d, const Aff& x) {
    if (x.k == 0 || d.k == 2) return false;
    if (d.k == 0) { d = x; return true; }
    if (x.k == 2 || !(x == d)) { d = Aff{2, 0, 0}; return true; }
    return false;
  };
  std::vector<uint8_t> work(N, 0);
  work[0] = 1;
  for (bool any = true; any;) {
    any = false;
    for (uint32_t pc = 0; pc < N; pc++) {
      if (!work[pc]) continue;
      work[pc] = 0;
      const Ins& I = P->code[pc];
      std::vector<Aff> v = A[pc];
      const Aff x = v[I.b < R ? I.b : 0], y = v[I.c < R ? I.c : 0];
      switch (I.op) {
        case RC_OP_CONST: v[I.a] = known(0, (uint32_t)I.imm); break;
        case RC_OP_TID: v[I.a] = known(1, S.gid * S.n); break;
        case RC_OP_LID: v[I.a] = known(1, 0); break;
        case RC_OP_GID: v[I.a] = known(0, S.gid); break;
        case RC_OP_LSIZE: v[I.a] = known(0, S.n); break;
        case RC_OP_SIZE: v[I.a] = known(0, S.size[I.b]); break;
        case RC_OP_MOV: v[I.a] = x; break;
        case RC_OP_ADDI: v[I.a] = x.k == 1 ? known(x.a, x.b + (uint32_t)I.imm) : x; break;
        case RC_OP_ADD: v[I.a] = (x.k == 1 && y.k == 1) ? known(x.a + y.a, x.b + y.b) : top; break;
        case RC_OP_SUB: v[I.a] = (x.k == 1 && y.k == 1) ? known(x.a - y.a, x.b - y.b) : top; break;
        case RC_OP_MUL:
          v[I.a] = (x.k == 1 && y.k == 1 && x.a == 0) ? known(x.b * y.a, x.b * y.b)
                   : (x.k == 1 && y.k == 1 && y.a == 0) ? known(x.a * y.b, x.b * y.b) : top;
          break;
        case RC_OP_ST: case RC_OP_BAR: case RC_OP_JMP: case RC_OP_EXIT: case RC_OP_ASSUME: case RC_OP_ASSERT:
        case RC_OP_BR: break;
        default: v[I.a] = top; break;  // LD and the other ALU ops
      }
      uint32_t s[2];
      int ns = 0;
      if (I.op == RC_OP_BR) { s[ns++] = (uint32_t)I.imm; s[ns++] = (uint32_t)I.b + 256u * I.c; }
      else if (I.op == RC_OP_JMP) s[ns++] = (uint32_t)I.imm;
      else if (I.op != RC_OP_EXIT && pc + 1 < N) s[ns++] = pc + 1;
      for (int j = 0; j < ns; j++) {
        bool ch = false;
        for (uint32_t r = 0; r < R; r++) ch |= join(A[s[j]][r], v[r]);
        if (ch) { work[s[j]] = 1; any = true; }
      }
    }
  }
  return A;
}

}  // namespace

std::string jit_source(const rc_program* P, const JitShape& S, int* n_carried) {
  const uint32_t N = P->n_instr;
  const Facts F = facts(P);
  const auto LIVE = live_in(P);
  const auto AFF = affine_in(P, S);
  // registers carried through HBM: live at some interval entry where their
  // value is not a known affine function of the local id (the others are
  // rematerialised at the entry and never stored)
  std::vector<uint8_t> carried(P->n_regs, 0);
  for (uint32_t e = 0; e < N; e++)
    if (F.entry[e])
      for (uint32_t r = 0; r < P->n_regs; r++)
        if (LIVE[e][r] && AFF[e][r].k != 1) carried[r] = 1;
  if (n_carried) *n_carried = (int)std::count(carried.begin(), carried.end(), (uint8_t)1);
  const int K = std::max(1, P->ovl_cap);
  const bool D = S.direct;
  std::ostringstream o;
  o << "// K1c for one program (" << N << " instructions) and shape " << shape_key(S) << " (generated by jit.cpp)\n"
    << "typedef unsigned int u32; typedef int i32; typedef unsigned long long u64; typedef unsigned char u8;\n"
    << "typedef unsigned short u16;\n"
    << RC_STR_(RC_K1C_PARAMS_DECL) << "\n"
    << "struct Rep { u32 instance, interval; i32 array, index; u32 tid1, tid2; u16 kind, flags; u32 reserved; };\n"
    << "#define FULL 0xFFFFFFFFu\n"
    << "__device__ __noinline__ void k1c_report(const K1cParams* pp, u32 inst, i32 arr, i32 idx, u32 tid, u32 kind) {\n"
    << "  const u64 pos = atomicAdd(pp->report_count, 1ull);\n"
    << "  if (pos < pp->report_cap) {\n"
    << "    Rep r; r.instance = pp->inst_base + inst; r.interval = pp->interval; r.array = arr; r.index = idx;\n"
    << "    r.tid1 = " << S.gid * S.n << "u + tid; r.tid2 = 0xFFFFFFFFu; r.kind = (u16)kind; r.flags = 0; r.reserved = 0;\n"
    << "    ((Rep*)pp->reports)[pos] = r;\n"
    << "  }\n"
    << "}\n"
    << "__device__ __forceinline__ u64 wsum(u64 v) {\n"
    << "  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);\n"
    << "  return v;\n"
    << "}\n"
    << "extern \"C\" __global__ void __launch_bounds__(" << JIT_THREADS << ", " << jit_min_blocks()
    << ") rc_k1c(const __grid_constant__ K1cParams p) {\n"
    << "  if (*p.abort) return;  // speculative interval (DevCounters::abort)\n"
    << "  __shared__ u32 s_done;  // warps of the block finished (the report-count snapshot)\n"
    << "  if (p.snapshot) { if (threadIdx.x == 0) s_done = 0; __syncthreads(); }  // (converged: the kernel start)\n"
    << "  const u32 lane = threadIdx.x & 31u;\n"
    << "  " << (S.narrow ? "u32" : "u64") << " s_instr = 0, s_loads = 0, s_stores = 0, s_recs = 0, s_wrec = 0;"
    << (S.narrow ? "  // (per-thread sums < 2^32: the host's step bound)" : "") << "\n"
    << "  bool s_wait = false, s_bail = false, s_bover = false;\n"
    << "  u32 a4_inst = 0xFFFFFFFFu; i32 a4_lo = 0, a4_hi = 0;\n";
  if (!D)
    o << "  if (blockIdx.x == 0 && threadIdx.x == 0) {\n"
      << "    *p.stage_count = (u64)p.planes * p.lane_pad;\n"
      << "    if ((u64)p.planes * p.lane_pad > p.stage_cap) *p.log_overflow = 1;  // the host grows the buffer, re-runs\n"
      << "  }\n"
      << "  if ((u64)p.planes * p.lane_pad > p.stage_cap) return;\n";
  // the next lane's state is loaded while this lane runs (software pipeline:
  // its latency overlaps the heap loads and the writes of the current one)
  auto prefetch = [&](const char* gexpr, const char* cond) {
    o << "    { const u32 g2 = " << gexpr << "; n_st = " << (int)L_EXITED << "; n_pc = 0u;\n"
      << "      if (p.fresh) {  // a batch's first interval: RUNNING at pc 0, registers 0 (reading L18)\n"
      << "        if (" << cond << " && g2 < p.n_lanes) n_st = " << (int)L_RUNNING << ";\n";
    for (uint32_t r = 0; r < P->n_regs; r++)
      if (carried[r]) o << "        n_r" << r << " = 0;\n";
    o << "      }\n"
      << "      else if (" << cond << " && g2 < p.n_lanes) {\n"
      << "        n_st = p.status_in[g2]; n_pc = p.pc_in[g2];\n";
    for (uint32_t r = 0; r < P->n_regs; r++)
      if (carried[r]) o << "        n_r" << r << " = p.regs_in[(u64)" << r << " * p.reg_stride + g2];\n";
    o << "      } }\n";
  };
  // lanes -> warps: blocked (a warp walks a contiguous run of 32-lane
  // groups), so the warps in flight at any moment are spread over the whole
  // batch and seldom meet on one bucket cursor (cyclic: every warp of the
  // grid in the same few buckets; RC_JIT_CYCLIC=1 is the A/B knob)
  const bool cyc = getenv("RC_JIT_CYCLIC") != nullptr;
  if (cyc)
    o << "  const u32 stride = gridDim.x * blockDim.x;\n"
      << "  u32 base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u);\n"
      << "  const u32 base_end = p.lane_pad;\n";
  else
    o << "  const u32 stride = 32u;\n"
      << "  const u32 n_w = gridDim.x * (blockDim.x >> 5), w_id = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);\n"
      << "  const u32 n_grp = p.lane_pad >> 5, per_w = (n_grp + n_w - 1) / n_w;\n"
      << "  u32 base = min(w_id * per_w, n_grp) * 32u;\n"
      << "  const u32 base_end = min((w_id + 1) * per_w, n_grp) * 32u;\n";
  o
    << "  u8 n_st; u32 n_pc;";
  for (uint32_t r = 0; r < P->n_regs; r++)
    if (carried[r]) o << " i32 n_r" << r << " = 0;";
  o << "\n";
  // (RC_JIT_NOPF=1, A/B knob: load each lane's state when it starts.  With
  // every register carried the prefetch cost occupancy — 87.6 vs 82.4 ms/step;
  // with the rematerialised registers only status, pc and the carried ones
  // are in flight: 57.1 vs 70.7 ms/step)
  const bool pf = getenv("RC_JIT_NOPF") == nullptr;
  if (pf) prefetch("base + lane", "base < base_end");

  o << "  for (; base < base_end; base += stride) {\n"
    << "    const u32 g = base + lane;\n"
    << "    const bool valid = g < p.n_lanes;\n";
  if (!pf) prefetch("g", "true");
  o << "    u8 st = n_st;\n"
    << "    u32 pc = n_pc;\n";
  for (uint32_t r = 0; r < P->n_regs; r++) {
    o << "    i32 r" << r << " = " << (carried[r] ? "n_r" + std::to_string(r) : std::string("0")) << ";\n";
  }
  if (pf) prefetch("g + stride", "base + stride < base_end");
  o << "    if (st == " << (int)L_EXITED_NOW << ") st = " << (int)L_EXITED << ";\n"
    << "    const bool running = valid && (st == " << (int)L_RUNNING << " || st == " << (int)L_WAITING << ");\n"
    << "    const u32 inst = valid ? g / " << S.n << "u : 0u;\n"
    << "    const u32 tid = g - inst * " << S.n << "u;\n"
    << "    const u32 cb = inst * " << S.cpi << "u;\n"
    << "    " << (S.fuel ? "u64" : "u32") << " steps = 0;\n"
    << "    u32 nl = 0, ns = 0, nrec = 0, ro = 0, n_own = 0;\n";
  for (int j = 0; j < K; j++) o << "    u32 oc" << j << " = 0; i32 ov" << j << " = 0;\n";
  o    << "    if (running) {\n"
    << "      st = " << (int)L_RUNNING << ";\n";
  if (S.ro_skip && !D)
    o << "      const bool rodiv = !(p.check_div && p.inst_div[inst]);  // the instance did not diverge\n";
  o << "      switch (pc) {\n";
  for (uint32_t e = 0; e < N; e++) {
    if (!F.entry[e]) continue;
    const uint32_t ro = P->entry_ro.empty() ? 0u : P->entry_ro[e];
    o << "        case " << e << "u: ";
    if (S.ro_skip && !D) o << "ro = rodiv ? " << ro << "u : 0u; ";
    for (uint32_t r = 0; r < P->n_regs; r++)  // rematerialised registers
      if (LIVE[e][r] && AFF[e][r].k == 1)
        o << "r" << r << " = (i32)(" << AFF[e][r].a << "u * tid + " << AFF[e][r].b << "u); ";
    o << "goto L" << e << ";\n";
  }
  o << "        default: s_bail = true; goto Lend;  // not an interval entry (never: K1 would not get here either)\n"
    << "      }\n";
  auto R = [](int r) { return "r" + std::to_string(r); };
  for (uint32_t pc = 0; pc < N; pc++) {
    const Ins& I = P->code[pc];
    if (F.own_in[pc] < 0) continue;  // unreachable inside any interval
    if (F.entry[pc] || F.target[pc]) o << "    L" << pc << ":;\n";
    o << "      {  // pc " << pc << "\n";
    if (S.fuel)
      o << "        if (steps == p.fuel) { k1c_report(&p, inst, -1, " << pc << ", tid, " << RC_FUEL << "); st = "
        << (int)L_FUEL << "; pc = " << pc << "u; goto Lend; }\n";
    o << "        steps++;\n";
    const std::string a = R(I.a), b = R(I.b), c = R(I.c);
    const int m = F.own_in[pc];
    switch (I.op) {
      case RC_OP_CONST: o << "        " << a << " = " << I.imm << ";\n"; break;
      case RC_OP_MOV: o << "        " << a << " = " << b << ";\n"; break;
      case RC_OP_TID: o << "        " << a << " = (i32)(" << S.gid * S.n << "u + tid);\n"; break;
      case RC_OP_LID: o << "        " << a << " = (i32)tid;\n"; break;
      case RC_OP_GID: o << "        " << a << " = " << (int32_t)S.gid << ";\n"; break;
      case RC_OP_LSIZE: o << "        " << a << " = " << (int32_t)S.n << ";\n"; break;
      case RC_OP_SIZE: o << "        " << a << " = " << (int32_t)S.size[I.b] << ";\n"; break;
      case RC_OP_ADDI: o << "        " << a << " = (i32)((u32)" << b << " + " << (uint32_t)I.imm << "u);\n"; break;
#define BIN(OPC, EXPR) \
  case OPC: o << "        { const i32 x = " << b << ", y = " << c << "; " << a << " = " << EXPR << "; }\n"; break;
      BIN(RC_OP_ADD, "(i32)((u32)x + (u32)y)")
      BIN(RC_OP_SUB, "(i32)((u32)x - (u32)y)")
      BIN(RC_OP_MUL, "(i32)((u32)x * (u32)y)")
      BIN(RC_OP_MIN, "min(x, y)")
      BIN(RC_OP_MAX, "max(x, y)")
      BIN(RC_OP_AND, "x & y")
      BIN(RC_OP_OR, "x | y")
      BIN(RC_OP_XOR, "x ^ y")
      BIN(RC_OP_LT, "(i32)(x < y)")
      BIN(RC_OP_EQ, "(i32)(x == y)")
      BIN(RC_OP_LAND, "(i32)(x != 0 && y != 0)")
#undef BIN
      case RC_OP_DIV: case RC_OP_MOD:
        o << "        { const i32 x = " << b << ", y = " << c << ";\n"
          << "          if (y == 0) { k1c_report(&p, inst, -1, " << pc << ", tid, " << RC_DIV0 << "); st = " << (int)L_DIV0
          << "; pc = " << pc << "u; goto Lend; }\n"
          << "          " << a << " = "
          << (I.op == RC_OP_DIV ? "(y == -1) ? (i32)(0u - (u32)x) : x / y" : "(y == -1) ? 0 : x % y") << "; }\n";
        break;
      case RC_OP_LNOT: o << "        " << a << " = (i32)(" << b << " == 0);\n"; break;
      case RC_OP_LD: {
        const uint32_t arr = I.b;
        o << "        const i32 idx = " << c << ";\n"
          << "        if ((u32)idx >= " << S.size[arr] << "u) { k1c_report(&p, inst, " << arr << ", idx, tid, " << RC_OOB
          << "); st = " << (int)L_OOB << "; pc = " << pc << "u; goto Lend; }\n"
          << "        const u32 cell = cb + " << S.off[arr] << "u + (u32)idx;\n"
          << "        i32 v = 0; bool f = false;\n";
        if (F.stored[arr])
          for (int j = 0; j < m && j < K; j++)
            o << "        if (n_own > " << j << "u && oc" << j << " == cell) { v = ov" << j << "; f = true; }\n";
        o << "        if (!f) v = " << (D ? "p.heap[cell]" : "__ldg(p.heap + cell)") << ";\n"
          << "        nl++;\n";
        if (!D) {
          o << "        if (" << (arr >= 31 ? std::string("true") : "!((ro >> " + std::to_string(arr) + ") & 1u)") << ") {\n"
            << "          if (nrec < p.planes) p.stage[(u64)nrec * p.lane_pad + g] = ((u64)cell << 32) | (g << 5); else s_bail = true;\n"
            << "          nrec++;\n"
            << "        }\n";
        }
        o << "        " << a << " = v;\n";
        break;
      }
      case RC_OP_ST: {
        const uint32_t arr = I.a;
        o << "        const i32 idx = " << b << ";\n"
          << "        if ((u32)idx >= " << S.size[arr] << "u) { k1c_report(&p, inst, " << arr << ", idx, tid, " << RC_OOB
          << "); st = " << (int)L_OOB << "; pc = " << pc << "u; goto Lend; }\n"
          << "        const u32 cell = cb + " << S.off[arr] << "u + (u32)idx;\n"
          << "        const i32 v = " << c << ";\n";
        if (m == 0) {
          o << "        oc0 = cell; ov0 = v; n_own = 1;\n";
        } else {
          o << "        bool hit = false;\n";
          for (int j = 0; j < m && j < K; j++)
            o << "        if (!hit && n_own > " << j << "u && oc" << j << " == cell) { ov" << j << " = v; hit = true; }\n";
          o << "        if (!hit) {\n";
          for (int j = 0; j <= m && j < K; j++)
            o << "          if (n_own == " << j << "u) { oc" << j << " = cell; ov" << j << " = v; }\n";
          o << "          n_own++;\n"
            << "        }\n";
        }
        o << "        ns++;\n";
        break;
      }
      case RC_OP_BAR:
        // the registers the work-item resumes with at pc + 1 (the carried ones)
        if (pc + 1 < N)
          for (uint32_t r = 0; r < P->n_regs; r++)
            if (LIVE[pc + 1][r] && AFF[pc + 1][r].k != 1)
              o << "        p.regs_out[(u64)" << r << " * p.reg_stride + g] = r" << r << ";\n";
        o << "        pc = " << pc + 1 << "u; st = " << (int)L_WAITING << "; goto Lend;\n";
        break;
      case RC_OP_EXIT:
        o << "        pc = " << pc << "u; st = " << (int)L_EXITED_NOW << "; goto Lend;\n";
        break;
      case RC_OP_ASSUME:
        o << "        if (" << a << " == 0) { st = " << (int)L_PRUNED << "; pc = " << pc << "u; goto Lend; }\n";
        break;
      case RC_OP_ASSERT:
        o << "        if (" << a << " == 0) { k1c_report(&p, inst, -1, " << pc << ", tid, " << RC_ASSERT << "); st = "
          << (int)L_ASSERT << "; pc = " << pc << "u; goto Lend; }\n";
        break;
      case RC_OP_BR:
        o << "        if (" << a << " != 0) goto L" << (uint32_t)I.imm << "; else goto L" << (uint32_t)I.b + 256u * I.c
          << ";\n";
        break;
      case RC_OP_JMP: o << "        goto L" << (uint32_t)I.imm << ";\n"; break;
      default: o << "        s_bail = true; goto Lend;\n"; break;
    }
    o << "      }\n";
  }
  o << "    Lend:;\n"
    << "    }\n";
  // lane state out
  o << "    if (valid) {\n"
    << "      p.status_out[g] = st;\n"
    << "      p.pc_out[g] = pc;\n";
  o << "    }\n";
  // the interval's writes: write records (final value, reading L3, to wval;
  // the write-set map) — or, in direct mode, the commit itself
  if (S.wbucket) o << "    __syncwarp();\n";
  for (int j = 0; j < K; j++) {
    if (S.wbucket && !D) {
      // straight into the bucket regions: lanes of one bucket
      // take their slots with one atomic on the bucket's cursor
      o << "    { const bool has = n_own > " << j << "u; const u32 act = __ballot_sync(FULL, has);\n"
        << "      if (has) {\n"
        << "        const u32 b = oc" << j << " >> 12;\n"
        << "        const u32 m = __match_any_sync(act, b);\n"
        << "        const u32 leader = __ffs(m) - 1;\n"
        << "        u32 pos = 0;\n"
        << "        if (lane == leader) pos = atomicAdd(p.bcur + b, (u32)__popc(m));\n"
        << "        pos = __shfl_sync(m, pos, leader) + __popc(m & ((1u << lane) - 1u));\n"
        << "        if (pos < p.region) p.bucket_out[(u64)b * p.region + pos] = ((u64)oc" << j << " << 32) | (g << 5) | "
        << (j << 1 | 1) << "u; else s_bover = true;\n"
        << "        if (pos < p.region) p.bucket_val[(u64)b * p.region + pos] = ov" << j
        << ";  // (beside the record; detect fills wval for multi-record cells)\n"
        << "        if (!(ro >> 31)) p.wmap[oc" << j << "] = (u8)p.wtag;\n"
        << "        s_wrec++;\n"
        << "      } }\n";
      continue;
    }
    o << "    if (n_own > " << j << "u) {\n";
    if (D) {
      o << "      p.heap_w[oc" << j << "] = ov" << j << ";\n";
    } else {
      o << "      if (nrec < p.planes) p.stage[(u64)nrec * p.lane_pad + g] = ((u64)oc" << j << " << 32) | (g << 5) | "
        << (j << 1 | 1) << "u; else s_bail = true;\n"
        << "      nrec++;\n"
        << "      p.wval[(u64)" << j << " * p.n_lanes + g] = ov" << j << ";\n"
        << "      if (!(ro >> 31)) p.wmap[oc" << j << "] = (u8)p.wtag;\n";
    }
    o << "    }\n";
  }
  if (!D)
    o << "    s_recs += min(nrec, p.planes);\n"
      << "    for (u32 k = nrec; k < p.planes; k++) p.stage[(u64)k * p.lane_pad + g] = ~0ull;\n";
  // fused A4 (K1's logic): per-instance arrival-node range
  o << "    __syncwarp();\n"
    << "    {\n"
    << "      const bool arrived = valid && (st == " << (int)L_WAITING << " || st == " << (int)L_EXITED_NOW << ");\n"
    << "      const i32 node = st == " << (int)L_WAITING << " ? (i32)pc - 1 : -1;\n"
    << "      const u32 inst0 = __shfl_sync(FULL, inst, 0);\n"
    << "      if (__all_sync(FULL, !valid || inst == inst0)) {\n"
    << "        const u32 nmin = __reduce_min_sync(FULL, arrived ? (u32)(node + 1) : 0xFFFFFFFFu);\n"
    << "        const u32 nmax = __reduce_max_sync(FULL, arrived ? (u32)(node + 1) : 0u);\n"
    << "        const i32 lo_ = (i32)(nmin - 1), hi_ = (i32)(nmax - 1);\n"
    << "        if (nmin != 0xFFFFFFFFu && !(inst0 == a4_inst && lo_ >= a4_lo && hi_ <= a4_hi)) {\n"
    << "          if (inst0 != a4_inst) { a4_inst = inst0; a4_lo = lo_; a4_hi = hi_; }\n"
    << "          else { a4_lo = min(a4_lo, lo_); a4_hi = max(a4_hi, hi_); }\n"
    << "          if (lane == 0) { atomicMin(p.node_min + inst0, lo_); atomicMax(p.node_max + inst0, hi_); }\n"
    << "        }\n"
    << "      } else if (arrived) {\n"
    << "        atomicMin(p.node_min + inst, node);\n"
    << "        atomicMax(p.node_max + inst, node);\n"
    << "      }\n"
    << "    }\n"
    << "    s_instr += steps; s_loads += nl; s_stores += ns;\n"
    << "    s_wait |= st == " << (int)L_WAITING << ";\n"
    << "  }\n";
  o << "  const u64 w_instr = wsum(s_instr), w_loads = wsum(s_loads), w_stores = wsum(s_stores), w_recs = wsum(s_recs);\n"
    << "  const u64 w_wrec = wsum(s_wrec);\n"
    << "  const bool any_bail = __any_sync(FULL, s_bail), any_wait = __any_sync(FULL, s_wait), any_bover = __any_sync(FULL, s_bover);\n"
    << "  if (lane == 0) {\n"
    << "    if (w_instr) atomicAdd(p.iv_instr, w_instr);\n"
    << "    if (w_loads) atomicAdd(p.iv_loads, w_loads);\n"
    << "    if (w_stores) atomicAdd(p.iv_stores, w_stores);\n"
    << "    if (w_recs) atomicAdd(p.staged_recs, w_recs);\n"
    << "    if (w_wrec) { atomicAdd(p.kept_count, w_wrec); atomicAdd(p.kept_writes, w_wrec); }  // (bucket writes)\n"
    << "    if (any_bail) { *p.jit_bail = 1; *p.log_overflow = 1; }\n"
    << "    if (any_wait) *p.any_waiting = 1;\n"
    << "    if (any_bover) *p.bucket_overflow = 1;  // the host re-runs the interval with K1\n"
    << "  }\n"
    // no scatter runs after this launch: its last block takes the scatter's
    // snapshot of the report count after K1 (a detect-only re-run rolls back to it)
    // (per warp, no block barrier: after the goto-structured code a warp's
    // lanes need not have reconverged for an aligned __syncthreads; the warp
    // is converged here — the reductions above are full-warp — and every
    // report a lane emitted took its slot with a returning atomic)
    << "  if (p.snapshot && lane == 0) {\n"
    << "    __threadfence();\n"
    << "    if (atomicAdd(&s_done, 1u) == (blockDim.x >> 5) - 1 && atomicAdd(p.k1c_done, 1u) == gridDim.x - 1)\n"
    << "      *p.k1_reports = atomicAdd(p.report_count, 0ull);  // the block's last warp, the grid's last block\n"
    << "  }\n"
    << "}\n";
  // rc_k1c_fix: before K1 (the interpreter, which reads every live register
  // row) runs on lane state K1c produced, write the rematerialised registers
  // of every work-item waiting at an interval entry into the rows
  o << "extern \"C\" __global__ void __launch_bounds__(256) rc_k1c_fix(const __grid_constant__ K1cParams p) {\n"
    << "  for (u32 g = blockIdx.x * blockDim.x + threadIdx.x; g < p.n_lanes; g += gridDim.x * blockDim.x) {\n"
    << "    const u8 st = p.status_in[g];\n"
    << "    if (st != " << (int)L_RUNNING << " && st != " << (int)L_WAITING << ") continue;\n"
    << "    const u32 inst = g / " << S.n << "u, tid = g - inst * " << S.n << "u;\n"
    << "    switch (p.pc_in[g]) {\n";
  for (uint32_t e = 0; e < N; e++) {
    if (!F.entry[e]) continue;
    o << "      case " << e << "u:";
    for (uint32_t r = 0; r < P->n_regs; r++)
      if (LIVE[e][r] && AFF[e][r].k == 1)
        o << " p.regs_out[(u64)" << r << " * p.reg_stride + g] = (i32)(" << AFF[e][r].a << "u * tid + " << AFF[e][r].b
          << "u);";
    o << " break;\n";
  }
  o << "      default: break;\n"
    << "    }\n"
    << "  }\n"
    << "}\n";
  return o.str();
}

bool jit_get(rc_program* P, const JitShape& S, JitKernel* out, std::string* why) {
  auto no = [&](const std::string& w) {
    if (why) *why = w;
    return false;
  };
  if (P->may_spill) return no("the own-write overlay may spill");
  if (P->n_instr > JIT_MAX_INSTR) return no("program too large");
  if (!S.direct) {
    const int planes = S.wbucket ? (S.ro_skip ? P->read_bound_ro : P->read_bound)
                                 : (S.ro_skip ? P->rec_bound_ro : P->rec_bound);
    if (planes < 0 || planes > JIT_MAX_PLANES) return no("no small static bound on records per interval");
  }
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return no("no device");
  if (!P->jit) P->jit = new JitCache();
  JitCache& C = *static_cast<JitCache*>(P->jit);
  const std::string key = shape_key(S);
  for (auto& e : C.v)
    if (e->device == dev && e->key == key) {
      if (!e->ok) return no(e->why);
      *out = e->k;
      return true;
    }
  C.v.push_back(std::make_unique<JitEntry>());
  JitEntry& E = *C.v.back();
  E.device = dev;
  E.key = key;
  Api& A = api();
  if (!A.ok) {
    E.why = A.why;
    return no(E.why);
  }
  const std::string src = jit_source(P, S, &E.k.carried);
  if (const char* dump = getenv("RC_JIT_DUMP")) {
    if (FILE* f = fopen(dump, "w")) {
      fputs(src.c_str(), f);
      fclose(f);
    }
  }
  nvrtcProgram prog = nullptr;
  if (A.create(&prog, src.c_str(), "rc_k1c.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    E.why = "nvrtcCreateProgram failed";
    return no(E.why);
  }
  const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo", "-w"};
  const nvrtcResult cr = A.compile(prog, 4, opts);
  if (cr != NVRTC_SUCCESS) {
    size_t n = 0;
    A.log_size(prog, &n);
    std::string log(n, '\0');
    if (n) A.get_log(prog, &log[0]);
    A.destroy(&prog);
    E.why = "NVRTC: " + log.substr(0, 2000);
    return no(E.why);
  }
  size_t nb = 0;
  A.cubin_size(prog, &nb);
  std::vector<char> cubin(nb);
  A.get_cubin(prog, cubin.data());
  A.destroy(&prog);
  CUfunction fn = nullptr, fix = nullptr;
  if (A.load(&E.mod, cubin.data()) != CUDA_SUCCESS || A.get_fn(&fn, E.mod, "rc_k1c") != CUDA_SUCCESS ||
      A.get_fn(&fix, E.mod, "rc_k1c_fix") != CUDA_SUCCESS) {
    E.why = "cuModuleLoadData / cuModuleGetFunction failed";
    return no(E.why);
  }
  int per_sm = 1, nsm = 148;
  A.occupancy(&per_sm, fn, JIT_THREADS, 0);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  E.k.fn = fn;
  E.k.fix = fix;
  E.k.grid = std::max(1, per_sm) * nsm;
  E.ok = true;
  *out = E.k;
  return true;
}

cudaError_t jit_launch(const JitKernel& k, const K1cParams& p, cudaStream_t s) {
  const uint32_t blocks = (p.lane_pad + JIT_THREADS - 1) / JIT_THREADS;
  const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>(blocks, (uint32_t)k.grid));
  K1cParams q = p;
  void* args[] = {&q};
  const CUresult r = api().launch(static_cast<CUfunction>(k.fn), grid, 1, 1, JIT_THREADS, 1, 1, 0,
                                  reinterpret_cast<CUstream>(s), args, nullptr);
  launched();
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorLaunchFailure;
}

cudaError_t jit_fix(const JitKernel& k, const K1cParams& p, cudaStream_t s) {
  const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>((p.n_lanes + 255) / 256, (uint32_t)k.grid));
  K1cParams q = p;
  void* args[] = {&q};
  const CUresult r = api().launch(static_cast<CUfunction>(k.fix), grid, 1, 1, 256, 1, 1, 0,
                                  reinterpret_cast<CUstream>(s), args, nullptr);
  launched();
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorLaunchFailure;
}

void jit_release(rc_program* P) {
  if (!P->jit) return;
  JitCache* C = static_cast<JitCache*>(P->jit);
  int prev = -1;
  cudaGetDevice(&prev);
  for (auto& e : C->v)
    if (e->mod) {
      cudaSetDevice(e->device);
      api().unload(e->mod);
    }
  if (prev >= 0) cudaSetDevice(prev);
  delete C;
  P->jit = nullptr;
}

}  // namespace rc

extern "C" {
// test hook (not in include/rc.h): the K1c source for a loaded program and
// shape, for inspection without a GPU; returns the byte length (0 if none)
RC_API size_t rc_debug_jit_source(const rc_program* P, uint32_t n, const uint32_t* sizes, uint32_t n_arrays,
                                  uint32_t flags, char* buf, size_t cap) {
  if (!P || n_arrays != P->n_arrays) return 0;
  rc::JitShape S;
  S.n = n;
  uint32_t cpi = 0;
  for (uint32_t a = 0; a < n_arrays; a++) {
    S.off.push_back(cpi);
    S.size.push_back(sizes[a]);
    cpi += sizes[a];
  }
  S.cpi = cpi;
  S.direct = (flags & 1u) != 0;
  S.fuel = (flags & 2u) != 0;
  S.ro_skip = (flags & 4u) != 0;
  S.wbucket = (flags & 8u) != 0;
  S.narrow = (flags & 16u) != 0;
  const std::string src = rc::jit_source(P, S);
  if (buf && cap) {
    const size_t k = std::min(cap - 1, src.size());
    memcpy(buf, src.data(), k);
    buf[k] = '\0';
  }
  return src.size();
}
}

extern "C" {
// test hook (not in include/rc.h): K1c kernels compiled and loaded for this
// program (any shape, any device) — the tests check that K1c really ran
RC_API int rc_debug_jit_kernels(const rc_program* P) {
  if (!P || !P->jit) return 0;
  int k = 0;
  for (auto& e : static_cast<const rc::JitCache*>(P->jit)->v) k += e->ok ? 1 : 0;
  return k;
}
}
