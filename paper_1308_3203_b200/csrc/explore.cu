// explore.cu — rc_explore: every interleaving of one barrier interval on the
// GPU (the paper's own global semantics, PAPER.md:
// 204-227: one work-item steps at a time on the SHARED heap, immediate
// visibility; an interval ends when no work-item can step).
//
// Schedules are indexed, not searched.  A schedule is the sequence of choices
// "which runnable work-item steps next"; index i decodes in mixed radix, the
// radix of step k being r_k = the number of runnable work-items in the state
// reached so far: d_k = i mod r_k, i /= r_k, step the d_k-th runnable one.
// Every index therefore replays SOME complete schedule; it is counted only
// when the quotient left at the end is 0, which makes index -> schedule a
// bijection onto the schedules whose radix product P(s) exceeds the index.
// One GPU thread replays one index at a time (grid-stride, persistent), so
// the exploration is embarrassingly parallel and needs no memo table.
// Coverage: if every examined index i < E has P(path(i)) <= E then every
// schedule has an index < E (a schedule first leaving [0, E) at step j would
// share its first j+1 states with the index of its j-digit prefix, whose
// product then exceeds E) — reported as max_product / complete.
//
// RC_EXPLORE_REDUCED schedules only the shared-heap accesses (LD / ST): the
// private instructions of a work-item (ALU, branches, BAR, EXIT, assume,
// assert) touch only its own state and commute with every step of another
// work-item, so running them eagerly reaches the same set of terminal states
// with far fewer schedules.  Without the flag every instruction is a step and
// n_schedules equals the number of interleavings of the paper's semantics.
//
// Per-thread state (heap + lanes, the oracle enumerator's row layout: heap
// cells, then per work-item pc, status, 0, 0, registers) is word-interleaved
// across threads ([word][thread]: conflict-free / coalesced) in shared memory
// when a block's rows fit in 96 KB, else in a global scratch slice.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "rc_internal.h"

namespace rc {
int fail(int code, const char* fmt, ...);
extern std::atomic<uint64_t> g_launches;

namespace {

// lane status, the same numbering as the enumerator rows
enum : int32_t { X_RUNNING = 0, X_WAITING, X_EXITED, X_PRUNED, X_OOB, X_ASSERT, X_DIV0, X_FUEL };
constexpr uint32_t X_MAX_N = 32;      // work-items per explored interval
constexpr uint32_t X_MAX_ROW = 4096;  // words per state row

struct ExploreParams {
  const Ins* code;
  uint32_t n, n_regs, n_arrays, cells, row_words;
  const uint32_t* arr_off;   // [n_arrays + 1] cell offset of each array (device)
  const int32_t* start;      // [row_words] start state row (device)
  const int32_t* ref_heap;   // [cells] schedule 0's terminal heap (main pass)
  uint64_t fuel, index_begin, index_end;
  bool reduced;
  int32_t* scratch;          // [row_words][G]
  uint64_t G;                // threads in the grid (index stride)
  uint64_t scr_stride;       // word stride of the global scratch rows (G, or 1 when the grid uses shared memory)
  unsigned long long* ctr;   // [0] n_schedules [1] n_differ [2] witness [3] max_product [4] n_terminal
  int32_t* terminals;        // [cap][row_words] or null
  uint64_t cap;
  uint32_t* wsched;          // witness choices or null
  uint32_t max_len;
  uint32_t* wlen;            // [1]
};

// A work-item's words in a strided state row.  Instruction semantics as
// include/rc.h (the opcode table) and DESIGN.md §3 readings L5-L7, L17.
struct Lane {
  int32_t* base;  // first word of this lane in the row (pc) — strided by G
  uint64_t G;
  __device__ int32_t& w(uint32_t i) const { return base[(uint64_t)i * G]; }
  __device__ int32_t& pc() const { return w(0); }
  __device__ int32_t& st() const { return w(1); }
  __device__ int32_t& r(uint32_t i) const { return w(4 + i); }
};

__device__ __forceinline__ int32_t wrap_add(int32_t x, int32_t y) { return (int32_t)((uint32_t)x + (uint32_t)y); }

// Execute one instruction of lane `L` (tid t) on the heap `H` (strided by G).
// The fuel check precedes every instruction (reading L17).
__device__ void step(const ExploreParams& p, int32_t* H, const Lane& L, uint32_t t, uint64_t& steps) {
  if (steps == p.fuel) { L.st() = X_FUEL; return; }
  steps++;
  const Ins I = p.code[(uint32_t)L.pc()];
  int32_t x, y, v = 0;
  switch (I.op) {
    case RC_OP_CONST: L.r(I.a) = I.imm; break;
    case RC_OP_MOV: L.r(I.a) = L.r(I.b); break;
    case RC_OP_TID: L.r(I.a) = (int32_t)t; break;
    // one work-group is explored (group 0 of p.n work-items, reading L20)
    case RC_OP_GID: L.r(I.a) = 0; break;
    case RC_OP_LID: L.r(I.a) = (int32_t)t; break;
    case RC_OP_LSIZE: L.r(I.a) = (int32_t)p.n; break;
    case RC_OP_SIZE: L.r(I.a) = (int32_t)(p.arr_off[I.b + 1] - p.arr_off[I.b]); break;
    case RC_OP_ADDI: L.r(I.a) = wrap_add(L.r(I.b), I.imm); break;
    case RC_OP_ADD: case RC_OP_SUB: case RC_OP_MUL: case RC_OP_DIV: case RC_OP_MOD: case RC_OP_MIN:
    case RC_OP_MAX: case RC_OP_AND: case RC_OP_OR: case RC_OP_XOR: case RC_OP_LT: case RC_OP_EQ:
    case RC_OP_LAND:
      x = L.r(I.b);
      y = L.r(I.c);
      switch (I.op) {
        case RC_OP_ADD: v = wrap_add(x, y); break;
        case RC_OP_SUB: v = (int32_t)((uint32_t)x - (uint32_t)y); break;
        case RC_OP_MUL: v = (int32_t)((uint32_t)x * (uint32_t)y); break;
        case RC_OP_DIV:
        case RC_OP_MOD:
          if (y == 0) { L.st() = X_DIV0; return; }  // ⊥: pc stays (reading L5)
          if (I.op == RC_OP_DIV) v = (y == -1) ? (int32_t)(0u - (uint32_t)x) : x / y;
          else v = (y == -1) ? 0 : x % y;
          break;
        case RC_OP_MIN: v = x < y ? x : y; break;
        case RC_OP_MAX: v = x > y ? x : y; break;
        case RC_OP_AND: v = x & y; break;
        case RC_OP_OR: v = x | y; break;
        case RC_OP_XOR: v = x ^ y; break;
        case RC_OP_LT: v = x < y; break;
        case RC_OP_EQ: v = x == y; break;
        default: v = (x != 0) && (y != 0); break;  // LAND
      }
      L.r(I.a) = v;
      break;
    case RC_OP_LNOT: L.r(I.a) = L.r(I.b) == 0; break;
    case RC_OP_BR: L.pc() = L.r(I.a) != 0 ? I.imm : (int32_t)(I.b + 256u * I.c); return;
    case RC_OP_JMP: L.pc() = I.imm; return;
    case RC_OP_LD: {
      const int32_t idx = L.r(I.c);
      const uint32_t size = p.arr_off[I.b + 1] - p.arr_off[I.b];
      if (idx < 0 || (uint32_t)idx >= size) { L.st() = X_OOB; return; }
      L.r(I.a) = H[(uint64_t)(p.arr_off[I.b] + (uint32_t)idx) * L.G];
      break;
    }
    case RC_OP_ST: {
      const int32_t idx = L.r(I.b);
      const uint32_t size = p.arr_off[I.a + 1] - p.arr_off[I.a];
      if (idx < 0 || (uint32_t)idx >= size) { L.st() = X_OOB; return; }
      H[(uint64_t)(p.arr_off[I.a] + (uint32_t)idx) * L.G] = L.r(I.c);
      break;
    }
    case RC_OP_BAR: L.st() = X_WAITING; break;            // suspended τ⊡σ, pc past the BAR
    case RC_OP_EXIT: L.st() = X_EXITED; return;           // implicit final barrier
    case RC_OP_ASSUME: if (L.r(I.a) == 0) { L.st() = X_PRUNED; return; } break;  // ⊤
    case RC_OP_ASSERT: if (L.r(I.a) == 0) { L.st() = X_ASSERT; return; } break;  // ⊥
    default: L.st() = X_ASSERT; return;                   // unreachable: validated bytecode
  }
  L.pc() = L.pc() + 1;
}

__device__ __forceinline__ bool is_shared(const ExploreParams& p, const Lane& L) {
  const uint8_t op = p.code[(uint32_t)L.pc()].op;
  return op == RC_OP_LD || op == RC_OP_ST;
}

// run lane L's private instructions until it is at a shared access or stops
__device__ void run_private(const ExploreParams& p, int32_t* H, const Lane& L, uint32_t t, uint64_t& steps) {
  while (L.st() == X_RUNNING && !is_shared(p, L)) step(p, H, L, t, steps);
}

__device__ __forceinline__ unsigned long long sat_mul(unsigned long long a, unsigned long long b) {
  return (b != 0 && a > ~0ull / b) ? ~0ull : a * b;
}

// Replay schedule `idx` in the thread's scratch slice.  Returns the quotient
// left over (0 = idx is this schedule's own index) and the radix product.
// `choices` (nullable) receives the chosen tids.
__device__ unsigned long long replay(const ExploreParams& p, int32_t* S, uint64_t sst, unsigned long long idx,
                                     unsigned long long& prod, uint32_t* choices, uint32_t max_len,
                                     uint32_t& len) {
  for (uint32_t wd = 0; wd < p.row_words; wd++) S[(uint64_t)wd * sst] = p.start[wd];
  uint64_t steps[X_MAX_N];
  const uint32_t LW = 4 + p.n_regs;
  auto lane = [&](uint32_t t) { return Lane{S + (uint64_t)(p.cells + t * LW) * sst, sst}; };
  for (uint32_t t = 0; t < p.n; t++) steps[t] = 0;
  if (p.reduced)
    for (uint32_t t = 0; t < p.n; t++) run_private(p, S, lane(t), t, steps[t]);
  prod = 1;
  len = 0;
  for (;;) {
    uint32_t runnable = 0, r = 0;
    for (uint32_t t = 0; t < p.n; t++)
      if (lane(t).st() == X_RUNNING) { runnable |= 1u << t; r++; }
    if (!r) break;
    const uint32_t d = (uint32_t)(idx % r);
    idx /= r;
    prod = sat_mul(prod, r);
    uint32_t m = runnable;
    for (uint32_t k = 0; k < d; k++) m &= m - 1;
    const uint32_t t = __ffs(m) - 1;
    if (choices && len < max_len) choices[len] = t;
    len++;
    const Lane L = lane(t);
    step(p, S, L, t, steps[t]);
    if (p.reduced) run_private(p, S, L, t, steps[t]);
  }
  return idx;
}

// schedule 0 (always the lowest runnable work-item): the reference terminal heap
__global__ void explore_ref_kernel(ExploreParams p, int32_t* ref) {
  unsigned long long prod;
  uint32_t len;
  replay(p, p.scratch, p.scr_stride, 0, prod, nullptr, 0, len);
  for (uint32_t c = 0; c < p.cells; c++) ref[c] = p.scratch[(uint64_t)c * p.scr_stride];
}

// SMEM: the state rows live in shared memory ([word][thread] per block),
// else in the global scratch ([word][grid thread]).
template <bool SMEM>
__global__ void __launch_bounds__(128) explore_kernel(ExploreParams p) {
  extern __shared__ int32_t s_rows[];
  const uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int32_t* S = SMEM ? s_rows + threadIdx.x : p.scratch + g;
  const uint64_t sst = SMEM ? blockDim.x : p.G;
  unsigned long long n_sched = 0, n_diff = 0, wit = ~0ull, maxp = 0;
  for (uint64_t i = p.index_begin + g; i < p.index_end; i += p.G) {
    unsigned long long prod;
    uint32_t len;
    const unsigned long long rem = replay(p, S, sst, i, prod, nullptr, 0, len);
    maxp = prod > maxp ? prod : maxp;
    if (rem) continue;  // a duplicate of schedule i mod P(s)
    n_sched++;
    bool differ = false;
    for (uint32_t c = 0; c < p.cells; c++) differ |= S[(uint64_t)c * sst] != p.ref_heap[c];
    if (differ) {
      n_diff++;
      wit = i < wit ? i : wit;
    }
    if (p.terminals) {
      const unsigned long long slot = atomicAdd(&p.ctr[4], 1ull);
      if (slot < p.cap) {
        int32_t* row = p.terminals + slot * p.row_words;
        for (uint32_t wd = 0; wd < p.row_words; wd++) row[wd] = S[(uint64_t)wd * sst];
        for (uint32_t t = 0; t < p.n; t++) {  // steps are not observable (enumerator rows zero them)
          row[p.cells + t * (4 + p.n_regs) + 2] = 0;
          row[p.cells + t * (4 + p.n_regs) + 3] = 0;
        }
      }
    }
  }
  // warp-aggregated counters
  for (int o = 16; o; o >>= 1) {
    n_sched += __shfl_xor_sync(0xFFFFFFFFu, n_sched, o);
    n_diff += __shfl_xor_sync(0xFFFFFFFFu, n_diff, o);
    const unsigned long long w2 = __shfl_xor_sync(0xFFFFFFFFu, wit, o);
    const unsigned long long m2 = __shfl_xor_sync(0xFFFFFFFFu, maxp, o);
    wit = w2 < wit ? w2 : wit;
    maxp = m2 > maxp ? m2 : maxp;
  }
  if ((threadIdx.x & 31) == 0) {
    if (n_sched) atomicAdd(&p.ctr[0], n_sched);
    if (n_diff) atomicAdd(&p.ctr[1], n_diff);
    if (wit != ~0ull) atomicMin(&p.ctr[2], wit);
    if (maxp) atomicMax(&p.ctr[3], maxp);
  }
}

// the witness schedule's choice sequence (one thread; after the main pass)
__global__ void explore_witness_kernel(ExploreParams p) {
  const unsigned long long w = p.ctr[2];
  if (w == ~0ull) { *p.wlen = 0; return; }
  unsigned long long prod;
  uint32_t len;
  replay(p, p.scratch, p.scr_stride, w, prod, p.wsched, p.max_len, len);
  *p.wlen = len;
}

}  // namespace

void ExploreCache::release() {
  for (int i = 0; i < 3; i++) {
    if (p[i]) cudaFree(p[i]);
    p[i] = nullptr;
    cap[i] = 0;
  }
  device = -1;
}
}  // namespace rc

using namespace rc;

extern "C" int rc_explore(const rc_program* prog, uint32_t n, const uint32_t* sizes, const int32_t* heap,
                          const int32_t* regs, const uint32_t* pc, const uint8_t* status, uint64_t fuel,
                          uint64_t index_begin, uint64_t index_end, uint32_t flags, int32_t* terminals,
                          uint64_t cap, uint32_t* witness_sched, uint32_t max_len, void* cuda_stream,
                          rc_explore_result* out) {
  if (out) memset(out, 0, sizeof *out);
  if (!prog || !out) return fail(RC_EINVAL, "program or out is NULL");
  if (n == 0 || n > X_MAX_N) return fail(RC_EINVAL, "rc_explore: work_group_size %u not in 1..%u", n, X_MAX_N);
  if (prog->n_arrays && !sizes) return fail(RC_EINVAL, "rc_explore: sizes is NULL");
  if (!pc || !status || (prog->n_regs && !regs)) return fail(RC_EINVAL, "rc_explore: lane state is NULL");
  if (index_end < index_begin) return fail(RC_EINVAL, "rc_explore: index_end < index_begin");
  if (flags & ~RC_EXPLORE_REDUCED) return fail(RC_EINVAL, "rc_explore: unknown flags 0x%x", flags);
  if (cap && !terminals) return fail(RC_EINVAL, "rc_explore: terminals is NULL with cap %llu", (unsigned long long)cap);
  if (max_len && !witness_sched) return fail(RC_EINVAL, "rc_explore: witness_sched is NULL with max_len %u", max_len);
  std::vector<uint32_t> off(prog->n_arrays + 1, 0);
  uint64_t cells = 0;
  for (uint32_t a = 0; a < prog->n_arrays; a++) {
    off[a] = (uint32_t)cells;
    cells += sizes[a];
    if (cells > X_MAX_ROW) break;
  }
  off[prog->n_arrays] = (uint32_t)cells;
  const uint32_t LW = 4 + prog->n_regs;
  const uint64_t row_words = cells + (uint64_t)n * LW;
  if (row_words > X_MAX_ROW)
    return fail(RC_ELIMIT, "rc_explore: state row of %llu words > %u", (unsigned long long)row_words, X_MAX_ROW);
  if (cells && !heap) return fail(RC_EINVAL, "rc_explore: heap is NULL");
  // start row (heap | per lane pc, status, 0, 0, regs): gathered to the host
  // (at most X_MAX_ROW words) and uploaded once
  cudaStream_t s = static_cast<cudaStream_t>(cuda_stream);
  std::vector<int32_t> row(row_words, 0), regs_h((uint64_t)n * prog->n_regs);
  std::vector<uint32_t> pc_h(n);
  std::vector<uint8_t> st_h(n);
  bool ok = true;
  if (cells) ok &= cudaMemcpyAsync(row.data(), heap, cells * 4, cudaMemcpyDefault, s) == cudaSuccess;
  if (prog->n_regs) ok &= cudaMemcpyAsync(regs_h.data(), regs, regs_h.size() * 4, cudaMemcpyDefault, s) == cudaSuccess;
  ok &= cudaMemcpyAsync(pc_h.data(), pc, n * 4, cudaMemcpyDefault, s) == cudaSuccess;
  ok &= cudaMemcpyAsync(st_h.data(), status, n, cudaMemcpyDefault, s) == cudaSuccess;
  ok &= cudaStreamSynchronize(s) == cudaSuccess;
  if (!ok) return fail(RC_ECUDA, "rc_explore: reading the start state failed");
  for (uint32_t t = 0; t < n; t++) {
    if (st_h[t] > X_FUEL) return fail(RC_EINVAL, "rc_explore: status[%u] = %u is not a lane status", t, st_h[t]);
    if (pc_h[t] >= prog->n_instr) return fail(RC_EINVAL, "rc_explore: pc[%u] = %u out of range", t, pc_h[t]);
    int32_t* L = row.data() + cells + (uint64_t)t * LW;
    L[0] = (int32_t)pc_h[t];
    L[1] = st_h[t];
    for (uint32_t r = 0; r < prog->n_regs; r++) L[4 + r] = regs_h[(uint64_t)t * prog->n_regs + r];
  }
  int dev = 0, nsm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return fail(RC_ECUDA, "rc_explore: no CUDA device");
  const uint64_t todo = index_end - index_begin;
  const size_t row_b = row_words * 4;
  // state rows in shared memory when a block's rows fit (small problems: all
  // the explorer is for), else in the L1/L2-cached global scratch
  const size_t smem = row_b * 128;
  const bool use_smem = smem <= 96 * 1024 && !getenv("RC_DEBUG_EXPLORE_GLOBAL") &&  // (test hook)
                        cudaFuncSetAttribute(explore_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem) == cudaSuccess;
  // resident blocks per SM (latency of the dependent state loads): as many as
  // fit, up to 16 x 128 threads
  int per_sm = 8;
  if (use_smem && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, explore_kernel<true>, 128, smem) != cudaSuccess)
    per_sm = 8;
  if (getenv("RC_EXPLORE_BPS")) per_sm = atoi(getenv("RC_EXPLORE_BPS"));  // (A/B knob)
  per_sm = std::max(1, std::min(per_sm, 16));
  uint64_t blocks = (uint64_t)nsm * per_sm;
  while (blocks > 1 && blocks * 128 / 2 >= todo) blocks /= 2;
  // global-scratch rows: one per thread; keep the scratch within 256 MB
  // (the grid-stride loop covers every index with any grid)
  while (!use_smem && blocks > 1 && row_b * blocks * 128 > (256ull << 20)) blocks /= 2;
  const uint64_t G = blocks * 128;

  // device buffers cached on the program (grow-only; rc_release_workspace /
  // rc_free_program free them); the program is not re-entrant (include/rc.h)
  rc_program* P = const_cast<rc_program*>(prog);
  std::lock_guard<std::mutex> lk(P->mu);
  if (P->xc.device != dev) {
    if (P->xc.device >= 0) {
      int cur = dev;
      cudaSetDevice(P->xc.device);
      P->xc.release();
      cudaSetDevice(cur);
    }
    P->xc.device = dev;
  }
  auto buf = [&](int i, size_t bytes) -> void* {
    if (P->xc.cap[i] < bytes) {
      if (P->xc.p[i]) cudaFree(P->xc.p[i]);
      P->xc.p[i] = nullptr;
      P->xc.cap[i] = 0;
      if (cudaMalloc(&P->xc.p[i], bytes) != cudaSuccess) return nullptr;
      P->xc.cap[i] = bytes;
    }
    return P->xc.p[i];
  };
  const uint64_t scr_stride = use_smem ? 1 : G;
  void* b0 = buf(0, row_b + cells * 4 + (prog->n_arrays + 2) * 4 + prog->n_instr * sizeof(Ins));
  void* b1 = buf(1, row_words * scr_stride * 4);
  void* b2 = buf(2, 64);
  if (!b0 || !b1 || !b2) return fail(RC_ENOMEM, "rc_explore: device allocation failed");
  int32_t* start = static_cast<int32_t*>(b0);
  int32_t* ref = start + row_words;
  uint32_t* d_off = reinterpret_cast<uint32_t*>(ref + cells);
  Ins* d_code = reinterpret_cast<Ins*>(d_off + prog->n_arrays + 2);
  unsigned long long* ctr = static_cast<unsigned long long*>(b2);
  uint32_t* d_wlen = reinterpret_cast<uint32_t*>(ctr + 5);
  const unsigned long long init[6] = {0, 0, ~0ull, 0, 0, 0};
  ok &= cudaMemcpyAsync(start, row.data(), row_b, cudaMemcpyHostToDevice, s) == cudaSuccess;
  ok &= cudaMemcpyAsync(d_off, off.data(), off.size() * 4, cudaMemcpyHostToDevice, s) == cudaSuccess;
  ok &= cudaMemcpyAsync(d_code, prog->code.data(), prog->n_instr * sizeof(Ins), cudaMemcpyHostToDevice, s) == cudaSuccess;
  ok &= cudaMemcpyAsync(ctr, init, sizeof init, cudaMemcpyHostToDevice, s) == cudaSuccess;
  if (!ok) return fail(RC_ECUDA, "rc_explore: staging the program failed");

  ExploreParams p{};
  p.code = d_code;
  p.n = n;
  p.n_regs = prog->n_regs;
  p.n_arrays = prog->n_arrays;
  p.cells = (uint32_t)cells;
  p.row_words = (uint32_t)row_words;
  p.arr_off = d_off;
  p.start = start;
  p.ref_heap = ref;
  p.fuel = fuel ? fuel : (1ull << 20);
  p.index_begin = index_begin;
  p.index_end = index_end;
  p.reduced = (flags & RC_EXPLORE_REDUCED) != 0;
  p.scratch = static_cast<int32_t*>(b1);
  p.G = G;
  p.scr_stride = scr_stride;
  p.ctr = ctr;
  p.terminals = cap ? terminals : nullptr;
  p.cap = cap;
  p.wsched = witness_sched;
  p.max_len = max_len;
  p.wlen = d_wlen;
  explore_ref_kernel<<<1, 1, 0, s>>>(p, ref);
  if (todo && use_smem) explore_kernel<true><<<(unsigned)blocks, 128, smem, s>>>(p);
  else if (todo) explore_kernel<false><<<(unsigned)blocks, 128, 0, s>>>(p);
  explore_witness_kernel<<<1, 1, 0, s>>>(p);
  g_launches += todo ? 3 : 2;
  unsigned long long h[6];
  if (cudaGetLastError() != cudaSuccess || cudaMemcpyAsync(h, ctr, sizeof h, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return fail(RC_ECUDA, "rc_explore: kernel failed: %s", cudaGetErrorString(cudaGetLastError()));
  out->n_schedules = h[0];
  out->n_differ = h[1];
  out->witness = h[2];
  out->max_product = h[3];
  out->n_terminal = h[4] < cap ? h[4] : cap;
  out->witness_len = (uint32_t)(h[5] & 0xFFFFFFFFu);
  // complete: every schedule has an index in [0, index_end) — only known when
  // something was examined (schedule 0 always exists)
  out->complete = index_begin == 0 && todo > 0 && h[3] <= index_end;
  return RC_OK;
}
