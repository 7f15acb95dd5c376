// interp.cu — K1: one barrier interval of the §4 thread-local semantics for
// every live work-item of an instance batch, fused with the interval-boundary
// bookkeeping (A4) and the write-set map.
//
// One simulated work-item = one lane; a CUDA thread runs H lanes (H = 2 for
// large batches: lanes t and t + T of a tile of H·T lanes).  A warp is one
// instruction stream: each step it executes the instruction at the minimum pc
// among its running lanes (one redux.sync, a uniform fetch of the pre-decoded
// instruction from shared memory, a flat jump table), lanes at that pc
// execute it, the rest wait — a lane's result never depends on the order
// because, inside an interval, lanes only see the interval-start heap plus
// their own writes (delayed visibility, reading L2).  The grid is persistent:
// a block walks tiles, so the program is staged once and statistics are
// flushed once per block.
//
// Per lane: registers (Locals) live in shared memory laid out
// [reg][lane] (a warp touching one register hits 32 distinct banks),
// addressed through 32-bit shared-window addresses; only the registers live
// across a barrier (program.cpp analyze()) travel between intervals, as TMA
// bulk copies (the next tile's rows land while this tile runs).  The
// own-write overlay (cell, value), sized by the static bound on stores per
// interval, also lives in shared memory.  A heap LD is a cp.async straight
// into the destination register; the lane waits only before an instruction
// the static pending-load analysis flagged (OP_WAIT).
//
// Rules implemented: assign (170), store (176/179) into the
// overlay, load (182/185, reading L11) from the overlay else the interval-start
// heap, assert (188) -> ⊥ report, assume (194) -> ⊤, barrier (200) -> suspend.
// ⊥ halts only the faulting lane (reading L5).  Every executed instruction
// costs one unit of fuel (reading L17); the check is compiled out when the
// static longest barrier-free path fits in the fuel.
//
// Log: a read record per performed LD (unless static write-set elision
// proves the array unwritten in this interval), and at the end of the
// interval one write record per distinct cell the lane wrote (its final
// value, reading L3, goes to the side table wval[slot][lane]; the cell is
// marked in the tagged write-set map).  Records are staged per warp in shared
// memory, and each warp's slice leaves as one TMA bulk store into the block's
// chunk of the staging buffer (one atomic per 8192 slots); the write-set
// filter (filter.cu) compacts it for the sort.
//
// Fused A4 (reading L9): per instance the min / max arrival
// node (BAR pc, or -1 for exit) of the lanes that arrived in this interval —
// equal min and max means every arrival reached the same barrier — pushed
// only when it widens what the warp pushed before, and a global "some lane is
// suspended" flag.
#include <cstdlib>
#include <type_traits>

#include "rc_internal.h"

#ifndef INTERP_T  // threads per block (<= 256)
#define INTERP_T 256
#endif
#ifndef INTERP_H  // work-items per thread for large batches (>= 2)
#define INTERP_H 2
#endif
#ifndef INTERP_MIN_BLOCKS_H  // resident blocks per SM of the 2-work-items-per-thread kernel
#define INTERP_MIN_BLOCKS_H 3
#endif
#ifndef LS_NB  // lane-state buffers (TMA prefetch pipeline depth + 1)
#define LS_NB 2
#endif
#ifndef INTERP_MIN_BLOCKS
#define INTERP_MIN_BLOCKS 3
#endif
#ifndef INTERP_SMEM_CAP  // dynamic shared memory per block (the block size halves until it fits)
#define INTERP_SMEM_CAP (96 * 1024)
#endif

namespace rc {

namespace {
constexpr unsigned FULL = 0xFFFFFFFFu;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// rare path: reads what it needs from the kernel's parameter block through a
// pointer (__grid_constant__), so the interpreter loop keeps none of it live
__device__ __noinline__ void emit_report_(const InterpParams* pp, uint32_t inst, int32_t arr, int32_t idx,
                                          uint32_t t1, uint32_t kind) {
  unsigned long long pos = atomicAdd(&pp->ctr->report_count, 1ull);
  if (pos < pp->report_cap) {
    rc_report r;
    r.instance = pp->inst_base + inst;
    r.interval = pp->interval;
    r.array = arr;
    r.index = idx;
    r.tid1 = pp->gbase + t1;  // global id (work-group base + local id, reading L20)
    r.tid2 = NOTID;
    r.kind = (uint16_t)kind;
    r.flags = 0;
    r.reserved = 0;
    pp->reports[pos] = r;
  }
}
#define emit_report(p, inst, arr, idx, t1, kind) emit_report_(&(p), inst, arr, idx, t1, kind)

// a value the compiler must keep in a register (loop invariants it would
// otherwise re-derive from the parameter block every interpreter step)
__device__ __forceinline__ uint32_t pin(uint32_t v) {
  asm volatile("mov.b32 %0, %0;" : "+r"(v));
  return v;
}

struct Stage {
  uint64_t* recs;  // this warp's staging area
  uint32_t fill;   // warp-uniform
  uint32_t cap;
};

// the parts of InterpParams the log write-out needs (passed by value so the
// kernel's parameter block is never copied to local memory)
struct LogOut {
  uint64_t* stage;
  uint8_t* wmap;
  DevCounters* ctr;
  unsigned long long cap;
};

// Copy `cnt` staged records of this warp to stage[base, base + cnt).  Whole
// warp (rare path; the tile write-out is a bulk copy).
__device__ __forceinline__ void write_out(const LogOut& p, const uint64_t* recs, uint32_t cnt,
                                          unsigned long long base, int lane, bool* over) {
  for (uint32_t i = lane; i < cnt; i += 32) {
    const uint64_t rec = recs[i];
    if (base + i < p.cap) p.stage[base + i] = rec;
    else *over = true;
  }
}

// mid-interval overflow of a warp's staging buffer: flush it on its own
__device__ __noinline__ uint32_t flush_warp_(const LogOut p, const uint64_t* recs, uint32_t fill, int lane) {
  __syncwarp();
  unsigned long long base = 0;
  const uint32_t even = (fill + 1) & ~1u;  // slot counts stay even (16-byte bulk copies)
  if (lane == 0) {
    base = atomicAdd(&p.ctr->stage_count, (unsigned long long)even);
    atomicAdd(&p.ctr->staged_recs, (unsigned long long)fill);
  }
  base = __shfl_sync(FULL, base, 0);
  bool over = false;
  write_out(p, recs, fill, base, lane, &over);
  if (even != fill && lane == 0 && base + fill < p.cap) p.stage[base + fill] = REC_SENTINEL;
  if (__any_sync(FULL, over) && lane == 0) p.ctr->log_overflow = 1;
  __syncwarp();
  return 0;
}

#ifndef STAGE_CHUNK_OPT
#define STAGE_CHUNK_OPT 8192
#endif
constexpr uint32_t STAGE_CHUNK = STAGE_CHUNK_OPT;  // staging slots a block reserves at a time

__device__ __forceinline__ unsigned long long warp_sum64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// heap load as an asynchronous copy straight into the lane's destination
// register in shared memory (LDGSTS): the lane keeps executing; it waits
// (cp.async.wait_all) only before an instruction program.cpp flagged OP_WAIT
// (one that may touch a register with an outstanding load) and at the end of
// its interval.
__device__ __forceinline__ void ld_async(uint32_t dst_smem, const int32_t* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst_smem), "l"(src) : "memory");
}
__device__ __forceinline__ void ld_async_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ int32_t wadd(int32_t x, int32_t y) { return (int32_t)((uint32_t)x + (uint32_t)y); }

// ---- TMA bulk copies (cp.async.bulk) of lane-state rows ---------------------
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(mbar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(unsigned long long* mbar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(mbar)), "r"(parity)
        : "memory");
}

// one thread: load the lane state (status, pc, live register rows) of `tile`
// into shared-memory buffer b; rows are padded so every copy is 16-B aligned
__device__ __forceinline__ void prefetch_lanes(const InterpParams& p, uint32_t tile, int T, uint8_t* st, uint32_t* pcs,
                                               int32_t* regs, const uint8_t* live, unsigned long long* mbar) {
  const uint32_t bytes = (uint32_t)T * (1 + 4 + 4 * p.n_live);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes) : "memory");
  const size_t g0 = (size_t)tile * T;
  bulk_g2s(st, p.status_in + g0, (uint32_t)T, mbar);
  bulk_g2s(pcs, p.pc_in + g0, (uint32_t)T * 4, mbar);
  for (uint32_t i = 0; i < p.n_live; i++) {
    const uint32_t r = live[i];
    bulk_g2s(regs + (size_t)r * T, p.regs_in + (size_t)r * p.reg_stride + g0, (uint32_t)T * 4, mbar);
  }
}

// shared-memory accesses through 32-bit shared-window addresses (the
// register file, overlay and program are addressed once per tile, not
// re-derived from generic pointers every step)
__device__ __forceinline__ int32_t lds32(uint32_t a) {
  int32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, int32_t v) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// Pre-decoded instruction (24 B, shared memory: a 16-B head and an 8-B tail
// in two arrays).  Register operands become byte offsets r*T*4 into the
// [reg][thread] register file; LD/ST/SIZE fold in the array's cell offset and
// size, BR its false target.
//   head.x: op (bit 7 = OP_WAIT) | aux(array id) << 8    head.y/z/w: a/b/c byte offsets
//   tail.x: imm, or the array's cell offset (LD/ST), or size (SIZE)
//   tail.y: BR false target, or the array's size (LD/ST)
struct Dec {
  uint4 h;
  uint2 t;
};
// Work-group ids (reading L20) are launch constants: TID becomes "local id +
// imm" with imm = the group's first global tid, LID the same with imm = 0,
// GID and LSIZE become CONST.
__device__ __forceinline__ Dec predecode(uint2 raw, int T, const uint32_t* s_off, const uint32_t* s_size,
                                         const InterpParams& p) {
  uint32_t op = raw.x & 0x7F;
  const uint32_t a = (raw.x >> 8) & 0xFF, b = (raw.x >> 16) & 0xFF, c = raw.x >> 24;
  uint32_t aux = 0, z = raw.y, w = 0;
  if (op == RC_OP_TID) { z = p.gbase; }
  else if (op == RC_OP_LID) { op = RC_OP_TID; z = 0; }
  else if (op == RC_OP_GID) { op = RC_OP_CONST; z = p.gid; }
  else if (op == RC_OP_LSIZE) { op = RC_OP_CONST; z = p.n; }
  if (op == RC_OP_LD) { aux = b; z = s_off[b]; w = s_size[b]; }
  else if (op == RC_OP_ST) { aux = a; z = s_off[a]; w = s_size[a]; }
  else if (op == RC_OP_SIZE) { z = s_size[b]; }
  else if (op == RC_OP_BR) { w = b + 256u * c; }
  const uint32_t rb = 4u * (uint32_t)T;  // bytes per register row
  Dec d;
  d.h = make_uint4(op | (raw.x & OP_WAIT) | (aux << 8), a * rb, b * rb, c * rb);  // op keeps its OP_WAIT bit
  d.t = make_uint2(z, w);
  return d;
}

}  // namespace

// dev-only per-phase cycle accounting (build with -DINTERP_PHASE_TIMING; the
// runtime prints the totals to stderr when RC_PHASES is set)
#ifdef INTERP_PHASE_TIMING
__device__ unsigned long long g_iphase[8];
void interp_phase_io(unsigned long long* out, bool reset) {
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_iphase, z, sizeof z);
  } else {
    cudaMemcpyFromSymbol(out, g_iphase, sizeof(unsigned long long) * 8);
  }
}
#define IPHASE(i)                                 \
  do {                                            \
    if (t == 0) {                                 \
      const long long now_ = clock64();           \
      atomicAdd(&g_iphase[i], now_ - tprev_);     \
      tprev_ = now_;                              \
    }                                             \
  } while (0)
#else
#define IPHASE(i) do {} while (0)
#endif

// FUEL: per-instruction fuel check (reading L17).  Off when the program's
// longest barrier-free path (program.cpp analyze()) fits in the fuel, so no
// work-item can run out in any interval.
// H: work-items per thread.  Thread t runs lanes t, t + T, ... of a tile of
// H*T lanes side by side: one instruction fetch, decode, dispatch and warp
// vote serve H lanes, and each lane's heap loads add to the memory-level
// parallelism of the warp.
// MODE 1 (ALT): the RW-classification re-run (reads of alt_mask cells see
// alt_heap); MODE 2 (DIRECT): rc_prove proved the run conflict-free
// (RC_OPT_PREPASS): writes are committed at the end of each work-item's
// interval and nothing is logged.
// SPILL: a work-item may write more distinct cells in one interval than the
// shared-memory overlay holds (program.cpp may_spill): the spill-list paths.
template <bool CODE_SMEM, bool FUEL, int H, int MODE, bool SPILL>
__global__ void __launch_bounds__(INTERP_T, H == 1 ? INTERP_MIN_BLOCKS : INTERP_MIN_BLOCKS_H)
    interp_kernel(const __grid_constant__ InterpParams p) {
  constexpr bool ALT = MODE == 1;     // RW-classification re-run
  constexpr bool DIRECT = MODE == 2;  // RC_OPT_PREPASS: commit at the interval end, log nothing
  extern __shared__ __align__(16) unsigned char smem[];
  if (p.ctr->abort) return;  // speculative interval (DevCounters::abort)
  const int T = (int)p.lay.T;    // == blockDim.x
  const int TL = (int)p.lay.TL;  // lanes per tile (H * T)
  const int W = (int)p.lay.W;
  const int t = threadIdx.x;
  const int warp = t >> 5, lane = t & 31;
  const uint32_t R = p.n_regs, OV = p.ovl_cap;
  const uint32_t SW = H * p.stage_warp;  // staged records per warp
  const LogOut lo{p.stage, p.wmap, p.ctr, p.stage_cap};
  (void)R;

  // ---- shared memory carve-up (k1_layout): register files [reg][lane],
  // status and pc rows, LS_NB-buffered (TMA: the next tile's state lands
  // while this one runs; a buffer is refilled only after the bulk stores of
  // its previous tile have read it); buffer b is addressed arithmetically
  // from these bases (a runtime-indexed array of pointers would lose the
  // shared address space)
  int32_t* const sregs0 = reinterpret_cast<int32_t*>(smem + p.lay.regs);
  uint32_t* const spc0 = reinterpret_cast<uint32_t*>(smem + p.lay.spc);
  uint8_t* const sstat0 = smem + p.lay.sstat;
#define SREGS(b) (reinterpret_cast<int32_t*>(reinterpret_cast<unsigned char*>(sregs0) + (size_t)(b) * p.lay.regs_buf))
#define SPC(b) (spc0 + (size_t)(b) * TL)
#define SSTAT(b) (sstat0 + (size_t)(b) * TL)
  // mbar[b]: the lane state of buffer b landed (TMA)
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(smem + p.lay.mbar);
  uint64_t* st_recs = reinterpret_cast<uint64_t*>(smem + p.lay.recs);
  uint4* s_code = reinterpret_cast<uint4*>(smem + p.lay.code);   // heads + pad entry
  uint2* s_tail = reinterpret_cast<uint2*>(smem + p.lay.tail);   // tails + pad
  uint32_t* s_ro = reinterpret_cast<uint32_t*>(smem + p.lay.ro);  // entry_ro
  uint32_t* ocell = reinterpret_cast<uint32_t*>(smem + p.lay.ocell);
  int32_t* oval = reinterpret_cast<int32_t*>(smem + p.lay.oval);
  uint32_t* s_off = reinterpret_cast<uint32_t*>(smem + p.lay.soff);
  uint32_t* s_size = reinterpret_cast<uint32_t*>(smem + p.lay.ssize);
  uint8_t* s_live = smem + p.lay.live;
  uint32_t* wcnt = reinterpret_cast<uint32_t*>(smem + p.lay.wcnt);  // per-warp staged records, pad count
  unsigned long long* wbase = reinterpret_cast<unsigned long long*>(smem + p.lay.wbase);  // [W], pad start

  for (uint32_t a = t; a < p.n_arrays; a += T) {
    s_off[a] = p.arr_off[a];
    s_size[a] = p.arr_size[a];
  }
  __syncthreads();  // s_off / s_size before the pre-decode
  if (CODE_SMEM) {
    for (uint32_t i = t; i < p.n_instr; i += T) {
      const Dec d = predecode(__ldg(reinterpret_cast<const uint2*>(p.code) + i), TL, s_off, s_size, p);
      s_code[i] = d.h;
      s_tail[i] = d.t;
      s_ro[i] = __ldg(p.entry_ro + i);
    }
    if (t == 0) {  // pad entry (never executed)
      s_code[p.n_instr] = make_uint4(0, 0, 0, 0);
      s_tail[p.n_instr] = make_uint2(0, 0);
    }
  }
  const uint32_t code_h = pin(smem_u32(s_code)), code_t = pin(smem_u32(s_tail));
  for (uint32_t i = t; i < p.n_live; i += T) s_live[i] = p.live[i];
  const uint32_t n_tiles = (p.n_lanes + TL - 1) / TL;
  if (t == 0) {
    for (int b = 0; b < LS_NB; b++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (t == 0 && blockIdx.x < n_tiles)
    prefetch_lanes(p, blockIdx.x, TL, SSTAT(0), SPC(0), SREGS(0), s_live, &mbar[0]);

  // per-lane totals, reduced once at the end of the kernel
  unsigned long long b_instr = 0, b_loads = 0, b_stores = 0;
  bool b_wait = false, b_over = false, b_ovl = false;
  // the block's current staging chunk (thread 0)
  unsigned long long c_base = 0;
  uint32_t c_used = 0, c_cap = 0;

  uint32_t a4_inst = 0xFFFFFFFFu;  // arrival-node range this warp pushed (warp-uniform)
  int32_t a4_lo = 0, a4_hi = 0;
  unsigned long long b_staged = 0;  // thread 0: records staged by the block
  uint32_t parity = 0;  // bit b: expected phase of mbar[b]
  int cur = 0;
#ifdef INTERP_PHASE_TIMING
  long long tprev_ = clock64();
#endif
  for (uint32_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, cur = cur + 1 == LS_NB ? 0 : cur + 1) {
    IPHASE(0);
    // per-lane state, lane h*T + t of the tile
    uint32_t g[H], pc[H], inst[H], tid[H], cell_base[H];
    uint32_t div[H];  // the instance's previous interval diverged (loaded before the lane state lands)
    // a tile of TL <= n lanes spans at most two instances: one division per tile
    const uint32_t inst_t = fast_div(tile * (uint32_t)TL, p.n_magic);
    const uint32_t next_t = (inst_t + 1) * p.n;  // first lane of the next instance
#pragma unroll
    for (int h = 0; h < H; h++) {
      g[h] = tile * (uint32_t)TL + h * T + t;
      inst[h] = g[h] >= p.n_lanes ? 0u
                : (p.n >= (uint32_t)TL ? inst_t + (g[h] >= next_t ? 1u : 0u) : fast_div(g[h], p.n_magic));
      div[h] = (!ALT && p.ro_skip && p.interval > 0 && g[h] < p.n_lanes) ? __ldg(p.inst_div + inst[h]) : 0u;
    }
    mbar_wait_parity(&mbar[cur], (parity >> cur) & 1u);
    parity ^= 1u << cur;
    IPHASE(1);
    uint8_t* const sstat = SSTAT(cur);
    uint32_t* const spc = SPC(cur);
    uint8_t status[H];
    bool valid[H], running[H];
    int n_own[H];
    // instructions each lane executed in the interval (< 2^31 when !FUEL)
    typename std::conditional<FUEL, unsigned long long, uint32_t>::type steps[H];
    uint32_t nloads[H], nstores[H];
    bool ovl_over[H];
    uint32_t ro[H];  // arrays whose reads this lane need not log (static write-set elision)
#pragma unroll
    for (int h = 0; h < H; h++) {
      const int l = h * T + t;
      valid[h] = g[h] < p.n_lanes;
      status[h] = valid[h] ? sstat[l] : (uint8_t)L_EXITED;
      pc[h] = valid[h] ? spc[l] : 0;
      if (status[h] == L_EXITED_NOW) status[h] = L_EXITED;
      running[h] = valid[h] && (status[h] == L_RUNNING || status[h] == L_WAITING);
      if (running[h]) status[h] = L_RUNNING;
      tid[h] = valid[h] ? g[h] - inst[h] * p.n : 0;
      cell_base[h] = inst[h] * p.cpi;
      // every running lane of the instance starts this interval at the same
      // entry (interval 0, or no barrier divergence in the previous one): no
      // lane writes an array its region never stores to (program.cpp (5))
      ro[h] = (!ALT && p.ro_skip && running[h] && !div[h])
                  ? (CODE_SMEM ? s_ro[pc[h]] : __ldg(p.entry_ro + pc[h])) : 0u;
      n_own[h] = 0;
      steps[h] = 0;
      nloads[h] = 0;
      nstores[h] = 0;
      ovl_over[h] = false;
    }
    const uint32_t orow = 4u * (uint32_t)TL;  // overlay row stride (bytes)
    // byte address of lane t's register 0 (lane h*T + t: + 4*T*h); register r
    // is at + r*TL*4 (the live ones arrived by TMA); the overlay cells and
    // values likewise (oval follows ocell)
    const uint32_t rg0 = pin(smem_u32(SREGS(cur)) + 4u * (uint32_t)t);
    const uint32_t oc0 = pin(smem_u32(ocell) + 4u * (uint32_t)t);
    const uint32_t ovd = OV * orow;  // ocell -> oval
#define RG(h) (rg0 + (uint32_t)(h) * 4u * (uint32_t)T)
#define OC(h) (oc0 + (uint32_t)(h) * 4u * (uint32_t)T)
#define OVL(h) (OC(h) + ovd)
    // the previous tile's bulk store of this warp's staged records has read them
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncwarp();
    Stage S{st_recs + (size_t)warp * SW, 0, SW};

    for (;;) {
      bool ex[H];
      uint32_t mine = 0xFFFFFFFFu;
#pragma unroll
      for (int h = 0; h < H; h++)
        if (running[h]) mine = min(mine, pc[h]);
      const uint32_t minpc = __reduce_min_sync(FULL, mine);
      if (minpc == 0xFFFFFFFFu) break;  // no lane of the warp is running (pcs are < 65536)
#pragma unroll
      for (int h = 0; h < H; h++) ex[h] = running[h] && pc[h] == minpc;
      uint4 eh;
      uint2 et;
      if (CODE_SMEM) {
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(eh.x), "=r"(eh.y), "=r"(eh.z), "=r"(eh.w)
                     : "r"(code_h + 16u * minpc)
                     : "memory");
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(et.x), "=r"(et.y) : "r"(code_t + 8u * minpc) : "memory");
      } else {
        const Dec d = predecode(__ldg(reinterpret_cast<const uint2*>(p.code) + minpc), TL, s_off, s_size, p);
        eh = d.h;
        et = d.t;
      }
      const uint32_t op = eh.x & 0x7F;
      const int32_t imm = (int32_t)et.x;
      if (eh.x & OP_WAIT) ld_async_wait();  // warp-uniform
#pragma unroll
      for (int h = 0; h < H; h++) {
        if (FUEL && ex[h]) {  // fuel check before executing (reading L17)
          if (steps[h] == p.fuel) {
            emit_report(p, inst[h], -1, (int32_t)pc[h], tid[h], RC_FUEL);
            running[h] = false;
            status[h] = L_FUEL;
            ex[h] = false;
          } else {
            steps[h]++;
          }
        }
        if (!FUEL) steps[h] += ex[h];
      }
      // this lane's operand registers
#define RA(h) (RG(h) + eh.y)
#define RB(h) (RG(h) + eh.z)
#define RC(h) (RG(h) + eh.w)
#define EACH(...) \
  _Pragma("unroll") for (int h = 0; h < H; h++) if (ex[h]) { __VA_ARGS__; }
      // dispatch (warp-uniform): the heap accesses first, the rest through a switch
      if (op == RC_OP_LD) {
#pragma unroll
        for (int h = 0; h < H; h++) {
          bool ok = false;
          uint32_t cell = 0;
          if (ex[h]) {
            const int32_t idx = lds32(RC(h));
            if ((uint32_t)idx >= et.y) {  // also catches idx < 0
              emit_report(p, inst[h], (int32_t)((eh.x >> 8) & 0xFF), idx, tid[h], RC_OOB);
              running[h] = false;
              status[h] = L_OOB;
            } else {
              cell = cell_base[h] + et.x + (uint32_t)idx;
              int32_t v = 0;
              bool found = false;
              const int n_sm = SPILL ? min(n_own[h], (int)OV) : n_own[h];
              for (int j = 0; j < n_sm; j++)
                if ((uint32_t)lds32(OC(h) + j * orow) == cell) { v = lds32(OVL(h) + j * orow); found = true; }
              if (SPILL && n_own[h] > (int)OV && !found) {  // the lane's spill list (rare)
                for (int j = 0; j < n_own[h] - (int)OV; j++)
                  if (p.spill_cell[(size_t)j * p.n_lanes + g[h]] == cell) {
                    v = p.spill_val[(size_t)j * p.n_lanes + g[h]];
                    found = true;
                  }
              }
              if (found) {
                sts32(RA(h), v);
              } else {
                const int32_t* src = p.heap + cell;
                if (ALT && p.alt_mask[cell]) src = p.alt_heap + cell;  // writers-first visibility
                ld_async(RA(h), src);
              }
              pc[h]++;
              nloads[h]++;
              const uint32_t arr = (eh.x >> 8) & 0xFF;
              ok = !DIRECT && (arr >= 31 || !((ro[h] >> arr) & 1u));  // a read of a written-in-no-way array is not logged
            }
          }
          const unsigned m = __ballot_sync(FULL, ok);
          if (m) {
            if (S.fill + __popc(m) > S.cap) S.fill = flush_warp_(lo, S.recs, S.fill, lane);
            if (ok) S.recs[S.fill + __popc(m & lanemask_lt())] = make_rec(cell, g[h], 0, 0);
            S.fill += __popc(m);
          }
        }
      } else if (op == RC_OP_ST) {
        EACH({
          const int32_t idx = lds32(RB(h));
          if ((uint32_t)idx >= et.y) {  // also catches idx < 0
            emit_report(p, inst[h], (int32_t)((eh.x >> 8) & 0xFF), idx, tid[h], RC_OOB);
            running[h] = false;
            status[h] = L_OOB;
          } else {
            const uint32_t cell = cell_base[h] + et.x + (uint32_t)idx;
            const int n_sm = SPILL ? min(n_own[h], (int)OV) : n_own[h];
            int j = 0;
            while (j < n_sm && (uint32_t)lds32(OC(h) + j * orow) != cell) j++;
            if (j < n_sm) {
              sts32(OVL(h) + j * orow, lds32(RC(h)));
            } else if (!SPILL || n_own[h] < (int)OV) {  // (!SPILL: the static bound fits the overlay)
              sts32(OC(h) + j * orow, (int32_t)cell);
              n_own[h]++;
              sts32(OVL(h) + j * orow, lds32(RC(h)));
            } else {  // beyond the smem overlay: the lane's spill list in HBM (rare)
              const int ns = n_own[h] - (int)OV;
              int k = 0;
              while (k < ns && p.spill_cell[(size_t)k * p.n_lanes + g[h]] != cell) k++;
              if (k == ns) {
                if ((uint32_t)ns < p.spill_cap) {
                  p.spill_cell[(size_t)k * p.n_lanes + g[h]] = cell;
                  n_own[h]++;
                } else {
                  ovl_over[h] = true;  // full: the interval is re-run with a larger list
                  k = -1;
                }
              }
              if (k >= 0) p.spill_val[(size_t)k * p.n_lanes + g[h]] = lds32(RC(h));
            }
            pc[h]++;
            nstores[h]++;
          }
        })
      } else switch (op & 31) {
        case RC_OP_LD: case RC_OP_ST: break;  // handled above
        case 0: case 28: case 29: case 30: case 31: break;  // (GID / LID / LSIZE are pre-decoded away)
        case RC_OP_CONST: EACH({ sts32(RA(h), imm); pc[h]++; }) break;
        case RC_OP_MOV: EACH({ sts32(RA(h), lds32(RB(h))); pc[h]++; }) break;
        case RC_OP_TID: EACH({ sts32(RA(h), wadd(imm, (int32_t)tid[h])); pc[h]++; }) break;  // imm: pre-decode
        case RC_OP_SIZE: EACH({ sts32(RA(h), imm); pc[h]++; }) break;
        case RC_OP_ADDI: EACH({ sts32(RA(h), wadd(lds32(RB(h)), imm)); pc[h]++; }) break;
        // binary ALU ops, one case each (a flat jump table; int32 wrap, reading L7)
#define ALU2(OPC, EXPR)                                \
  case OPC:                                            \
    EACH({                                             \
      const int32_t x = lds32(RB(h)), y = lds32(RC(h)); \
      sts32(RA(h), (EXPR));                            \
      pc[h]++;                                         \
    })                                                 \
    break;
        ALU2(RC_OP_ADD, wadd(x, y))
        ALU2(RC_OP_SUB, (int32_t)((uint32_t)x - (uint32_t)y))
        ALU2(RC_OP_MUL, (int32_t)((uint32_t)x * (uint32_t)y))
        ALU2(RC_OP_MIN, min(x, y))
        ALU2(RC_OP_MAX, max(x, y))
        ALU2(RC_OP_AND, x & y)
        ALU2(RC_OP_OR, x | y)
        ALU2(RC_OP_XOR, x ^ y)
        ALU2(RC_OP_LT, (int32_t)(x < y))
        ALU2(RC_OP_EQ, (int32_t)(x == y))
        ALU2(RC_OP_LAND, (int32_t)((x != 0) && (y != 0)))
#undef ALU2
        case RC_OP_DIV: case RC_OP_MOD:
          EACH({
            const int32_t x = lds32(RB(h)), y = lds32(RC(h));
            if (y == 0) {
              emit_report(p, inst[h], -1, (int32_t)pc[h], tid[h], RC_DIV0);
              running[h] = false;
              status[h] = L_DIV0;
            } else {
              int32_t v;
              if (op == RC_OP_DIV) v = (y == -1) ? (int32_t)(0u - (uint32_t)x) : x / y;
              else v = (y == -1) ? 0 : x % y;
              sts32(RA(h), v);
              pc[h]++;
            }
          })
          break;
        case RC_OP_LNOT: EACH({ sts32(RA(h), lds32(RB(h)) == 0); pc[h]++; }) break;
        case RC_OP_BAR: EACH({ pc[h]++; running[h] = false; status[h] = L_WAITING; }) break;
        case RC_OP_EXIT: EACH({ running[h] = false; status[h] = L_EXITED_NOW; }) break;
        case RC_OP_ASSUME:
          EACH({
            if (lds32(RA(h)) == 0) { running[h] = false; status[h] = L_PRUNED; }
            else pc[h]++;
          })
          break;
        case RC_OP_ASSERT:
          EACH({
            if (lds32(RA(h)) == 0) {
              emit_report(p, inst[h], -1, (int32_t)pc[h], tid[h], RC_ASSERT);
              running[h] = false;
              status[h] = L_ASSERT;
            } else {
              pc[h]++;
            }
          })
          break;
        case RC_OP_BR: EACH({ pc[h] = lds32(RA(h)) != 0 ? (uint32_t)imm : et.y; }) break;
        case RC_OP_JMP: EACH({ pc[h] = (uint32_t)imm; }) break;
      }
#undef EACH
#undef RA
#undef RB
#undef RC
#undef RG
#undef OC
#undef OVL
    }

    IPHASE(2);
    // prefetch the next tile's lane state into the next buffer once the bulk
    // stores of its previous use (LS_NB - 1 tiles back) have read it: issued
    // after this warp's interpretation, when those stores (from the end of
    // the previous tile) are long done, so thread 0 does not wait on them;
    // the copy still lands during this tile's write-out
    if (t == 0 && tile + gridDim.x < n_tiles) {
      const int nx = cur + 1 == LS_NB ? 0 : cur + 1;
      if (LS_NB == 2) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      else asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      prefetch_lanes(p, tile + gridDim.x, TL, SSTAT(nx), SPC(nx), SREGS(nx), s_live, &mbar[nx]);
    }
    ld_async_wait();  // registers of suspended lanes are saved below

    // write records: one per distinct written cell; its final value (reading
    // L3) goes to the side table wval[slot][lane] read by detect.  Direct
    // mode (rc_prove proved the run conflict-free, RC_OPT_PREPASS): no other
    // work-item touches the cell in this interval, so the final value is
    // committed right away and nothing is logged.
    if (DIRECT) {
#pragma unroll
      for (int h = 0; h < H; h++) {
        const int l = h * T + t;
        for (int j = 0; j < n_own[h]; j++) {
          if (!SPILL || j < (int)OV) {
            p.heap_w[ocell[j * TL + l]] = oval[j * TL + l];
          } else {
            const size_t k = (size_t)(j - (int)OV) * p.n_lanes + g[h];
            p.heap_w[p.spill_cell[k]] = p.spill_val[k];
          }
        }
      }
    }
#pragma unroll
    for (int h = 0; h < H && !DIRECT; h++) {
      const int l = h * T + t;
      const int max_own = __reduce_max_sync(FULL, (unsigned)n_own[h]);
      for (int j = 0; j < max_own; j++) {
        const bool has = j < n_own[h];
        const unsigned m = __ballot_sync(FULL, has);
        if (S.fill + __popc(m) > S.cap) S.fill = flush_warp_(lo, S.recs, S.fill, lane);
        if (has) {
          uint32_t cell, slot;
          if (!SPILL || j < (int)OV) {
            cell = ocell[j * TL + l];
            slot = (uint32_t)j;
            p.wval[(size_t)j * p.n_lanes + g[h]] = oval[j * TL + l];
          } else {  // spilled: detect looks the value up in the lane's list
            cell = p.spill_cell[(size_t)(j - (int)OV) * p.n_lanes + g[h]];
            slot = SLOT_SPILL;
          }
          S.recs[S.fill + __popc(m & lanemask_lt())] = make_rec(cell, g[h], slot, 1);
          // write-set map (the filter's dynamic half): not needed when no
          // read of this instance's region is logged (entry_ro bit 31)
          if (!(ro[h] >> 31)) p.wmap[cell] = p.wtag;
        }
        S.fill += __popc(m);
      }
      if (SPILL && n_own[h] > (int)OV) p.spill_n[g[h]] = (uint32_t)(n_own[h] - (int)OV);
    }

    IPHASE(3);
    // fused A4: arrival node range per instance (fire-and-forget atomics,
    // pushed only when they widen what this warp already pushed), suspended flag
#pragma unroll
    for (int h = 0; h < H; h++) {
      const bool arrived = valid[h] && (status[h] == L_WAITING || status[h] == L_EXITED_NOW);
      const int32_t node = status[h] == L_WAITING ? (int32_t)pc[h] - 1 : NODE_EXIT;
      const uint32_t inst0 = __shfl_sync(FULL, inst[h], 0);
      const bool warp_uniform = __all_sync(FULL, !valid[h] || inst[h] == inst0);
      if (warp_uniform) {
        // nodes are >= -1; bias by 1 so unsigned reductions apply
        const uint32_t nmin = __reduce_min_sync(FULL, arrived ? (uint32_t)(node + 1) : 0xFFFFFFFFu);
        const uint32_t nmax = __reduce_max_sync(FULL, arrived ? (uint32_t)(node + 1) : 0u);
        // min/max atomics are idempotent: ~one pair per warp and instance
        const int32_t lo_ = (int32_t)(nmin - 1), hi_ = (int32_t)(nmax - 1);
        if (nmin != 0xFFFFFFFFu && !(inst0 == a4_inst && lo_ >= a4_lo && hi_ <= a4_hi)) {
          if (inst0 != a4_inst) { a4_inst = inst0; a4_lo = lo_; a4_hi = hi_; }
          else { a4_lo = min(a4_lo, lo_); a4_hi = max(a4_hi, hi_); }
          if (lane == 0) {
            atomicMin(p.node_min + inst0, lo_);
            atomicMax(p.node_max + inst0, hi_);
          }
        }
      } else if (arrived) {  // small work-groups: per-lane atomics
        atomicMin(p.node_min + inst[h], node);
        atomicMax(p.node_max + inst[h], node);
      }
      // statistics stay per lane until the end of the kernel
      b_instr += steps[h];
      b_loads += nloads[h];
      b_stores += nstores[h];
      b_ovl |= ovl_over[h];
      b_wait |= status[h] == L_WAITING;
    }

    // ---- tile write-out into the block's staging chunk (a new chunk — one
    //      atomic — only when the current one is full; its tail is padded)
    if (S.fill & 1) {  // even record counts: every warp's slice is a 16-byte bulk copy
      if (lane == 0) S.recs[S.fill] = REC_SENTINEL;
      S.fill++;
    }
    if (lane == 0) wcnt[warp] = S.fill;
    __syncthreads();
    IPHASE(4);
    if (warp == 0) {
      const uint32_t c = lane < W ? wcnt[lane] : 0u;
      uint32_t x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
      }
      const uint32_t tot = __shfl_sync(FULL, x, 31);
      unsigned long long pad_from = 0;
      uint32_t pad_n = 0;
      if (lane == 0 && tot) {
        if (c_used + tot > c_cap) {  // pad the rest of the current chunk, take a new one
          pad_from = c_base + c_used;
          pad_n = c_cap - c_used;
          const uint32_t sz = max(STAGE_CHUNK, tot);
          c_base = atomicAdd(&p.ctr->stage_count, (unsigned long long)sz);
          c_used = 0;
          c_cap = sz;
        }
        b_staged += tot;
      }
      const unsigned long long cb = __shfl_sync(FULL, c_base + c_used, 0);
      if (lane < W) wbase[lane] = cb + x - c;
      if (lane == 0) {
        c_used += tot;
        wbase[W] = pad_from;
        wcnt[W] = pad_n;
      }
    }
    // lane state out: status / pc into the shared rows (the live register
    // rows already are), then bulk stores of every row
#pragma unroll
    for (int h = 0; h < H; h++) {
      sstat[h * T + t] = valid[h] ? status[h] : (uint8_t)L_EXITED;
      spc[h * T + t] = pc[h];
    }
    __syncthreads();
    IPHASE(5);
    if (t == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const size_t g0 = (size_t)tile * TL;
      bulk_s2g(p.status_out + g0, sstat, (uint32_t)TL);
      bulk_s2g(p.pc_out + g0, spc, (uint32_t)TL * 4);
      for (uint32_t i = 0; i < p.n_live; i++) {
        const uint32_t r = s_live[i];
        bulk_s2g(p.regs_out + (size_t)r * p.reg_stride + g0, SREGS(cur) + (size_t)r * TL, (uint32_t)TL * 4);
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    // this warp's records: one bulk copy (its lane 0 waits for the read before
    // the next tile stages records again)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0 && S.fill) {
      const unsigned long long b = wbase[warp];
      if (b + S.fill <= p.stage_cap) {
        bulk_s2g(p.stage + b, S.recs, S.fill * 8u);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      } else {
        b_over = true;
      }
    }
    for (uint32_t i = t; i < wcnt[W]; i += T)  // sentinels in the abandoned chunk tail
      if (wbase[W] + i < p.stage_cap) p.stage[wbase[W] + i] = REC_SENTINEL;
    IPHASE(6);
    // no block barrier here: the next tile's first __syncthreads orders every
    // shared word a warp could overwrite early (wcnt / wbase are rewritten only
    // after it; lane-state buffers are refilled only after their bulk stores
    // have read them)
    IPHASE(7);
  }

  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // record / lane-state stores complete
  if (t == 0) {
    if (b_staged) atomicAdd(&p.ctr->staged_recs, b_staged);
  }
  // ---- block flush: sentinels in the last chunk's tail, statistics, flags
  // (the barrier: other warps may still be padding the last tile's abandoned
  // chunk from wbase[W] / wcnt[W])
  __syncthreads();
  if (t == 0) {
    wbase[W] = c_base + c_used;
    wcnt[W] = c_cap - c_used;
  }
  __syncthreads();
  for (uint32_t i = t; i < wcnt[W]; i += T)
    if (wbase[W] + i < p.stage_cap) p.stage[wbase[W] + i] = REC_SENTINEL;
  if (__any_sync(FULL, b_over) && lane == 0) p.ctr->log_overflow = 1;
  {  // per-warp totals
    b_instr = warp_sum64(b_instr);
    b_loads = warp_sum64(b_loads);
    b_stores = warp_sum64(b_stores);
    const bool any_ovl = __any_sync(FULL, b_ovl);
    if (lane == 0) {
      if (b_instr) atomicAdd(&p.ctr->iv_instr, b_instr);
      if (b_loads) atomicAdd(&p.ctr->iv_loads, b_loads);
      if (b_stores) atomicAdd(&p.ctr->iv_stores, b_stores);
      if (any_ovl) p.ctr->ovl_overflow = 1;
    }
  }
  if (__any_sync(FULL, b_wait) && lane == 0) p.ctr->any_waiting = 1;
#undef SREGS
#undef SPC
#undef SSTAT
}

// The carve-up of K1's dynamic shared memory for T threads and H lanes per
// thread (offsets in bytes; every buffer a TMA copy touches is 16-B aligned).
K1Layout k1_layout(const InterpParams& p, int T, bool code_in_smem, int H) {
  K1Layout L;
  const uint32_t W = (uint32_t)T / 32, TL = (uint32_t)(H * T);
  L.T = (uint32_t)T;
  L.TL = TL;
  L.W = W;
  uint32_t q = 0;
  L.regs = q; L.regs_buf = p.n_regs * TL * 4; q += LS_NB * L.regs_buf;  // register files (LS_NB buffers)
  L.spc = q; q += LS_NB * TL * 4;                                        // pc rows
  L.sstat = q; q += LS_NB * TL;                                          // status rows
  q = (q + 15) & ~15u;
  L.mbar = q; q += (16 * LS_NB + 15) & ~15;                              // mbarriers
  L.recs = q; q += W * (uint32_t)H * p.stage_warp * 8;                   // staging
  L.code = q; q += code_in_smem ? (p.n_instr + 1) * 16 : 0;              // pre-decoded heads + pad entry
  L.tail = q; q += code_in_smem ? (p.n_instr + 1) * 8 : 0;               // tails + pad
  L.ro = q; q += code_in_smem ? (p.n_instr + 1) * 4 : 0;                 // entry_ro
  q = (q + 15) & ~15u;
  L.ocell = q; q += p.ovl_cap * TL * 4;                                  // overlay cells
  L.oval = q; q += p.ovl_cap * TL * 4;                                   // overlay values
  L.soff = q; q += p.n_arrays * 4;                                       // array offsets
  L.ssize = q; q += p.n_arrays * 4;                                      // array sizes
  L.live = q; q += (p.n_live + 3) & ~3u;                                 // live register list
  L.wcnt = q; q += W * 4 + 8;                                            // warp counts, pad count
  q = (q + 7) & ~7u;
  L.wbase = q; q += (W + 1) * 8;                                         // warp bases, pad start
  L.total = q;
  return L;
}

size_t interp_smem_bytes(const InterpParams& p, int T, bool code_in_smem, int H) {
  return k1_layout(p, T, code_in_smem, H).total;
}

namespace {
template <int H, int MODE, bool SPILL>
cudaError_t launch_interp_h(const InterpParams& p, cudaStream_t s, int nsm) {
  const bool code_smem = p.n_instr <= 2048;
  int T = INTERP_T;
  while (T > 32 && interp_smem_bytes(p, T, code_smem, H) > INTERP_SMEM_CAP) T >>= 1;
  InterpParams q = p;
  q.lay = k1_layout(p, T, code_smem, H);
  const size_t sm = q.lay.total;
  auto kern = code_smem ? (p.fuel_check ? interp_kernel<true, true, H, MODE, SPILL> : interp_kernel<true, false, H, MODE, SPILL>)
                        : (p.fuel_check ? interp_kernel<false, true, H, MODE, SPILL> : interp_kernel<false, false, H, MODE, SPILL>);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, sm);
  const uint32_t tiles = (p.n_lanes + H * T - 1) / (H * T);
  const uint32_t grid = std::min<uint32_t>(tiles, (uint32_t)std::max(1, per_sm) * nsm);
  kern<<<grid, T, sm, s>>>(q);
  launched();
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_interp(const InterpParams& p, cudaStream_t s) {
  if (p.n_lanes == 0) return cudaSuccess;
  static DeviceSetup setup;
  static int nsm_of[RC_MAX_DEVICES];
  int dev = 0;
  cudaError_t se = setup.run(
      [](int d) -> cudaError_t {
#define RC_K1_VARIANTS(M, SP)                                                                                \
  interp_kernel<true, true, 1, M, SP>, interp_kernel<false, true, 1, M, SP>,                                 \
      interp_kernel<true, false, 1, M, SP>, interp_kernel<false, false, 1, M, SP>,                           \
      interp_kernel<true, true, INTERP_H, M, SP>, interp_kernel<false, true, INTERP_H, M, SP>,               \
      interp_kernel<true, false, INTERP_H, M, SP>, interp_kernel<false, false, INTERP_H, M, SP>
        for (auto f : {RC_K1_VARIANTS(0, false), RC_K1_VARIANTS(0, true), RC_K1_VARIANTS(2, false),
                       RC_K1_VARIANTS(2, true), interp_kernel<true, true, 1, 1, true>,
                       interp_kernel<false, true, 1, 1, true>, interp_kernel<true, false, 1, 1, true>,
                       interp_kernel<false, false, 1, 1, true>}) {
#undef RC_K1_VARIANTS
          cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
          if (e != cudaSuccess) return e;
          cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        }
        return cudaDeviceGetAttribute(&nsm_of[d], cudaDevAttrMultiProcessorCount, d);
      },
      &dev);
  if (se != cudaSuccess) return se;
  const int nsm = nsm_of[dev];
  // two work-items per thread when the batch has enough lanes to fill the GPU
  // (test hook RC_DEBUG_INTERP_H=1|2 forces one variant; results never differ)
  const char* force = getenv("RC_DEBUG_INTERP_H");
  const int h = force ? (force[0] != '1' ? INTERP_H : 1)
                      : (INTERP_H >= 2 && p.n_lanes >= (uint32_t)INTERP_H * 256u * (uint32_t)nsm ? INTERP_H : 1);
  if (p.alt_mask) return launch_interp_h<1, 1, true>(p, s, nsm);  // classification re-run (rare)
  if (p.direct) {
    if (p.may_spill)
      return h > 1 ? launch_interp_h<INTERP_H, 2, true>(p, s, nsm) : launch_interp_h<1, 2, true>(p, s, nsm);
    return h > 1 ? launch_interp_h<INTERP_H, 2, false>(p, s, nsm) : launch_interp_h<1, 2, false>(p, s, nsm);
  }
  if (p.may_spill)
    return h > 1 ? launch_interp_h<INTERP_H, 0, true>(p, s, nsm) : launch_interp_h<1, 0, true>(p, s, nsm);
  return h > 1 ? launch_interp_h<INTERP_H, 0, false>(p, s, nsm) : launch_interp_h<1, 0, false>(p, s, nsm);
}

}  // namespace rc
