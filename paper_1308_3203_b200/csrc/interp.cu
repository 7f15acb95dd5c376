// interp.cu — K1: one barrier interval of the §4 thread-local semantics for
// every live work-item of an instance batch.
//
// One CUDA thread = one simulated work-item (lane).  A warp is one instruction
// stream: each step it executes the instruction at the minimum pc among its
// running lanes (uniform fetch/decode), lanes at that pc execute it, the rest
// wait — a lane's result never depends on the order because, inside an
// interval, lanes only see the interval-start heap plus their own writes
// (delayed visibility, reading L2).
//
// Per lane: registers (Locals) live in shared memory laid out
// [reg][thread] (a warp touching one register hits 32 distinct banks); the
// own-write overlay (cell, value) also lives in shared memory.
//
// Rules implemented: assign (170), store (176/179) into the
// overlay, load (182/185, reading L11) from the overlay else the interval-start
// heap, assert (188) -> ⊥ report, assume (194) -> ⊤, barrier (200) -> suspend.
// ⊥ halts only the faulting lane (reading L5).  Every executed instruction
// costs one unit of fuel (reading L17).
//
// Log: a read record per performed LD, and at the end of the interval one
// write record per distinct cell the lane wrote carrying its final value
// (reading L3).  Records are staged per warp in shared memory and written out
// by the block with ONE global atomic per block (per-warp atomics on a single
// counter would serialise ~10^7 times per interval at config 5).
#include "rc_internal.h"

namespace rc {

namespace {
constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr int STAGE = 256;  // records staged per warp

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ void emit_report(const InterpParams& p, uint32_t inst, int32_t arr, int32_t idx,
                                            uint32_t t1, uint32_t t2, uint16_t kind) {
  unsigned long long pos = atomicAdd(&p.ctr->report_count, 1ull);
  if (pos < p.report_cap) {
    rc_report r;
    r.instance = p.inst_base + inst;
    r.interval = p.interval;
    r.array = arr;
    r.index = idx;
    r.tid1 = t1;
    r.tid2 = t2;
    r.kind = kind;
    r.flags = 0;
    r.reserved = 0;
    p.reports[pos] = r;
  }
}

struct Stage {
  uint32_t* keys;  // this warp's staging area
  uint64_t* vals;
  uint32_t fill;   // warp-uniform
};

// write this warp's staged records to the global log (mid-interval overflow path)
__device__ __noinline__ void flush_warp(const InterpParams& p, Stage& S, int lane) {
  __syncwarp();
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(&p.ctr->log_count, (unsigned long long)S.fill);
  base = __shfl_sync(FULL, base, 0);
  bool over = false;
  for (uint32_t i = lane; i < S.fill; i += 32) {
    unsigned long long pos = base + i;
    if (pos < p.log_cap) {
      p.log_keys[pos] = S.keys[i];
      p.log_vals[pos] = S.vals[i];
    } else {
      over = true;
    }
  }
  if (__any_sync(FULL, over) && lane == 0) p.ctr->log_overflow = 1;
  __syncwarp();
  S.fill = 0;
}

// warp-aggregated append of one record per lane in `m` (must be called by the whole warp)
__device__ __forceinline__ void stage_append(const InterpParams& p, Stage& S, int lane, unsigned m, bool mine,
                                             uint32_t key, uint64_t val) {
  uint32_t cnt = __popc(m);
  if (S.fill + cnt > STAGE) flush_warp(p, S, lane);
  if (mine) {
    uint32_t pos = S.fill + __popc(m & lanemask_lt());
    S.keys[pos] = key;
    S.vals[pos] = val;
  }
  S.fill += cnt;
}

__device__ __forceinline__ unsigned long long warp_sum64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

__device__ __forceinline__ int32_t wadd(int32_t x, int32_t y) { return (int32_t)((uint32_t)x + (uint32_t)y); }

}  // namespace

__global__ void __launch_bounds__(256) interp_kernel(const InterpParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int T = blockDim.x;
  const int W = T >> 5;
  const int t = threadIdx.x;
  const int warp = t >> 5, lane = t & 31;
  const uint32_t R = p.n_regs;

  uint64_t* st_vals = reinterpret_cast<uint64_t*>(smem);
  uint32_t* st_keys = reinterpret_cast<uint32_t*>(st_vals + (size_t)W * STAGE);
  int32_t* sregs = reinterpret_cast<int32_t*>(st_keys + (size_t)W * STAGE);
  uint32_t* ocell = reinterpret_cast<uint32_t*>(sregs + (size_t)R * T);
  int32_t* oval = reinterpret_cast<int32_t*>(ocell + (size_t)OVL_CAP * T);
  uint32_t* s_off = reinterpret_cast<uint32_t*>(oval + (size_t)OVL_CAP * T);
  uint32_t* s_size = s_off + p.n_arrays;
  uint32_t* wcnt = s_size + p.n_arrays;       // [W]
  unsigned long long* wbase = reinterpret_cast<unsigned long long*>(
      (reinterpret_cast<uintptr_t>(wcnt + W) + 7) & ~uintptr_t(7));  // [W]
  unsigned long long* wstat = wbase + W;      // [3][W]

  for (uint32_t a = t; a < p.n_arrays; a += T) {
    s_off[a] = p.arr_off[a];
    s_size[a] = p.arr_size[a];
  }

  const uint32_t g = blockIdx.x * (uint32_t)T + t;
  const bool valid = g < p.n_lanes;
  uint8_t status = valid ? p.status_in[g] : (uint8_t)L_EXITED;
  bool running = valid && (status == L_RUNNING || status == L_WAITING);
  const uint32_t inst = valid ? g / p.n : 0;
  const uint32_t tid = valid ? g - inst * p.n : 0;
  const uint32_t cell_base = inst * p.cpi;
  uint32_t pc = running ? p.pc_in[g] : 0;
  int32_t* Rg = sregs + t;  // register r of this lane = Rg[r*T]
  if (running)
    for (uint32_t r = 0; r < R; r++) Rg[r * T] = p.regs_in[(size_t)r * p.n_lanes + g];
  __syncthreads();

  if (running) status = L_RUNNING;
  int n_own = 0;
  int32_t node = NODE_NONE;
  unsigned long long steps = 0;
  uint32_t nloads = 0, nstores = 0;
  bool ovl_over = false;
  Stage S{st_keys + (size_t)warp * STAGE, st_vals + (size_t)warp * STAGE, 0};

  for (;;) {
    if (__ballot_sync(FULL, running) == 0) break;
    const uint32_t minpc = __reduce_min_sync(FULL, running ? pc : 0xFFFFFFFFu);
    bool ex = running && pc == minpc;
    const Ins I = p.code[minpc];
    if (ex) {  // fuel check before executing (reading L17)
      if (steps == p.fuel) {
        emit_report(p, inst, -1, (int32_t)pc, tid, NOTID, RC_FUEL);
        running = false;
        status = L_FUEL;
        ex = false;
      } else {
        steps++;
      }
    }
    switch (I.op) {  // warp-uniform
      case RC_OP_CONST: if (ex) { Rg[I.a * T] = I.imm; pc++; } break;
      case RC_OP_MOV: if (ex) { Rg[I.a * T] = Rg[I.b * T]; pc++; } break;
      case RC_OP_TID: if (ex) { Rg[I.a * T] = (int32_t)tid; pc++; } break;
      case RC_OP_SIZE: if (ex) { Rg[I.a * T] = (int32_t)s_size[I.b]; pc++; } break;
      case RC_OP_ADDI: if (ex) { Rg[I.a * T] = wadd(Rg[I.b * T], I.imm); pc++; } break;
      case RC_OP_ADD: case RC_OP_SUB: case RC_OP_MUL: case RC_OP_MIN: case RC_OP_MAX: case RC_OP_AND:
      case RC_OP_OR: case RC_OP_XOR: case RC_OP_LT: case RC_OP_EQ: case RC_OP_LAND:
        if (ex) {
          const int32_t x = Rg[I.b * T], y = Rg[I.c * T];
          int32_t v;
          switch (I.op) {
            case RC_OP_ADD: v = wadd(x, y); break;
            case RC_OP_SUB: v = (int32_t)((uint32_t)x - (uint32_t)y); break;
            case RC_OP_MUL: v = (int32_t)((uint32_t)x * (uint32_t)y); break;
            case RC_OP_MIN: v = min(x, y); break;
            case RC_OP_MAX: v = max(x, y); break;
            case RC_OP_AND: v = x & y; break;
            case RC_OP_OR: v = x | y; break;
            case RC_OP_XOR: v = x ^ y; break;
            case RC_OP_LT: v = x < y; break;
            case RC_OP_EQ: v = x == y; break;
            default: v = (x != 0) && (y != 0); break;
          }
          Rg[I.a * T] = v;
          pc++;
        }
        break;
      case RC_OP_DIV: case RC_OP_MOD:
        if (ex) {
          const int32_t x = Rg[I.b * T], y = Rg[I.c * T];
          if (y == 0) {
            emit_report(p, inst, -1, (int32_t)pc, tid, NOTID, RC_DIV0);
            running = false;
            status = L_DIV0;
          } else {
            int32_t v;
            if (I.op == RC_OP_DIV) v = (y == -1) ? (int32_t)(0u - (uint32_t)x) : x / y;
            else v = (y == -1) ? 0 : x % y;
            Rg[I.a * T] = v;
            pc++;
          }
        }
        break;
      case RC_OP_LNOT: if (ex) { Rg[I.a * T] = Rg[I.b * T] == 0; pc++; } break;
      case RC_OP_LD: {
        bool ok = false;
        uint32_t cell = 0;
        if (ex) {
          const int32_t idx = Rg[I.c * T];
          if (idx < 0 || (uint32_t)idx >= s_size[I.b]) {
            emit_report(p, inst, (int32_t)I.b, idx, tid, NOTID, RC_OOB);
            running = false;
            status = L_OOB;
          } else {
            cell = cell_base + s_off[I.b] + (uint32_t)idx;
            int32_t v = 0;
            bool found = false;
            for (int j = 0; j < n_own; j++)
              if (ocell[j * T + t] == cell) { v = oval[j * T + t]; found = true; }
            if (!found) v = __ldg(p.heap + cell);
            Rg[I.a * T] = v;
            pc++;
            nloads++;
            ok = true;
          }
        }
        const unsigned m = __ballot_sync(FULL, ok);
        if (m) stage_append(p, S, lane, m, ok, cell, (uint64_t)(tid << 1));
        break;
      }
      case RC_OP_ST:
        if (ex) {
          const int32_t idx = Rg[I.b * T];
          if (idx < 0 || (uint32_t)idx >= s_size[I.a]) {
            emit_report(p, inst, (int32_t)I.a, idx, tid, NOTID, RC_OOB);
            running = false;
            status = L_OOB;
          } else {
            const uint32_t cell = cell_base + s_off[I.a] + (uint32_t)idx;
            int j = 0;
            while (j < n_own && ocell[j * T + t] != cell) j++;
            if (j == n_own) {
              if (n_own < OVL_CAP) { ocell[j * T + t] = cell; n_own++; }
              else { ovl_over = true; j = -1; }
            }
            if (j >= 0) oval[j * T + t] = Rg[I.c * T];
            pc++;
            nstores++;
          }
        }
        break;
      case RC_OP_BAR: if (ex) { node = (int32_t)pc; pc++; running = false; status = L_WAITING; } break;
      case RC_OP_EXIT: if (ex) { node = NODE_EXIT; running = false; status = L_EXITED; } break;
      case RC_OP_ASSUME:
        if (ex) {
          if (Rg[I.a * T] == 0) { running = false; status = L_PRUNED; }
          else pc++;
        }
        break;
      case RC_OP_ASSERT:
        if (ex) {
          if (Rg[I.a * T] == 0) {
            emit_report(p, inst, -1, (int32_t)pc, tid, NOTID, RC_ASSERT);
            running = false;
            status = L_ASSERT;
          } else {
            pc++;
          }
        }
        break;
      case RC_OP_BR: if (ex) pc = Rg[I.a * T] != 0 ? (uint32_t)I.imm : (uint32_t)I.b + 256u * I.c; break;
      case RC_OP_JMP: if (ex) pc = (uint32_t)I.imm; break;
      default: break;  // unreachable: the validator rejects unknown opcodes
    }
  }

  // write records: one per distinct written cell, final value (reading L3)
  const int max_own = __reduce_max_sync(FULL, (unsigned)n_own);
  for (int j = 0; j < max_own; j++) {
    const bool has = j < n_own;
    const unsigned m = __ballot_sync(FULL, has);
    uint64_t v = 0;
    uint32_t c = 0;
    if (has) {
      c = ocell[j * T + t];
      v = ((uint64_t)(uint32_t)oval[j * T + t] << 32) | (uint64_t)(tid << 1) | 1ull;
    }
    stage_append(p, S, lane, m, has, c, v);
  }

  // lane state out
  if (valid) {
    p.status_out[g] = status;
    p.node_out[g] = node;
    if (status == L_WAITING) {
      p.pc_out[g] = pc;
      for (uint32_t r = 0; r < R; r++) p.regs_out[(size_t)r * p.n_lanes + g] = Rg[r * T];
    }
  }

  // block-level log write-out: one atomic per block
  unsigned long long s0 = warp_sum64(steps), s1 = warp_sum64(nloads), s2 = warp_sum64(nstores);
  const bool any_ovl = __any_sync(FULL, ovl_over);
  if (lane == 0) {
    wcnt[warp] = S.fill;
    wstat[warp] = s0;
    wstat[W + warp] = s1;
    wstat[2 * W + warp] = s2;
    if (any_ovl) p.ctr->ovl_overflow = 1;
  }
  __syncthreads();
  if (t == 0) {
    unsigned long long tot = 0, a0 = 0, a1 = 0, a2 = 0;
    for (int w = 0; w < W; w++) {
      wbase[w] = tot;
      tot += wcnt[w];
      a0 += wstat[w];
      a1 += wstat[W + w];
      a2 += wstat[2 * W + w];
    }
    const unsigned long long base = tot ? atomicAdd(&p.ctr->log_count, tot) : 0ull;
    for (int w = 0; w < W; w++) wbase[w] += base;
    if (base + tot > p.log_cap) p.ctr->log_overflow = 1;
    if (a0) atomicAdd(&p.ctr->iv_instr, a0);
    if (a1) atomicAdd(&p.ctr->iv_loads, a1);
    if (a2) atomicAdd(&p.ctr->iv_stores, a2);
  }
  __syncthreads();
  const unsigned long long base = wbase[warp];
  for (uint32_t i = lane; i < S.fill; i += 32) {
    const unsigned long long pos = base + i;
    if (pos < p.log_cap) {
      p.log_keys[pos] = S.keys[i];
      p.log_vals[pos] = S.vals[i];
    }
  }
}

int interp_threads(uint32_t n_regs) {
  // keep the per-block shared memory within ~96 KB so >= 2 blocks fit per SM
  for (int T = 256; T >= 32; T >>= 1)
    if (interp_smem_bytes(n_regs, T) <= 96 * 1024) return T;
  return 32;
}

size_t interp_smem_bytes(uint32_t n_regs, int T) {
  const int W = T / 32;
  size_t b = (size_t)W * STAGE * (8 + 4);         // staging
  b += (size_t)n_regs * T * 4;                     // registers
  b += (size_t)OVL_CAP * T * 8;                    // overlay
  b += 2 * 256 * 4;                                // array offsets / sizes
  b += (size_t)W * 4 + 8;                          // warp counts (+align)
  b += (size_t)W * 8 * 4;                          // warp bases + 3 stats
  return b;
}

cudaError_t launch_interp(const InterpParams& p, cudaStream_t s) {
  if (p.n_lanes == 0) return cudaSuccess;
  const int T = interp_threads(p.n_regs);
  const size_t sm = interp_smem_bytes(p.n_regs, T);
  static bool attr_set = false;  // per process; the attribute is per function
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(interp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const uint32_t grid = (p.n_lanes + T - 1) / T;
  interp_kernel<<<grid, T, sm, s>>>(p);
  launched();
  return cudaGetLastError();
}

}  // namespace rc
