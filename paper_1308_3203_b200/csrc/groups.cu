// groups.cu — inter-group races (reading L20).
//
// With options->n_groups = G > 1 an instance runs G work-groups of n
// work-items (work-items are grouped in work-groups with their
// own ids; a barrier synchronises one work-group).  The canonical schedule
// runs the groups one after another in ascending order, each under the
// paper's semantics on the heap the previous ones left (runtime.cu), so
// intra-group races are the per-interval reports of K1/K4.  No barrier orders
// two groups: two work-items of different groups that access one cell
// anywhere in the kernel, at least one writing, race.  Because global tids
// ascend with the group (tid = gid * n + lid), the lexicographically smallest
// such pair can be folded in group by group:
//
//   per group pass h, per cell: rh / wh = smallest reader / writer tid of h
//     (ig_accumulate: atomicMin over every access record K1 logged);
//   after the pass (ig_combine), with r1 / w1 the smallest reader / writer of
//   the earlier groups:
//     IG_RW candidate  a = min(r1 if h writes, w1 if h reads),
//                      b = wh if a is r1 only, rh if a is w1 only, min of both
//                      if a is both; the pair = lexicographic min over passes;
//     IG_WW pair       (w1, wh) at the first pass h that writes after an
//                      earlier group wrote;
//     benign test      the cell's committed value after pass h is group h's
//                      last written value; non-benign iff two groups' last
//                      values differ (the final value of a write-only cell is
//                      the last value of whichever group writes last);
//   after every pass (ig_emit): one IG_RW and one IG_WW_* report per cell.
#include "rc_internal.h"

namespace rc {

namespace {
constexpr uint32_t INF = 0xFFFFFFFFu;

// per-cell state, IG_FIELDS u32 planes of `cells` words each
enum { CUR_R = 0, CUR_W, R1, W1, RW_A, RW_B, WW_A, WW_B, VAL, VFLAGS, IG_FIELDS_ };
static_assert(IG_FIELDS_ == IG_FIELDS, "state planes");
constexpr uint32_t VF_HAS = 1, VF_DIFFER = 2;

__global__ void ig_accumulate_kernel(const uint64_t* __restrict__ stage, const DevCounters* ctr, uint64_t cap,
                                     uint32_t* __restrict__ st, uint64_t cells, uint32_t n, uint32_t cpi,
                                     uint32_t gbase) {
  const uint64_t cnt = min((unsigned long long)cap, ctr->stage_count);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = stage[i];
    if (r == REC_SENTINEL) continue;
    const uint32_t cell = (uint32_t)(r >> REC_CELL_SHIFT);
    const uint32_t lane = ((uint32_t)r >> 5) & (MAX_WG - 1);
    const uint32_t tid = lane - (cell / cpi) * n + gbase;  // global tid
    atomicMin(st + (size_t)((r & 1) ? CUR_W : CUR_R) * cells + cell, tid);
  }
}

__global__ void ig_combine_kernel(uint32_t* __restrict__ st, const int32_t* __restrict__ heap, uint64_t cells) {
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += (uint64_t)gridDim.x * blockDim.x) {
#define F(k) st[(size_t)(k) * cells + c]
    const uint32_t rh = F(CUR_R), wh = F(CUR_W);
    if (rh == INF && wh == INF) continue;
    F(CUR_R) = INF;
    F(CUR_W) = INF;
    const uint32_t r1 = F(R1), w1 = F(W1);
    uint32_t a = INF, b = INF;
    if (wh != INF && r1 != INF) { a = r1; b = wh; }
    if (rh != INF && w1 != INF) {
      if (w1 < a) { a = w1; b = rh; }
      else if (w1 == a) b = min(b, rh);
    }
    if (a != INF) {
      const uint32_t pa = F(RW_A), pb = F(RW_B);
      if (a < pa || (a == pa && b < pb)) { F(RW_A) = a; F(RW_B) = b; }
    }
    if (wh != INF && w1 != INF && F(WW_A) == INF) { F(WW_A) = w1; F(WW_B) = wh; }
    if (wh != INF) {  // this group's last value of the cell is the committed one
      const int32_t v = heap[c];
      const uint32_t vf = F(VFLAGS);
      if (!(vf & VF_HAS)) { F(VAL) = (uint32_t)v; F(VFLAGS) = vf | VF_HAS; }
      else if ((int32_t)F(VAL) != v) F(VFLAGS) = vf | VF_DIFFER;
    }
    if (r1 == INF) F(R1) = rh;  // earlier groups have smaller tids: set once
    if (w1 == INF) F(W1) = wh;
#undef F
  }
}

__device__ __forceinline__ void ig_push(rc_report* reports, unsigned long long cap, DevCounters* ctr, const rc_report& r) {
  const unsigned long long pos = atomicAdd(&ctr->report_count, 1ull);
  if (pos < cap) reports[pos] = r;
}

__global__ void ig_emit_kernel(const uint32_t* __restrict__ st, uint64_t cells, uint32_t cpi,
                               const uint32_t* __restrict__ arr_off, uint32_t n_arrays, uint32_t inst_base,
                               rc_report* reports, unsigned long long cap, DevCounters* ctr) {
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cells; c += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t rw_a = st[(size_t)RW_A * cells + c], ww_a = st[(size_t)WW_A * cells + c];
    if (rw_a == INF && ww_a == INF) continue;
    const uint32_t inst = (uint32_t)(c / cpi), rem = (uint32_t)(c - (uint64_t)inst * cpi);
    uint32_t a = 0;
    while (a + 1 < n_arrays && arr_off[a + 1] <= rem) a++;
    rc_report r;
    r.instance = inst_base + inst;
    r.interval = RC_IG_INTERVAL;
    r.array = (int32_t)a;
    r.index = (int32_t)(rem - arr_off[a]);
    r.flags = 0;
    r.reserved = 0;
    if (rw_a != INF) {
      r.tid1 = rw_a;
      r.tid2 = st[(size_t)RW_B * cells + c];
      r.kind = RC_IG_RW;
      ig_push(reports, cap, ctr, r);
    }
    if (ww_a != INF) {
      r.tid1 = ww_a;
      r.tid2 = st[(size_t)WW_B * cells + c];
      r.kind = (st[(size_t)VFLAGS * cells + c] & VF_DIFFER) ? RC_IG_WW_NONBENIGN : RC_IG_WW_BENIGN;
      ig_push(reports, cap, ctr, r);
    }
  }
}

unsigned grid_for(uint64_t items) { return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((items + 255) / 256, 148ull * 16)); }
}  // namespace

cudaError_t ig_reset(uint32_t* st, uint64_t cells, cudaStream_t s) {
  // every plane INF except the value flags
  cudaError_t e = cudaMemsetAsync(st, 0xFF, (size_t)IG_FIELDS * cells * 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(st + (size_t)VFLAGS * cells, 0, cells * 4, s);
  return e;
}

cudaError_t launch_ig_accumulate(const uint64_t* stage, const DevCounters* ctr, uint64_t cap, uint32_t* st,
                                 uint64_t cells, uint32_t n, uint32_t cpi, uint32_t gbase, cudaStream_t s) {
  if (!cells || !cpi) return cudaSuccess;
  ig_accumulate_kernel<<<grid_for(cap), 256, 0, s>>>(stage, ctr, cap, st, cells, n, cpi, gbase);
  launched();
  return cudaGetLastError();
}

cudaError_t launch_ig_combine(uint32_t* st, const int32_t* heap, uint64_t cells, cudaStream_t s) {
  if (!cells) return cudaSuccess;
  ig_combine_kernel<<<grid_for(cells), 256, 0, s>>>(st, heap, cells);
  launched();
  return cudaGetLastError();
}

cudaError_t launch_ig_emit(const uint32_t* st, uint64_t cells, uint32_t cpi, const uint32_t* arr_off, uint32_t n_arrays,
                           uint32_t inst_base, rc_report* reports, unsigned long long cap, DevCounters* ctr,
                           cudaStream_t s) {
  if (!cells || !cpi) return cudaSuccess;
  ig_emit_kernel<<<grid_for(cells), 256, 0, s>>>(st, cells, cpi, arr_off, n_arrays, inst_base, reports, cap, ctr);
  launched();
  return cudaGetLastError();
}

}  // namespace rc
