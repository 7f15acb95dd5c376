// detect.cu — K4+K5: segmented race detection over the sorted access log,
// fused with the barrier-release commit.
//
// A segment is the run of records of one cell c.  For it the race rule of
// PAPER.md:224-229 (reading L1) and the benign test of PAPER.md:23, 229 are
// applied with the pair rule of reading L4:
//   WW  if |W(c)| >= 2: non-benign iff two writers' final values differ; pair
//       = (min W, min{w : val_w != val_{min W}}), else (two smallest writers);
//   RW  if some r in R(c), w in W(c), r != w: pair = lexicographically smallest
//       (t1 < t2) with one reading and the other writing.
// and the barrier release PAPER.md:220-222 commits heap[c] <- val of the
// max-tid writer (invariant I4 of DESIGN.md §3).
//
// Every statistic is an order-independent reduction (min / second-min / max /
// membership), so the within-cell order the sort leaves does not matter.
// RW pair from first-pass statistics:
//   t1 = min(r1 if r1 < wmax, w1 if w1 < rmax),   t1 <= r1 and t1 <= w1,
//   t2 = min(t1 == r1 ? (w1 > t1 ? w1 : w2) : INF, t1 == w1 ? (r1 > t1 ? r1 : r2) : INF).
#include "rc_internal.h"

namespace rc {

namespace {
constexpr uint32_t INF = 0xFFFFFFFFu;

__device__ __forceinline__ void emit(const DetectParams& p, uint32_t cell, uint32_t t1, uint32_t t2, uint16_t kind,
                                  uint16_t flags) {
  const uint32_t inst = cell / p.cpi;
  const uint32_t rem = cell - inst * p.cpi;
  uint32_t a = 0;
  while (a + 1 < p.n_arrays && __ldg(p.arr_off + a + 1) <= rem) a++;
  unsigned long long pos = atomicAdd(&p.ctr->report_count, 1ull);
  if (pos < p.report_cap) {
    rc_report r;
    r.instance = p.inst_base + inst;
    r.interval = p.interval;
    r.array = (int32_t)a;
    r.index = (int32_t)(rem - __ldg(p.arr_off + a));
    r.tid1 = t1;
    r.tid2 = t2;
    r.kind = kind;
    r.flags = flags;
    r.reserved = 0;
    p.reports[pos] = r;
  }
}

// Emit the RW / WW reports of one cell.
__device__ __forceinline__ void finish_cell(const DetectParams& p, uint32_t key, uint32_t w1, uint32_t w2,
                                            uint32_t nw, uint32_t t1, uint32_t t2, uint32_t nb, bool t1r,
                                            bool t2r, bool t2w, bool w1r, bool w2r, bool nbr) {
  if (t1 != INF)  // t1 <= w1, so t1 writes iff t1 == w1
    emit(p, key, t1, t2, RC_RW, (t1r ? 1 : 0) | (t1 == w1 ? 2 : 0) | (t2r ? 4 : 0) | (t2w ? 8 : 0));
  if (nw >= 2) {
    if (nb != INF) emit(p, key, w1, nb, RC_WW_NONBENIGN, (w1r ? 1 : 0) | 2 | (nbr ? 4 : 0) | 8);
    else emit(p, key, w1, w2, RC_WW_BENIGN, (w1r ? 1 : 0) | 2 | (w2r ? 4 : 0) | 8);
  }
}

// RW pair from the first-pass statistics (see header comment)
__device__ __forceinline__ void rw_pair(bool hasr, uint32_t r1, uint32_t r2, uint32_t rmax, uint32_t w1,
                                        uint32_t w2, uint32_t wmax, uint32_t* t1, uint32_t* t2) {
  *t1 = INF;
  *t2 = INF;
  if (!hasr) return;
  const uint32_t c1 = r1 < wmax ? r1 : INF;
  const uint32_t c2 = w1 < rmax ? w1 : INF;
  *t1 = min(c1, c2);
  if (*t1 != INF) {
    const uint32_t mw = w1 > *t1 ? w1 : w2;
    const uint32_t mr = r1 > *t1 ? r1 : r2;
    *t2 = min(*t1 == r1 ? mw : INF, *t1 == w1 ? mr : INF);
  }
}

// Serial path for a segment that does not fit one 32-record round: the head
// thread walks it (pass 1: statistics; pass 2: first differing writer and
// membership flags; pass 3 only for a non-benign pair with readers).
__device__ __forceinline__ void serial_segment(const DetectParams& p, uint32_t i) {
  const uint32_t key = __ldg(p.keys + i);
  uint32_t r1 = INF, r2 = INF, rmax = 0, w1 = INF, w2 = INF, wmax = 0, nw = 0;
  bool hasr = false;
  int32_t vw1 = 0, vwmax = 0;
  uint32_t end = i;
  do {
    const uint64_t v = __ldg(p.vals + end);
    const uint32_t tid = (uint32_t)v >> 1;
    if (v & 1) {
      const int32_t val = (int32_t)(v >> 32);
      if (tid < w1) { w2 = w1; w1 = tid; vw1 = val; }
      else if (tid < w2) w2 = tid;
      if (nw == 0 || tid > wmax) { wmax = tid; vwmax = val; }
      nw++;
    } else {
      if (tid < r1) { r2 = r1; r1 = tid; }
      else if (tid > r1 && tid < r2) r2 = tid;
      if (!hasr || tid > rmax) rmax = tid;
      hasr = true;
    }
    end++;
  } while (end < p.n_records && __ldg(p.keys + end) == key);
  if (nw == 0) return;  // only reads: no conflict, nothing to commit
  p.heap[key] = vwmax;  // barrier release: max-tid writer wins
  uint32_t t1, t2;
  rw_pair(hasr, r1, r2, rmax, w1, w2, wmax, &t1, &t2);
  if (t1 == INF && nw < 2) return;
  uint32_t nb = INF;
  bool t1r = false, t2r = false, t2w = false, w1r = false, w2r = false;
  for (uint32_t j = i; j < end; j++) {
    const uint64_t v = __ldg(p.vals + j);
    const uint32_t tid = (uint32_t)v >> 1;
    if (v & 1) {
      if ((int32_t)(v >> 32) != vw1 && tid < nb) nb = tid;
      t2w |= tid == t2;
    } else {
      t1r |= tid == t1;
      t2r |= tid == t2;
      w1r |= tid == w1;
      w2r |= tid == w2;
    }
  }
  bool nbr = false;
  if (nb != INF && hasr)
    for (uint32_t j = i; j < end; j++) {
      const uint64_t v = __ldg(p.vals + j);
      if (!(v & 1) && ((uint32_t)v >> 1) == nb) nbr = true;
    }
  finish_cell(p, key, w1, w2, nw, t1, t2, nb, t1r, t2r, t2w, w1r, w2r, nbr);
}
}  // namespace

constexpr uint32_t DET_ROUNDS = 8;  // 32-record rounds per warp
constexpr uint32_t DET_CHUNK = 32 * DET_ROUNDS;

// Warp-cooperative detection: a warp owns DET_CHUNK consecutive records and
// reads them 32 at a time (coalesced).  __match_any_sync groups the lanes of
// one cell; a cell whose whole segment lies in the round is reduced with
// redux.sync / ballot / shfl over its group mask (groups run their collectives
// concurrently, each with its own mask); a segment that starts in the round
// but continues past it goes to serial_segment on its head lane; records of a
// segment that started earlier belong to that segment's head.
__global__ void __launch_bounds__(256) detect_kernel(const DetectParams p) {
  const unsigned FULL = 0xFFFFFFFFu;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t wg = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t c0 = wg * DET_CHUNK;
  if (c0 >= p.n_records) return;  // whole warp
  const uint64_t c1 = min((uint64_t)p.n_records, c0 + DET_CHUNK);
  for (uint64_t b = c0; b < c1; b += 32) {
    const uint64_t r = b + lane;
    const bool inb = r < c1;
    const uint32_t key = inb ? __ldg(p.keys + r) : 0xFFFFFFFFu;  // cell ids are < 0xFFFFFFFF
    const uint64_t v = inb ? __ldg(p.vals + r) : 0ull;
    uint32_t prev = __shfl_up_sync(FULL, key, 1);
    if (lane == 0) prev = b > 0 ? __ldg(p.keys + b - 1) : ~key;
    uint32_t next = __shfl_down_sync(FULL, key, 1);
    if (lane == 31) next = r + 1 < p.n_records ? __ldg(p.keys + r + 1) : ~key;
    const bool head = inb && prev != key;
    const bool tail = inb && next != key;
    const unsigned peers = __match_any_sync(FULL, key);
    const int lo = __ffs(peers) - 1, hi = 31 - __clz(peers);
    const bool lo_head = __shfl_sync(FULL, head, lo);
    const bool hi_tail = __shfl_sync(FULL, tail, hi);
    if (head && !hi_tail) serial_segment(p, (uint32_t)r);  // segment continues past this round
    if (!(inb && lo_head && hi_tail)) continue;             // not a complete segment of this round
    const uint32_t tid = (uint32_t)v >> 1;
    const bool isw = (v & 1) != 0;
    const int32_t val = (int32_t)(v >> 32);
    const uint32_t wmaxp1 = __reduce_max_sync(peers, isw ? tid + 1 : 0u);
    if (wmaxp1 == 0) continue;  // only reads: no conflict, nothing to commit
    const uint32_t r1 = __reduce_min_sync(peers, isw ? INF : tid);
    const uint32_t r2 = __reduce_min_sync(peers, (!isw && tid != r1) ? tid : INF);
    const uint32_t rmaxp1 = __reduce_max_sync(peers, isw ? 0u : tid + 1);
    const uint32_t w1 = __reduce_min_sync(peers, isw ? tid : INF);
    const uint32_t w2 = __reduce_min_sync(peers, (isw && tid != w1) ? tid : INF);
    const uint32_t wmax = wmaxp1 - 1;
    const unsigned wmask = __ballot_sync(peers, isw);
    const int32_t vw1 = __shfl_sync(peers, val, __ffs(__ballot_sync(peers, isw && tid == w1)) - 1);
    const int32_t vwmax = __shfl_sync(peers, val, __ffs(__ballot_sync(peers, isw && tid == wmax)) - 1);
    uint32_t t1, t2;
    rw_pair(rmaxp1 != 0, r1, r2, rmaxp1 - 1, w1, w2, wmax, &t1, &t2);
    const uint32_t nb = __reduce_min_sync(peers, (isw && val != vw1) ? tid : INF);
    const bool t1r = __ballot_sync(peers, !isw && tid == t1) != 0;
    const bool t2r = __ballot_sync(peers, !isw && tid == t2) != 0;
    const bool t2w = __ballot_sync(peers, isw && tid == t2) != 0;
    const bool w1r = __ballot_sync(peers, !isw && tid == w1) != 0;
    const bool w2r = __ballot_sync(peers, !isw && tid == w2) != 0;
    const bool nbr = __ballot_sync(peers, !isw && tid == nb) != 0;
    if ((int)lane == lo) {
      p.heap[key] = vwmax;  // barrier release: max-tid writer wins
      finish_cell(p, key, w1, w2, __popc(wmask), t1, t2, nb, t1r, t2r, t2w, w1r, w2r, nbr);
    }
  }
}

cudaError_t launch_detect(const DetectParams& p, cudaStream_t s) {
  if (p.n_records == 0) return cudaSuccess;
  const uint64_t warps = (p.n_records + DET_CHUNK - 1) / DET_CHUNK;
  detect_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(p);
  launched();
  return cudaGetLastError();
}

}  // namespace rc
