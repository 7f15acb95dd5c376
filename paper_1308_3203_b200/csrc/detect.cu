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
}  // namespace

__global__ void __launch_bounds__(256) detect_kernel(const DetectParams p) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.n_records) return;
  const uint32_t key = __ldg(p.keys + i);
  if (i > 0 && __ldg(p.keys + i - 1) == key) return;  // not a segment head

  // pass 1: top-2 minima and maxima of readers and writers
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

  // barrier release: max-tid writer wins
  p.heap[key] = vwmax;

  uint32_t t1 = INF, t2 = INF;
  if (hasr) {
    const uint32_t c1 = r1 < wmax ? r1 : INF;
    const uint32_t c2 = w1 < rmax ? w1 : INF;
    t1 = min(c1, c2);
    if (t1 != INF) {
      const uint32_t mw = w1 > t1 ? w1 : w2;
      const uint32_t mr = r1 > t1 ? r1 : r2;
      t2 = min(t1 == r1 ? mw : INF, t1 == w1 ? mr : INF);
    }
  }
  if (t1 == INF && nw < 2) return;

  // pass 2: first differing writer, membership flags
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
  if (t1 != INF)  // t1 <= w1, so t1 writes iff t1 == w1
    emit(p, key, t1, t2, RC_RW, (t1r ? 1 : 0) | (t1 == w1 ? 2 : 0) | (t2r ? 4 : 0) | (t2w ? 8 : 0));
  if (nw >= 2) {
    if (nb != INF) {
      bool nbr = false;
      if (hasr)
        for (uint32_t j = i; j < end; j++) {
          const uint64_t v = __ldg(p.vals + j);
          if (!(v & 1) && ((uint32_t)v >> 1) == nb) nbr = true;
        }
      emit(p, key, w1, nb, RC_WW_NONBENIGN, (w1r ? 1 : 0) | 2 | (nbr ? 4 : 0) | 8);
    } else {
      emit(p, key, w1, w2, RC_WW_BENIGN, (w1r ? 1 : 0) | 2 | (w2r ? 4 : 0) | 8);
    }
  }
}

cudaError_t launch_detect(const DetectParams& p, cudaStream_t s) {
  if (p.n_records == 0) return cudaSuccess;
  detect_kernel<<<(p.n_records + 255) / 256, 256, 0, s>>>(p);
  launched();
  return cudaGetLastError();
}

}  // namespace rc
