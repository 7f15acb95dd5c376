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

// record fields (rc_internal.h make_rec); a write's final value lives in the
// side table wval[slot][lane], lane = (cell / cpi) * n + tid
__device__ __forceinline__ uint32_t rec_cell(uint64_t r) { return (uint32_t)(r >> REC_CELL_SHIFT); }
// the batch lane of the access (inst_local * n + tid): inside one cell (one
// instance) lanes order exactly like tids, so every statistic below is kept on
// lanes and emit() turns them into tids
__device__ __forceinline__ uint32_t rec_tid(uint64_t r) { return ((uint32_t)r >> 5) & (MAX_WG - 1); }
__device__ __forceinline__ bool rec_w(uint64_t r) { return (r & 1) != 0; }
// a spilled write (slot SLOT_SPILL): the value is in the lane's spill list (rare)
__device__ __noinline__ int32_t spilled_val(const DetectParams& p, uint64_t r) {
  const uint32_t lane = rec_tid(r), cell = rec_cell(r), ns = p.spill_n[lane];
  for (uint32_t j = 0; j < ns; j++)
    if (p.spill_cell[(size_t)j * p.n_lanes + lane] == cell) return p.spill_val[(size_t)j * p.n_lanes + lane];
  return 0;  // unreachable: K1 wrote the record from this list
}
template <bool SPILL>
__device__ __forceinline__ int32_t rec_val(const DetectParams& p, uint64_t r) {
  // slot * n_lanes + lane < 15 * 2^27: 32-bit index arithmetic
  const uint32_t slot = ((uint32_t)r >> 1) & 0xF;
  if (SPILL && slot == SLOT_SPILL) return spilled_val(p, r);
  // (L2, not the read-only path: with bval the bucket kernels fill wval for
  // the multi-record cells in this very launch)
  return __ldcg(p.wval + (slot * p.n_lanes + rec_tid(r)));
}
// K1c in region mode writes each value beside its record (bval) and no wval:
// the multi-record cells' write values are put where rec_val looks for them
__device__ __forceinline__ void put_val(const DetectParams& p, uint64_t r, int32_t v) {
  p.wval[(((uint32_t)r >> 1) & 0xF) * p.n_lanes + rec_tid(r)] = v;
}

__device__ __forceinline__ void emit(const DetectParams& p, uint32_t cell, uint32_t t1, uint32_t t2, uint16_t kind,
                                  uint16_t flags) {
  if (p.quiet) return;  // classification re-run: commit only
  if (kind == RC_RW) atomicAdd(&p.ctr->rw_reports, 1ull);
  const uint32_t inst = fast_div(cell, p.cpi_magic);
  const uint32_t rem = cell - inst * p.cpi;
  t1 = t1 - inst * p.n + p.gbase;  // batch lanes -> (global) tids
  if (t2 != INF) t2 = t2 - inst * p.n + p.gbase;
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

// Where a detection reads its sorted records from: the global sorted log
// (read-only for the kernel: non-coherent loads), a bucket sorted into
// global scratch by the same kernel (L2 loads), or a bucket in shared memory.
struct SrcLdg {
  const uint64_t* p;
  __device__ __forceinline__ uint64_t operator[](uint32_t i) const { return __ldg(p + i); }
};
struct SrcCg {
  const uint64_t* p;
  __device__ __forceinline__ uint64_t operator[](uint32_t i) const { return __ldcg(p + i); }
};
struct SrcSmem {
  const uint64_t* p;
  __device__ __forceinline__ uint64_t operator[](uint32_t i) const { return p[i]; }
};

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
// (out of line: the rare path stays out of the streaming loop's instruction footprint)
template <class Src>
__device__ __noinline__ void serial_segment(const DetectParams& p, const Src recs, uint32_t i, uint32_t n_records) {
  const uint32_t key = rec_cell(recs[i]);
  uint32_t r1 = INF, r2 = INF, rmax = 0, w1 = INF, w2 = INF, wmax = 0, nw = 0;
  bool hasr = false;
  int32_t vw1 = 0, vwmax = 0;
  uint32_t end = i;
  do {
    const uint64_t v = recs[end];
    const uint32_t tid = rec_tid(v);
    if (rec_w(v)) {
      const int32_t val = rec_val<true>(p, v);
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
  } while (end < n_records && rec_cell(recs[end]) == key);
  if (nw == 0) return;  // only reads: no conflict, nothing to commit
  p.heap[key] = vwmax;  // barrier release: max-tid writer wins
  uint32_t t1, t2;
  rw_pair(hasr, r1, r2, rmax, w1, w2, wmax, &t1, &t2);
  if (t1 == INF && nw < 2) return;
  uint32_t nb = INF;
  bool t1r = false, t2r = false, t2w = false, w1r = false, w2r = false;
  for (uint32_t j = i; j < end; j++) {
    const uint64_t v = recs[j];
    const uint32_t tid = rec_tid(v);
    if (rec_w(v)) {
      if (rec_val<true>(p, v) != vw1 && tid < nb) nb = tid;
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
      const uint64_t v = recs[j];
      if (!rec_w(v) && rec_tid(v) == nb) nbr = true;
    }
  finish_cell(p, key, w1, w2, nw, t1, t2, nb, t1r, t2r, t2w, w1r, w2r, nbr);
}
}  // namespace

#ifndef DET_MINB  // resident blocks per SM (register cap)
#define DET_MINB 2
#endif
#ifndef DET_ROUNDS_OPT
#define DET_ROUNDS_OPT 8
#endif
constexpr uint32_t DET_ROUNDS = DET_ROUNDS_OPT;  // 32-record rounds per warp (all prefetched)
constexpr uint32_t DET_CHUNK = 32 * DET_ROUNDS;

// Associative per-segment summary.  A cell is SIMPLE when it has at most one
// writer and no reader other than that writer: it can produce no report and
// only its commit is needed.  Everything else (>= 2 writers, or a reader that
// is not the writer) is COMPLEX and goes to serial_segment (reports).
struct Seg {
  uint32_t rmin, rmax;  // reader tids (rmin = INF: no reader)
  uint32_t w;           // a writer tid (the only one when nw == 1)
  int32_t vw;           // its value
  uint32_t nw;          // writers, saturating at 2
};
__device__ __forceinline__ Seg seg_merge(const Seg& a, const Seg& b) {
  Seg r;
  r.rmin = min(a.rmin, b.rmin);
  r.rmax = max(a.rmax, b.rmax);
  r.nw = min(2u, a.nw + b.nw);
  r.w = a.nw ? a.w : b.w;
  r.vw = a.nw ? a.vw : b.vw;
  return r;
}
__device__ __forceinline__ bool seg_complex(const Seg& s) {
  return s.nw >= 2 || (s.nw == 1 && s.rmin != INF && (s.rmin != s.w || s.rmax != s.w));
}
__device__ __forceinline__ Seg seg_shfl_down(const Seg& a, int off) {
  const unsigned FULL = 0xFFFFFFFFu;
  Seg r;
  r.rmin = __shfl_down_sync(FULL, a.rmin, off);
  r.rmax = __shfl_down_sync(FULL, a.rmax, off);
  r.w = __shfl_down_sync(FULL, a.w, off);
  r.vw = __shfl_down_sync(FULL, a.vw, off);
  r.nw = __shfl_down_sync(FULL, a.nw, off);
  return r;
}
__device__ __forceinline__ Seg seg_shfl(const Seg& a, int src) {
  const unsigned FULL = 0xFFFFFFFFu;
  Seg r;
  r.rmin = __shfl_sync(FULL, a.rmin, src);
  r.rmax = __shfl_sync(FULL, a.rmax, src);
  r.w = __shfl_sync(FULL, a.w, src);
  r.vw = __shfl_sync(FULL, a.vw, src);
  r.nw = __shfl_sync(FULL, a.nw, src);
  return r;
}

// Warp-cooperative detection.  A warp owns DET_CHUNK consecutive sorted
// records; all of them (and the final values of its write records) are loaded
// up front so the loads overlap, then processed 32 at a time.  Segment heads /
// tails come from comparing neighbouring keys (shuffles + the two boundary
// keys); each lane's suffix summary over its segment is built by a segmented
// shuffle reduction (log2(longest segment in the round) steps).  A segment
// that crosses a round boundary is carried (warp-uniform state) into the next
// round; one that crosses the chunk end, and every COMPLEX cell, is handled by
// serial_segment from the segment's head.  Segments that start before the
// chunk belong to the previous warp.
// The records of chunk wg (and its two boundary keys), issued as independent
// loads: the caller fetches the next chunk while it processes this one.
template <int ROUNDS = DET_ROUNDS>
struct Chunk {
  uint64_t vr[ROUNDS];
  uint32_t key_before, key_after;
};
template <class Src, int ROUNDS>
__device__ __forceinline__ void load_chunk(const Src recs, uint64_t wg, uint32_t n_records, Chunk<ROUNDS>& ch) {
  const int lane = threadIdx.x & 31;
  // record indices are < 2^32 (n_records is): 32-bit index arithmetic
  const uint32_t c0 = (uint32_t)wg * (32 * ROUNDS);
  const uint32_t c1 = min(n_records, c0 + 32 * ROUNDS);
#pragma unroll
  for (int rd = 0; rd < ROUNDS; rd++) {
    const uint32_t r = c0 + rd * 32 + lane;
    ch.vr[rd] = r < c1 ? recs[r] : ~0ull;
  }
  ch.key_before = c0 > 0 ? rec_cell(recs[c0 - 1]) : 0xFFFFFFFFu;
  ch.key_after = c1 < n_records ? rec_cell(recs[c1]) : 0xFFFFFFFFu;
}

template <bool SPILL, class Src, int ROUNDS>
__device__ __forceinline__ void detect_chunk(const DetectParams& p, const Src recs, uint64_t wg, uint32_t n_records,
                                             const Chunk<ROUNDS>& ch) {
  const unsigned FULL = 0xFFFFFFFFu;
  const int lane = threadIdx.x & 31;
  const uint32_t c0 = (uint32_t)wg * (32 * ROUNDS);
  const uint32_t c1 = min(n_records, c0 + 32 * ROUNDS);
  const uint64_t(&vr)[ROUNDS] = ch.vr;
  const uint32_t key_before = ch.key_before, key_after = ch.key_after;
  // final values of the chunk's write records (all gathers in flight at once)
  int32_t wv[ROUNDS];
#pragma unroll
  for (int rd = 0; rd < ROUNDS; rd++) wv[rd] = (vr[rd] != ~0ull && rec_w(vr[rd])) ? rec_val<SPILL>(p, vr[rd]) : 0;

  const Seg ident{INF, 0u, 0u, 0, 0u};
  bool carry = false;       // an open segment started in an earlier round of this chunk
  uint32_t carry_start = 0;
  Seg cs = ident;
  uint32_t last_key = key_before;  // key of the record before this round
#pragma unroll
  for (int rd = 0; rd < ROUNDS; rd++) {
    const uint32_t b = c0 + rd * 32;
    if (b >= c1) break;  // warp-uniform
    const uint32_t r = b + lane;
    const bool inb = r < c1;
    const uint64_t v = vr[rd];
    const uint32_t key = rec_cell(v);  // invalid lanes: 0xFFFFFFFF (cell ids are smaller)
    uint32_t prev = __shfl_up_sync(FULL, key, 1);
    if (lane == 0) prev = b > 0 ? last_key : ~key;
    uint32_t next = __shfl_down_sync(FULL, key, 1);
    const uint32_t next_round_first = rd + 1 < ROUNDS ? rec_cell(__shfl_sync(FULL, vr[rd + 1 < ROUNDS ? rd + 1 : rd], 0)) : 0u;
    if (lane == 31) next = r + 1 < c1 ? next_round_first : (r + 1 < n_records ? key_after : ~key);
    last_key = __shfl_sync(FULL, key, 31);
    const bool head = inb && prev != key;
    const bool tail = inb && next != key;  // last record of its segment (possibly beyond c1)
    const unsigned heads = __ballot_sync(FULL, head);
    const unsigned tails = __ballot_sync(FULL, tail);
    const unsigned inbm = __ballot_sync(FULL, inb);
    if (!carry && (heads & tails) == inbm) {
      // fast path: every record of the round is alone in its cell — a lone
      // writer only commits (no report is possible), a lone read does nothing
      if (inb && rec_w(v)) p.heap[key] = wv[rd];
      continue;
    }
    // hi = last lane of my segment inside this round
    const unsigned t_at_or_after = tails & (~0u << lane);
    const int last_inb = 31 - __clz(inbm);
    const int hi = t_at_or_after ? __ffs(t_at_or_after) - 1 : last_inb;
    const bool closes = (tails >> hi) & 1;  // segment ends inside this round
    // per-record summary, then segmented suffix reduction over [lane, hi]
    const uint32_t tid = rec_tid(v);
    Seg S = ident;
    if (inb) {
      if (rec_w(v)) { S.w = tid; S.vw = wv[rd]; S.nw = 1; }
      else { S.rmin = tid; S.rmax = tid; }
    }
    const bool starter = head || lane == 0;  // lanes whose suffix summary is consumed
    const uint32_t len = (starter && inb) ? (uint32_t)(hi - lane + 1) : 1u;
    const uint32_t maxlen = __reduce_max_sync(FULL, len);
    for (uint32_t off = 1; off < maxlen; off <<= 1) {
      const Seg T = seg_shfl_down(S, (int)off);
      if (lane + (int)off <= hi) S = seg_merge(S, T);
    }
    // lane 0's segment: continues the carried one, or belongs to the previous warp
    const Seg S0 = seg_shfl(S, 0);
    const bool l0_head = heads & 1u;
    const bool l0_closes = __shfl_sync(FULL, closes, 0);
    if (!l0_head && carry) {
      const Seg M = seg_merge(cs, S0);
      if (l0_closes) {
        if (lane == 0) {
          if (seg_complex(M)) serial_segment(p, recs, (uint32_t)carry_start, n_records);
          else if (M.nw == 1) p.heap[key] = M.vw;
        }
        carry = false;
      } else {
        cs = M;  // the whole round continues the carried segment
      }
    }
    // segments starting in this round
    if (head && closes) {
      if (seg_complex(S)) serial_segment(p, recs, (uint32_t)r, n_records);
      else if (S.nw == 1) p.heap[key] = S.vw;
    }
    // the last segment of the round stays open: carry it
    const bool opens = head && !closes;
    const unsigned om = __ballot_sync(FULL, opens);
    if (om) {
      const int h = __ffs(om) - 1;
      cs = seg_shfl(S, h);
      carry_start = b + h;
      carry = true;
    }
  }
  if (carry && lane == 0) serial_segment(p, recs, (uint32_t)carry_start, n_records);  // continues into the next chunk
}

// A4 fused as the tail of K4 (readings L9, L17): the
// last WARP to finish (a grid-wide warp counter, no block barrier: warps of a
// block finish independently) checks, per instance, whether the work-items
// that arrived in this interval reached more than one barrier node (K1
// reduced the min / max arrival node), resets the ranges, and takes the
// interval's verdict: `abort` when the host must act before the next interval
// may run (DevCounters::abort).  Called by converged full warps.
__device__ __forceinline__ void boundary_tail(const DetectParams& p) {
  DevCounters* c = p.ctr;
  const uint32_t lane = threadIdx.x & 31;
  uint32_t done = 0;
  if (lane == 0) {
    __threadfence();
    done = atomicAdd(&c->bdone, 1u);
  }
  done = __shfl_sync(0xFFFFFFFFu, done, 0);
  if (done != ((gridDim.x * blockDim.x) >> 5) - 1) return;
  __threadfence();
  // an interval that will be re-run (its log or K1's reports overflowed)
  // leaves the divergence flags of the previous interval in place: the re-run
  // of K1 reads them (static write-set elision, InterpParams::inst_div)
  const volatile DevCounters* cv = c;
  const bool rerun = cv->log_overflow || cv->ovl_overflow || cv->k1_reports > p.report_cap;
  bool any_div = false;
  for (uint32_t inst = lane; inst < p.n_inst; inst += 32) {
    const int32_t lo = p.node_min[inst], hi = p.node_max[inst];
    p.node_min[inst] = 0x7FFFFFFF;
    p.node_max[inst] = (int32_t)0x80000000;
    if (rerun) continue;
    const bool div = lo < hi;
    p.inst_flag[inst] = div;
    any_div |= div;
  }
  if (__any_sync(0xFFFFFFFFu, any_div) && lane == 0) c->diverged = 1;
  __syncwarp();
  if (lane == 0) {
    __threadfence();
    c->bdone = 0;
    const volatile DevCounters* v = c;
    const bool need_host = v->log_overflow || v->ovl_overflow || v->k1_reports > p.report_cap || v->bucket_overflow ||
                           v->report_count > p.report_cap || v->diverged || !v->any_waiting ||
                           (p.classify && v->rw_reports > 0);
    if (need_host) c->abort = 1;
  }
}

// Persistent: warps stride over the chunks; the record count is read from
// device memory (no host sync).  Skips the detection (no commit) when this
// interval's log, a spill list or K1's reports overflowed: the host then
// re-runs the interval from the saved lane state on an untouched heap.
template <bool SPILL>
__global__ void __launch_bounds__(256, DET_MINB) detect_kernel(const DetectParams p) {
  if (p.ctr->abort) return;  // speculative interval after one that needs the host (grid-uniform)
  if (!(p.ctr->log_overflow || p.ctr->ovl_overflow || p.ctr->k1_reports > p.report_cap)) {
    const uint32_t n_records = (uint32_t)p.ctr->kept_count;
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint64_t wg = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const SrcLdg recs{p.recs};
    Chunk<> cur, nxt;
    if (wg * DET_CHUNK < n_records) load_chunk(recs, wg, n_records, cur);
    for (; wg * DET_CHUNK < n_records; wg += warps) {
      // software pipeline: the next chunk's records load while this one is processed
      if ((wg + warps) * DET_CHUNK < n_records) load_chunk(recs, wg + warps, n_records, nxt);
      detect_chunk<SPILL>(p, recs, wg, n_records, cur);
      cur = nxt;
    }
  }
  __syncwarp();
  if (p.with_boundary) boundary_tail(p);
}

// ---- K4+K5 on the bucket path -------------------------------
// A bucket = the records of BUCKET_CELLS consecutive cells (bucket_scatter,
// sort.cu, grouped them in arbitrary order).  Block j takes buckets j,
// j + G, j + 2G, ... (G blocks).  A bucket of <= BD_CAP records is loaded into registers and
// counted per cell in shared memory; a cell with one record only commits (a
// lone writer can race with nobody, a lone read does nothing); the records of
// the other cells are placed by cell into shared memory (a counting sort on
// the low BUCKET_BITS bits) and run through the segmented detection above.
// A larger bucket is counting-sorted into global scratch (`tmp`) and detected
// there.  Any order inside a cell is fine: every statistic is
// order-independent.
#ifndef BD_THREADS_OPT
#define BD_THREADS_OPT 512
#endif
constexpr int BD_THREADS = BD_THREADS_OPT;
constexpr int BD_ITEMS = 16;
#ifndef BD_MINB_OPT
#define BD_MINB_OPT (1024 / BD_THREADS_OPT)
#endif
constexpr int BD_MINB = BD_MINB_OPT;  // resident blocks per SM (1024 threads: 64 registers per thread)
#ifndef BD_SORTED_OPT
#define BD_SORTED_OPT (BD_THREADS_OPT * 16)
#endif
constexpr uint32_t BD_SORTED = BD_SORTED_OPT;  // multi-record cells' records placed in shared memory
constexpr uint32_t BD_CAP = BD_THREADS * BD_ITEMS;  // records of a bucket held in registers
constexpr int BD_WARPS = BD_THREADS / 32;
constexpr int BD_ROUNDS = 2;  // 32-record rounds per detection chunk (the records are in shared memory / L2)
struct BucketSmem {
  uint64_t sorted[BD_SORTED];   // records of the bucket's multi-record cells, by cell (global path: u32 offsets)
  uint32_t cnt[BUCKET_CELLS + 4];  // per cell: record count (bits 0-15), then | start << 16 during the
                                   // placement; [BUCKET_CELLS]: the spare counter of absent items
  uint32_t wsum[BD_WARPS];
  uint32_t ls0[32], lm[32];     // the block's non-empty buckets: start, record count
  uint32_t nlist;
};
constexpr int BD_LIST = 32;  // buckets per block (blockIdx.x + i * gridDim.x, i < BD_LIST)
// block barrier that does not assume a converged warp (barrier.sync without
// .aligned): it follows detect_chunk, whose serial path runs on some lanes only
__device__ __forceinline__ void block_sync() { asm volatile("barrier.sync 0;" ::: "memory"); }
__device__ __forceinline__ uint32_t bucket_low(uint64_t r) {
  return (uint32_t)(r >> REC_CELL_SHIFT) & (BUCKET_CELLS - 1);
}

// exclusive scan over the 4096 per-cell values v[] (8 consecutive per thread);
// returns this thread's start, *total = the sum (synchronises the block)
__device__ __forceinline__ uint32_t bd_scan8(const uint32_t (&v)[BUCKET_CELLS / BD_THREADS], uint32_t* wsum,
                                             uint32_t* total) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  uint32_t sum = 0;
#pragma unroll
  for (int k = 0; k < (int)(BUCKET_CELLS / BD_THREADS); k++) sum += v[k];
  uint32_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  uint32_t run = x - sum, tot = 0;
#pragma unroll
  for (int i = 0; i < BD_WARPS; i++) {
    const uint32_t c = wsum[i];
    run += i < w ? c : 0u;
    tot += c;
  }
  *total = tot;
  return run;
}

// The bucket's cells with more than one record (S.cnt holds every cell's
// count): their records, re-read from L2, are placed by cell into shared
// memory (a counting sort on the low BUCKET_BITS bits) and run through the
// segmented detection.  Out of line: the single-record path stays lean.
template <bool SPILL>
__device__ __noinline__ void bucket_multi(const DetectParams& p, BucketSmem& S, uint32_t s0, uint32_t m) {
  const int t = threadIdx.x;
  constexpr int PER = BUCKET_CELLS / BD_THREADS;
  uint32_t v[PER];
#pragma unroll
  for (int k = 0; k < PER; k++) {
    const uint32_t c = S.cnt[t * PER + k] & 0xFFFFu;
    v[k] = c > 1 ? c : 0u;
  }
  uint32_t M = 0;
  uint32_t run = bd_scan8(v, S.wsum, &M);
#pragma unroll
  for (int k = 0; k < PER; k++)
    if (v[k]) {
      S.cnt[t * PER + k] = (run << 16) | v[k];
      run += v[k];
    }
  __syncthreads();
  // (more than BD_SORTED such records: placed in the global scratch instead)
  uint64_t* dst = M <= BD_SORTED ? S.sorted : p.tmp + s0;
  for (uint32_t i = t; i < m; i += BD_THREADS) {
    const uint64_t r = __ldcg(p.recs + s0 + i);
    uint32_t* c = &S.cnt[bucket_low(r)];
    if ((*c & 0xFFFFu) > 1u) dst[atomicAdd(c, 1u << 16) >> 16] = r;
  }
  __syncthreads();
  // segmented detection over dst[0, M): warps take 64-record chunks
  if (M <= BD_SORTED) {
    const SrcSmem src{S.sorted};
    for (uint32_t wg = (uint32_t)t >> 5; wg * (32 * BD_ROUNDS) < M; wg += BD_WARPS) {
      Chunk<BD_ROUNDS> ch;
      load_chunk(src, wg, M, ch);
      detect_chunk<SPILL>(p, src, wg, M, ch);
    }
  } else {
    const SrcCg src{p.tmp + s0};
    for (uint32_t wg = (uint32_t)t >> 5; wg * (32 * BD_ROUNDS) < M; wg += BD_WARPS) {
      Chunk<BD_ROUNDS> ch;
      load_chunk(src, wg, M, ch);
      detect_chunk<SPILL>(p, src, wg, M, ch);
    }
  }
  block_sync();
}

// returns true (block-uniform) when the segmented detection ran (its lanes
// may not have reconverged: the caller then uses the non-aligned barrier)
template <bool SPILL, int ITEMS>
__device__ __forceinline__ bool bucket_smem(const DetectParams& p, BucketSmem& S, uint32_t s0, uint32_t m) {
  const int t = threadIdx.x;
  uint64_t r[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; j++) {
    const uint32_t i = t + j * BD_THREADS;
    r[j] = i < m ? __ldg(p.recs + s0 + i) : REC_SENTINEL;
  }
  // the final values of the write records, gathered while the cells are
  // counted (used for the lone writers' commits; detect_chunk re-reads the
  // others')
  int32_t val[ITEMS];
  if (p.bval) {  // K1c wrote each value beside its record: no dependent gather
#pragma unroll
    for (int j = 0; j < ITEMS; j++) {
      const uint32_t i = t + j * BD_THREADS;
      val[j] = i < m ? __ldg(p.bval + s0 + i) : 0;
    }
  } else {
#pragma unroll
    for (int j = 0; j < ITEMS; j++) val[j] = (r[j] != REC_SENTINEL && rec_w(r[j])) ? rec_val<SPILL>(p, r[j]) : 0;
  }
  // (an absent item counts into the spare counter: no branch per item)
#pragma unroll
  for (int j = 0; j < ITEMS; j++) atomicAdd(&S.cnt[r[j] != REC_SENTINEL ? bucket_low(r[j]) : BUCKET_CELLS], 1u);
  __syncthreads();
  // single-record cells: the commit of a lone writer (barrier release)
  bool multi = false;
#pragma unroll
  for (int j = 0; j < ITEMS; j++) {
    const bool ok = r[j] != REC_SENTINEL;
    const bool lone = (S.cnt[ok ? bucket_low(r[j]) : BUCKET_CELLS] & 0xFFFFu) == 1u;
    if (ok && lone && rec_w(r[j])) p.heap[rec_cell(r[j])] = val[j];
    if (p.bval && ok && !lone && rec_w(r[j])) put_val(p, r[j], val[j]);  // (visible to the block after the barrier)
    multi |= ok && !lone;
  }
  __syncwarp();
  const bool any_multi = __syncthreads_or(multi);
  if (any_multi) bucket_multi<SPILL>(p, S, s0, m);
  // (the records are dead here: the counters are cleared whole, 8 per thread)
#pragma unroll
  for (int k = 0; k < (int)(BUCKET_CELLS / BD_THREADS); k++) S.cnt[t + k * BD_THREADS] = 0u;  // (the caller synchronises)
  if (t == 0) S.cnt[BUCKET_CELLS] = 0u;
  return any_multi;
}

// a bucket larger than BD_CAP: counting sort by cell into tmp[s0, s0 + m), then detect there
template <bool SPILL>
__device__ __noinline__ void bucket_global(const DetectParams& p, BucketSmem& S, uint32_t s0, uint32_t m) {
  const int t = threadIdx.x;
  for (uint32_t i = t; i < m; i += BD_THREADS) {
    const uint64_t r = __ldcg(p.recs + s0 + i);
    atomicAdd(&S.cnt[bucket_low(r)], 1u);
    if (p.bval && rec_w(r)) put_val(p, r, __ldcg(p.bval + s0 + i));
  }
  __syncthreads();
  constexpr int PER = BUCKET_CELLS / BD_THREADS;
  uint32_t* offs = reinterpret_cast<uint32_t*>(S.sorted);
  uint32_t v[PER];
#pragma unroll
  for (int k = 0; k < PER; k++) v[k] = S.cnt[t * PER + k];
  uint32_t tot = 0;
  uint32_t run = bd_scan8(v, S.wsum, &tot);
#pragma unroll
  for (int k = 0; k < PER; k++) {
    offs[t * PER + k] = run;
    run += v[k];
  }
  __syncthreads();
  for (uint32_t i = t; i < m; i += BD_THREADS) {
    const uint64_t r = __ldcg(p.recs + s0 + i);
    const uint32_t l = bucket_low(r);
    p.tmp[s0 + offs[l] + atomicSub(&S.cnt[l], 1u) - 1u] = r;  // (counts return to 0)
  }
  __syncthreads();  // the block's global stores are visible to the block
  const SrcCg src{p.tmp + s0};
  for (uint32_t wg = (uint32_t)t >> 5; wg * (32 * BD_ROUNDS) < m; wg += BD_WARPS) {
    Chunk<BD_ROUNDS> ch;
    load_chunk(src, wg, m, ch);
    detect_chunk<SPILL>(p, src, wg, m, ch);
  }
}

template <bool SPILL>
__global__ void __launch_bounds__(BD_THREADS, BD_MINB) bucket_detect_kernel(const DetectParams p) {
  extern __shared__ __align__(16) unsigned char bd_smem_raw[];
  BucketSmem& S = *reinterpret_cast<BucketSmem*>(bd_smem_raw);
  if (p.ctr->abort) return;  // speculative interval after one that needs the host (grid-uniform)
  const int t = threadIdx.x;
  if (!(p.ctr->log_overflow || p.ctr->ovl_overflow || p.ctr->k1_reports > p.report_cap ||
        (p.ctr->bucket_overflow && !p.region_rerun))) {
    for (uint32_t i = t; i < BUCKET_CELLS + 4; i += BD_THREADS) S.cnt[i] = 0u;
    // the block's buckets (static round robin: no claim round trips; empty
    // buckets — e.g. those of an array the interval does not write — drop out)
    if (t < 32) {
      const uint32_t b = blockIdx.x + (uint32_t)t * gridDim.x;
      uint32_t s0 = 0, m = 0;
      if (b < p.nb) {
        if (p.region) {  // region mode: bucket b = recs[b * region, + min(rcur[b], region))
          s0 = b * p.region;
          if (p.region_rerun) {
            m = p.rend[b] - s0;
          } else {
            m = min(__ldcg(p.rcur + b), p.region);
            p.rend[b] = s0 + m;  // (for a detect-only re-run: the next interval resets rcur)
          }
        } else {
          s0 = __ldg(p.bstart + b);
          m = __ldg(p.bend + b) - s0;
        }
      }
      const unsigned nz = __ballot_sync(0xFFFFFFFFu, m != 0);
      if (m) {
        const int k = __popc(nz & ((1u << t) - 1u));
        S.ls0[k] = s0;
        S.lm[k] = m;
      }
      if (t == 0) S.nlist = __popc(nz);
    }
    __syncthreads();
    const uint32_t nl = S.nlist;
    for (uint32_t i = 0; i < nl; i++) {
      const uint32_t s0 = S.ls0[i], m = S.lm[i];
      bool ran = true;
      if (m > BD_CAP) bucket_global<SPILL>(p, S, s0, m);
      else if (m <= BD_CAP / 2) ran = bucket_smem<SPILL, BD_ITEMS / 2>(p, S, s0, m);
      else ran = bucket_smem<SPILL, BD_ITEMS>(p, S, s0, m);
      if (ran) block_sync();  // (after detect_chunk the lanes of a warp need not have reconverged)
      else __syncthreads();
    }
  }
  __syncwarp();
  if (p.with_boundary) boundary_tail(p);
}

// ---- RW value classification helpers (DESIGN.md §3 reading L19) -----------
__global__ void rw_mark_kernel(const rc_report* __restrict__ reports, uint64_t r0, uint64_t r1, uint32_t inst_base,
                               uint32_t cpi, const uint32_t* __restrict__ arr_off, uint8_t* __restrict__ mask) {
  const uint64_t i = r0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r1) return;
  const rc_report r = reports[i];
  if (r.kind != RC_RW) return;
  mask[(uint64_t)(r.instance - inst_base) * cpi + arr_off[r.array] + (uint32_t)r.index] = 1;
}

// per instance (instances are independent runs): do the two heaps differ?
__global__ void heap_compare_kernel(const int32_t* __restrict__ a, const int32_t* __restrict__ b, uint64_t n,
                                    uint32_t cpi, uint32_t* __restrict__ diff) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    if (a[i] != b[i]) diff[i / cpi] = 1;
}

__global__ void rw_flag_kernel(rc_report* __restrict__ reports, uint64_t r0, uint64_t r1, uint32_t inst_base,
                               const uint32_t* __restrict__ diff) {
  const uint64_t i = r0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r1 || reports[i].kind != RC_RW) return;
  reports[i].flags |= diff[reports[i].instance - inst_base] ? 0x20 : 0x10;
}

cudaError_t launch_rw_mark(const rc_report* reports, uint64_t r0, uint64_t r1, uint32_t inst_base, uint32_t cpi,
                           const uint32_t* arr_off, uint8_t* mask, cudaStream_t s) {
  if (r1 <= r0) return cudaSuccess;
  rw_mark_kernel<<<(unsigned)((r1 - r0 + 255) / 256), 256, 0, s>>>(reports, r0, r1, inst_base, cpi, arr_off, mask);
  launched();
  return cudaGetLastError();
}
cudaError_t launch_heap_compare(const int32_t* a, const int32_t* b, uint64_t n, uint32_t cpi, uint32_t* diff,
                                cudaStream_t s) {
  if (!n) return cudaSuccess;
  heap_compare_kernel<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 8), 256, 0, s>>>(a, b, n, cpi, diff);
  launched();
  return cudaGetLastError();
}
cudaError_t launch_rw_flag(rc_report* reports, uint64_t r0, uint64_t r1, uint32_t inst_base, const uint32_t* diff,
                           cudaStream_t s) {
  if (r1 <= r0) return cudaSuccess;
  rw_flag_kernel<<<(unsigned)((r1 - r0 + 255) / 256), 256, 0, s>>>(reports, r0, r1, inst_base, diff);
  launched();
  return cudaGetLastError();
}

cudaError_t launch_bucket_detect(const DetectParams& p, cudaStream_t s) {
  static DeviceSetup setup;
  static int nsm_of[RC_MAX_DEVICES], per_sm_of[RC_MAX_DEVICES];
  int dev = 0;
  cudaError_t se = setup.run(
      [](int d) -> cudaError_t {
        const void* ks[2] = {(const void*)bucket_detect_kernel<false>, (const void*)bucket_detect_kernel<true>};
        for (const void* k : ks) {
          cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(BucketSmem));
          if (e != cudaSuccess) return e;
        }
        int per_sm = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bucket_detect_kernel<false>, BD_THREADS,
                                                                      sizeof(BucketSmem));
        if (e != cudaSuccess) return e;
        per_sm_of[d] = std::max(per_sm, 1);
        return cudaDeviceGetAttribute(&nsm_of[d], cudaDevAttrMultiProcessorCount, d);
      },
      &dev);
  if (se != cudaSuccess) return se;
  // one resident wave, but never more than BD_LIST buckets per block
  const unsigned grid = (unsigned)std::max<uint64_t>({uint64_t{1}, std::min<uint64_t>(p.nb, (uint64_t)nsm_of[dev] * per_sm_of[dev]),
                                                      (p.nb + BD_LIST - 1) / BD_LIST});
  if (p.spill_n) bucket_detect_kernel<true><<<grid, BD_THREADS, sizeof(BucketSmem), s>>>(p);
  else bucket_detect_kernel<false><<<grid, BD_THREADS, sizeof(BucketSmem), s>>>(p);
  launched();
  return cudaGetLastError();
}

cudaError_t launch_detect(const DetectParams& p, cudaStream_t s) {
  if (p.nb) return launch_bucket_detect(p, s);
  if (p.n_records == 0 && !p.with_boundary) return cudaSuccess;
  static DeviceSetup setup;
  static int nsm_of[RC_MAX_DEVICES], per_sm_of[RC_MAX_DEVICES];
  int dev = 0;
  cudaError_t se = setup.run(
      [](int d) -> cudaError_t {
        int per_sm = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, detect_kernel<false>, 256, 0);
        if (e != cudaSuccess) return e;
        per_sm_of[d] = std::max(per_sm, 1);
        return cudaDeviceGetAttribute(&nsm_of[d], cudaDevAttrMultiProcessorCount, d);
      },
      &dev);
  if (se != cudaSuccess) return se;
  const int nsm = nsm_of[dev], per_sm = per_sm_of[dev];
  // one resident wave (persistent warps stride over the chunks)
  const uint64_t warps = (p.n_records + DET_CHUNK - 1) / DET_CHUNK;  // upper bound
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((warps + 7) / 8, (uint64_t)nsm * per_sm));
  if (p.spill_n) detect_kernel<true><<<grid, 256, 0, s>>>(p);  // (spill_n: set iff the program may spill)
  else detect_kernel<false><<<grid, 256, 0, s>>>(p);
  launched();
  return cudaGetLastError();
}

}  // namespace rc
