// filter.cu — write-set filter / compaction between K1 and the sort.
//
// K1 staged the interval's access records in per-block chunks of one staging
// buffer (unused chunk tails hold REC_SENTINEL) and marked every written cell
// in the byte map wmap with this interval's tag.  This pass keeps every write
// record and the read
// records of written cells and writes them densely to the sort buffer.  A read
// of a cell that no work-item wrote in this interval can take part in no RW
// report (P:224-229 needs a writer), no WW report and no commit, so
// dropping it is exact: R(c) and W(c) of every cell with W(c) != {} are
// unchanged, and cells with W(c) = {} produce no output.
//
// Also computes the sort's digit histograms of the kept records (fused K2).
#include "rc_internal.h"

#ifndef F_ITEMS_OPT
#define F_ITEMS_OPT 4
#endif
namespace rc {

namespace {
constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr int F_THREADS = 256, F_ITEMS = F_ITEMS_OPT;
static_assert(F_ITEMS % 2 == 0, "two records per 16-byte load");

}  // namespace

__global__ void __launch_bounds__(F_THREADS) filter_kernel(const FilterParams p) {
  __shared__ uint32_t bh[4 * 256];
  __shared__ uint32_t wcnt[F_THREADS / 32];
  __shared__ unsigned long long sbase;
  __shared__ uint64_t sbuf[F_THREADS * F_ITEMS + 8 * F_ITEMS];
  if (p.ctr->abort) return;  // speculative interval (DevCounters::abort)
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  for (int i = t; i < p.passes * 256; i += F_THREADS) bh[i] = 0;
  if (blockIdx.x == 0 && t == 0) p.ctr->k1_reports = p.ctr->report_count;  // K1 is complete here
  if (p.ctr->log_overflow || p.ctr->ovl_overflow) return;  // the interval will be re-run
  // slots reserved past the buffer end only ever held sentinel padding (a real
  // record there sets log_overflow): clamp to the capacity
  // (slot indices < n_slots < 2^32: 32-bit index arithmetic)
  const uint32_t nr = (uint32_t)min(p.ctr->stage_count, (unsigned long long)p.n_slots);
  const uint32_t step = gridDim.x * F_THREADS * F_ITEMS;
  uint32_t kept_w = 0;  // kept write records (profile: detect's value gathers and commits)
  __syncthreads();
  for (uint32_t b0 = blockIdx.x * F_THREADS * F_ITEMS; b0 < nr; b0 = nr - b0 > step ? b0 + step : nr) {
    // F_ITEMS consecutive slots per thread (the block's slots in order), so
    // the kept records keep the staging order and a thread's records are
    // mostly consecutive cells: its digit counts go in runs
    uint64_t rec[F_ITEMS];
    bool keep[F_ITEMS];
    const uint32_t i0 = b0 + (uint32_t)t * F_ITEMS;
    if (i0 + F_ITEMS <= nr) {
#pragma unroll
      for (int j = 0; j < F_ITEMS; j += 2) {
        const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(p.stage + i0 + j));
        rec[j] = v.x;
        rec[j + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < F_ITEMS; j++) rec[j] = i0 + j < nr ? __ldg(p.stage + i0 + j) : REC_SENTINEL;
    }
#pragma unroll
    for (int j = 0; j < F_ITEMS; j++) {
      keep[j] = rec[j] != REC_SENTINEL &&
                (p.keep_all || (rec[j] & 1) || __ldg(p.wmap + (rec[j] >> REC_CELL_SHIFT)) == p.wtag);
    }
    uint32_t mine = 0;
#pragma unroll
    for (int j = 0; j < F_ITEMS; j++) {
      mine += keep[j];
      kept_w += keep[j] && (rec[j] & 1);
    }
    // digit histograms of the kept records: one shared add per run of equal digits
    if (mine) {
      for (int ps = 0; ps < p.passes; ps++) {
        const int sh = REC_CELL_SHIFT + 8 * ps;
        uint32_t cur = 0xFFFFFFFFu, run = 0;
#pragma unroll
        for (int j = 0; j < F_ITEMS; j++) {
          if (!keep[j]) continue;
          const uint32_t d = (uint32_t)(rec[j] >> sh) & 0xFF;
          if (d == cur) {
            run++;
          } else {
            if (run) atomicAdd(&bh[ps * 256 + cur], run);
            cur = d;
            run = 1;
          }
        }
        atomicAdd(&bh[ps * 256 + cur], run);
      }
    }
    // block-exclusive offsets of this thread's kept records
    uint32_t x = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wcnt[w] = x;
    __syncthreads();
    uint32_t woff = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < F_THREADS / 32; i++) {
      const uint32_t c = wcnt[i];
      woff += i < w ? c : 0u;
      tot += c;
    }
    if (t == 0) sbase = tot ? atomicAdd(&p.ctr->kept_count, (unsigned long long)tot) : 0ull;
    // block-local compaction in shared memory, then coalesced stores, F_ITEMS-
    // way interleaved: output F_ITEMS*m + r <- kept record r*Q + m (Q = tot /
    // F_ITEMS), so records F_THREADS slots apart — in lane-ordered staging,
    // cells a multiple of 256 apart: the same low digit — sit next to each
    // other, which the onesweep ranking's warp matching merges.  Any order is
    // correct (a stable sort by cell; detect reduces each cell's segment
    // order-independently).  Group r lives at r*(Q+8) in sbuf: the 8-word skew
    // keeps a warp's interleaved reads at two wavefronts.
    const uint32_t Q = tot / F_ITEMS, QF = Q * F_ITEMS;
    uint32_t pos = woff + x - mine;
#pragma unroll
    for (int j = 0; j < F_ITEMS; j++)
      if (keep[j]) {
        uint32_t r = 0;
#pragma unroll
        for (int g = 1; g <= F_ITEMS; g++) r += pos >= (uint32_t)g * Q;
        sbuf[pos + 8 * r] = rec[j];
        pos++;
      }
    __syncthreads();
    const unsigned long long base = sbase;
    for (uint32_t i = t; i < tot; i += F_THREADS)
      p.out[base + i] = sbuf[i < QF ? (i % F_ITEMS) * (Q + 8) + i / F_ITEMS : i + 8 * F_ITEMS];
    __syncthreads();  // wcnt / sbase / sbuf reuse
  }
  for (int i = t; i < p.passes * 256; i += F_THREADS)
    if (bh[i]) atomicAdd(&p.hist[i], bh[i]);
  for (int o = 16; o > 0; o >>= 1) kept_w += __shfl_xor_sync(FULL, kept_w, o);
  if (lane == 0 && kept_w) atomicAdd(&p.ctr->kept_writes, (unsigned long long)kept_w);
}

cudaError_t launch_filter(const FilterParams& p, cudaStream_t s) {
  if (p.n_slots == 0) return cudaSuccess;
  static DeviceSetup setup;
  static int nsm_of[RC_MAX_DEVICES];
  int dev = 0;
  cudaError_t se = setup.run(
      [](int d) -> cudaError_t { return cudaDeviceGetAttribute(&nsm_of[d], cudaDevAttrMultiProcessorCount, d); },
      &dev);
  if (se != cudaSuccess) return se;
  const int nsm = nsm_of[dev];
  const uint64_t per_block = (uint64_t)F_THREADS * F_ITEMS;
  const uint32_t grid = (uint32_t)std::min<uint64_t>((p.n_slots + per_block - 1) / per_block, (uint64_t)nsm * 8);
  filter_kernel<<<grid, F_THREADS, 0, s>>>(p);
  launched();
  return cudaGetLastError();
}

}  // namespace rc
