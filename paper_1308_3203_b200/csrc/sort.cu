// sort.cu — K2/K3: onesweep LSD radix sort of the access log by cell.
//
// Groups the interval's access records by cell so that
// the race rule can be applied per cell.  A record is one
// u64 (rc_internal.h make_rec) whose high 32 bits are the batch-local cell id;
// only the live cell bits are sorted (8-bit digits).  The sort is stable, and
// the detector only uses order-independent reductions inside a cell.
//
// Onesweep (Adinets & Merrill): the digit histograms of every pass come
// first (fused into the write-set filter; hist_kernel otherwise), then each
// pass (K3) is a single persistent kernel, 2 blocks per SM:
//   * each block scans the pass's digit counts (global digit starts),
//   * a block claims tile t from an atomic counter (in-order claiming gives
//     forward progress to the look-back) only after its previous tile's
//     look-back; the tile (4096 records, 32 KB) arrives by a TMA bulk copy
//     (cp.async.bulk + mbarrier) while the previous tile is written out,
//   * digit peers per warp round through shared-memory lane masks (atomicOr,
//     three rotating mask sets), stable in-tile ranking from per-warp digit
//     counters,
//   * per digit: publish the tile's count (AGGREGATE), look back over
//     predecessors (4 per L2 round trip) until an INCLUSIVE prefix is found,
//     publish INCLUSIVE,
//   * scatter to shared memory in digit order and write out coalesced runs.
// Status words carry an epoch so the look-back array is re-zeroed only when
// the epoch wraps (32-bit words for sorts of < 2^26 records, else 64-bit).
#include <cstdlib>

#include "rc_internal.h"

#ifndef SORT_LB
#define SORT_LB 4
#endif
#ifndef SORT_W32  // 1: 32-bit look-back status words for sorts of < 2^26 records
#define SORT_W32 1
#endif
#ifndef SORT_MINB  // resident blocks per SM of the persistent pass (smem: ~72 KB each)
#define SORT_MINB 2
#endif

namespace rc {

namespace {
constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr int RADIX = 256;
constexpr int WARPS = SORT_THREADS / 32;
constexpr int WARP_ITEMS = SORT_ITEMS * 32;
constexpr uint32_t FLAG_AGG = 1, FLAG_INC = 2;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// Decoupled look-back status word: flag (AGGREGATE / INCLUSIVE), epoch (so
// the array is never re-zeroed between passes), value.
//   64-bit: flag 2 | epoch 22 | value 40
//   32-bit: flag 2 | epoch 4  | value 26   (sorts of < 2^26 records: half the
//           look-back bytes per predecessor)
template <typename W>
struct LB;
template <>
struct LB<unsigned long long> {
  __device__ static unsigned long long make(uint32_t flag, uint32_t ep, unsigned long long v) {
    return ((unsigned long long)flag << 62) | ((unsigned long long)(ep & 0x3FFFFF) << 40) | v;
  }
  __device__ static bool ready(unsigned long long w, uint32_t ep) {
    return ((w >> 40) & 0x3FFFFF) == (ep & 0x3FFFFF) && (w >> 62) != 0;
  }
  __device__ static bool inclusive(unsigned long long w) { return (w >> 62) == 2; }
  __device__ static unsigned long long value(unsigned long long w) { return w & ((1ull << 40) - 1); }
};
template <>
struct LB<unsigned> {
  __device__ static unsigned make(uint32_t flag, uint32_t ep, unsigned long long v) {
    return (flag << 30) | ((ep & 0xF) << 26) | (unsigned)v;
  }
  __device__ static bool ready(unsigned w, uint32_t ep) { return ((w >> 26) & 0xF) == (ep & 0xF) && (w >> 30) != 0; }
  __device__ static bool inclusive(unsigned w) { return (w >> 30) == 2; }
  __device__ static unsigned long long value(unsigned w) { return w & ((1u << 26) - 1); }
};
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// exclusive scan of one value per thread over a 256-thread block
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* warp_tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  uint32_t off = 0;
  for (int i = 0; i < w; i++) off += warp_tot[i];
  __syncthreads();
  return off + x - v;
}
}  // namespace

#ifdef SORT_PHASE_TIMING
__device__ unsigned long long g_phase_cycles[12];
void sort_phase_io(unsigned long long* out, bool reset) {
  if (reset) {
    unsigned long long z[12] = {0};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof z);
  } else {
    cudaMemcpyFromSymbol(out, g_phase_cycles, 12 * sizeof(unsigned long long));
  }
}
#define PHASE_T(i)                                       \
  do {                                                   \
    if (t == 0) {                                        \
      const long long now_ = clock64();                  \
      atomicAdd(&g_phase_cycles[i], now_ - tprev_);      \
      tprev_ = now_;                                     \
    }                                                    \
  } while (0)
#else
#define PHASE_T(i) do {} while (0)
#endif

// ---- K2: all digit histograms in one read (fallback; K1 fuses it) ----------
__device__ __forceinline__ uint32_t dev_count(uint32_t n_host, const unsigned long long* n_a,
                                              const unsigned long long* n_b) {
  if (!n_a) return n_host;
  // the device count may exceed the buffer when the interval overflowed (K1
  // reserves sort-buffer room with atomics; the interval is then re-run and
  // this sort's output unused): never walk past the buffer / look-back words
  return (uint32_t)umin64(*n_a + (n_b ? *n_b : 0ull), n_host);
}

__global__ void __launch_bounds__(256) hist_kernel(const uint64_t* __restrict__ recs, uint32_t n_host,
                                                   const unsigned long long* n_a, const unsigned long long* n_b,
                                                   int passes, uint32_t* __restrict__ hist) {
  const uint32_t n = dev_count(n_host, n_a, n_b);
  __shared__ uint32_t h[4][RADIX];
  for (int i = threadIdx.x; i < 4 * RADIX; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  const uint32_t chunk = 16;  // consecutive records per thread; count runs of equal digits
  for (uint64_t b = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * chunk; b < n;
       b += (uint64_t)gridDim.x * blockDim.x * chunk) {
    uint32_t k[16];
    const uint32_t m = (uint32_t)umin64(chunk, n - b);
#pragma unroll
    for (int j = 0; j < 16; j++) k[j] = j < (int)m ? (uint32_t)(__ldg(recs + b + j) >> REC_CELL_SHIFT) : 0u;
    for (int p = 0; p < passes; p++) {
      const int sh = 8 * p;
      uint32_t cur = (k[0] >> sh) & 0xFF, run = 1;
#pragma unroll
      for (int j = 1; j < 16; j++) {
        if (j < (int)m) {
          const uint32_t d = (k[j] >> sh) & 0xFF;
          if (d == cur) run++;
          else { atomicAdd(&h[p][cur], run); cur = d; run = 1; }
        }
      }
      atomicAdd(&h[p][cur], run);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * RADIX; i += blockDim.x) {
    const uint32_t v = (&h[0][0])[i];
    if (v) atomicAdd(&hist[i], v);
  }
}


// ---- K3: one onesweep digit pass -------------------------------------------
// Persistent: a resident grid of blocks claims tiles in order from an atomic
// counter (claiming one tile ahead to hide the atomic); each block keeps two
// tile buffers and prefetches (TMA) the next claimed tile while it processes
// the current one.
struct SortSmem {
  uint64_t buf[2][SORT_TILE];
  uint32_t whist[WARPS][RADIX];  // per-warp digit counters (ranking; <= 512 per warp)
  uint32_t wmask[3][WARPS][RADIX];  // per-warp digit lane masks (zero between uses)
  uint32_t thist[2][RADIX];      // early tile counts (two copies: fewer atomic conflicts)
  uint32_t glob_base[RADIX];
  uint32_t bin_base[RADIX];      // global exclusive start of each digit (this pass)
  uint32_t wt[WARPS];
  uint32_t tile[2];
  unsigned long long mbar[2];
};

__device__ __forceinline__ void tile_fetch(uint64_t* dst, unsigned long long* mbar, const uint64_t* src,
                                           uint32_t cnt) {
  // one elected thread: bulk copy of the 16-byte-aligned part (cnt & ~1 records)
  const uint32_t c2 = cnt & ~1u;
  const uint32_t bar = smem_u32(mbar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(c2 * 8) : "memory");
  if (c2)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(c2 * 8), "r"(bar)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* mbar, uint32_t phase) {
  const uint32_t bar = smem_u32(mbar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(phase)
        : "memory");
  }
}

// Persistent: a resident grid, two tile buffers per block, the next tile
// prefetched (TMA) while the current one is processed.
template <typename SWORD>
__global__ void __launch_bounds__(SORT_THREADS, SORT_MINB) onesweep_kernel(const uint64_t* __restrict__ in,
                                                                   uint64_t* __restrict__ out, uint32_t n_host,
                                                                   const unsigned long long* n_a,
                                                                   const unsigned long long* n_b, int shift,
                                                                   const uint32_t* __restrict__ hist,
                                                                   SWORD* __restrict__ status,
                                                                   uint32_t* __restrict__ tile_ctr, uint32_t epoch) {
  using L = LB<SWORD>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  SortSmem& S = *reinterpret_cast<SortSmem*>(smem_raw);
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const uint32_t n = dev_count(n_host, n_a, n_b);
  const uint32_t n_tiles = (uint32_t)((n + SORT_TILE - 1) / SORT_TILE);
  const int dsh = REC_CELL_SHIFT + shift;

  for (int i = t; i < 3 * WARPS * RADIX; i += SORT_THREADS) (&S.wmask[0][0][0])[i] = 0u;
  if (t == 0) {
    for (int b = 0; b < 2; b++)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&S.mbar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t t0 = atomicAdd(tile_ctr, 1u);
    S.tile[0] = t0;
    if (t0 < n_tiles) {
      tile_fetch(S.buf[0], &S.mbar[0], in + (uint64_t)t0 * SORT_TILE,
                 (uint32_t)umin64(SORT_TILE, n - (uint64_t)t0 * SORT_TILE));
    }
  }
  {  // global start of every digit of this pass: exclusive scan of its counts
    const uint32_t e = block_excl_scan(t < RADIX ? hist[t] : 0u, S.wt);  // (synchronises the block)
    if (t < RADIX) S.bin_base[t] = e;
  }
  __syncthreads();
  uint32_t phase = 0;  // bit b = expected parity of buffer b's mbarrier
  int cur = 0;
#ifdef SORT_PHASE_TIMING
  long long tprev_ = clock64();
#endif
  for (;;) {
    const uint32_t tile = S.tile[cur];
    if (tile >= n_tiles) break;  // block-uniform
    for (int i = t; i < WARPS * RADIX; i += SORT_THREADS) (&S.whist[0][0])[i] = 0;
    if (t < RADIX) {
      S.thist[0][t] = 0;
      S.thist[1][t] = 0;
    }
    const uint64_t base = (uint64_t)tile * SORT_TILE;
    const uint32_t cnt = (uint32_t)umin64(SORT_TILE, n - base);
    uint64_t* B = S.buf[cur];
    PHASE_T(0);
    mbar_wait(&S.mbar[cur], (phase >> cur) & 1u);
    phase ^= 1u << cur;
    if ((cnt & 1u) && t == 0) B[cnt - 1] = in[base + cnt - 1];  // odd tail of the last tile
    __syncthreads();
    PHASE_T(1);

    // ---- records to registers; digit groups of all items up front (the 16
    //      MATCH.ANY are independent, so their latencies overlap)
    uint64_t k[SORT_ITEMS];
    uint32_t pm[SORT_ITEMS];  // peer mask, later the rank within the warp
#pragma unroll
    for (int j = 0; j < SORT_ITEMS; j++) {
      const uint32_t idx = w * WARP_ITEMS + j * 32 + lane;
      k[j] = idx < cnt ? B[idx] : ~0ull;  // invalid items: digit 0x100 below
    }
#define DIGIT(j) ((w * WARP_ITEMS + (j) * 32 + lane) < cnt ? (uint32_t)(k[j] >> dsh) & 0xFF : 0x100u)
    PHASE_T(2);
    {
      const unsigned vm = cnt >= (uint32_t)(w * WARP_ITEMS + WARP_ITEMS) ? FULL : 0u;
#pragma unroll
      for (int j = 0; j < SORT_ITEMS; j++) {
        const uint32_t dd = DIGIT(j);
        // peers through shared-memory lane masks: three mask sets rotate so
        // one __syncwarp per round suffices (set j%3 is cleared in round j+1,
        // after that round's __syncwarp, and reused in round j+3)
        (void)vm;
        if (dd < RADIX) atomicOr(&S.wmask[j % 3][w][dd], 1u << lane);
        __syncwarp();
        const unsigned m = dd < RADIX ? S.wmask[j % 3][w][dd] : 0u;
        if (j > 0) {
          const uint32_t dp = DIGIT(j - 1);
          if (dp < RADIX && lane == __ffs(pm[j - 1]) - 1) S.wmask[(j - 1) % 3][w][dp] = 0u;
        }
        pm[j] = m;
      }
    }
    __syncwarp();
    {
      const uint32_t dp = DIGIT(SORT_ITEMS - 1);
      if (dp < RADIX && lane == __ffs(pm[SORT_ITEMS - 1]) - 1) S.wmask[(SORT_ITEMS - 1) % 3][w][dp] = 0u;
    }
    PHASE_T(3);
    // early tile counts: one shared atomic per digit group, then publish AGGREGATE
#pragma unroll
    for (int j = 0; j < SORT_ITEMS; j++) {
      const uint32_t dd = DIGIT(j);
      if (dd < RADIX && lane == __ffs(pm[j]) - 1) atomicAdd(&S.thist[w & 1][dd], (uint32_t)__popc(pm[j]));
    }
    __syncthreads();
    // per-digit steps: thread d < RADIX owns digit d
    const int d = t < RADIX ? t : RADIX - 1;
    const bool dig = t < RADIX;
    const uint32_t tile_cnt = dig ? S.thist[0][d] + S.thist[1][d] : 0u;
    SWORD* my_status = status + (size_t)tile * RADIX + d;
    if (dig) st_relaxed(my_status, L::make(tile == 0 ? FLAG_INC : FLAG_AGG, epoch, tile_cnt));
    const uint32_t excl_tile = block_excl_scan(tile_cnt, S.wt);  // tile-local start of digit d
    PHASE_T(4);

    // ---- stable in-tile ranking (warp w owns items [w*512, w*512+512), striped)
#pragma unroll
    for (int j = 0; j < SORT_ITEMS; j++) {
      const uint32_t dd = DIGIT(j);
      const bool valid = dd < RADIX;
      uint32_t prev = 0;
      if (valid) prev = S.whist[w][dd];
      __syncwarp();
      if (valid && lane == __ffs(pm[j]) - 1) S.whist[w][dd] = (prev + __popc(pm[j]));
      __syncwarp();
      pm[j] = prev + __popc(pm[j] & lanemask_lt());
    }
    __syncthreads();
    if (dig) {  // per digit: tile-local start of each warp's items of digit d
      uint32_t run = excl_tile;
#pragma unroll
      for (int ww = 0; ww < WARPS; ww++) {
        const uint32_t c = S.whist[ww][d];
        S.whist[ww][d] = run;
        run += c;
      }
    }
    __syncthreads();
    PHASE_T(5);

    // ---- scatter into shared memory in digit order (stable), in place
#pragma unroll
    for (int j = 0; j < SORT_ITEMS; j++) {
      const uint32_t dd = DIGIT(j);
      if (dd < RADIX) B[S.whist[w][dd] + pm[j]] = k[j];
    }
#undef DIGIT
    PHASE_T(6);

    // ---- look-back (after the scatter: predecessors had time to publish
    //      INCLUSIVE), then publish our INCLUSIVE prefix
    unsigned long long excl = 0;
    if (tile > 0 && dig) {
      constexpr int LBN = SORT_LB;  // predecessors per L2 round trip
      int64_t tp = (int64_t)tile - 1;
      bool done = false;
#ifdef SORT_PHASE_TIMING
      uint32_t st_rounds = 0, st_notready = 0, st_walk = 0;
#endif
      while (!done) {
#ifdef SORT_PHASE_TIMING
        st_rounds++;
#endif
        SWORD sw[LBN];
#pragma unroll
        for (int j = 0; j < LBN; j++) sw[j] = tp - j >= 0 ? ld_relaxed(status + (size_t)(tp - j) * RADIX + d) : (SWORD)0;
#pragma unroll
        for (int j = 0; j < LBN; j++) {
          if (done) break;
          const bool ready = L::ready(sw[j], epoch);
          if (!ready) {  // re-poll from this predecessor
#ifdef SORT_PHASE_TIMING
            st_notready++;
#endif
            break;
          }
          excl += L::value(sw[j]);
          tp--;
          if (L::inclusive(sw[j])) done = true;
        }
      }
      st_relaxed(my_status, L::make(FLAG_INC, epoch, excl + tile_cnt));
#ifdef SORT_PHASE_TIMING
      st_walk = (uint32_t)((int64_t)tile - 1 - tp);
      {
        uint32_t a = st_rounds, b = st_notready, c = st_walk;
        for (int o = 16; o; o >>= 1) {
          a += __shfl_xor_sync(FULL, a, o); b += __shfl_xor_sync(FULL, b, o); c += __shfl_xor_sync(FULL, c, o);
        }
        if (lane == 0) { atomicAdd(&g_phase_cycles[9], a); atomicAdd(&g_phase_cycles[10], b); atomicAdd(&g_phase_cycles[11], c); }
      }
#endif
    }
    if (dig) S.glob_base[d] = (uint32_t)(S.bin_base[d] + excl) - excl_tile;
    // claim the next tile only now (its AGGREGATE follows within a few
    // thousand cycles, so successors' look-backs never wait on a tile claimed
    // long before it is processed); its TMA load overlaps the write-out
    if (t == 0) {
      const uint32_t tn = atomicAdd(tile_ctr, 1u);
      S.tile[cur ^ 1] = tn;
      if (tn < n_tiles)
        tile_fetch(S.buf[cur ^ 1], &S.mbar[cur ^ 1], in + (uint64_t)tn * SORT_TILE,
                   (uint32_t)umin64(SORT_TILE, n - (uint64_t)tn * SORT_TILE));
    }
    __syncthreads();
    PHASE_T(7);

    // ---- coalesced write-out: sorted position i goes to glob_base[digit] + i
    if (cnt == SORT_TILE) {
#pragma unroll
      for (int j = 0; j < SORT_ITEMS; j++) k[j] = B[t + j * SORT_THREADS];
#pragma unroll
      for (int j = 0; j < SORT_ITEMS; j++)
        out[S.glob_base[(uint32_t)(k[j] >> dsh) & 0xFF] + t + j * SORT_THREADS] = k[j];
    } else {
      for (uint32_t i = t; i < cnt; i += SORT_THREADS) {
        const uint64_t kk = B[i];
        out[S.glob_base[(uint32_t)(kk >> dsh) & 0xFF] + i] = kk;
      }
    }
    __syncthreads();  // buffer `cur`, whist, glob_base free for reuse
    PHASE_T(8);
    cur ^= 1;
  }
}

size_t sort_tiles(size_t n) { return (n + SORT_TILE - 1) / SORT_TILE; }

cudaError_t onesweep_sort(uint64_t* recs, uint32_t n, const unsigned long long* n_a, const unsigned long long* n_b,
                          int bits, SortWorkspace& ws, cudaStream_t s, bool* in_alt, Profiler* prof,
                          bool hist_ready) {
  *in_alt = false;  // n: upper bound of the record count (exact when n_a == NULL)
  if (n == 0 || bits <= 0) return cudaSuccess;
  const int passes = (bits + 7) / 8;
  static DeviceSetup setup;
  static int nsm_of[RC_MAX_DEVICES], per_sm_of[RC_MAX_DEVICES];
  int dev = 0;
  cudaError_t se = setup.run(
      [](int d) -> cudaError_t {
        const void* ks[2] = {(const void*)onesweep_kernel<unsigned long long>, (const void*)onesweep_kernel<unsigned>};
        for (int i = 0; i < 2; i++) {
          cudaError_t e = cudaFuncSetAttribute(ks[i], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SortSmem));
          if (e != cudaSuccess) return e;
          cudaFuncSetAttribute(ks[i], cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        }
        int per_sm = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, onesweep_kernel<unsigned long long>, SORT_THREADS, sizeof(SortSmem));
        if (e != cudaSuccess) return e;
        per_sm_of[d] = per_sm < 1 ? 1 : per_sm;
        return cudaDeviceGetAttribute(&nsm_of[d], cudaDevAttrMultiProcessorCount, d);
      },
      &dev);
  if (se != cudaSuccess) return se;
  const int nsm = nsm_of[dev], per_sm = per_sm_of[dev];
  if (ws.reset_tile_ctr) cudaMemsetAsync(ws.tile_ctr, 0, 4 * sizeof(uint32_t), s);
  if (!hist_ready) {  // (each pass scans its digit counts itself)
    if (prof) prof->begin(s);
    cudaMemsetAsync(ws.hist, 0, 4 * RADIX * sizeof(uint32_t), s);
    const uint32_t hist_grid = (uint32_t)umin64((uint64_t)nsm * 8, (n + 256 * 16 - 1) / (256 * 16));
    hist_kernel<<<hist_grid, 256, 0, s>>>(recs, n, n_a, n_b, passes, ws.hist);
    launched();
    if (prof) prof->end(RC_PROF_HIST, s, (uint64_t)n * 8, n);
  }
  const uint32_t tiles = (uint32_t)sort_tiles(n);
  // persistent: never more blocks than can be resident (look-back progress)
  const uint32_t grid = (uint32_t)umin64(tiles, (uint64_t)per_sm * nsm);
  uint64_t* kin = recs;
  uint64_t* kout = ws.alt;
  // 32-bit look-back words when every prefix fits 26 bits
  // (test hook RC_DEBUG_SORT_W64 forces the 64-bit words; results never differ)
  const int fmt = (SORT_W32 && n < (1u << 26) && !getenv("RC_DEBUG_SORT_W64")) ? 1 : 0;
  const uint32_t epochs = fmt ? 16u : (1u << 22);
  for (int p = 0; p < passes; p++) {
    if (fmt != ws.status_fmt || ++ws.epoch >= epochs) {  // format switch or epoch wrap: clear the words once
      cudaMemsetAsync(ws.status, 0, ws.status_tiles * RADIX * sizeof(unsigned long long), s);
      ws.epoch = 1;
      ws.status_fmt = fmt;
    }
    if (prof) prof->begin(s);
    const dim3 g(grid), b(SORT_THREADS);
    const uint32_t* h = ws.hist + p * RADIX;
    uint32_t* tc = ws.tile_ctr + p;
    unsigned* st32 = reinterpret_cast<unsigned*>(ws.status);
    if (fmt)
      onesweep_kernel<unsigned><<<g, b, sizeof(SortSmem), s>>>(kin, kout, n, n_a, n_b, 8 * p, h, st32, tc, ws.epoch);
    else
      onesweep_kernel<unsigned long long><<<g, b, sizeof(SortSmem), s>>>(kin, kout, n, n_a, n_b, 8 * p, h, ws.status, tc, ws.epoch);
    launched();
    if (prof) prof->end(RC_PROF_SORT, s, (uint64_t)n * 16, n);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    std::swap(kin, kout);
  }
  *in_alt = (passes & 1) != 0;
  return cudaGetLastError();
}

// ---- K2 on the bucket path: bucket counts of the kept records + starts ------
// The staging buffer is read as by the scatter (same slots, same write-set
// filter rule); a warp's rounds of one bucket are summed in registers and
// flushed when the bucket changes (records come in lane order: long runs),
// other rounds add per group of equal buckets (__match_any_sync).  The last
// block to finish turns the counts into the buckets' exclusive starts
// (bstart) and the scatter's cursors (bcur).
constexpr int BC_THREADS = 512;
#ifndef BC_ROUNDS_OPT
#define BC_ROUNDS_OPT 4
#endif
constexpr int BC_ROUNDS = BC_ROUNDS_OPT;  // 16-byte loads per lane and chunk
constexpr int BC_ITEMS = 2 * BC_ROUNDS;
#ifndef BC_MINB
#define BC_MINB 1
#endif
// A warp's chunk of 64 * ROUNDS staging slots: 16-byte loads, lane L of round
// j takes slots c0 + 64 j + 2 L, + 1 into items 2 j, 2 j + 1 (slots >= n:
// REC_SENTINEL).  Any order of a chunk's records inside a bucket is fine.
template <int ROUNDS>
__device__ __forceinline__ void load_chunk2(const uint64_t* __restrict__ stage, uint32_t c0, uint32_t n, int lane,
                                            uint64_t (&r)[2 * ROUNDS]) {
#pragma unroll
  for (int j = 0; j < ROUNDS; j++) {
    const uint32_t i = c0 + 64 * j + 2 * lane;
    if (i + 1 < n) {
      const ulonglong2 v = __ldcs(reinterpret_cast<const ulonglong2*>(stage + i));
      r[2 * j] = v.x;
      r[2 * j + 1] = v.y;
    } else {
      r[2 * j] = i < n ? __ldcs(stage + i) : REC_SENTINEL;
      r[2 * j + 1] = REC_SENTINEL;
    }
  }
}

// the write-set filter over a warp's chunk (records -> REC_SENTINEL when
// dropped): the map is looked up only when the chunk holds read records
// (none at all when K1 elided every read statically)
template <int ROUNDS>
__device__ __forceinline__ void filter_chunk(const ScatterParams& p, uint64_t (&r)[ROUNDS]) {
  bool rd = false;
#pragma unroll
  for (int j = 0; j < ROUNDS; j++) rd |= r[j] != REC_SENTINEL && !(r[j] & 1);
  if (p.keep_all || !__any_sync(FULL, rd)) return;
#pragma unroll
  for (int j = 0; j < ROUNDS; j++)
    if (r[j] != REC_SENTINEL && !(r[j] & 1) && __ldg(p.wmap + (uint32_t)(r[j] >> REC_CELL_SHIFT)) != p.wtag)
      r[j] = REC_SENTINEL;
}
__global__ void __launch_bounds__(BC_THREADS, BC_MINB) bucket_count_kernel(const ScatterParams p, uint32_t* __restrict__ hist,
                                                                   uint32_t nb, uint32_t* __restrict__ bstart) {
  DevCounters* ctr = p.ctr;
  if (ctr->abort || ctr->log_overflow || ctr->ovl_overflow) return;  // grid-uniform
  const uint32_t n = (uint32_t)umin64(ctr->stage_count, p.n_slots);
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const uint32_t warps = gridDim.x * (BC_THREADS / 32);
  uint32_t run_b = 0xFFFFFFFFu, run_n = 0;  // (warp-uniform) the open run of one-bucket rounds
  for (uint32_t c = blockIdx.x * (BC_THREADS / 32) + w; (uint64_t)c * (64 * BC_ROUNDS) < n; c += warps) {
    uint64_t r[BC_ITEMS];
    load_chunk2<BC_ROUNDS>(p.stage, c * (64 * BC_ROUNDS), n, lane, r);
    filter_chunk<BC_ITEMS>(p, r);
    // the common case first: every kept record of the chunk in one bucket
    uint32_t bmin = 0xFFFFFFFFu, bmax = 0, nk = 0;
#pragma unroll
    for (int j = 0; j < BC_ITEMS; j++) {
      const bool ok = r[j] != REC_SENTINEL;
      const uint32_t b = (uint32_t)(r[j] >> (REC_CELL_SHIFT + BUCKET_BITS));
      bmin = min(bmin, ok ? b : 0xFFFFFFFFu);
      bmax = max(bmax, ok ? b : 0u);
      nk += ok;
    }
    bmin = __reduce_min_sync(FULL, bmin);
    bmax = __reduce_max_sync(FULL, bmax);
    if (bmin == bmax) {
      const uint32_t k = __reduce_add_sync(FULL, nk);
      if (bmin != run_b) {
        if (lane == 0 && run_n) atomicAdd(hist + run_b, run_n);
        run_b = bmin;
        run_n = 0;
      }
      run_n += k;
      continue;
    }
    if (bmin > bmax) continue;  // nothing kept
#pragma unroll
    for (int j = 0; j < BC_ITEMS; j++) {
      const bool keep = r[j] != REC_SENTINEL;
      const uint32_t b = keep ? (uint32_t)(r[j] >> (REC_CELL_SHIFT + BUCKET_BITS)) : 0xFFFFFFFFu;
      const unsigned km = __ballot_sync(FULL, keep);
      if (!km) continue;
      const uint32_t b0 = __shfl_sync(FULL, b, __ffs(km) - 1);
      if (__all_sync(FULL, !keep || b == b0)) {
        if (b0 != run_b) {
          if (lane == 0 && run_n) atomicAdd(hist + run_b, run_n);
          run_b = b0;
          run_n = 0;
        }
        run_n += __popc(km);
      } else {
        const unsigned peers = __match_any_sync(FULL, b);
        if (keep && (peers & lanemask_lt()) == 0) atomicAdd(hist + b, (uint32_t)__popc(peers));
      }
    }
  }
  if (lane == 0 && run_n) atomicAdd(hist + run_b, run_n);
  // the last block: exclusive scan of the counts (nb <= NB_MAX)
  __shared__ uint32_t wsum[BC_THREADS / 32];
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (t == 0) last = atomicAdd(&ctr->count_done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  constexpr int PER = NB_MAX / BC_THREADS;
  uint32_t sum = 0;  // (the counts are re-read below, not held in registers: PER is large)
#pragma unroll 8
  for (int k = 0; k < PER; k++) {
    const uint32_t b = (uint32_t)t * PER + k;
    sum += b < nb ? __ldcg(hist + b) : 0u;
  }
  uint32_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  uint32_t run = x - sum;
  for (int i = 0; i < w; i++) run += wsum[i];
#pragma unroll 8
  for (int k = 0; k < PER; k++) {
    const uint32_t b = (uint32_t)t * PER + k;
    if (b < nb) {
      bstart[b] = run;
      p.bcur[b] = run;
      run += __ldcg(hist + b);
    }
  }
}

cudaError_t launch_bucket_count(const ScatterParams& p, uint32_t* hist, uint32_t nb, uint32_t* bstart,
                                cudaStream_t s, Profiler* prof) {
  if (nb == 0 || nb > NB_MAX) return nb ? cudaErrorInvalidValue : cudaSuccess;
  static DeviceSetup setup;
  static int nsm_of[RC_MAX_DEVICES], per_sm_of[RC_MAX_DEVICES];
  int dev = 0;
  cudaError_t se = setup.run(
      [](int d) -> cudaError_t {
        int per_sm = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bucket_count_kernel, BC_THREADS, 0);
        if (e != cudaSuccess) return e;
        per_sm_of[d] = std::max(per_sm, 1);
        return cudaDeviceGetAttribute(&nsm_of[d], cudaDevAttrMultiProcessorCount, d);
      },
      &dev);
  if (se != cudaSuccess) return se;
  const uint64_t chunks = ((uint64_t)std::max<uint32_t>(p.n_slots, 1) + 64 * BC_ROUNDS - 1) / (64 * BC_ROUNDS);
  const uint32_t grid = (uint32_t)std::max<uint64_t>(
      1, std::min<uint64_t>((chunks + BC_THREADS / 32 - 1) / (BC_THREADS / 32), (uint64_t)nsm_of[dev] * per_sm_of[dev]));
  if (prof) prof->begin(s);
  bucket_count_kernel<<<grid, BC_THREADS, 0, s>>>(p, hist, nb, bstart);
  launched();
  if (prof) prof->end(RC_PROF_HIST, s, (uint64_t)p.n_slots * 8, p.n_slots);
  return cudaGetLastError();
}

// ---- K3 on the bucket path: one MSD scatter on the high cell bits ----------
// Fused with the write-set filter (filter.cu, the same rule): from the
// staging buffer every write record and every read of a cell written in this
// interval goes to out[bcur[bucket]++], bucket = cell >> BUCKET_BITS (bucket_count
// counted the kept records per bucket and set bcur to the buckets' starts).
// Sentinels and the other reads are dropped: a read of a cell no work-item
// wrote can take part in no report and no commit.  The
// order inside a bucket is arbitrary (bucket_detect sorts each bucket by its
// low bits; the detection only uses order-independent reductions inside a
// cell).  A warp takes 64 * BS_ROUNDS consecutive slots (16-byte loads, all in
// flight), groups each round's kept lanes by bucket (one vote when the round
// is one bucket — the common case, K1 stages in lane order — else
// __match_any_sync), and the group leader reserves the group's slots with one
// atomic; the atomics of all rounds are issued before any result is used.
#ifndef BS_ROUNDS_OPT
#define BS_ROUNDS_OPT 4
#endif
constexpr int BS_ROUNDS = BS_ROUNDS_OPT;  // 16-byte loads per lane and chunk
constexpr int BS_ITEMS = 2 * BS_ROUNDS;
#ifndef BS_MINB
#define BS_MINB 4
#endif
constexpr int BS_THREADS = 256;
// store record r at position pos of bucket b (count mode: pos is absolute;
// region mode: pos is relative to the bucket's region, b * BUCKET_REGION)
template <bool REGION>
__device__ __forceinline__ void place(const ScatterParams& p, uint32_t b, uint32_t pos, uint64_t r) {
  if (!REGION) {
    __stcs(p.out + pos, r);
  } else if (pos < BUCKET_REGION) {
    __stcs(p.out + (b * BUCKET_REGION + pos), r);  // (< 2^26: 32-bit arithmetic)
  } else {
    p.ctr->bucket_overflow = 1;  // (idempotent; the host regroups the interval with the counts)
  }
}
template <bool REGION>
__global__ void __launch_bounds__(BS_THREADS, BS_MINB) bucket_scatter_kernel(const ScatterParams p) {
  const DevCounters* ctr = p.ctr;
  if (ctr->abort) return;  // speculative interval (DevCounters::abort)
  if (blockIdx.x == 0 && threadIdx.x == 0) p.ctr->k1_reports = p.ctr->report_count;  // K1 is complete here
  if (ctr->log_overflow || ctr->ovl_overflow) return;  // the interval will be re-run
  // slots reserved past the buffer end only ever held sentinel padding (a
  // real record there sets log_overflow): clamp to the capacity
  const uint32_t n = (uint32_t)umin64(ctr->stage_count, p.n_slots);
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (BS_THREADS / 32);
  const unsigned lt = lanemask_lt();
  uint32_t kept = 0, kept_w = 0;  // lane 0: the warp's kept records / write records
  for (uint32_t c = blockIdx.x * (BS_THREADS / 32) + (threadIdx.x >> 5); (uint64_t)c * (64 * BS_ROUNDS) < n;
       c += warps) {
    uint64_t r[BS_ITEMS];
    load_chunk2<BS_ROUNDS>(p.stage, c * (64 * BS_ROUNDS), n, lane, r);
    filter_chunk<BS_ITEMS>(p, r);  // the write-set filter
    uint32_t bmin = 0xFFFFFFFFu, bmax = 0, nk = 0;
#pragma unroll
    for (int j = 0; j < BS_ITEMS; j++) {
      const bool ok = r[j] != REC_SENTINEL;
      const uint32_t b = (uint32_t)(r[j] >> (REC_CELL_SHIFT + BUCKET_BITS));
      bmin = min(bmin, ok ? b : 0xFFFFFFFFu);
      bmax = max(bmax, ok ? b : 0u);
      nk += ok;
    }
    bmin = __reduce_min_sync(FULL, bmin);
    bmax = __reduce_max_sync(FULL, bmax);
    if (bmin > bmax) continue;  // nothing kept
    if (bmin == bmax) {  // the common case: one bucket, one reservation for the chunk
      uint32_t base = 0;
      const uint32_t k = __reduce_add_sync(FULL, nk);
      if (lane == 0) base = atomicAdd(p.bcur + bmin, k);
      base = __shfl_sync(FULL, base, 0);
#pragma unroll
      for (int j = 0; j < BS_ITEMS; j++) {
        const unsigned m = __ballot_sync(FULL, r[j] != REC_SENTINEL);
        if (r[j] != REC_SENTINEL) place<REGION>(p, bmin, base + __popc(m & lt), r[j]);
        base += __popc(m);
        kept_w += __popc(__ballot_sync(FULL, r[j] != REC_SENTINEL && (r[j] & 1)));
      }
      kept += k;
      continue;
    }
    uint32_t base[BS_ITEMS], rank[BS_ITEMS], lead[BS_ITEMS];
#pragma unroll
    for (int j = 0; j < BS_ITEMS; j++) {
      const uint32_t b = (uint32_t)(r[j] >> (REC_CELL_SHIFT + BUCKET_BITS));  // sentinel: 0xFFFFF (no bucket)
      const uint32_t b0 = __shfl_sync(FULL, b, 0);
      unsigned peers;
      if (__all_sync(FULL, b == b0)) peers = FULL;
      else peers = __match_any_sync(FULL, b);
      lead[j] = __ffs(peers) - 1;
      rank[j] = __popc(peers & lt);
      base[j] = 0;
      if (r[j] != REC_SENTINEL && rank[j] == 0) base[j] = atomicAdd(p.bcur + b, (uint32_t)__popc(peers));
      kept += __popc(__ballot_sync(FULL, r[j] != REC_SENTINEL));
      kept_w += __popc(__ballot_sync(FULL, r[j] != REC_SENTINEL && (r[j] & 1)));
    }
#pragma unroll
    for (int j = 0; j < BS_ITEMS; j++) {
      const uint32_t bb = __shfl_sync(FULL, base[j], lead[j]);
      if (r[j] != REC_SENTINEL) place<REGION>(p, (uint32_t)(r[j] >> (REC_CELL_SHIFT + BUCKET_BITS)), bb + rank[j], r[j]);
    }
  }
  if (lane == 0 && kept) {
    atomicAdd(&p.ctr->kept_count, (unsigned long long)kept);
    if (kept_w) atomicAdd(&p.ctr->kept_writes, (unsigned long long)kept_w);
  }
}

cudaError_t launch_bucket_scatter(const ScatterParams& p, cudaStream_t s, Profiler* prof) {
  if (p.n_slots == 0) return cudaSuccess;
  static DeviceSetup setup;
  static int nsm_of[RC_MAX_DEVICES], per_sm_of[RC_MAX_DEVICES];
  int dev = 0;
  cudaError_t se = setup.run(
      [](int d) -> cudaError_t {
        int per_sm = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bucket_scatter_kernel<true>, BS_THREADS, 0);
        if (e != cudaSuccess) return e;
        per_sm_of[d] = std::max(per_sm, 1);
        return cudaDeviceGetAttribute(&nsm_of[d], cudaDevAttrMultiProcessorCount, d);
      },
      &dev);
  if (se != cudaSuccess) return se;
  const uint64_t chunks = ((uint64_t)p.n_slots + 64 * BS_ROUNDS - 1) / (64 * BS_ROUNDS);
  const uint32_t grid = (uint32_t)std::max<uint64_t>(
      1, std::min<uint64_t>((chunks + BS_THREADS / 32 - 1) / (BS_THREADS / 32), (uint64_t)nsm_of[dev] * per_sm_of[dev]));
  if (prof) prof->begin(s);
  if (p.region) {
    if (p.region != BUCKET_REGION) return cudaErrorInvalidValue;
    bucket_scatter_kernel<true><<<grid, BS_THREADS, 0, s>>>(p);
  } else {
    bucket_scatter_kernel<false><<<grid, BS_THREADS, 0, s>>>(p);
  }
  launched();
  if (prof) prof->end(RC_PROF_SORT, s, (uint64_t)p.n_slots * 16, p.n_slots);
  return cudaGetLastError();
}

}  // namespace rc
