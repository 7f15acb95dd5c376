// sortbench.cu — dev tool: time the onesweep sort (sort.cu) in isolation on
// access-log-shaped keys, verify the result, and (with -DSORT_PHASE_TIMING)
// print the per-tile cycle split of the onesweep pass.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude \
//        -Ipaper_1308_3203_b200/csrc [-DSORT_PHASE_TIMING] \
//        tools/sortbench.cu paper_1308_3203_b200/csrc/sort.cu -o build/sortbench
//   build/sortbench [n_records] [bits] [pattern: stencil|random] [reps]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "rc_internal.h"

namespace rc {
std::atomic<uint64_t> g_launches{0};
size_t Profiler::next() { return 0; }
void Profiler::begin(cudaStream_t) {}
void Profiler::end(int, cudaStream_t, uint64_t, uint64_t) {}
void Profiler::collect(rc_profile*) {}
Profiler::~Profiler() {}
#ifdef SORT_PHASE_TIMING
void sort_phase_io(unsigned long long* out, bool reset);
#endif
}  // namespace rc

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

int main(int argc, char** argv) {
  const uint32_t n = argc > 1 ? (uint32_t)atoll(argv[1]) : 29360128u;
  const int bits = argc > 2 ? atoi(argv[2]) : 24;
  const std::string pat = argc > 3 ? argv[3] : "stencil";
  const int reps = argc > 4 ? atoi(argv[4]) : 10;
  std::vector<uint64_t> hk(n);
  // stencil-like log (config 5 even interval): per 32-lane warp: reads of
  // A[c-1], A[c], A[c+1] then the write of B[c]; instance-major
  const uint64_t mask = bits >= 32 ? 0xFFFFFFFFull : ((1ull << bits) - 1);
  uint64_t x = 88172645463325252ull;
  const uint32_t lanes = n / 4;
  const uint32_t half = (uint32_t)((mask + 1) / 2);
  for (uint32_t i = 0; i < n; i++) {
    uint32_t key;
    if (pat == "random") {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      key = (uint32_t)(x & mask);
    } else {
      const uint32_t w = i / 128, r = i % 128, kind = r / 32, l = r % 32;
      const uint32_t lane = w * 32 + l;
      const uint32_t c = lane + 1;
      key = kind < 3 ? (c - 1 + kind) % half : half + c % half;
      (void)lanes;
    }
    hk[i] = ((uint64_t)key << 32) | i;  // low word: source index (checks permutation / stability)
  }
  uint64_t *dk, *dk2;
  CK(cudaMalloc(&dk, n * 8ull)); CK(cudaMalloc(&dk2, n * 8ull));
  rc::SortWorkspace ws;
  CK(cudaMalloc(&ws.hist, 4096 * 4));
  ws.bin_off = ws.hist + 1024;
  ws.tile_ctr = ws.bin_off + 1024;
  ws.status_tiles = rc::sort_tiles(n) + 1;
  CK(cudaMalloc(&ws.status, ws.status_tiles * 256 * 8));
  CK(cudaMemset(ws.status, 0, ws.status_tiles * 256 * 8));
  ws.alt = dk2;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<float> times;
  bool in_alt = false;
  for (int it = 0; it < reps + 2; it++) {
    CK(cudaMemcpy(dk, hk.data(), n * 8ull, cudaMemcpyHostToDevice));
#ifdef SORT_PHASE_TIMING
    rc::sort_phase_io(nullptr, true);
#endif
    cudaEventRecord(e0);
    CK(rc::onesweep_sort(dk, n, nullptr, nullptr, bits, ws, 0, &in_alt, nullptr, false));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it >= 2) times.push_back(ms);
  }
  std::sort(times.begin(), times.end());
  const float med = times[times.size() / 2];
  const int passes = (bits + 7) / 8;
  printf("n=%u bits=%d pattern=%s passes=%d: median %.3f ms  -> %.1f GB/s sort-alg (16 B/rec/pass + 8 B hist)\n",
         n, bits, pat.c_str(), passes, med, (double)n * (16.0 * passes + 8) / (med * 1e-3) / 1e9);
#ifdef SORT_PHASE_TIMING
  unsigned long long ph[12];
  rc::sort_phase_io(ph, false);
  const double tiles = (double)rc::sort_tiles(n) * passes;
  const char* names[] = {"claim+prefetch", "tma wait", "load keys", "match", "count+publish", "rank", "scatter",
                         "lookback", "writeout", "", "", ""};
  double tot = 0;
  for (int i = 0; i < 9; i++) tot += ph[i];
  for (int i = 0; i < 9; i++)
    printf("  phase %-16s %9.0f cycles/tile (%.1f%%)\n", names[i], ph[i] / tiles, 100.0 * ph[i] / tot);
  printf("  look-back per digit-tile: %.2f rounds, %.2f not-ready polls, %.2f predecessors walked\n",
         ph[9] / (tiles * 256), ph[10] / (tiles * 256), ph[11] / (tiles * 256));
#endif
  // verify: sorted by cell bits, a permutation, stable (low word = source index)
  std::vector<uint64_t> ok(n);
  CK(cudaMemcpy(ok.data(), in_alt ? dk2 : dk, n * 8ull, cudaMemcpyDeviceToHost));
  bool good = true;
  std::vector<uint8_t> seen(n, 0);
  for (uint32_t i = 0; i < n && good; i++) {
    const uint64_t a = (ok[i] >> 32) & mask, pa = i ? (ok[i - 1] >> 32) & mask : 0;
    if (i && pa > a) { printf("NOT SORTED at %u\n", i); good = false; }
    const uint32_t src = (uint32_t)ok[i];
    if (src >= n || seen[src] || hk[src] != ok[i]) { printf("BAD PERMUTATION at %u\n", i); good = false; }
    else seen[src] = 1;
    if (i && pa == a && (uint32_t)ok[i - 1] > src) { printf("NOT STABLE at %u\n", i); good = false; }
  }
  printf("verify: %s\n", good ? "ok" : "FAILED");
  return good ? 0 : 1;
}
