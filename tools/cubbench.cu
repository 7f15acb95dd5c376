// cubbench.cu — dev tool: CUB's device radix sort (the library onesweep) on
// the same access-log-shaped keys as tools/sortbench.cu, sorting the same
// cell bits [32, 32 + bits) of u64 records, as a library baseline for K3.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/cubbench.cu -o build/cubbench
//   build/cubbench [n_records] [bits] [pattern: stencil|random] [reps]
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e = (x);                                                                \
    if (e != cudaSuccess) {                                                             \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                          \
    }                                                                                   \
  } while (0)

int main(int argc, char** argv) {
  const uint32_t n = argc > 1 ? (uint32_t)atoll(argv[1]) : 29360128u;
  const int bits = argc > 2 ? atoi(argv[2]) : 24;
  const std::string pat = argc > 3 ? argv[3] : "stencil";
  const int reps = argc > 4 ? atoi(argv[4]) : 10;
  std::vector<unsigned long long> hk(n);
  const uint64_t mask = bits >= 32 ? 0xFFFFFFFFull : ((1ull << bits) - 1);
  uint64_t x = 88172645463325252ull;
  const uint32_t half = (uint32_t)((mask + 1) / 2);
  for (uint32_t i = 0; i < n; i++) {  // same generator as sortbench.cu
    uint32_t key;
    if (pat == "random") {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      key = (uint32_t)(x & mask);
    } else {
      const uint32_t w = i / 128, r = i % 128, kind = r / 32, l = r % 32;
      const uint32_t c = w * 32 + l + 1;
      key = kind < 3 ? (c - 1 + kind) % half : half + c % half;
    }
    hk[i] = ((unsigned long long)key << 32) | i;
  }
  unsigned long long *d_in, *d_out;
  CK(cudaMalloc(&d_in, n * 8ull));
  CK(cudaMalloc(&d_out, n * 8ull));
  size_t tmp_bytes = 0;
  CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, d_in, d_out, (int)n, 32, 32 + bits));
  void* tmp;
  CK(cudaMalloc(&tmp, tmp_bytes));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<float> times;
  for (int it = 0; it < reps + 2; it++) {
    CK(cudaMemcpy(d_in, hk.data(), n * 8ull, cudaMemcpyHostToDevice));
    cudaEventRecord(e0);
    CK(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, d_in, d_out, (int)n, 32, 32 + bits));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it >= 2) times.push_back(ms);
  }
  std::sort(times.begin(), times.end());
  const float med = times[times.size() / 2];
  const int passes = (bits + 7) / 8;
  printf("CUB %d.%d.%d SortKeys n=%u bits=%d pattern=%s: median %.3f ms -> %.1f GB/s (16 B/rec/pass + 8 B hist, %d passes)\n",
         CUB_MAJOR_VERSION, CUB_MINOR_VERSION, CUB_SUBMINOR_VERSION, n, bits, pat.c_str(), med,
         (double)n * (16.0 * passes + 8) / (med * 1e-3) / 1e9, passes);
  std::vector<unsigned long long> ok(n);
  CK(cudaMemcpy(ok.data(), d_out, n * 8ull, cudaMemcpyDeviceToHost));
  bool good = true;
  for (uint32_t i = 1; i < n && good; i++)
    if (((ok[i - 1] >> 32) & mask) > ((ok[i] >> 32) & mask)) good = false;
  printf("verify: %s\n", good ? "ok" : "FAILED");
  return good ? 0 : 1;
}
