// boundary.cu — A4 interval boundary bookkeeping and K6 report finalize.
//
// A4 (readings L9, L17): per instance, which work-items
// are suspended at a barrier (released next interval), whether the work-items
// that arrived in this interval all reached the same barrier node
// (BARRIER_DIVERGENCE, "the same instruction barrier"), and the
// instance-level max_intervals stop.
// K6: reports of the whole run sorted into canonical order
// (instance, interval, array, index, kind, tid1, tid2) by a bitonic network.
#include "rc_internal.h"

namespace rc {

namespace {
constexpr unsigned FULL = 0xFFFFFFFFu;

__device__ __forceinline__ void push_report(rc_report* reps, unsigned long long cap, DevCounters* ctr,
                                            const rc_report& r) {
  unsigned long long pos = atomicAdd(&ctr->report_count, 1ull);
  if (pos < cap) reps[pos] = r;
}
}  // namespace

__device__ __forceinline__ bool arrived_node(uint8_t st, uint32_t pc, int32_t* node) {
  if (st == L_WAITING) { *node = (int32_t)pc - 1; return true; }
  if (st == L_EXITED_NOW) { *node = NODE_EXIT; return true; }
  return false;
}

// per instance: did the arrivals of this interval reach more than one node?
// (K1 reduced min / max arrival node per instance.)  Resets the range.  The
// last block to finish takes the interval's verdict: `abort` when the host must
// act before the next interval may run (DevCounters::abort).
__global__ void boundary_check_kernel(const BoundaryParams p) {
  DevCounters* c = p.ctr;
  if (c->abort) return;  // speculative interval after one that needs the host
  const uint32_t inst = blockIdx.x * blockDim.x + threadIdx.x;
  if (inst < p.n_inst) {
    const int32_t lo = p.node_min[inst], hi = p.node_max[inst];
    p.node_min[inst] = 0x7FFFFFFF;
    p.node_max[inst] = (int32_t)0x80000000;
    const bool div = lo < hi;
    p.inst_flag[inst] = div;
    if (div) c->diverged = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&c->bdone, 1u) == gridDim.x - 1) {
      __threadfence();
      c->bdone = 0;
      const volatile DevCounters* v = c;
      const bool need_host = v->log_overflow || v->ovl_overflow || v->k1_reports > p.report_cap ||
                             v->report_count > p.report_cap || v->diverged || !v->any_waiting;
      if (need_host) c->abort = 1;
    }
  }
}

// rare path 1: first arrived tid of each diverged instance
__global__ void div_first_kernel(const BoundaryParams p) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= p.n_lanes) return;
  const uint32_t inst = g / p.n;
  int32_t nd;
  if (!p.inst_flag[inst] || !arrived_node(p.status[g], p.pc[g], &nd)) return;
  atomicMin(&p.first_tid[inst], g - inst * p.n);
}

// rare path 2: min arrived tid at a node different from the first arrival's
__global__ void div_second_kernel(const BoundaryParams p) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= p.n_lanes) return;
  const uint32_t inst = g / p.n;
  int32_t nd, n1;
  if (!p.inst_flag[inst] || !arrived_node(p.status[g], p.pc[g], &nd)) return;
  const size_t f = (size_t)inst * p.n + p.first_tid[inst];
  arrived_node(p.status[f], p.pc[f], &n1);
  if (nd != n1) atomicMin(&p.second_tid[inst], g - inst * p.n);
}

__global__ void div_report_kernel(const BoundaryParams p) {
  const uint32_t inst = blockIdx.x * blockDim.x + threadIdx.x;
  if (inst >= p.n_inst || !p.inst_flag[inst]) return;
  const uint32_t t1 = p.first_tid[inst];
  const size_t f = (size_t)inst * p.n + t1;
  int32_t n1 = NODE_NONE;
  arrived_node(p.status[f], p.pc[f], &n1);
  rc_report r;
  r.instance = p.inst_base + inst;
  r.interval = p.interval;
  r.array = -1;
  r.index = n1;
  r.tid1 = p.gbase + t1;  // global ids (reading L20)
  r.tid2 = p.gbase + p.second_tid[inst];
  r.kind = RC_BARRIER_DIVERGENCE;
  r.flags = 0;
  r.reserved = 0;
  push_report(p.reports, p.report_cap, p.ctr, r);
}

// instance-level FUEL when max_intervals stops a batch with suspended work-items
__global__ void waiting_scan_kernel(const BoundaryParams p) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= p.n_lanes) return;
  if (p.status[g] == L_WAITING) p.inst_flag[g / p.n] = 1;
}

__global__ void max_intervals_kernel(const BoundaryParams p) {
  const uint32_t inst = blockIdx.x * blockDim.x + threadIdx.x;
  if (inst >= p.n_inst || !p.inst_flag[inst]) return;
  rc_report r;
  r.instance = p.inst_base + inst;
  r.interval = p.interval;
  r.array = -1;
  r.index = -1;
  r.tid1 = NOTID;
  r.tid2 = NOTID;
  r.kind = RC_FUEL;
  r.flags = 0;
  r.reserved = 0;
  push_report(p.reports, p.report_cap, p.ctr, r);
}

__global__ void lane_hist_kernel(const uint8_t* __restrict__ status, uint32_t n_lanes, DevCounters* ctr) {
  __shared__ unsigned int h[8];
  if (threadIdx.x < 8) h[threadIdx.x] = 0;
  __syncthreads();
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < n_lanes; g += gridDim.x * blockDim.x) {
    const uint8_t s = status[g];
    int slot;
    switch (s) {
      case L_EXITED: case L_EXITED_NOW: slot = 0; break;
      case L_PRUNED: slot = 1; break;
      case L_OOB: slot = 2; break;
      case L_ASSERT: slot = 3; break;
      case L_DIV0: slot = 4; break;
      case L_FUEL: slot = 5; break;
      default: slot = 6; break;  // still suspended when max_intervals stopped the batch
    }
    atomicAdd(&h[slot], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 8 && h[threadIdx.x]) atomicAdd(&ctr->lanes_final[threadIdx.x], (unsigned long long)h[threadIdx.x]);
}

cudaError_t launch_boundary(const BoundaryParams& p, cudaStream_t s) {
  if (p.n_inst == 0) return cudaSuccess;
  boundary_check_kernel<<<(p.n_inst + 255) / 256, 256, 0, s>>>(p);
  launched();
  return cudaGetLastError();
}

cudaError_t launch_divergence(const BoundaryParams& p, cudaStream_t s) {
  if (p.n_inst == 0 || p.n_lanes == 0) return cudaSuccess;
  cudaMemsetAsync(p.first_tid, 0xFF, p.n_inst * sizeof(uint32_t), s);
  cudaMemsetAsync(p.second_tid, 0xFF, p.n_inst * sizeof(uint32_t), s);
  const uint32_t grid = (p.n_lanes + 255) / 256;
  div_first_kernel<<<grid, 256, 0, s>>>(p);
  div_second_kernel<<<grid, 256, 0, s>>>(p);
  div_report_kernel<<<(p.n_inst + 255) / 256, 256, 0, s>>>(p);
  launched(3);
  return cudaGetLastError();
}

cudaError_t launch_max_intervals(const BoundaryParams& p, cudaStream_t s) {
  if (p.n_inst == 0) return cudaSuccess;
  cudaMemsetAsync(p.inst_flag, 0, p.n_inst * sizeof(uint32_t), s);
  if (p.n_lanes) {
    waiting_scan_kernel<<<(p.n_lanes + 255) / 256, 256, 0, s>>>(p);
    launched();
  }
  max_intervals_kernel<<<(p.n_inst + 255) / 256, 256, 0, s>>>(p);
  launched();
  return cudaGetLastError();
}

cudaError_t launch_lane_hist(const uint8_t* status, uint32_t n_lanes, DevCounters* ctr, cudaStream_t s) {
  if (n_lanes == 0) return cudaSuccess;
  const uint32_t grid = (uint32_t)std::min<uint64_t>(1184, (n_lanes + 255) / 256);
  lane_hist_kernel<<<grid, 256, 0, s>>>(status, n_lanes, ctr);
  launched();
  return cudaGetLastError();
}

// ---- K6: canonical order -----------------------------------------------------
namespace {
__device__ __forceinline__ bool rep_less(const rc_report& a, const rc_report& b) {
  if (a.instance != b.instance) return a.instance < b.instance;
  if (a.interval != b.interval) return a.interval < b.interval;
  if (a.array != b.array) return a.array < b.array;
  if (a.index != b.index) return a.index < b.index;
  if (a.kind != b.kind) return a.kind < b.kind;
  if (a.tid1 != b.tid1) return a.tid1 < b.tid1;
  return a.tid2 < b.tid2;
}
constexpr int BLK = 1024;  // threads per block; a block sorts 2*BLK entries in smem
}  // namespace

__global__ void pad_kernel(rc_report* a, uint64_t n, uint64_t n2) {
  const uint64_t i = n + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n2) return;
  rc_report r;
  r.instance = 0xFFFFFFFFu; r.interval = 0xFFFFFFFFu; r.array = 0x7FFFFFFF; r.index = 0x7FFFFFFF;
  r.tid1 = 0xFFFFFFFFu; r.tid2 = 0xFFFFFFFFu; r.kind = 0xFFFF; r.flags = 0xFFFF; r.reserved = 0xFFFFFFFFu;
  a[i] = r;
}

// one global compare-exchange step (k, j) with j >= 2*BLK
__global__ void bitonic_global(rc_report* a, uint64_t n2, uint64_t k, uint64_t j) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n2) return;
  const uint64_t l = i ^ j;
  if (l <= i) return;
  const bool up = (i & k) == 0;
  rc_report x = a[i], y = a[l];
  if (rep_less(y, x) == up) { a[i] = y; a[l] = x; }
}

// steps j = jstart .. 1 of stage k, inside blocks of 2*BLK entries
__global__ void __launch_bounds__(BLK) bitonic_local(rc_report* a, uint64_t k_lo, uint64_t k_hi, uint64_t jstart) {
  extern __shared__ rc_report sh[];
  const uint64_t base = (uint64_t)blockIdx.x * 2 * BLK;
  sh[threadIdx.x] = a[base + threadIdx.x];
  sh[threadIdx.x + BLK] = a[base + threadIdx.x + BLK];
  __syncthreads();
  // k_lo..k_hi: all stages handled here (k_lo == k_hi unless presorting blocks)
  for (uint64_t k = k_lo; k <= k_hi; k <<= 1) {
    for (uint64_t j = (k == k_lo ? jstart : k >> 1); j > 0; j >>= 1) {
      const uint32_t t = threadIdx.x;
      const uint32_t i = 2 * t - (t & (uint32_t)(j - 1));  // lower index of this thread's pair
      const uint32_t l = i + (uint32_t)j;
      const bool up = ((base + i) & k) == 0;
      rc_report x = sh[i], y = sh[l];
      if (rep_less(y, x) == up) { sh[i] = y; sh[l] = x; }
      __syncthreads();
    }
  }
  a[base + threadIdx.x] = sh[threadIdx.x];
  a[base + threadIdx.x + BLK] = sh[threadIdx.x + BLK];
}

cudaError_t finalize_reports(rc_report* reports, uint64_t n, rc_report* scratch, cudaStream_t s) {
  if (n <= 1) return cudaSuccess;
  uint64_t n2 = 2 * BLK;
  while (n2 < n) n2 <<= 1;
  static DeviceSetup setup;
  int dev = 0;
  cudaError_t se = setup.run(
      [](int) -> cudaError_t {
        return cudaFuncSetAttribute(bitonic_local, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    2 * BLK * (int)sizeof(rc_report));
      },
      &dev);
  if (se != cudaSuccess) return se;
  cudaMemcpyAsync(scratch, reports, n * sizeof(rc_report), cudaMemcpyDeviceToDevice, s);
  if (n2 > n) { pad_kernel<<<(unsigned)((n2 - n + 255) / 256), 256, 0, s>>>(scratch, n, n2); launched(); }
  const unsigned blocks_local = (unsigned)(n2 / (2 * BLK));
  const size_t smem = 2 * BLK * sizeof(rc_report);
  // all stages k <= 2*BLK inside blocks
  bitonic_local<<<blocks_local, BLK, smem, s>>>(scratch, 2, 2 * BLK, 1);
  launched();
  for (uint64_t k = 4 * BLK; k <= n2; k <<= 1) {
    uint64_t j = k >> 1;
    for (; j >= 2 * BLK; j >>= 1)
    {
      bitonic_global<<<(unsigned)((n2 + 255) / 256), 256, 0, s>>>(scratch, n2, k, j);
      launched();
    }
    bitonic_local<<<blocks_local, BLK, smem, s>>>(scratch, k, k, j);
    launched();
  }
  cudaMemcpyAsync(reports, scratch, n * sizeof(rc_report), cudaMemcpyDeviceToDevice, s);
  return cudaGetLastError();
}

}  // namespace rc
