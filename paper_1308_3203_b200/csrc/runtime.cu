// runtime.cu — rc_run: device workspace, instance batching and the barrier
// interval loop.
//
// Per instance batch:
//   A2  heap init: the caller's arrays are copied into one working heap laid
//       out [instance][cells], array a at offset off[a] (cell id
//       = inst_local * cpi + off[a] + index, a u32 key for the sort).
//       (double-buffered: the next batch's inputs copy in on a second stream)
//   per interval k, queued one interval ahead of the host:
//     K1  interpret every live work-item until it suspends / exits / stops;
//         log reads and final writes (interp.cu)
//     F   write-set filter + the sort's digit histograms (filter.cu)
//     K3  onesweep sort of the log by cell (sort.cu)
//     K4+K5 segmented detection + commit, A4 tail: divergence check and the
//         interval's verdict (detect.cu); rare paths (overflow re-runs,
//         divergence lane scans, RW classification) on the host's word
//   until no work-item is suspended at a barrier.
// After all batches: K6 canonical report order, copy to the host buffer.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

#include <array>

#include <nvtx3/nvToolsExt.h>  // header-only; the ranges cost a pointer test unless a tool is attached

#include "rc_internal.h"

namespace rc {
int fail(int code, const char* fmt, ...);
#ifdef INTERP_PHASE_TIMING
void interp_phase_io(unsigned long long* out, bool reset);
#endif
std::atomic<uint64_t> g_launches{0};

size_t Profiler::next() {
  if (used == pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    pool.push_back(e);
  }
  return used++;
}
void Profiler::begin(cudaStream_t s) {
  if (!on) return;
  if (last_end != (size_t)-1 && end_stream == s && launches_at_end == g_launches.load()) {
    open_ev = last_end;
    return;
  }
  open_ev = next();
  cudaEventRecord(pool[open_ev], s);
}
void Profiler::end(int cls, cudaStream_t s, uint64_t bytes, uint64_t items) {
  if (!on) return;
  size_t e1 = next();
  cudaEventRecord(pool[e1], s);
  marks.push_back({cls, open_ev, e1, bytes, items});
  last_end = e1;
  end_stream = s;
  launches_at_end = g_launches.load();
}
void Profiler::collect(rc_profile* out) {
  for (const Mark& m : marks) {
    float ms = 0;
    cudaEventElapsedTime(&ms, pool[m.e0], pool[m.e1]);
    out->launches[m.cls] += 1;
    out->ms[m.cls] += ms;
    out->alg_bytes[m.cls] += m.bytes;
    out->items[m.cls] += m.items;
  }
}
Profiler::~Profiler() {
  for (cudaEvent_t e : pool) cudaEventDestroy(e);
}

}  // namespace rc

using namespace rc;

// NVTX range for the host span of rc_run, a batch, an interval enqueue
// (SURVEY §5 tracing; visible under nsys / ncu --nvtx)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// grow-only device buffer
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t need, bool keep = false, cudaStream_t s = 0) {
    if (need <= bytes) return cudaSuccess;
    size_t nb = std::max(need, bytes + bytes / 2);
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, nb);
    if (e != cudaSuccess) {
      nb = need;  // retry without slack
      cudaGetLastError();
      e = cudaMalloc(&q, nb);
      if (e != cudaSuccess) return e;
    }
    if (keep && p && bytes) {
      cudaMemcpyAsync(q, p, bytes, cudaMemcpyDeviceToDevice, s);
      cudaStreamSynchronize(s);
    }
    if (p) cudaFree(p);
    p = q;
    bytes = nb;
    return cudaSuccess;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

// interval scratch layout (one memset per interval attempt): digit / bucket
// histograms [NB_MAX] u32 (LSD: [4][256]), sort tile counters, then DevCounters
constexpr size_t CTR_OFF = NB_MAX * 4 + 64;

struct rc_workspace {
  int device = -1;
  DevBuf code, arr_off, arr_size, heap, heap2;  // working heaps of alternate batches (A2 double-buffered)
  cudaStream_t copy_stream = nullptr;            // A2: the next batch's inputs copy in while this one runs
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr}, ev_start = nullptr;
  DevBuf regs[2], pc[2], status[2], live, entry_ro;
  DevBuf log, log_alt, wval, wmap, sort_status, ctr_block;
  DevBuf buckets;  // bucket path: [NB_MAX] starts | [NB_MAX] scatter cursors
  DevBuf bval;     // K1c region mode: the write records' final values beside them (W.log slot -> value)
  DevBuf spill_cell, spill_val, spill_n;  // own-write overlay spill lists (grown on demand)
  DevBuf ig;                              // inter-group race state (groups.cu), IG_FIELDS planes
  uint32_t spill_cap = 0;                 // entries per lane the spill buffers hold
  uint8_t wtag = 0;  // write-set map tag of the last interval attempt
  bool prove_valid = false;     // cached rc_prove verdict (RC_OPT_PREPASS) for prove_key
  std::vector<uint64_t> prove_key;
  uint32_t prove_verdict = 0;
  bool region_ok = true;        // bucket region mode for the cached plan (cleared after a bucket overflow)
  bool plan_valid = false;      // cached batch plan (rc_run)
  uint64_t plan_key[4] = {0, 0, 0, 0};
  uint32_t plan_ib = 0;
  DevBuf reports, reports_scratch;
  DevBuf inst_tmp;  // node_min | node_max | first_tid | second_tid | inst_flag  ([I_b] each)
  // RW classification: interval-start heaps (two slots), the re-run's heap,
  // the RW-cell mask, the re-run's (discarded) lane state
  DevBuf heap_snap[2], heapB, amap, regs_b, pc_b, status_b, cmp_inst;
  DevBuf ctr;
  DevCounters* h_ctr = nullptr;  // pinned [4]: interval slots 0/1, synchronous reads 2, copy source 3
  cudaEvent_t iv_done[2] = {nullptr, nullptr};  // interval k's counters landed in h_ctr[k & 1]
  SortWorkspace sort;
  Profiler prof;
  ~rc_workspace() {
    for (cudaEvent_t e : {ev_in[0], ev_in[1], ev_free[0], ev_free[1], ev_start})
      if (e) cudaEventDestroy(e);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    for (DevBuf* b : {&code, &arr_off, &arr_size, &heap, &heap2, &regs[0], &regs[1], &pc[0], &pc[1], &status[0],
                      &status[1], &live, &entry_ro, &log, &log_alt, &wval, &wmap, &sort_status, &buckets,
                      &ctr_block, &reports, &reports_scratch, &inst_tmp, &heap_snap[0], &heap_snap[1], &heapB, &amap,
                      &regs_b, &pc_b, &status_b, &cmp_inst, &spill_cell, &spill_val, &spill_n, &ig})  // (ctr: a view)
      b->release();
    if (h_ctr) cudaFreeHost(h_ctr);
    for (cudaEvent_t e : iv_done)
      if (e) cudaEventDestroy(e);
  }
};

namespace {

#define CK(call)                                                                                     \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess)                                                                           \
      return fail(e_ == cudaErrorMemoryAllocation ? RC_ENOMEM : RC_ECUDA, "%s failed: %s (%s:%d)",   \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                                \
  } while (0)

int bits_for(uint64_t x) {  // bits needed for values in [0, x)
  if (x <= 1) return 0;
  int b = 0;
  uint64_t v = x - 1;
  while (v) { b++; v >>= 1; }
  return b;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Instance batch size: a batch's cells must fit the u32 key
// (bucket path: the NB_MAX buckets); LSD path: prefer the fewest 8-bit sort
// passes that still give >= ~4M lanes per batch, then the largest batch with
// that pass count, within a memory budget.
uint32_t plan_batch(uint32_t n_inst, uint32_t n, uint64_t cpi, uint32_t n_regs, uint32_t max_batch,
                    size_t free_bytes, bool groups, bool bucket) {
  if (n_inst == 0) return 0;
  const uint64_t cells_cap = cpi ? (uint64_t)0xFFFFFFFFull / cpi : (uint64_t)n_inst;
  const uint64_t lane_cap = n ? ((uint64_t)1 << 27) / n : (uint64_t)n_inst;  // batch lanes fit the record's 27 bits
  // bytes per lane: 2x lane state + node + ~6 log records (keys+vals, double buffered)
  const uint64_t per_lane = 2 * (4ull * n_regs + 5) + 4 + 6 * 24;
  const uint64_t per_inst = (uint64_t)n * per_lane + cpi * 4 * (groups ? 1 + IG_FIELDS : 1) + 16;
  const uint64_t mem_cap = std::max<uint64_t>(1, (uint64_t)(free_bytes * 0.5) / std::max<uint64_t>(per_inst, 1));
  uint64_t hi = std::min<uint64_t>({(uint64_t)n_inst, cells_cap, lane_cap, mem_cap});
  if (max_batch) hi = std::min<uint64_t>(hi, max_batch);
  hi = std::max<uint64_t>(hi, 1);
  // bucket path: the largest batch whose cells fit the NB_MAX buckets (fewer
  // batches: fewer interval launches for the same work)
  if (bucket) return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(hi, BUCKET_PATH_CELLS / std::max<uint64_t>(cpi, 1)));
  const uint64_t target_lanes = 1ull << 22;
  uint64_t need = n ? (target_lanes + n - 1) / n : hi;
  need = std::min(std::max<uint64_t>(need, 1), hi);
  const int passes = (bits_for(need * std::max<uint64_t>(cpi, 1)) + 7) / 8;
  uint64_t best = need;
  // largest batch <= hi with the same pass count
  uint64_t lim = passes >= 4 ? hi : std::min<uint64_t>(hi, ((1ull << (8 * passes)) / std::max<uint64_t>(cpi, 1)));
  best = std::max(best, lim);
  best = std::min(best, hi);
  return (uint32_t)std::max<uint64_t>(best, 1);
}

}  // namespace

extern "C" {

void rc_free_program(rc_program* P) {
  if (!P) return;
  if (P->ws || P->xc.device >= 0) {
    int prev = -1;
    cudaGetDevice(&prev);
    if (P->ws) {
      if (P->ws->device >= 0) cudaSetDevice(P->ws->device);
      delete P->ws;
    }
    if (P->xc.device >= 0) {
      cudaSetDevice(P->xc.device);
      P->xc.release();
    }
    if (prev >= 0) cudaSetDevice(prev);
  }
  rc::jit_release(P);
  delete P;
}

int rc_release_workspace(rc_program* P) {
  if (!P) return fail(RC_EINVAL, "program is NULL");
  std::lock_guard<std::mutex> lk(P->mu);
  if (P->ws) {
    DeviceGuard g(P->ws->device);
    delete P->ws;
    P->ws = nullptr;
  }
  if (P->xc.device >= 0) {
    DeviceGuard g(P->xc.device);
    P->xc.release();
  }
  jit_release(P);
  return RC_OK;
}

int rc_run(const rc_program* prog, uint32_t n, const rc_array* arrays, uint32_t n_arrays, uint32_t n_inst,
           const rc_options* options, rc_report* out, uint64_t capacity, uint64_t* n_reports_total,
           rc_stats* stats, int32_t* const* final_heaps) {
  if (n_reports_total) *n_reports_total = 0;
  if (stats) memset(stats, 0, sizeof *stats);
  if (!prog) return fail(RC_EINVAL, "program is NULL");
  rc_program* P = const_cast<rc_program*>(prog);
  if (n_arrays != P->n_arrays) return fail(RC_EINVAL, "n_arrays %u != program's %u", n_arrays, P->n_arrays);
  if (n_arrays && !arrays) return fail(RC_EINVAL, "arrays is NULL");
  if (n > MAX_WG) return fail(RC_EINVAL, "work_group_size %u > 2^27", n);
  if (capacity && !out) return fail(RC_EINVAL, "out is NULL with capacity %llu", (unsigned long long)capacity);
  rc_options opt;
  memset(&opt, 0, sizeof opt);
  if (options) opt = *options;
  if (!opt.max_intervals) opt.max_intervals = 65536;
  if (!opt.fuel_per_interval) opt.fuel_per_interval = 1ull << 20;
  const bool host_io = (opt.flags & RC_OPT_HOST_IO) != 0;
  const uint32_t G = opt.n_groups ? opt.n_groups : 1;  // work-groups per instance (reading L20)
  if ((uint64_t)G * n > 0xFFFFFFFEull) return fail(RC_EINVAL, "n_groups * work_group_size exceeds 2^32 - 2");
  const bool classify = (opt.flags & RC_OPT_CLASSIFY_RW) != 0;  // RW value classification (reading L19)
  uint64_t cpi = 0;
  std::vector<uint32_t> off(n_arrays + 1, 0), size(n_arrays + 1, 0);
  for (uint32_t a = 0; a < n_arrays; a++) {
    if (arrays[a].size >= (1u << 31)) return fail(RC_EINVAL, "array %u: size %u >= 2^31", a, arrays[a].size);
    if (arrays[a].size && n_inst && !arrays[a].data) return fail(RC_EINVAL, "array %u: data is NULL", a);
    off[a] = (uint32_t)cpi;
    size[a] = arrays[a].size;
    cpi += arrays[a].size;
    if (cpi > 0xFFFFFFFFull) return fail(RC_ELIMIT, "cells per instance exceed 2^32");
  }
  if (final_heaps)
    for (uint32_t a = 0; a < n_arrays; a++)
      if (arrays[a].size && n_inst && !final_heaps[a]) return fail(RC_EINVAL, "final_heaps[%u] is NULL", a);

  std::lock_guard<std::mutex> lk(P->mu);
  DeviceGuard dg(opt.device);
  NvtxRange nvtx_run("rc_run");
  cudaStream_t s = static_cast<cudaStream_t>(opt.cuda_stream);
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (opt.device < 0 || opt.device >= ndev) return fail(RC_EINVAL, "device %d not present", opt.device);
  if (P->ws && P->ws->device != opt.device) {
    delete P->ws;
    P->ws = nullptr;
  }
  if (!P->ws) {
    P->ws = new (std::nothrow) rc_workspace();
    if (!P->ws) return fail(RC_ENOMEM, "host allocation failed");
    P->ws->device = opt.device;
    rc_workspace& W = *P->ws;
    CK(W.code.ensure(P->code.size() * sizeof(Ins)));
    CK(cudaMemcpy(W.code.p, P->dev_code.data(), P->dev_code.size() * sizeof(Ins), cudaMemcpyHostToDevice));
    CK(W.entry_ro.ensure(P->entry_ro.size() * 4));
    CK(cudaMemcpy(W.entry_ro.p, P->entry_ro.data(), P->entry_ro.size() * 4, cudaMemcpyHostToDevice));
    CK(W.live.ensure(std::max<size_t>(1, P->live_regs.size())));
    if (!P->live_regs.empty())
      CK(cudaMemcpy(W.live.p, P->live_regs.data(), P->live_regs.size(), cudaMemcpyHostToDevice));
    // interval scratch in one allocation, zeroed by one memset per interval:
    // [digit / bucket histograms 32 KB][sort tile counters, 64 B][DevCounters]
    CK(W.ctr_block.ensure(CTR_OFF + sizeof(DevCounters)));
    CK(W.buckets.ensure(2 * NB_MAX * sizeof(uint32_t)));
    W.ctr.p = static_cast<char*>(W.ctr_block.p) + CTR_OFF;
    W.ctr.bytes = sizeof(DevCounters);
    CK(cudaMallocHost(&W.h_ctr, 4 * sizeof(DevCounters)));
    for (cudaEvent_t& e : W.iv_done) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaStreamCreateWithFlags(&W.copy_stream, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&W.ev_in[0], &W.ev_in[1], &W.ev_free[0], &W.ev_free[1], &W.ev_start})
      CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    W.sort.hist = W.ctr_block.as<uint32_t>();
    W.sort.bin_off = nullptr;  // each pass scans its counts itself
    W.sort.tile_ctr = W.sort.hist + NB_MAX;
    W.sort.reset_tile_ctr = false;
  }
  rc_workspace& W = *P->ws;
  W.prof.reset();
  W.prof.on = opt.profile != nullptr;
  const uint32_t prof_every = opt.profile ? (opt.profile->sample_every ? opt.profile->sample_every : 7u) : 1u;
  uint64_t prof_intervals = 0;  // interval enqueues so far (sampling clock)
  if (opt.profile) memset(opt.profile, 0, sizeof(rc_profile));
  const uint64_t launches0 = g_launches.load();
  cudaEvent_t t_begin = nullptr, t_end = nullptr;
  if (W.prof.on) {
    cudaEventCreate(&t_begin);
    cudaEventCreate(&t_end);
    cudaEventRecord(t_begin, s);
  }

  CK(W.arr_off.ensure((n_arrays + 1) * 4));
  CK(W.arr_size.ensure((n_arrays + 1) * 4));
  CK(cudaMemcpyAsync(W.arr_off.p, off.data(), (n_arrays + 1) * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(W.arr_size.p, size.data(), (n_arrays + 1) * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(W.ctr.p, 0, sizeof(DevCounters), s));

  // batch plan, cached per shape: cudaMemGetInfo can take milliseconds (it
  // was the largest host stall between back-to-back runs)
  // the bucket path groups the log by cell whenever one
  // instance's cells fit its buckets; else (and under the A/B hook
  // RC_SORT_LSD=1) the onesweep LSD sort
  const bool bucket = cpi <= BUCKET_PATH_CELLS && getenv("RC_SORT_LSD") == nullptr;
  const uint64_t plan_key[4] = {n_inst, n, cpi,
                                (uint64_t)opt.max_batch_instances | (uint64_t)(G > 1) << 32 | (uint64_t)bucket << 33};
  if (!W.plan_valid || memcmp(plan_key, W.plan_key, sizeof plan_key) != 0) {
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    W.plan_ib = plan_batch(n_inst, n, cpi, P->n_regs, opt.max_batch_instances, free_b, G > 1, bucket);
    W.region_ok = true;
    memcpy(W.plan_key, plan_key, sizeof plan_key);
    W.plan_valid = true;
  }
  // with host inputs (RC_OPT_HOST_IO) the run is bound by the host->device
  // copies, overlapped batch by batch (A2): the last batch's work is the part
  // no copy hides, so the batch is capped at 1/16 of the run (config 5: 32
  // instances; 4 batches of 128 left 25% of the step exposed)
  const uint32_t I_b = (host_io && !opt.max_batch_instances && n_inst >= 32)
                           ? std::min<uint32_t>(W.plan_ib, (n_inst + 15) / 16)
                           : W.plan_ib;
  // RC_OPT_PREPASS: a run proved conflict-free by the
  // symbolic pre-pass interprets its intervals in direct-commit mode
  bool direct = false;
  if ((opt.flags & RC_OPT_PREPASS) && G == 1 && !classify && n_inst) {
    std::vector<uint64_t> key{n, opt.fuel_per_interval, opt.max_intervals};
    key.insert(key.end(), size.begin(), size.begin() + n_arrays);
    if (!W.prove_valid || W.prove_key != key) {
      rc_prove_result pr;
      const int pe = rc_prove(P, n, size.data(), n_arrays, opt.fuel_per_interval, 0, &pr);
      if (pe != RC_OK) return pe;
      // (an interval count beyond max_intervals is the host's instance-level FUEL report, unchanged)
      W.prove_verdict = pr.verdict;
      W.prove_key = key;
      W.prove_valid = true;
    }
    direct = W.prove_verdict == RC_PROVE_NO_CONFLICT;
  }
  const uint64_t L_max = (uint64_t)I_b * n;
  const uint64_t L_pad = (L_max + LANE_PAD - 1) / LANE_PAD * LANE_PAD + LANE_PAD;  // TMA rows, + a spare tile
  const int key_bits = bits_for((uint64_t)I_b * std::max<uint64_t>(cpi, 1));

  // batch-sized buffers
  if (I_b) {
    CK(W.heap.ensure(std::max<uint64_t>(1, (uint64_t)I_b * cpi) * 4));
    if (n_inst > I_b) CK(W.heap2.ensure(std::max<uint64_t>(1, (uint64_t)I_b * cpi) * 4));
    for (int b = 0; b < 2; b++) {
      CK(W.regs[b].ensure(L_pad * P->n_regs * 4));
      CK(W.pc[b].ensure(L_pad * 4));
      CK(W.status[b].ensure(L_pad));
    }
    CK(W.inst_tmp.ensure((uint64_t)I_b * 20));
    if (classify) {
      const uint64_t hb = std::max<uint64_t>(1, (uint64_t)I_b * cpi) * 4;
      CK(W.heap_snap[0].ensure(hb));
      CK(W.heap_snap[1].ensure(hb));
      CK(W.heapB.ensure(hb));
      CK(W.amap.ensure(hb / 4));
      CK(W.regs_b.ensure(L_pad * P->n_regs * 4));
      CK(W.pc_b.ensure(L_pad * 4));
      CK(W.status_b.ensure(L_pad));
      CK(W.cmp_inst.ensure((uint64_t)I_b * 4));
    }
    CK(W.wval.ensure(std::max<uint64_t>(1, L_max * (uint64_t)P->ovl_cap) * 4));
    if (P->may_spill) CK(W.spill_n.ensure(L_pad * 4));
    if (G > 1) CK(W.ig.ensure(std::max<uint64_t>(1, (uint64_t)I_b * cpi) * 4 * IG_FIELDS));
    const void* wmap_before = W.wmap.p;
    CK(W.wmap.ensure(std::max<uint64_t>(1, (uint64_t)I_b * cpi)));
    if (W.wmap.p != wmap_before) W.wtag = 0;  // new memory: zero it before the next tag is used
  }
  const int passes = (key_bits + 7) / 8;
  // test hook: start from tiny log / report buffers so the grow-and-retry
  // paths run (results must not change)
  const bool small_buffers = getenv("RC_DEBUG_SMALL_BUFFERS") != nullptr;
  uint64_t log_cap = std::min(W.log.bytes, W.log_alt.bytes) / 8;
  {
    // ~4 records per lane plus the tails of the per-block staging chunks (K1 grid <= 4 blocks per SM)
    uint64_t want = std::max<uint64_t>(1u << 16, std::min<uint64_t>(L_max * 4 + 148ull * 4 * 8192, 0xFFFFFFFFull));
    if (small_buffers) want = 1024;
    if (log_cap < want) {
      CK(W.log.ensure(want * 8));
      CK(W.log_alt.ensure(want * 8));
      log_cap = std::min(W.log.bytes, W.log_alt.bytes) / 8;
    }
  }
  auto ensure_sort_status = [&](uint64_t cap) -> cudaError_t {
    const size_t tiles = sort_tiles(cap);
    if (W.sort_status.bytes < tiles * 256 * 8) {
      cudaError_t e = W.sort_status.ensure(tiles * 256 * 8);
      if (e != cudaSuccess) return e;
      e = cudaMemsetAsync(W.sort_status.p, 0, W.sort_status.bytes, s);
      W.sort.epoch = 0;
      W.sort.status_fmt = -1;
      if (e != cudaSuccess) return e;
    }
    W.sort.status = W.sort_status.as<unsigned long long>();
    W.sort.status_tiles = W.sort_status.bytes / (256 * 8);
    return cudaSuccess;
  };
  CK(ensure_sort_status(log_cap));
  // bucket region mode: bucket b owns W.log[b * BUCKET_REGION, + BUCKET_REGION)
  // — no count pass; an overflowing bucket makes the host regroup the interval with the counts
  bool region = bucket && W.region_ok && getenv("RC_BUCKET_COUNT") == nullptr;
  if (region) {
    const uint64_t nb_max = std::max<uint64_t>(1, ((uint64_t)I_b * cpi + BUCKET_CELLS - 1) / BUCKET_CELLS);
    CK(W.log.ensure(std::max<uint64_t>(W.log.bytes, nb_max * BUCKET_REGION * 8 + 64)));
  }
  // own-write overlay spill lists [spill_cap][L_max] (PAPER.md:176-179 puts no
  // bound on the cells a work-item writes in an interval): grown when K1
  // reports a full list, and the interval re-run
  auto ensure_spill = [&](uint32_t cap) -> cudaError_t {
    if (!P->may_spill || cap == 0) return cudaSuccess;
    cudaError_t e = W.spill_cell.ensure((uint64_t)cap * std::max<uint64_t>(L_max, 1) * 4);
    if (e == cudaSuccess) e = W.spill_val.ensure((uint64_t)cap * std::max<uint64_t>(L_max, 1) * 4);
    if (e == cudaSuccess) W.spill_cap = cap;
    return e;
  };
  CK(ensure_spill(W.spill_cap));  // (L_max may have grown since the capacity was set)
  auto grow_spill = [&]() -> int {
    const uint64_t want = W.spill_cap ? 4ull * W.spill_cap : 16ull;
    if (want > (1ull << 24) - OVL_CAP)
      return fail(RC_ELIMIT, "a work-item wrote more than 2^24 distinct cells in one barrier interval");
    CK(ensure_spill((uint32_t)want));
    return RC_OK;
  };
  uint64_t rep_cap = W.reports.bytes / sizeof(rc_report);
  if (rep_cap < (1u << 16) && !small_buffers) {
    CK(W.reports.ensure((1u << 16) * sizeof(rc_report)));
    rep_cap = W.reports.bytes / sizeof(rc_report);
  } else if (small_buffers && rep_cap == 0) {
    CK(W.reports.ensure(4 * sizeof(rc_report)));
    rep_cap = W.reports.bytes / sizeof(rc_report);
  }

  // K1c (jit.cpp): the intervals run in a kernel compiled for this program
  // and shape when the batches are large enough to repay the compile (once per
  // program and shape; RC_JIT=1 forces it for any size, RC_JIT=0 keeps K1).
  // Not with work-groups, RW classification re-runs (always K1) or programs
  // jit_get declines; a K1c interval that bails (jit_bail) is re-run by K1 and
  // K1 keeps the rest of the run.
  JitKernel jk;
  bool jit_on = false, jit_wbucket = false;
  int jit_planes = 0;
  const char* jit_env = getenv("RC_JIT");
  const uint64_t jit_min_lanes =
      getenv("RC_JIT_MIN_LANES") ? strtoull(getenv("RC_JIT_MIN_LANES"), nullptr, 10) : (1ull << 20);
  const bool jit_wanted = !(jit_env && jit_env[0] == '0') && G == 1 && I_b &&
                          ((jit_env && jit_env[0] == '1') || L_max >= jit_min_lanes);
  // the K1c variant for this run: wb = its write records go straight into the
  // bucket regions (region mode; the planes and the scatter carry only reads)
  auto select_jit = [&](bool wb) -> cudaError_t {
    JitShape S;
    S.n = n;
    S.gid = 0;
    S.cpi = (uint32_t)cpi;
    S.off.assign(off.begin(), off.begin() + n_arrays);
    S.size.assign(size.begin(), size.begin() + n_arrays);
    S.direct = direct;
    S.fuel = P->instr_bound < 0 || (uint64_t)P->instr_bound > opt.fuel_per_interval;
    S.ro_skip = (opt.flags & RC_OPT_KEEP_ALL_READS) == 0;
    // a thread runs <= 2^27 / (148 * 256) < 3600 lanes: 32-bit statistics
    // when no work-item can execute 2^20 instructions in one interval
    const uint64_t sb = P->instr_bound >= 0 ? std::min<uint64_t>((uint64_t)P->instr_bound, opt.fuel_per_interval)
                                            : opt.fuel_per_interval;
    S.narrow = sb < (1ull << 20);
    S.wbucket = wb && !direct;
    std::string why;
    jit_on = jit_get(P, S, &jk, &why);
    if (!jit_on && getenv("RC_JIT_VERBOSE")) fprintf(stderr, "rc: K1c not used: %s\n", why.c_str());
    jit_wbucket = S.wbucket;
    if (jit_on && jit_wbucket) {  // values beside the records: one int32 per region slot
      const uint64_t nb_max = std::max<uint64_t>(1, ((uint64_t)I_b * cpi + BUCKET_CELLS - 1) / BUCKET_CELLS);
      const cudaError_t e = W.bval.ensure(nb_max * BUCKET_REGION * 4 + 64);
      if (e != cudaSuccess) return e;
    }
    jit_planes = direct ? 0
                 : S.wbucket ? (S.ro_skip ? P->read_bound_ro : P->read_bound)
                             : (S.ro_skip ? P->rec_bound_ro : P->rec_bound);
    if (jit_on && jit_planes > 0) {  // fixed record slots: planes x (lanes rounded up to LANE_PAD)
      const uint64_t want = (uint64_t)jit_planes * ((L_max + LANE_PAD - 1) / LANE_PAD * LANE_PAD);
      if (log_cap < want) {
        cudaError_t e = W.log.ensure(std::max<uint64_t>(W.log.bytes, want * 8));
        if (e == cudaSuccess) e = W.log_alt.ensure(want * 8);
        if (e != cudaSuccess) return e;
        log_cap = std::min(W.log.bytes, W.log_alt.bytes) / 8;
        return ensure_sort_status(log_cap);
      }
    }
    return cudaSuccess;
  };
  if (jit_wanted) CK(select_jit(region && getenv("RC_JIT_NO_WBUCKET") == nullptr));
  bool jit_off = false;  // a K1c interval bailed: K1 for the rest of the run
  bool jit_fix_pending = false;  // lane state K1c produced has rematerialised registers missing from the rows
  bool jit_used_wb[2] = {false, false};  // interval k & 1 ran K1c with its writes in the buckets
  bool jit_used_iv[2] = {false, false};  // interval k & 1 ran K1c
  bool jit_ran = false;
  bool fresh_pending = false;  // this batch's initial lane state is not in the rows yet (K1c reads none)

  uint64_t tot_loads = 0, tot_stores = 0, tot_instr = 0, intervals_max = 0;
  uint64_t rep_count = 0;  // host mirror of ctr.report_count
  DevCounters* dctr = W.ctr.as<DevCounters>();

  auto read_ctr = [&]() -> cudaError_t {
    cudaError_t e = cudaMemcpyAsync(&W.h_ctr[2], dctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return e;
    return cudaStreamSynchronize(s);
  };
  auto set_report_count = [&](uint64_t v) -> cudaError_t {
    W.h_ctr[3].report_count = v;  // slot 3: only ever a copy source
    return cudaMemcpyAsync(&dctr->report_count, &W.h_ctr[3].report_count, 8, cudaMemcpyHostToDevice, s);
  };
  auto grow_reports = [&](uint64_t need) -> cudaError_t {
    cudaError_t e = W.reports.ensure(need * sizeof(rc_report) * 5 / 4, true, s);
    rep_cap = W.reports.bytes / sizeof(rc_report);
    return e;
  };

  // dev instrumentation (RC_GAPS=1): GPU time inside interval enqueues vs the whole run
  const bool gaps = getenv("RC_GAPS") != nullptr;
  std::vector<std::array<cudaEvent_t, 2>> gap_ev;
  std::vector<uint32_t> gap_b;  // batch of each recorded interval
  cudaEvent_t g0 = nullptr, g1 = nullptr;
  if (gaps) { cudaEventCreate(&g0); cudaEventCreate(&g1); cudaEventRecord(g0, s); }
  // A2, double-buffered: batch i's inputs are copied (2-D copies into the
  // instance-major working heap) on a copy stream into heap[i & 1] while batch
  // i - 1 runs; batch i waits for its copy, the copy of batch i + 2 waits for
  // batch i to release the buffer (after its final-heap copy).
  auto heap_buf = [&](uint64_t bi) -> int32_t* { return ((bi & 1) ? W.heap2 : W.heap).as<int32_t>(); };
  bool free_recorded[2] = {false, false};
  auto enqueue_inputs = [&](uint64_t bi, uint32_t b0) -> cudaError_t {
    const uint32_t nb = std::min(I_b, n_inst - b0);
    cudaError_t e = cudaSuccess;
    if (free_recorded[bi & 1]) e = cudaStreamWaitEvent(W.copy_stream, W.ev_free[bi & 1], 0);
    for (uint32_t a = 0; a < n_arrays && e == cudaSuccess; a++) {
      if (!size[a]) continue;
      e = cudaMemcpy2DAsync(heap_buf(bi) + off[a], cpi * 4, arrays[a].data + (uint64_t)b0 * size[a],
                            (size_t)size[a] * 4, (size_t)size[a] * 4, nb,
                            host_io ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, W.copy_stream);
    }
    if (e == cudaSuccess) e = cudaEventRecord(W.ev_in[bi & 1], W.copy_stream);
    return e;
  };
  if (n_inst && I_b) {
    CK(cudaEventRecord(W.ev_start, s));  // inputs the caller produced on its stream
    CK(cudaStreamWaitEvent(W.copy_stream, W.ev_start, 0));
    CK(enqueue_inputs(0, 0));
  }
  for (uint32_t b0 = 0, bi = 0; b0 < n_inst; b0 += I_b, bi++) {
    NvtxRange nvtx_batch("rc batch");
    const uint32_t nb = std::min(I_b, n_inst - b0);
    const uint32_t L = nb * n;
    const uint32_t inst_base = opt.instance_offset + b0;
    int32_t* const heap_cur = heap_buf(bi);  // this batch's working heap
    CK(cudaStreamWaitEvent(s, W.ev_in[bi & 1], 0));
    if (b0 + I_b < n_inst) CK(enqueue_inputs(bi + 1, b0 + I_b));  // overlaps this batch
    int32_t* node_min = W.inst_tmp.as<int32_t>();
    int32_t* node_max = node_min + I_b;
    uint32_t* first_tid = reinterpret_cast<uint32_t*>(node_max + I_b);
    uint32_t* second_tid = first_tid + I_b;
    uint32_t* inst_flag = second_tid + I_b;
    uint32_t gi = 0;  // work-group pass (reading L20; one pass when n_groups == 1)
    const uint64_t bcells = (uint64_t)nb * cpi;
    const uint64_t* sr = nullptr;  // sorted log of the last enqueued interval
    const uint32_t nbk = bucket ? (uint32_t)std::max<uint64_t>(1, (bcells + BUCKET_CELLS - 1) / BUCKET_CELLS) : 0u;
    // write-set filter + grouping of one interval's records by cell (K3): the
    // bucket scatter (filter fused), or the filter and the onesweep passes
    auto enqueue_sort = [&](Profiler* prof, bool keep_all, bool use_region) -> cudaError_t {
      if (bucket) {
        sr = W.log.as<uint64_t>();
        ScatterParams sp;
        sp.region = 0;
        sp.stage = W.log_alt.as<uint64_t>();
        sp.n_slots = (uint32_t)log_cap;  // upper bound; the kernel reads stage_count
        sp.wmap = W.wmap.as<uint8_t>();
        sp.wtag = W.wtag;
        sp.keep_all = keep_all;
        sp.out = W.log.as<uint64_t>();
        sp.bcur = W.buckets.as<uint32_t>() + NB_MAX;
        sp.ctr = dctr;
        if (use_region) {  // no count pass: the cursors (zeroed with the interval scratch) start at 0
          sp.region = BUCKET_REGION;
          sp.bcur = W.sort.hist;
          return launch_bucket_scatter(sp, s, prof);
        }
        cudaError_t e = launch_bucket_count(sp, W.sort.hist, nbk, W.buckets.as<uint32_t>(), s, prof);
        if (e != cudaSuccess) return e;
        return launch_bucket_scatter(sp, s, prof);
      }
      FilterParams fp;
      fp.stage = W.log_alt.as<uint64_t>();
      fp.wmap = W.wmap.as<uint8_t>();
      fp.wtag = W.wtag;
      fp.out = W.log.as<uint64_t>();
      fp.hist = W.sort.hist;
      fp.passes = passes;
      fp.ctr = dctr;
      fp.n_slots = (uint32_t)log_cap;  // upper bound; the kernel reads stage_count
      fp.keep_all = keep_all;
      if (prof) prof->begin(s);
      cudaError_t e = launch_filter(fp, s);
      if (prof) prof->end(RC_PROF_FILTER, s, 0, 0);
      if (e != cudaSuccess) return e;
      bool in_alt = false;
      W.sort.alt = W.log_alt.as<uint64_t>();
      e = onesweep_sort(W.log.as<uint64_t>(), (uint32_t)log_cap, &dctr->kept_count, nullptr, key_bits, W.sort, s,
                        &in_alt, prof, /*hist_ready=*/true);
      sr = in_alt ? W.log_alt.as<uint64_t>() : W.log.as<uint64_t>();
      return e;
    };
    if (G > 1) CK(ig_reset(W.ig.as<uint32_t>(), bcells, s));
    // the initial lane state as rows (status RUNNING, pc 0, the registers live
    // at pc 0 zero — reading L18: a register read before it is written in
    // interval 0 can observe it; the other rows are written before any read)
    auto materialize_fresh = [&](int cc) -> cudaError_t {
      const uint32_t rs = (uint32_t)((L + LANE_PAD - 1) / LANE_PAD * LANE_PAD);
      cudaError_t e = cudaMemsetAsync(W.status[cc].p, 0, rs, s);
      if (e == cudaSuccess) e = cudaMemsetAsync(W.pc[cc].p, 0, (size_t)rs * 4, s);
      for (uint8_t r : P->live_at_entry)
        if (e == cudaSuccess) e = cudaMemsetAsync(W.regs[cc].as<int32_t>() + (size_t)r * rs, 0, (size_t)rs * 4, s);
      fresh_pending = false;
      return e;
    };
    auto bparams = [&](uint32_t interval) {
      BoundaryParams bp;
      bp.n = n;
      bp.gbase = gi * n;
      bp.n_lanes = L;
      bp.n_inst = nb;
      bp.interval = interval;
      bp.inst_base = inst_base;
      bp.node_min = node_min;
      bp.node_max = node_max;
      bp.first_tid = first_tid;
      bp.second_tid = second_tid;
      bp.inst_flag = inst_flag;
      bp.reports = W.reports.as<rc_report>();
      bp.report_cap = rep_cap;
      bp.ctr = dctr;
      return bp;
    };
    int cur = 0;
    const uint32_t reg_stride = (uint32_t)((L + LANE_PAD - 1) / LANE_PAD * LANE_PAD);
    // ---- one interval = K1 → filter → sort → detect → A4 (+ verdict), then
    //      the counters to a pinned slot and an event.  No kernel needs a host
    //      count (each reads its record count from device memory).
    const uint32_t stage_warp =
        P->rec_bound > 0 ? (uint32_t)std::min(256, ((32 * P->rec_bound + 31) / 32) * 32) : 256u;
    auto detect_params = [&](uint32_t kk) {
      DetectParams dp;
      dp.recs = sr;
      dp.wval = W.wval.as<int32_t>();
      dp.spill_cell = P->may_spill ? W.spill_cell.as<uint32_t>() : nullptr;  // (null: no spilled record)
      dp.spill_val = P->may_spill ? W.spill_val.as<int32_t>() : nullptr;
      dp.spill_n = P->may_spill ? W.spill_n.as<uint32_t>() : nullptr;
      dp.n_lanes = L;
      dp.n = n;
      dp.gbase = gi * n;
      dp.n_records = (uint32_t)log_cap;  // upper bound; the kernel reads the exact count
      dp.heap = heap_cur;
      dp.cpi = (uint32_t)std::max<uint64_t>(cpi, 1);
      dp.cpi_magic = div_magic(dp.cpi);
      dp.n_arrays = n_arrays;
      dp.arr_off = W.arr_off.as<uint32_t>();
      dp.interval = kk;
      dp.inst_base = inst_base;
      dp.reports = W.reports.as<rc_report>();
      dp.report_cap = rep_cap;
      dp.ctr = dctr;
      dp.with_boundary = false;
      dp.classify = classify;
      dp.quiet = false;
      dp.n_inst = nb;
      dp.node_min = node_min;
      dp.node_max = node_max;
      dp.inst_flag = inst_flag;
      dp.nb = nbk;
      dp.bstart = W.buckets.as<uint32_t>();
      dp.bend = W.buckets.as<uint32_t>() + NB_MAX;
      dp.tmp = W.log_alt.as<uint64_t>();  // (the staging buffer: free once the scatter has read it)
      dp.region = region ? BUCKET_REGION : 0u;
      dp.rcur = W.sort.hist;
      dp.rend = W.buckets.as<uint32_t>() + NB_MAX;  // (free in region mode)
      dp.region_rerun = false;
      dp.bval = nullptr;
      return dp;
    };
    struct Marks { size_t m0 = 0, m1 = 0; };
    auto make_ip = [&](uint32_t kk, int cc) {
      InterpParams ip;
      ip.code = W.code.as<Ins>();
      ip.n_instr = P->n_instr;
      ip.n_regs = P->n_regs;
      ip.n_arrays = n_arrays;
      ip.n = n;
      ip.gid = gi;
      ip.gbase = gi * n;
      ip.n_magic = div_magic(n);
      ip.n_lanes = L;
      ip.cpi = (uint32_t)cpi;
      ip.fuel = opt.fuel_per_interval;
      ip.fuel_check = P->instr_bound < 0 || (uint64_t)P->instr_bound > opt.fuel_per_interval;
      ip.interval = kk;
      ip.inst_base = inst_base;
      ip.arr_off = W.arr_off.as<uint32_t>();
      ip.arr_size = W.arr_size.as<uint32_t>();
      ip.heap = heap_cur;
      ip.heap_w = heap_cur;
      ip.direct = direct;
      ip.reg_stride = reg_stride;
      ip.regs_in = W.regs[cc].as<int32_t>();
      ip.pc_in = W.pc[cc].as<uint32_t>();
      ip.status_in = W.status[cc].as<uint8_t>();
      ip.regs_out = W.regs[cc ^ 1].as<int32_t>();
      ip.pc_out = W.pc[cc ^ 1].as<uint32_t>();
      ip.status_out = W.status[cc ^ 1].as<uint8_t>();
      ip.live = W.live.as<uint8_t>();
      ip.n_live = (uint32_t)P->live_regs.size();
      ip.ovl_cap = (uint32_t)P->ovl_cap;
      ip.spill_cell = P->may_spill ? W.spill_cell.as<uint32_t>() : nullptr;
      ip.spill_val = P->may_spill ? W.spill_val.as<int32_t>() : nullptr;
      ip.spill_n = P->may_spill ? W.spill_n.as<uint32_t>() : nullptr;
      ip.spill_cap = P->may_spill ? W.spill_cap : 0;
      ip.may_spill = P->may_spill;
      ip.stage_warp = stage_warp;
      ip.node_min = node_min;
      ip.node_max = node_max;
      ip.stage = W.log_alt.as<uint64_t>();
      ip.stage_cap = log_cap;
      ip.wmap = W.wmap.as<uint8_t>();
      ip.wtag = W.wtag;
      ip.wval = W.wval.as<int32_t>();
      ip.reports = W.reports.as<rc_report>();
      ip.report_cap = rep_cap;
      ip.ctr = dctr;
      ip.alt_heap = nullptr;
      ip.alt_mask = nullptr;
      ip.entry_ro = W.entry_ro.as<uint32_t>();
      ip.inst_div = inst_flag;
      // (inter-group races need every read logged: no static elision with groups)
      ip.ro_skip = (opt.flags & RC_OPT_KEEP_ALL_READS) == 0 && G == 1;
      return ip;
    };
    // K1c's parameter block for the interval interpreter's parameters
    auto make_kp = [&](const InterpParams& ip, uint32_t kk) {
      K1cParams kp;
      kp.status_in = ip.status_in;
      kp.pc_in = ip.pc_in;
      kp.regs_in = ip.regs_in;
      kp.status_out = ip.status_out;
      kp.pc_out = ip.pc_out;
      kp.regs_out = ip.regs_out;
      kp.heap = ip.heap;
      kp.heap_w = ip.heap_w;
      kp.stage = reinterpret_cast<unsigned long long*>(ip.stage);
      kp.wval = ip.wval;
      kp.wmap = ip.wmap;
      kp.node_min = ip.node_min;
      kp.node_max = ip.node_max;
      kp.inst_div = ip.inst_div;
      kp.reports = ip.reports;
      kp.report_count = &dctr->report_count;
      kp.stage_count = &dctr->stage_count;
      kp.staged_recs = &dctr->staged_recs;
      kp.iv_loads = &dctr->iv_loads;
      kp.iv_stores = &dctr->iv_stores;
      kp.iv_instr = &dctr->iv_instr;
      kp.log_overflow = &dctr->log_overflow;
      kp.any_waiting = &dctr->any_waiting;
      kp.jit_bail = &dctr->jit_bail;
      kp.abort = &dctr->abort;
      kp.report_cap = ip.report_cap;
      kp.fuel = ip.fuel;
      kp.stage_cap = ip.stage_cap;
      kp.n_lanes = L;
      kp.lane_pad = reg_stride;
      kp.reg_stride = reg_stride;
      kp.interval = kk;
      kp.inst_base = inst_base;
      kp.planes = (uint32_t)jit_planes;
      kp.wtag = W.wtag;
      kp.check_div = ip.ro_skip && kk > 0;
      kp.bucket_out = reinterpret_cast<unsigned long long*>(W.log.as<uint64_t>());
      kp.bcur = W.sort.hist;
      kp.bucket_overflow = &dctr->bucket_overflow;
      kp.region = BUCKET_REGION;
      kp.bucket_val = W.bval.as<int32_t>();
      kp.kept_count = &dctr->kept_count;
      kp.k1c_done = &dctr->k1c_done;
      kp.k1_reports = &dctr->k1_reports;
      kp.snapshot = 0;
      kp.fresh = 0;
      kp.kept_writes = &dctr->kept_writes;
      return kp;
    };
    auto enqueue_interval = [&](uint32_t kk, int cc, Marks* mk) -> cudaError_t {
      NvtxRange nvtx_iv(jit_on && !jit_off ? "rc interval (K1c)" : "rc interval (K1)");
      cudaError_t e;
#define EQ(x) do { e = (x); if (e != cudaSuccess) return e; } while (0)
      if (gaps) { gap_ev.push_back({}); gap_b.push_back(bi); cudaEventCreate(&gap_ev.back()[0]); cudaEventCreate(&gap_ev.back()[1]); cudaEventRecord(gap_ev.back()[0], s); }
      if (opt.profile) W.prof.on = (prof_intervals++ % prof_every) == 0;  // sampled interval profile
      // write-set map: a fresh tag per interval attempt; zeroed only when the tags wrap
      if (++W.wtag == 0 || W.wtag == 1) {
        W.wtag = 1;
        if (cpi) EQ(cudaMemsetAsync(W.wmap.p, 0, W.wmap.bytes, s));
      }
      // histograms, sort tile counters and the per-attempt counters
      EQ(cudaMemsetAsync(W.ctr_block.p, 0, CTR_OFF + offsetof(DevCounters, report_count), s));
      // RW classification: the interval-start heap, kept until the host has
      // seen this interval (two slots: the speculative next interval's copy
      // must not overwrite it)
      if (classify && cpi)
        EQ(cudaMemcpyAsync(W.heap_snap[kk & 1].p, heap_cur, (size_t)nb * cpi * 4, cudaMemcpyDeviceToDevice, s));
      InterpParams ip = make_ip(kk, cc);
      mk->m0 = W.prof.marks.size();
      W.prof.cut();
      W.prof.begin(s);
      if (jit_on && !jit_off) {
        K1cParams kp = make_kp(ip, kk);
        // no scatter will run (writes in the buckets, no read record possible):
        // K1c's last block snapshots the report count after K1 itself
        kp.snapshot = jit_wbucket && jit_planes == 0 && !direct && !getenv("RC_JIT_NOSNAP");
        kp.fresh = fresh_pending && kk == 0;
        jit_fix_pending = true;
        EQ(jit_launch(jk, kp, s));
      } else {
        if (fresh_pending && kk == 0) EQ(materialize_fresh(cc));  // K1 reads the initial state
        if (jit_fix_pending) {  // K1 reads every live register row: write K1c's rematerialised ones
          K1cParams kp = make_kp(ip, kk);
          kp.regs_out = const_cast<int32_t*>(ip.regs_in);
          EQ(jit_fix(jk, kp, s));
          jit_fix_pending = false;
        }
        EQ(launch_interp(ip, s));
      }
      const bool wb = jit_on && !jit_off && jit_wbucket;
      jit_used_wb[kk & 1] = wb;
      jit_used_iv[kk & 1] = jit_on && !jit_off;
      if (jit_on && !jit_off) jit_ran = true;
      W.prof.end(RC_PROF_INTERP, s, 0, L);
      // inter-group races: this group's smallest reader / writer per cell
      // (from the staging buffer, before the sort reuses it)
      if (G > 1)
        EQ(launch_ig_accumulate(W.log_alt.as<uint64_t>(), dctr, log_cap, W.ig.as<uint32_t>(), bcells, n,
                                (uint32_t)cpi, gi * n, s));
      // ---- write-set filter: writes + reads of written cells, dense, with histograms
      // ---- write-set filter + K3: group the kept records by cell
      // (K1c with its writes in the buckets and no read record possible: nothing to scatter)
      if (!direct && !(wb && jit_planes == 0))
        EQ(enqueue_sort(W.prof.on ? &W.prof : nullptr, (opt.flags & RC_OPT_KEEP_ALL_READS) != 0, region));
      else if (wb) {
        sr = W.log.as<uint64_t>();  // the bucket regions K1c filled (its last block took the report snapshot)
        if (getenv("RC_JIT_NOSNAP"))
          EQ(cudaMemcpyAsync(&dctr->k1_reports, &dctr->report_count, 8, cudaMemcpyDeviceToDevice, s));
      }
      // ---- K4+K5 detect + commit, A4 check + verdict
      DetectParams dp = detect_params(kk);
      dp.with_boundary = true;  // A4 as detect's tail: consumes (and resets) K1's per-instance node ranges
      if (wb) dp.bval = W.bval.as<int32_t>();  // every write record's value is beside it
      if (direct) {  // nothing was logged: the kernel runs only its A4 tail (one block)
        dp.nb = 0;
        dp.n_records = 0;
      }
      W.prof.begin(s);
      EQ(launch_detect(dp, s));
      W.prof.end(RC_PROF_DETECT, s, 0, 0);
      mk->m1 = W.prof.marks.size();
      EQ(cudaMemcpyAsync(&W.h_ctr[kk & 1], dctr, sizeof(DevCounters), cudaMemcpyDeviceToHost, s));
      EQ(cudaEventRecord(W.iv_done[kk & 1], s));
      if (gaps) cudaEventRecord(gap_ev.back()[1], s);
      if (opt.profile) W.prof.on = true;  // batch-level marks (copies, finalize) are always recorded
#undef EQ
      return cudaSuccess;
    };
    auto clear_abort = [&]() { return cudaMemsetAsync(&dctr->abort, 0, sizeof(unsigned int), s); };

    // RW value classification of interval kk (DESIGN.md §3 reading L19): the
    // interval is re-run from its start state (lane state `cur`, heap snapshot)
    // with reads of its RW cells seeing the committed heap; the re-run commits
    // onto a copy of the snapshot, the two heaps are compared and the RW
    // reports in [r0, r1) get flag bit 4 or 5.  Nothing of the re-run survives
    // but the flags (its lane state goes to scratch rows, its reports are not
    // written, the report count and K1's node ranges are restored).  The host
    // reaches this with the speculative next interval aborted (the verdict
    // asks for it), so the interval's input lane state is intact.
    auto classify_interval = [&](uint32_t kk, uint64_t r0, uint64_t r1) -> cudaError_t {
      cudaError_t e;
#define EQ(x) do { e = (x); if (e != cudaSuccess) return e; } while (0)
      const size_t cells = (size_t)nb * cpi;
      EQ(cudaMemsetAsync(W.amap.p, 0, cells, s));
      EQ(launch_rw_mark(W.reports.as<rc_report>(), r0, r1, inst_base, (uint32_t)cpi, W.arr_off.as<uint32_t>(),
                        W.amap.as<uint8_t>(), s));
      for (int attempt = 0;; attempt++) {
        EQ(cudaMemcpyAsync(W.heapB.p, W.heap_snap[kk & 1].p, cells * 4, cudaMemcpyDeviceToDevice, s));
        if (++W.wtag == 0 || W.wtag == 1) {
          W.wtag = 1;
          EQ(cudaMemsetAsync(W.wmap.p, 0, W.wmap.bytes, s));
        }
        EQ(cudaMemsetAsync(W.ctr_block.p, 0, CTR_OFF + offsetof(DevCounters, report_count), s));
        InterpParams ip = make_ip(kk, cur);
        if (fresh_pending && kk == 0) EQ(materialize_fresh(cur));
        if (jit_on) {  // the interval's input lane state may be K1c's (rematerialised registers)
          K1cParams kp = make_kp(ip, kk);
          kp.regs_out = const_cast<int32_t*>(ip.regs_in);
          EQ(jit_fix(jk, kp, s));
        }
        ip.heap = W.heap_snap[kk & 1].as<int32_t>();  // interval-start heap
        ip.alt_heap = heap_cur;                       // committed heap (writers first)
        ip.alt_mask = W.amap.as<uint8_t>();
        ip.regs_out = W.regs_b.as<int32_t>();
        ip.pc_out = W.pc_b.as<uint32_t>();
        ip.status_out = W.status_b.as<uint8_t>();
        ip.report_cap = 0;  // error reports of the re-run are not written (the count is restored below)
        EQ(launch_interp(ip, s));
        EQ(enqueue_sort(nullptr, false, false));  // (the classified interval's own sorted log is not needed again)
        DetectParams dp = detect_params(kk);
        dp.region = 0;  // (count mode: a re-run never overflows a region)
        dp.heap = W.heapB.as<int32_t>();
        dp.quiet = true;
        dp.report_cap = ~0ull;  // (quiet: nothing is written; K1's uncounted reports never skip the commit)
        EQ(launch_detect(dp, s));
        EQ(read_ctr());
        if ((!W.h_ctr[2].log_overflow && !W.h_ctr[2].ovl_overflow) || attempt >= 16) break;
        if (W.h_ctr[2].ovl_overflow) {  // a spill list was full: grow it and re-run
          if (grow_spill() != RC_OK) return cudaErrorMemoryAllocation;
          continue;
        }
        const uint64_t n_all = W.h_ctr[2].stage_count;  // grow the log and re-run (as for an interval)
        const uint64_t want = std::min<uint64_t>(n_all + n_all / 4 + 1024, 0xFFFFFFFFull);
        EQ(W.log.ensure(want * 8));
        EQ(W.log_alt.ensure(want * 8));
        log_cap = std::min(W.log.bytes, W.log_alt.bytes) / 8;
        EQ(ensure_sort_status(log_cap));
      }
      if (W.h_ctr[2].log_overflow || W.h_ctr[2].ovl_overflow) return cudaErrorMemoryAllocation;
      EQ(cudaMemsetAsync(W.cmp_inst.p, 0, (size_t)nb * 4, s));
      EQ(launch_heap_compare(W.heapB.as<int32_t>(), heap_cur, cells, (uint32_t)cpi,
                             W.cmp_inst.as<uint32_t>(), s));
      EQ(launch_rw_flag(W.reports.as<rc_report>(), r0, r1, inst_base, W.cmp_inst.as<uint32_t>(), s));
      EQ(set_report_count(r1));
      EQ(cudaMemsetAsync(node_min, 0x7F, (size_t)nb * 4, s));
      EQ(cudaMemsetAsync(node_max, 0x80, (size_t)nb * 4, s));
#undef EQ
      return cudaSuccess;
    };

    // Speculative pipeline: interval k+1 is queued before the host looks at
    // interval k, so the GPU never waits for the host between intervals.  If
    // k needs the host (overflow, divergence, or no lane left waiting), its
    // verdict makes every kernel of k+1 return at entry; the host then acts
    // and queues k+1 again.
    for (gi = 0; gi < G; gi++) {  // work-groups one after another (reading L20)
    cur = 0;
    // K1c starts a batch from the initial state without reading it (every
    // lane RUNNING at pc 0, registers 0): the rows are written only if
    // something else reads them first (K1 after a hand-back, the
    // classification re-run) — materialize_fresh()
    fresh_pending = L && jit_on && !jit_off && !getenv("RC_JIT_NOFRESH");
    if (L && !fresh_pending) CK(materialize_fresh(cur));
    CK(cudaMemsetAsync(node_min, 0x7F, (size_t)nb * 4, s));  // large positive: "no arrival"
    CK(cudaMemsetAsync(node_max, 0x80, (size_t)nb * 4, s));  // large negative
    uint32_t k = 0;
    Marks mk_cur, mk_next;
    CK(enqueue_interval(k, cur, &mk_cur));
    for (;;) {
      const uint64_t rep_before = rep_count;
      const bool spec = (uint64_t)k + 1 < opt.max_intervals;
      if (spec) CK(enqueue_interval(k + 1, cur ^ 1, &mk_next));
      CK(cudaEventSynchronize(W.iv_done[k & 1]));
      const DevCounters h = W.h_ctr[k & 1];  // interval k's counters
      const bool next_aborted = h.abort != 0;
      if (spec && next_aborted) W.prof.marks.resize(mk_next.m0);  // k+1 did nothing
      const uint64_t n_all = h.stage_count;  // staging slots reserved (records + padding)
      const bool log_over = h.log_overflow != 0;  // a real record did not fit
      const bool k1_rep_over = h.k1_reports > rep_cap;
      const bool spill_over = h.ovl_overflow != 0;  // a work-item's spill list was full
      // a bucket outgrew its region while K1c wrote records straight into the
      // regions: the staging buffer does not hold them, so the interval is
      // re-run with K1 in count mode (K1 for the rest of the run)
      const bool jit_bucket_over = h.bucket_overflow && jit_used_wb[k & 1];
      if (log_over || k1_rep_over || spill_over || jit_bucket_over) {  // filter/detect skipped: grow and re-run
        if (h.jit_bail) jit_off = true;  // a K1c work-item had more records than its planes: K1 from here
        if (jit_bucket_over) {  // count mode from here; K1c places its write records in the planes again
          W.region_ok = false;
          region = false;
          if (!jit_off) CK(select_jit(false));
        }
        if (spill_over) {
          const int e = grow_spill();
          if (e != RC_OK) return e;
        }
        if (log_over && !h.jit_bail) {
          const uint64_t want = std::min<uint64_t>(n_all + n_all / 4 + 1024, 0xFFFFFFFFull);
          if (n_all > 0xFFFFFFFFull) return fail(RC_ELIMIT, "more than 2^32 access records in one interval");
          CK(W.log.ensure(want * 8));
          CK(W.log_alt.ensure(want * 8));
          log_cap = std::min(W.log.bytes, W.log_alt.bytes) / 8;
          CK(ensure_sort_status(log_cap));
        }
        if (k1_rep_over) CK(grow_reports(h.k1_reports));
        CK(set_report_count(rep_before));
        CK(clear_abort());
        W.prof.marks.resize(mk_cur.m0);
        CK(enqueue_interval(k, cur, &mk_cur));
        continue;
      }
      if (next_aborted) CK(clear_abort());  // k+1 (if queued) has drained as a no-op before this
      uint64_t rc_fix = UINT64_MAX;  // report count after a regrouping
      if (h.bucket_overflow) {
        // region mode: a bucket outgrew its region (detect skipped, K1's work
        // stands): regroup this interval from the staging buffer with the
        // bucket counts, and keep the count mode for this shape
        // (the speculative next interval's scratch reset has run: restore this
        // interval's staged-slot count; its write-set tag may be gone — the
        // map is re-tagged or wiped per attempt — so every read record is
        // kept, which changes no report and no commit)
        W.region_ok = false;
        region = false;
        W.h_ctr[3].stage_count = h.stage_count;
        CK(cudaMemcpyAsync(&dctr->stage_count, &W.h_ctr[3].stage_count, 8, cudaMemcpyHostToDevice, s));
        CK(cudaMemsetAsync(W.sort.hist, 0, NB_MAX * sizeof(uint32_t), s));
        CK(cudaMemsetAsync(&dctr->count_done, 0, sizeof(unsigned int), s));
        CK(cudaMemsetAsync(&dctr->bucket_overflow, 0, sizeof(unsigned int), s));
        CK(enqueue_sort(nullptr, /*keep_all=*/true, false));
        DetectParams dp = detect_params(k);
        CK(launch_detect(dp, s));
        CK(read_ctr());
        rc_fix = W.h_ctr[2].report_count;
      }
      tot_loads += h.iv_loads;
      tot_stores += h.iv_stores;
      tot_instr += h.iv_instr;
      const uint64_t Ns = h.kept_count, Nslots = h.stage_count;
      uint64_t rc = rc_fix != UINT64_MAX ? rc_fix : h.report_count;
      // detect reports overflowed: grow, re-run detect (idempotent commits).  A
      // speculative interval's counter reset may have run: restore the count.
      if (rc > rep_cap) {
        W.h_ctr[3].kept_count = Ns;
        CK(cudaMemcpyAsync(&dctr->kept_count, &W.h_ctr[3].kept_count, 8, cudaMemcpyHostToDevice, s));
        do {
          CK(grow_reports(rc));
          CK(set_report_count(h.k1_reports));
          DetectParams dp = detect_params(k);
          dp.region_rerun = dp.region != 0;  // (the region cursors were reset by the next interval's scratch)
          if (jit_used_wb[k & 1]) dp.bval = W.bval.as<int32_t>();
          CK(launch_detect(dp, s));
          CK(read_ctr());
          rc = W.h_ctr[2].report_count;
        } while (rc > rep_cap);
      }
      if (h.diverged) {  // rare path: lane scans for the divergence report (idempotent)
        const uint64_t before = rc;
        for (;;) {
          BoundaryParams bp = bparams(k);
          bp.status = W.status[cur ^ 1].as<uint8_t>();
          bp.pc = W.pc[cur ^ 1].as<uint32_t>();
          CK(launch_divergence(bp, s));
          CK(read_ctr());
          rc = W.h_ctr[2].report_count;
          if (rc <= rep_cap) break;
          CK(grow_reports(rc));
          CK(set_report_count(before));
        }
      }
      rep_count = rc;
      if (classify && h.rw_reports > 0 && cpi) CK(classify_interval(k, rep_before, rc));
      if (W.prof.on) {  // exact record counts are known now: fix this interval's profile bytes
        for (size_t i = mk_cur.m0; i < mk_cur.m1; i++) {
          Profiler::Mark& m = W.prof.marks[i];
          // the sort: LSD 16 B per record and pass; the bucket scatter reads
          // every staging slot and writes every kept record
          if (m.cls == RC_PROF_SORT) { m.bytes = bucket ? Nslots * 8 + Ns * 8 : Ns * 16; m.items = Ns; }
          // detect: every record read, a value gathered and a cell committed per write record
          if (m.cls == RC_PROF_DETECT) { m.bytes = Ns * 8 + h.kept_writes * 8; m.items = Ns; }
          if (m.cls == RC_PROF_HIST && bucket) { m.bytes = Nslots * 8; m.items = Nslots; }  // bucket counts
          if (m.cls == RC_PROF_FILTER) { m.bytes = Nslots * 8 + h.staged_recs + Ns * 8; m.items = Nslots; }
          // K1c: status + pc in and out, the carried
          // registers in and out, 4 B per performed load, 8 B per logged
          // read, 8 B record + 4 B final value per write record
          if (m.cls == RC_PROF_INTERP && jit_used_iv[k & 1]) {
            const uint64_t wrec = jit_wbucket ? h.kept_writes : h.iv_stores;
            m.bytes = (uint64_t)L * (10 + 8 * (uint64_t)jk.carried) + 4 * h.iv_loads + 8 * h.staged_recs + 12 * wrec;
          }
        }
      }
      cur ^= 1;  // the interval's lane state becomes current
      if (!h.any_waiting) break;
      k++;
      if (k >= opt.max_intervals) {  // instance-level FUEL (reading L17); nothing was speculated
        for (;;) {
          BoundaryParams bp = bparams(k);
          bp.status = W.status[cur].as<uint8_t>();
          bp.pc = W.pc[cur].as<uint32_t>();
          CK(launch_max_intervals(bp, s));
          CK(read_ctr());
          if (W.h_ctr[2].report_count <= rep_cap) break;
          CK(grow_reports(W.h_ctr[2].report_count));
          CK(set_report_count(rep_count));
        }
        rep_count = W.h_ctr[2].report_count;
        k--;  // intervals executed = max_intervals
        break;
      }
      if (next_aborted) {
        W.prof.marks.resize(std::min(W.prof.marks.size(), mk_next.m0));
        CK(enqueue_interval(k, cur, &mk_cur));  // the speculative copy did nothing: queue it for real
      } else {
        mk_cur = mk_next;
      }
    }
    intervals_max = std::max<uint64_t>(intervals_max, (uint64_t)k + 1);
    CK(launch_lane_hist(W.status[cur].as<uint8_t>(), L, dctr, s));
    if (G > 1) CK(launch_ig_combine(W.ig.as<uint32_t>(), heap_cur, bcells, s));
    }  // work-group passes
    if (G > 1) {  // inter-group reports of the batch's instances
      for (;;) {
        CK(launch_ig_emit(W.ig.as<uint32_t>(), bcells, (uint32_t)cpi, W.arr_off.as<uint32_t>(), n_arrays, inst_base,
                          W.reports.as<rc_report>(), rep_cap, dctr, s));
        CK(read_ctr());
        if (W.h_ctr[2].report_count <= rep_cap) break;
        CK(grow_reports(W.h_ctr[2].report_count));
        CK(set_report_count(rep_count));
      }
      rep_count = W.h_ctr[2].report_count;
    }
    // final heaps out
    if (final_heaps) {
      W.prof.cut();
      W.prof.begin(s);
      for (uint32_t a = 0; a < n_arrays; a++) {
        if (!size[a]) continue;
        CK(cudaMemcpy2DAsync(final_heaps[a] + (uint64_t)b0 * size[a], (size_t)size[a] * 4,
                             heap_cur + off[a], cpi * 4, (size_t)size[a] * 4, nb,
                             host_io ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
      }
      W.prof.end(RC_PROF_COPY, s, (uint64_t)nb * cpi * 4, (uint64_t)nb * cpi);
    }
    CK(cudaEventRecord(W.ev_free[bi & 1], s));  // this batch's working heap may be refilled
    free_recorded[bi & 1] = true;
  }

  if (gaps) {
    cudaEventRecord(g1, s);
    cudaEventSynchronize(g1);
    float tot = 0, iv = 0, gap_in = 0, gap_x = 0;
    cudaEventElapsedTime(&tot, g0, g1);
    for (size_t i = 0; i < gap_ev.size(); i++) {
      float x = 0;
      cudaEventElapsedTime(&x, gap_ev[i][0], gap_ev[i][1]);
      iv += x;
      if (i + 1 < gap_ev.size()) {
        float y = 0;
        cudaEventElapsedTime(&y, gap_ev[i][1], gap_ev[i + 1][0]);
        (gap_b[i + 1] == gap_b[i] ? gap_in : gap_x) += y;
      }
      cudaEventDestroy(gap_ev[i][0]);
      cudaEventDestroy(gap_ev[i][1]);
    }
    fprintf(stderr, "RC_GAPS run %.2f ms, %zu interval enqueues %.2f ms, between them %.2f ms in batches + %.2f ms across batches\n",
            tot, gap_ev.size(), iv, gap_in, gap_x);
  }
#ifdef INTERP_PHASE_TIMING
  if (getenv("RC_PHASES")) {
    unsigned long long ph[8];
    cudaStreamSynchronize(s);
    interp_phase_io(ph, false);
    const char* nm[8] = {"prefetch-issue", "lane-state wait", "interpret", "pending+writes", "A4+counts+sync",
                         "reserve+state", "write-out", "end sync"};
    double tot = 0;
    for (int i = 0; i < 8; i++) tot += (double)ph[i];
    for (int i = 0; i < 8; i++) fprintf(stderr, "K1 phase %-16s %6.1f%%\n", nm[i], 100.0 * ph[i] / (tot > 0 ? tot : 1));
    interp_phase_io(nullptr, true);
  }
#endif
  // K6: canonical order, then the first min(capacity, total) to the host
  if (rep_count > 1) {
    CK(W.reports_scratch.ensure(std::max<uint64_t>(rep_count, 2048) * 2 * sizeof(rc_report)));
    W.prof.cut();
    W.prof.begin(s);
    CK(finalize_reports(W.reports.as<rc_report>(), rep_count, W.reports_scratch.as<rc_report>(), s));
    W.prof.end(RC_PROF_FINALIZE, s, rep_count * 64, rep_count);
  }
  const uint64_t ncopy = std::min<uint64_t>(capacity, rep_count);
  if (ncopy) CK(cudaMemcpyAsync(out, W.reports.p, ncopy * sizeof(rc_report), cudaMemcpyDeviceToHost, s));
  CK(read_ctr());  // also waits for the report copy and lanes_final
  if (W.prof.on) {
    cudaEventRecord(t_end, s);
    cudaEventSynchronize(t_end);
    W.prof.collect(opt.profile);
    float ms = 0;
    cudaEventElapsedTime(&ms, t_begin, t_end);
    opt.profile->total_ms = ms;
    opt.profile->kernel_launches = g_launches.load() - launches0;
    opt.profile->sample_every = prof_every;
    opt.profile->flags = jit_ran ? 1u : 0u;
    cudaEventDestroy(t_begin);
    cudaEventDestroy(t_end);
  }
  if (stats) {
    stats->loads = tot_loads;
    stats->stores = tot_stores;
    stats->checked_accesses = tot_loads + tot_stores;
    stats->instructions = tot_instr;
    stats->intervals_max = intervals_max;
    for (int i = 0; i < 8; i++) stats->lanes_final[i] = W.h_ctr[2].lanes_final[i];
  }
  if (n_reports_total) *n_reports_total = rep_count;
  if (rep_count > capacity)
    return fail(RC_ETRUNC, "%llu reports, capacity %llu", (unsigned long long)rep_count,
                (unsigned long long)capacity);
  return RC_OK;
}

}  // extern "C"
