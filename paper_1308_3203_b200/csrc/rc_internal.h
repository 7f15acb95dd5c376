// rc_internal.h — shared definitions of the CUDA path (librc.so).  Not part of
// the ABI (include/rc.h is).  Nothing here is shared with oracle/.
#pragma once
#include <algorithm>
#include <cstddef>
#include <atomic>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "rc.h"

namespace rc {

// Per-device one-time setup of a launcher (kernel attribute opt-ins such as
// the large dynamic shared memory, the SM count, occupancy): attributes
// apply to one device context and rc_options.device selects any GPU, so the
// setup runs once per device, under std::call_once (values are published to
// other threads only after every one of them is computed).
constexpr int RC_MAX_DEVICES = 64;
struct DeviceSetup {
  std::once_flag once[RC_MAX_DEVICES];
  cudaError_t err[RC_MAX_DEVICES] = {};
  // f(dev) -> cudaError_t, run once for the current device; returns its device via *dev_out
  template <class F>
  cudaError_t run(F&& f, int* dev_out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= RC_MAX_DEVICES) return cudaErrorInvalidDevice;
    std::call_once(once[dev], [&] { err[dev] = f(dev); });
    *dev_out = dev;
    return err[dev];
  }
};

// count of librc kernel launches (reported in rc_profile.kernel_launches)
extern std::atomic<uint64_t> g_launches;
inline void launched(uint64_t k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

struct Ins {  // 8-byte RCB1 instruction, include/rc.h
  uint8_t op, a, b, c;
  int32_t imm;
};
static_assert(sizeof(Ins) == 8, "instruction is 8 bytes");
// device copy of the program only: the instruction may touch a register with an
// outstanding asynchronous load (program.cpp analyze() (4)); opcodes are < 0x80
constexpr uint8_t OP_WAIT = 0x80;

// work-item status (lane.status), DESIGN.md §5
enum LaneStatus : uint8_t {
  L_RUNNING = 0,
  L_WAITING = 1,  // suspended at a barrier (τ ⊡ σ)
  L_EXITED = 2,
  L_PRUNED = 3,   // assume(false): ⊤
  L_OOB = 4,      // ⊥ kinds
  L_ASSERT = 5,
  L_DIV0 = 6,
  L_FUEL = 7,
  L_EXITED_NOW = 8,  // reached EXIT in the interval just interpreted (arrived at the exit node)
};
// Arrival node of a work-item in the interval just run (reading L9): the pc of
// its BAR (= pc_out - 1 for L_WAITING), NODE_EXIT for L_EXITED_NOW.
constexpr int32_t NODE_NONE = -2;
constexpr int32_t NODE_EXIT = -1;
constexpr uint32_t NOTID = 0xFFFFFFFFu;
constexpr int OVL_CAP = 15;        // own-write overlay entries per work-item in shared memory
// A work-item's distinct written cells beyond the shared-memory overlay go to
// its HBM spill list (spill_cell / spill_val [spill_cap][n_lanes]); their
// write records carry this slot and detect finds the value in the list.  The
// capacity is not semantic: when a list is full the interval is re-run with a
// larger one (runtime.cu).
constexpr uint32_t SLOT_SPILL = 15;

// One access-log record is a single u64:
//   bits 63..32  cell id (batch-local; the sort key — only these bits are sorted)
//   bits 31..5   batch lane = inst_local * n + tid (< 2^27; within one cell —
//                one instance — lanes order like tids, and the lane indexes
//                the write-value side table without a division)
//   bits  4..1   overlay slot of a write (its final value is wval[slot][lane])
//   bit      0   1 = write, 0 = read
constexpr int REC_CELL_SHIFT = 32;
constexpr uint32_t LANE_PAD = 1024;  // lane-state rows are padded to multiples of this (K1 tiles of <= 1024 lanes)
constexpr uint32_t MAX_WG = 1u << 27;
// Division by a run-constant divisor d (work-group size, cells per instance):
// magic = ceil(2^64 / d) (0 for d == 1); x / d == umulhi64(x, magic) exactly
// for every x < 2^32 (the rounding error is x * (magic - 2^64/d) / 2^64 <
// 2^-32 <= 1/d).
inline uint64_t div_magic(uint32_t d) { return d <= 1 ? 0ull : ~0ull / d + 1; }
#ifdef __CUDACC__
__device__ __forceinline__ uint32_t fast_div(uint32_t x, uint64_t magic) {
  return magic ? (uint32_t)__umul64hi((uint64_t)x, magic) : x;
}
#endif
__host__ __device__ inline uint64_t make_rec(uint32_t cell, uint32_t lane, uint32_t slot, uint32_t w) {
  return ((uint64_t)cell << 32) | (lane << 5) | (slot << 1) | w;
}

static_assert(OVL_CAP < (int)SLOT_SPILL + 1 && SLOT_SPILL == 15, "the record's 4-bit slot: overlay slots, then the spill marker");

// Device counters of one run; zeroed per attempt where noted.
struct DevCounters {
  unsigned long long stage_count;   // staging slots reserved this interval (records + sentinels; per attempt)
  unsigned long long staged_recs;   // access records staged this interval (per attempt)
  unsigned long long kept_count;    // records the write-set filter passed to the sort
  unsigned long long iv_loads;      // per attempt
  unsigned long long iv_stores;
  unsigned long long iv_instr;
  unsigned int log_overflow;        // per attempt
  unsigned int ovl_overflow;        // per attempt: a work-item's spill list was full (re-run with a larger one)
  unsigned int any_waiting;         // per interval
  unsigned int diverged;            // per interval
  unsigned long long k1_reports;    // report_count after K1 (snapshot taken by the filter)
  unsigned long long rw_reports;    // RW reports emitted by detect (RC_OPT_CLASSIFY_RW)
  unsigned long long kept_writes;   // write records among the kept ones (profile bytes of detect)
  unsigned int count_done;          // bucket_count blocks finished (last-block pattern: the bucket starts)
  unsigned int bucket_overflow;     // region mode: a bucket got more records than its region holds
  unsigned int jit_bail;            // K1c: a work-item had more records than its planes (re-run interpreted)
  unsigned int k1c_done;            // K1c blocks finished (the last one snapshots k1_reports)
  // ---- fields above: zeroed per interval attempt (one memset, runtime.cu)
  unsigned long long report_count;  // reports appended (whole run, rolled back on retry)
  unsigned long long lanes_final[8];
  // Speculation (runtime.cu): the host queues interval k+1 before it has seen
  // interval k's counters.  A4's last warp sets `abort` when interval k needs
  // the host (overflow, divergence, nothing left waiting); every kernel of an
  // interval returns at entry while it is set, so a speculative interval
  // leaves no trace.  The host clears it.  Never zeroed per interval.
  unsigned int abort;
  unsigned int bdone;               // A4 blocks (K4 tail: warps) finished (last-one pattern; self-resetting)
};

// K1's shared-memory carve-up, computed on the host for the launch's block
// size (byte offsets from the dynamic shared-memory base; interp.cu
// k1_layout): kernel parameters live in the constant bank, so the tile loop
// addresses its buffers through constant operands instead of re-deriving them
// from blockDim and the program sizes in registers.
struct K1Layout {
  uint32_t T, TL, W;   // threads per block, lanes per tile, warps per block
  uint32_t regs;       // register files, LS_NB buffers of regs_buf bytes
  uint32_t regs_buf;   // n_regs * TL * 4
  uint32_t spc, sstat; // pc / status rows, LS_NB buffers of TL * 4 / TL bytes
  uint32_t mbar, recs, code, tail, ro, ocell, oval, soff, ssize, live, wcnt, wbase;
  uint32_t total;
};

// Parameters of the interval interpreter (K1), passed by value.
struct InterpParams {
  K1Layout lay;               // (filled by launch_interp)
  const Ins* code;
  uint32_t n_instr, n_regs, n_arrays;
  uint32_t n;                 // work-group size
  uint32_t gid, gbase;        // work-group of this pass and its first global tid (gid * n; reading L20)
  uint64_t n_magic;           // div_magic(n)
  uint32_t n_lanes;           // I_b * n
  uint32_t cpi;               // cells per instance
  uint64_t fuel;
  bool fuel_check;            // false: no work-item can exhaust its fuel (static bound <= fuel)
  uint32_t interval;
  uint32_t inst_base;         // global instance id of batch instance 0
  const uint32_t* arr_off;    // [n_arrays] cell offset of each array inside an instance
  const uint32_t* arr_size;   // [n_arrays]
  const int32_t* heap;        // interval-start shared heap [I_b][cpi]
  int32_t* heap_w;            // the same heap, written only in direct mode
  bool direct;                // RC_OPT_PREPASS proved the run conflict-free: commit writes at the end of each
                              // work-item's interval, log nothing (no grouping / detect kernels run)
  // lane state in / out (SoA)
  uint32_t reg_stride;        // row stride of the register arrays (>= n_lanes, multiple of 256)
  const int32_t* regs_in;     // [n_regs][reg_stride]; status / pc rows are padded to reg_stride too
  const uint32_t* pc_in;
  const uint8_t* status_in;
  int32_t* regs_out;
  uint32_t* pc_out;
  uint8_t* status_out;
  const uint8_t* live;        // registers saved / restored across barriers
  uint32_t n_live;
  uint32_t ovl_cap;           // own-write overlay entries per work-item in smem (static bound, <= OVL_CAP)
  uint32_t* spill_cell;       // [spill_cap][n_lanes] cells written beyond the smem overlay (null: none possible)
  int32_t* spill_val;         // [spill_cap][n_lanes] their values
  uint32_t* spill_n;          // [n_lanes] spill entries of a lane (written when > 0)
  uint32_t spill_cap;
  bool may_spill;             // the program may write more cells than the smem overlay holds (SPILL kernels)
  uint32_t stage_warp;        // records staged per warp in shared memory
  int32_t* node_min;          // [I_b] min / max arrival node (fused A4)
  int32_t* node_max;
  // log: records are staged in per-block chunks of one staging buffer
  // (unused chunk tails hold the sentinel ~0); the write-set filter compacts
  // it into the sort buffer
  uint64_t* stage;            // [stage_cap] records (make_rec) and sentinels
  unsigned long long stage_cap;
  // static write-set elision (program.cpp analyze() (5)): a lane of an
  // instance whose running lanes all start the interval at one entry does not
  // log reads of the arrays entry_ro[entry] marks
  const uint32_t* entry_ro;   // [n_instr]
  const uint32_t* inst_div;   // [I_b] the instance's previous interval diverged (A4)
  bool ro_skip;               // off with RC_OPT_KEEP_ALL_READS
  // RW classification re-run (null in a canonical run): a read of cell c with
  // alt_mask[c] set (and no own earlier write) returns alt_heap[c]
  const int32_t* alt_heap;
  const uint8_t* alt_mask;
  uint8_t* wmap;              // [I_b * cpi] == wtag: cell written in this interval
  uint8_t wtag;               // this interval's tag (1..255; the map is zeroed when tags wrap)
  int32_t* wval;              // [ovl_cap][n_lanes] final value of each written smem overlay slot
  rc_report* reports;
  unsigned long long report_cap;
  DevCounters* ctr;
};

// K1c (jit.cpp): the interval interpreter specialised to one program and run
// shape — the bytecode compiled to a CUDA kernel with NVRTC at first use.
// The parameter block is declared once here and handed to NVRTC as text, so
// the host and the generated kernel share one layout.
#define RC_K1C_PARAMS_DECL                                                                                \
  struct K1cParams {                                                                                      \
    const unsigned char* status_in; const unsigned int* pc_in; const int* regs_in;                        \
    unsigned char* status_out; unsigned int* pc_out; int* regs_out;                                       \
    const int* heap; int* heap_w; unsigned long long* stage; int* wval; unsigned char* wmap;             \
    int* node_min; int* node_max; const unsigned int* inst_div; void* reports;                            \
    unsigned long long* report_count; unsigned long long* stage_count; unsigned long long* staged_recs;   \
    unsigned long long* iv_loads; unsigned long long* iv_stores; unsigned long long* iv_instr;            \
    unsigned int* log_overflow; unsigned int* any_waiting; unsigned int* jit_bail; const unsigned int* abort; \
    unsigned long long report_cap; unsigned long long fuel; unsigned long long stage_cap;                 \
    unsigned long long* bucket_out; unsigned int* bcur; unsigned int* bucket_overflow; unsigned int region; \
    unsigned long long* kept_count; unsigned long long* kept_writes; int* bucket_val;                     \
    unsigned int* k1c_done; unsigned long long* k1_reports; unsigned int snapshot, fresh;                 \
    unsigned int n_lanes, lane_pad, reg_stride, interval, inst_base, planes, wtag, check_div;              \
  };
RC_K1C_PARAMS_DECL
#define RC_STR2_(...) #__VA_ARGS__
#define RC_STR_(x) RC_STR2_(x)

// What a K1c kernel is specialised to (besides the program): the cache key.
struct JitShape {
  uint32_t n = 0, gid = 0, cpi = 0;
  std::vector<uint32_t> off, size;  // per array
  bool direct = false;   // RC_OPT_PREPASS direct-commit mode (no log)
  bool fuel = false;     // per-instruction fuel check
  bool ro_skip = false;  // static write-set elision (off with RC_OPT_KEEP_ALL_READS / work-groups)
  bool wbucket = false;  // bucket region mode: write records go straight into their bucket regions
  bool narrow = false;   // per-thread statistics fit 32 bits (steps per work-item-interval < 2^20)
};
struct JitKernel {
  void* fn = nullptr;   // CUfunction
  void* fix = nullptr;  // CUfunction rc_k1c_fix (registers K1c rematerialises, written out for K1)
  int grid = 0;         // persistent grid (resident blocks per SM x SMs)
  int carried = 0;      // registers carried through HBM across barriers (the rest rematerialised)
};
// The program's K1c kernel for this shape on the current device: compiled and
// loaded on first use, cached on the program.  false (with a reason in *why)
// when the program is not eligible or NVRTC / the driver is unavailable; the
// caller then runs the interpreter.
bool jit_get(rc_program* P, const JitShape& S, JitKernel* out, std::string* why);
cudaError_t jit_launch(const JitKernel& k, const K1cParams& p, cudaStream_t s);
// K1c carries only the registers that are not an affine function of the
// local id at the entry; before K1 runs on K1c-produced lane state (a K1c
// interval handed back, the RW-classification re-run) this writes the others
// into the rows p.regs_out of the lanes p.status_in / p.pc_in describe
cudaError_t jit_fix(const JitKernel& k, const K1cParams& p, cudaStream_t s);
void jit_release(rc_program* P);  // unload the cached modules (on their devices)
// the K1c source for a program and shape (tests / RC_JIT_DUMP)
std::string jit_source(const rc_program* P, const JitShape& S, int* carried = nullptr);

struct DetectParams {
  const uint64_t* recs;       // sorted by cell; count = ctr->kept_count
  int32_t* wval;              // [ovl_cap][n_lanes] (written by the bucket kernels for multi-record cells when bval)
  const uint32_t* spill_cell; // slot SLOT_SPILL: the lane's spill list (K1)
  const int32_t* spill_val;
  const uint32_t* spill_n;
  uint32_t n_lanes, n;        // lane = inst_local * n + tid
  uint32_t gbase;             // global tid of local id 0 (work-group pass, reading L20)
  uint32_t n_records;         // host upper bound (grid size)
  int32_t* heap;
  uint32_t cpi, n_arrays;
  uint64_t cpi_magic;         // div_magic(cpi)
  const uint32_t* arr_off;
  uint32_t interval, inst_base;
  rc_report* reports;
  unsigned long long report_cap;
  DevCounters* ctr;
  // fused A4 tail (detect.cu boundary_tail); off for a detect-only re-run
  bool with_boundary;
  bool classify;              // the verdict also asks the host for RW classification
  bool quiet;                 // commit only (classification re-run): no reports
  uint32_t n_inst;
  int32_t* node_min;          // [n_inst] from K1, reset by the tail
  int32_t* node_max;
  uint32_t* inst_flag;        // [n_inst] diverged
  // bucket path (nb > 0): recs = the bucketed records; bucket b holds
  // recs[bstart[b], bend[b]) (bend = the scatter's cursors when it is done;
  // unlike the counts, which the speculative next interval's scratch reset
  // clears, they survive until the next scatter, so a detect-only re-run
  // still finds its buckets); tmp = scratch of the same size (a bucket too
  // large for shared memory is sorted there)
  uint32_t nb;
  const uint32_t* bstart;
  const uint32_t* bend;
  uint64_t* tmp;
  // region mode (ScatterParams::region): bucket b = recs[b * region, + min(rcur[b], region));
  // the kernel records that end in rend[b]; a detect-only re-run (region_rerun) reads rend
  uint32_t region;
  const uint32_t* rcur;
  uint32_t* rend;
  bool region_rerun;
  // K1c in region mode wrote every write record's final value beside it
  // (bval[slot] for recs[slot]): the lone writers' commits read it in the
  // same pass as the records (null: gather from wval by lane)
  const int32_t* bval;
};

// ---- launchers (defined in the .cu files) --------------------------------
size_t interp_smem_bytes(const InterpParams& p, int threads, bool code_in_smem, int lanes_per_thread);
cudaError_t launch_interp(const InterpParams& p, cudaStream_t s);

// Write-set filter / compaction: from the staging buffer keep every write
// record and the read records whose cell some work-item wrote in this
// interval (the others can produce no report and no commit), drop sentinels;
// write them densely to the sort buffer with their digit histograms (K2).
struct FilterParams {
  const uint64_t* stage;
  const uint8_t* wmap;
  uint8_t wtag;           // wmap[c] == wtag: c written in this interval
  uint64_t* out;          // sort buffer, [0, kept_count)
  uint32_t* hist;         // [4][256] digit counts
  int passes;

  DevCounters* ctr;
  uint32_t n_slots;       // staging buffer capacity (slots); the kernel reads stage_count
  bool keep_all;          // RC_OPT_KEEP_ALL_READS: only drop the sentinels
};
constexpr uint64_t REC_SENTINEL = ~0ull;  // cell 0xFFFFFFFF is never a real cell
cudaError_t launch_filter(const FilterParams& p, cudaStream_t s);

// ---- bucket path: the kept records are grouped by cell with
// one MSD scatter on the high cell bits (bucket = cell >> BUCKET_BITS, 4096
// cells) into the alt buffer, then bucket_detect sorts each bucket by its low
// bits in shared memory and runs the segmented detection on it.
constexpr int BUCKET_BITS = 12;
constexpr uint32_t BUCKET_CELLS = 1u << BUCKET_BITS;
constexpr uint32_t NB_MAX = 65536;                    // buckets per batch: cells per batch <= 2^28
constexpr uint64_t BUCKET_PATH_CELLS = (uint64_t)NB_MAX * BUCKET_CELLS;
constexpr uint32_t BUCKET_REGION = 2 * BUCKET_CELLS;  // region mode: record slots a bucket owns

struct SortWorkspace {
  uint64_t* alt = nullptr;         // ping-pong buffer
  uint32_t* hist = nullptr;        // [4][256] digit histograms
  uint32_t* bin_off = nullptr;     // [4][256] exclusive offsets
  unsigned long long* status = nullptr;  // [tiles][256] decoupled look-back words
  uint32_t* tile_ctr = nullptr;    // [4] dynamic tile counters
  size_t status_tiles = 0;
  uint32_t epoch = 0;              // look-back epoch (memory cleared only when it wraps)
  int status_fmt = -1;             // word format of the last pass (0: 64-bit, 1: 32-bit)
  bool reset_tile_ctr = true;      // false: the caller zeroes tile_ctr (per-interval memset)
};
#ifndef SORT_THREADS_OPT
#define SORT_THREADS_OPT 256
#endif
constexpr int SORT_THREADS = SORT_THREADS_OPT;  // >= 256 (one thread per digit for the per-digit steps)
#ifndef SORT_ITEMS_OPT
#define SORT_ITEMS_OPT 16
#endif
constexpr int SORT_ITEMS = SORT_ITEMS_OPT;
constexpr int SORT_TILE = SORT_THREADS * SORT_ITEMS;
size_t sort_tiles(size_t n);

// Live profile: CUDA events recorded on the launch stream around each kernel
// class; read back once at the end of rc_run (no per-kernel synchronisation).
struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  struct Mark { int cls; size_t e0, e1; uint64_t bytes, items; };
  std::vector<Mark> marks;
  size_t used = 0;
  size_t open_ev = 0;
  // the last end event doubles as the next begin when nothing was launched
  // in between (halves the event records per interval)
  size_t last_end = (size_t)-1;
  uint64_t launches_at_end = 0;
  cudaStream_t end_stream = nullptr;
  cudaEvent_t ev(size_t i) { return pool[i]; }
  size_t next();
  void begin(cudaStream_t s);
  void end(int cls, cudaStream_t s, uint64_t bytes, uint64_t items);
  void reset() { marks.clear(); used = 0; last_end = (size_t)-1; }
  void cut() { last_end = (size_t)-1; }  // host sync / memsets since the last end: fresh begin
  void collect(rc_profile* out);
  ~Profiler();
};

// Sort (keys, vals) by key bits [0, bits).  *in_alt tells whether the sorted
// data ended in the alt buffers of `ws`.
// hist_ready: ws.hist already holds the digit histograms (fused into K1 and
// the filter); otherwise an upfront histogram pass (K2) computes them.
// n_ub: host-side upper bound of the record count; the exact count is
// *n_a + *n_b (device memory, may be NULL) read by the kernels.
cudaError_t onesweep_sort(uint64_t* recs, uint32_t n_ub, const unsigned long long* n_a,
                          const unsigned long long* n_b, int bits, SortWorkspace& ws, cudaStream_t s, bool* in_alt,
                          Profiler* prof, bool hist_ready);

// bucket scatter (K3 on the bucket path, fused with the write-set filter):
// from the staging buffer keep every write record and the reads of cells
// written in this interval (as the filter), drop sentinels, and place each
// kept record at out[bcur[bucket]++] (any order inside a bucket)
struct ScatterParams {
  const uint64_t* stage;
  uint32_t n_slots;       // staging capacity; the kernel reads stage_count
  const uint8_t* wmap;
  uint8_t wtag;
  bool keep_all;          // RC_OPT_KEEP_ALL_READS
  uint64_t* out;
  uint32_t* bcur;
  DevCounters* ctr;
  // region mode (region > 0): bucket b owns out[b * region, (b + 1) * region)
  // and bcur[b] starts at 0 (no count pass); records beyond a region set
  // ctr->bucket_overflow and are dropped (the host then regroups the interval
  // with the counts).  0: count mode (bcur = the starts from bucket_count).
  uint32_t region;
};
cudaError_t launch_bucket_scatter(const ScatterParams& p, cudaStream_t s, Profiler* prof);
// bucket_count: the kept records of the staging buffer per bucket into
// hist[0, nb) (zeroed by the caller); the last block to finish writes the
// exclusive starts to bstart and bcur (= ScatterParams::bcur).
cudaError_t launch_bucket_count(const ScatterParams& p, uint32_t* hist, uint32_t nb, uint32_t* bstart,
                                cudaStream_t s, Profiler* prof);
cudaError_t launch_detect(const DetectParams& p, cudaStream_t s);
// RW classification helpers (detect.cu): mark the cells of the RW reports in
// reports[r0, r1) (instance ids relative to inst_base), compare two heaps per
// instance (diff[inst] = 1), set flag bit 4 / 5 on the RW reports of [r0, r1)
cudaError_t launch_rw_mark(const rc_report* reports, uint64_t r0, uint64_t r1, uint32_t inst_base, uint32_t cpi,
                           const uint32_t* arr_off, uint8_t* mask, cudaStream_t s);
cudaError_t launch_heap_compare(const int32_t* a, const int32_t* b, uint64_t n, uint32_t cpi, uint32_t* diff,
                                cudaStream_t s);
cudaError_t launch_rw_flag(rc_report* reports, uint64_t r0, uint64_t r1, uint32_t inst_base, const uint32_t* diff,
                           cudaStream_t s);

struct BoundaryParams {
  uint32_t n, n_lanes, n_inst, interval, inst_base;
  uint32_t gbase;          // global tid of local id 0 (reading L20)
  const uint8_t* status;   // status_out of the interval just run
  const uint32_t* pc;      // pc_out of the interval just run
  int32_t* node_min;       // [n_inst] from K1
  int32_t* node_max;
  uint32_t* first_tid;     // [n_inst]
  uint32_t* second_tid;    // [n_inst]
  uint32_t* inst_flag;     // [n_inst] diverged / waiting
  rc_report* reports;
  unsigned long long report_cap;
  DevCounters* ctr;
};
// per instance: divergence check on K1's node range, reset of the range
cudaError_t launch_boundary(const BoundaryParams& p, cudaStream_t s);
// rare path: lane scans for the divergence report of flagged instances
cudaError_t launch_divergence(const BoundaryParams& p, cudaStream_t s);
cudaError_t launch_max_intervals(const BoundaryParams& p, cudaStream_t s);
cudaError_t launch_lane_hist(const uint8_t* status, uint32_t n_lanes, DevCounters* ctr, cudaStream_t s);
cudaError_t launch_init_lanes(uint8_t* status, uint32_t* pc, int32_t* regs, uint32_t n_regs,
                              uint32_t n_lanes, cudaStream_t s);
cudaError_t finalize_reports(rc_report* reports, uint64_t n, rc_report* scratch, cudaStream_t s);

// inter-group races (groups.cu, reading L20): per-cell state of IG_FIELDS u32
// planes over the batch's cells
constexpr int IG_FIELDS = 10;
cudaError_t ig_reset(uint32_t* st, uint64_t cells, cudaStream_t s);
cudaError_t launch_ig_accumulate(const uint64_t* stage, const DevCounters* ctr, uint64_t cap, uint32_t* st,
                                 uint64_t cells, uint32_t n, uint32_t cpi, uint32_t gbase, cudaStream_t s);
cudaError_t launch_ig_combine(uint32_t* st, const int32_t* heap, uint64_t cells, cudaStream_t s);
cudaError_t launch_ig_emit(const uint32_t* st, uint64_t cells, uint32_t cpi, const uint32_t* arr_off, uint32_t n_arrays,
                           uint32_t inst_base, rc_report* reports, unsigned long long cap, DevCounters* ctr,
                           cudaStream_t s);

}  // namespace rc

// opaque program object (include/rc.h)
struct rc_workspace;
namespace rc {
struct ExploreCache {  // rc_explore's device buffers: grown on demand, freed with the program
  int device = -1;
  void* p[3] = {nullptr, nullptr, nullptr};
  size_t cap[3] = {0, 0, 0};
  void release();  // explore.cu (on the current device)
};
}  // namespace rc

struct rc_program {
  uint32_t n_regs = 0, n_arrays = 0, n_instr = 0;
  std::vector<rc::Ins> code;
  // static analysis (program.cpp analyze()): sizing only, no semantic effect
  std::vector<rc::Ins> dev_code;    // code with OP_WAIT flags (uploaded for K1)
  std::vector<uint8_t> live_regs;  // registers live across a barrier (+ live at pc 0)
  std::vector<uint8_t> live_at_entry;  // live_in(pc 0): the rows zeroed at a batch start (reading L18)
  std::vector<uint32_t> entry_ro;  // [n_instr] at interval entries: arrays (< 32) the region never stores to
  int ovl_cap = rc::OVL_CAP;       // smem overlay entries (max distinct cells written per work-item per interval, capped)
  bool may_spill = true;           // a work-item may write more than OVL_CAP distinct cells in one interval
  int rec_bound = -1;              // max log records per work-item per interval (-1 unbounded)
  int rec_bound_ro = -1;           // the same with the static write-set elision (5) applied (K1c record planes)
  int read_bound = -1, read_bound_ro = -1;  // read records alone (K1c with its writes straight into the buckets)
  int64_t instr_bound = -1;        // max instructions per work-item per interval (-1 unbounded)
  std::mutex mu;
  rc_workspace* ws = nullptr;
  rc::ExploreCache xc;
  void* jit = nullptr;             // K1c kernels compiled for this program (jit.cpp)
};
