/*
 * rc.h — C ABI of the B200 race checker (librc.so).
 *
 * What it computes: the concrete SIMD operational semantics of arXiv 1308.3203
 * §4 for a kernel written in the §3 language
 * (PAPER.md:85-107), run for one work-group of `work_group_size` work-items on
 * each of `n_instances` independent input heaps, with the race rule read as in
 * DESIGN.md §3 (delayed visibility inside a barrier interval, per-cell access
 * conflicts between distinct tids, write-write conflicts classified benign /
 * non-benign).
 *
 * Everything below is plain C: no C++ or torch types cross this boundary.
 * Pointers marked "device" are CUDA device pointers on options->device;
 * pointers marked "host" are ordinary host memory.  The library never aborts
 * the process; every entry point returns an rc_status and sets a thread-local
 * message readable with rc_last_error().
 *
 * Races and runtime errors in the USER kernel are reports, never call errors.
 */
#ifndef RC_H
#define RC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RC_ABI_VERSION 1

#if defined(__GNUC__)
#define RC_API __attribute__((visibility("default")))
#else
#define RC_API
#endif

/* ---- status codes ------------------------------------------------------- */
typedef enum {
  RC_OK = 0,
  RC_EINVAL = 1, /* malformed bytecode or arguments (message says which)    */
  RC_ENOMEM = 2, /* device or host allocation failed                         */
  RC_ECUDA = 3,  /* a CUDA runtime call failed (no device, launch error ...)  */
  RC_ETRUNC = 4, /* more reports than `capacity`; the first `capacity` were
                    written, *n_reports_total holds the full count (snprintf) */
  RC_ELIMIT = 5  /* an address-space limit was hit: cells per instance exceed
                    2^32, more than 2^32 access records in one interval, or
                    more distinct cells written by one work-item in one
                    interval than 2^24 (the own-write overlay itself spills
                    to device memory: its capacity is not semantic)          */
} rc_status;

/* ---- bytecode (RCB1) ----------------------------------------------------
 * The §3 grammar lowered to three-address CFG bytecode
 * (reading L10 in DESIGN.md).  Little-endian.
 *   header (16 B): u32 magic = 'R''C''B''1' (0x31424352), u16 version = 1,
 *                  u16 flags = 0, u16 n_regs (1..256), u16 n_arrays (0..256),
 *                  u32 n_instr (1..65536)
 *   then n_instr instructions of 8 B: {u8 op, u8 a, u8 b, u8 c, i32 imm}.
 * `start` is pc 0.  Registers are the private variables
 * `Locals`, zero-initialised (reading L18).  Arrays are the
 * shared `GVar` arrays passed as `Args`; shared scalars
 * are 1-element arrays (reading L12).  Values are int32, two's complement,
 * wrapping (reading L7).  Booleans are 0/1; any non-zero value is true.     */
#define RC_MAGIC 0x31424352u
enum rc_opcode {
  RC_OP_CONST = 1,  /* r[a] := imm                          v := c   */
  RC_OP_MOV = 2,    /* r[a] := r[b]                         v := v'   */
  RC_OP_TID = 3,    /* r[a] := tid  (0-based, reading L8)   tid   */
  RC_OP_SIZE = 4,   /* r[a] := size(array b)                size(v)   */
  RC_OP_ADD = 5,    /* r[a] := r[b] op r[c]                 op(e)   */
  RC_OP_SUB = 6,
  RC_OP_MUL = 7,
  RC_OP_DIV = 8,    /* truncating; r[c]==0 -> DIV0 report, work-item halts */
  RC_OP_MOD = 9,    /* C99 remainder; r[c]==0 -> DIV0; INT_MIN%-1 == 0      */
  RC_OP_MIN = 10,
  RC_OP_MAX = 11,
  RC_OP_AND = 12,   /* bitwise */
  RC_OP_OR = 13,
  RC_OP_XOR = 14,
  RC_OP_LT = 15,    /* r[a] := r[b] <  r[c] (signed)        e<e   */
  RC_OP_EQ = 16,    /* r[a] := r[b] == r[c]                 e=e   */
  RC_OP_LAND = 17,  /* r[a] := r[b]!=0 && r[c]!=0           b∧b   */
  RC_OP_LNOT = 18,  /* r[a] := r[b]==0                      ¬b   */
  RC_OP_LD = 19,    /* r[a] := array b [r[c]]               v:=a[v] */
  RC_OP_ST = 20,    /* array a [r[b]] := r[c]               a[v]:=e */
  RC_OP_BAR = 21,   /* barrier   */
  RC_OP_ASSUME = 22,/* r[a]==0 -> work-item stops silently (⊤)   */
  RC_OP_ASSERT = 23,/* r[a]==0 -> ASSERT report, work-item halts (⊥) */
  RC_OP_BR = 24,    /* r[a]!=0 ? pc=imm : pc=b+256*c  (assume(b)/assume(¬b)
                       successor pair of the CFG)          */
  RC_OP_JMP = 25,   /* pc = imm                                              */
  RC_OP_EXIT = 26,  /* the `exit` node; implicit final barrier */
  RC_OP_ADDI = 27,  /* r[a] := r[b] + imm   (op(v, c) with a constant)      */
  /* work-groups ("both threads and work-groups have a unique
     identifier ... threads can also query the size of the work-group";
     DESIGN.md reading L20).  RC_OP_TID is the global id gid * LSIZE + lid. */
  RC_OP_GID = 28,   /* r[a] := work-group id, 0 .. n_groups-1                  */
  RC_OP_LID = 29,   /* r[a] := id inside the work-group, 0 .. LSIZE-1          */
  RC_OP_LSIZE = 30  /* r[a] := work-group size (rc_run's work_group_size)      */
};

/* ---- report kinds -------------------------------------------------------- */
enum rc_kind {
  RC_RW = 1,           /* a cell read by one tid and written by another     */
  RC_WW_BENIGN = 2,    /* >= 2 writers, all final values equal  */
  RC_WW_NONBENIGN = 3, /* >= 2 writers with different final values  */
  RC_OOB = 4,          /* index outside [0,size): ⊥; array/index set */
  RC_ASSERT = 5,       /* assert(false): ⊥; array=-1, index=pc      */
  RC_DIV0 = 6,         /* division by zero: ⊥; array=-1, index=pc           */
  RC_FUEL = 7,         /* per-interval fuel exhausted (tid1=tid, index=pc), or
                          max_intervals reached (tid1=tid2=0xFFFFFFFF,
                          index=-1, interval=max_intervals)                 */
  RC_BARRIER_DIVERGENCE = 8, /* arrived work-items at different barrier nodes
                          ("the same instruction barrier"); array=-1,
                          index = pc of tid1's BAR or -1 for exit; tid1 = min
                          arrived tid, tid2 = min arrived tid at another node */
  /* inter-group races (options->n_groups > 1, reading L20): no
     barrier orders two work-groups, so accesses of two work-items of
     different groups to one cell, anywhere in the kernel, at least one a
     write, race.  interval = RC_IG_INTERVAL, flags = 0, tid1 < tid2 global
     ids of different groups, the lexicographically smallest such pair.    */
  RC_IG_RW = 9,        /* one reads, the other writes                        */
  RC_IG_WW_BENIGN = 10,/* both write; every group's last value of the cell equal */
  RC_IG_WW_NONBENIGN = 11 /* both write; two groups' last values differ       */
};
#define RC_IG_INTERVAL 0xFFFFFFFFu

/* 32-byte report.  Canonical order = ascending (instance, interval, array
 * (signed), index (signed), kind, tid1, tid2); the array returned by rc_run is
 * in that order.  For RW / WW_*: (tid1 < tid2) is the lexicographically
 * smallest conflicting pair (reading L4); flags bit0 = tid1 read
 * the cell, bit1 = tid1 wrote it, bit2 = tid2 read, bit3 = tid2 wrote (all in
 * this interval).  With RC_OPT_CLASSIFY_RW an RW report also carries bit4
 * (0x10: re-running its interval with writers-first visibility of the RW
 * cells commits the same heap — the read values do not matter for this
 * input) or bit5 (0x20: the committed heap differs), DESIGN.md §3 reading
 * L19.  For error kinds tid2 = 0xFFFFFFFF and flags = 0.                    */
typedef struct {
  uint32_t instance; /* global instance id (includes options->instance_offset) */
  uint32_t interval; /* barrier interval k (0-based)                          */
  int32_t array;     /* array id, or -1                                       */
  int32_t index;     /* cell index (may be out of bounds for OOB), or pc      */
  uint32_t tid1, tid2;
  uint16_t kind, flags;
  uint32_t reserved; /* 0 */
} rc_report;

/* Exact counters; part of parity with the oracle. */
typedef struct {
  uint64_t checked_accesses; /* performed LD + ST (in-bounds) of all work-items */
  uint64_t loads, stores;
  uint64_t instructions;     /* executed bytecode instructions (the one refused
                                by the fuel check is not counted)               */
  uint64_t intervals_max;    /* max over instances of intervals executed        */
  uint64_t lanes_final[8];   /* final work-item status histogram:
                                [0] EXITED [1] PRUNED (assume false) [2] OOB
                                [3] ASSERT [4] DIV0 [5] FUEL
                                [6] still waiting when max_intervals stopped it
                                [7] 0                                          */
} rc_stats;

/* Optional live profile (options->profile), filled when non-NULL: per kernel
 * class, launches, summed CUDA-event time on the launch stream, and the
 * ALGORITHMIC bytes those launches must move.               */
enum rc_prof_class {
  RC_PROF_INTERP = 0,   /* K1  interval interpretation + log append          */
  RC_PROF_HIST = 1,     /* K2  digit histograms / bucket counts + starts     */
  RC_PROF_SORT = 2,     /* K3  onesweep passes / bucket scatter              */
  RC_PROF_DETECT = 3,   /* K4+K5 segmented detect + commit                   */
  RC_PROF_BOUNDARY = 4, /* A4  barrier bookkeeping, divergence               */
  RC_PROF_FINALIZE = 5, /* K6  canonical report sort                         */
  RC_PROF_COPY = 6,     /* heap init / final-heap copies                     */
  RC_PROF_FILTER = 7,   /* write-set filter of the read records  */
  RC_PROF_N = 8
};
typedef struct {
  uint64_t launches[RC_PROF_N];
  double ms[RC_PROF_N];
  uint64_t alg_bytes[RC_PROF_N];
  uint64_t items[RC_PROF_N]; /* records / lanes processed                    */
  double total_ms;           /* whole rc_run on the stream                    */
  uint64_t kernel_launches;  /* librc kernels launched by this rc_run         */
  /* in: record the per-interval kernels of every k-th interval only (0 = the
   * default, 7: coprime with the 2-interval period of alternating kernels);
   * out: the k used.  launches/ms/alg_bytes/items of the
   * per-interval classes cover the sampled intervals only (per-launch
   * averages are unbiased; totals scale by k).  Event bookkeeping for every
   * interval would cost the host more than the GPU work of small intervals. */
  uint32_t sample_every;
  uint32_t flags;            /* out: bit 0 = intervals ran K1c, the interval
                                kernel compiled for the program;
                                its alg_bytes[RC_PROF_INTERP] are then the lane
                                state, heap loads and log it must move       */
} rc_profile;

/* One shared array of the kernel (an element of Args).
 * `data` holds n_instances consecutive copies of the array:
 * data[inst * size + i], int32.  Borrowed, read-only; the library copies it
 * into its own working heap.  Device pointer unless RC_OPT_HOST_IO.         */
typedef struct {
  const int32_t* data;
  uint32_t size; /* element count, < 2^31; size(v) of PAPER.md:87           */
} rc_array;

#define RC_OPT_HOST_IO 1u /* arrays[].data and final_heaps[] are HOST pointers;
                             rc_run does the host<->device copies itself     */
#define RC_OPT_KEEP_ALL_READS 2u /* sort every read record, also those of cells no
                             work-item wrote in the interval (which can produce
                             no report or commit; by default they are dropped
                             before the sort) — same results     */
#define RC_OPT_CLASSIFY_RW 4u /* RW value classification:
                             every interval with an RW report is re-run under a
                             second visibility and the RW reports get flag bit 4
                             or 5 (see rc_report); costs a heap snapshot per
                             interval and one extra pass per racy interval     */

#define RC_OPT_PREPASS 8u /* run rc_prove on the run's shape first (cached per
                             shape); when it proves RC_PROVE_NO_CONFLICT no
                             report is possible, so the intervals run without
                             logging: each work-item's writes are committed at
                             the end of its interval (exact: no other work-item
                             touches those cells in it) and the grouping /
                             detect kernels are skipped.  Same reports (none),
                             final heaps and stats.  Ignored with n_groups > 1
                             or RC_OPT_CLASSIFY_RW.                         */

typedef struct {
  uint32_t instance_offset;    /* added to report.instance (multi-GPU shards) */
  uint32_t max_intervals;      /* default 65536 (reading L17)                  */
  uint64_t fuel_per_interval;  /* per work-item per interval; default 2^20     */
  int32_t device;              /* CUDA device ordinal; default 0               */
  uint32_t flags;              /* RC_OPT_*                                     */
  void* cuda_stream;           /* cudaStream_t; NULL = legacy default stream  */
  uint32_t max_batch_instances;/* 0 = library chooses the instance batch      */
  uint32_t n_groups;           /* work-groups per instance (0 = 1), each of
                                  work_group_size work-items; they run one
                                  after another in ascending order on the
                                  instance's heap (reading L20)              */
  rc_profile* profile;         /* nullable                                     */
} rc_options;

typedef struct rc_program rc_program; /* opaque, library-owned */

/* Decode + validate bytecode (host only; no CUDA call, so it works without a
 * GPU).  On success *out owns a copy of the program until rc_free_program.
 * RC_EINVAL (+ message) for: bad magic/version/flags, size mismatch, n_regs
 * or n_arrays or n_instr out of range, unknown opcode, register >= n_regs,
 * array >= n_arrays, branch target >= n_instr, execution that can fall off
 * the end, no EXIT reachable from pc 0.                                     */
RC_API int rc_load_program(const void* bytecode, size_t nbytes, rc_program** out);
RC_API void rc_free_program(rc_program* prog);
/* n_regs, n_arrays, n_instr of a loaded program (any pointer may be NULL). */
RC_API int rc_program_info(const rc_program* prog, uint32_t* n_regs, uint32_t* n_arrays,
                    uint32_t* n_instr);

/* Run `prog` with `work_group_size` work-items (tids 0..n-1) on each of
 * `n_instances` instances (with options->n_groups = G > 1: G work-groups of
 * `work_group_size` work-items each, global tids 0..G*n-1, see RC_OP_GID).  `arrays` has exactly the program's n_arrays
 * entries.  Reports go to the HOST buffer `out` (caller-owned, `capacity`
 * entries, may be NULL when capacity == 0) in canonical order;
 * *n_reports_total is always set (nullable).  `stats` (host, nullable).
 * `final_heaps` (nullable): n_arrays pointers, each to n_instances*size int32
 * (device, or host with RC_OPT_HOST_IO) receiving the final shared heap.
 * Stream-ordered on options->cuda_stream; returns after the reports are on
 * the host (synchronises that stream).  Not re-entrant on the same program
 * object from two threads at once (the program caches device workspace).  */
RC_API int rc_run(const rc_program* prog, uint32_t work_group_size, const rc_array* arrays,
           uint32_t n_arrays, uint32_t n_instances, const rc_options* options,
           rc_report* out, uint64_t capacity, uint64_t* n_reports_total,
           rc_stats* stats, int32_t* const* final_heaps);

/* Thread-local message describing the last non-OK status of this thread. */
RC_API const char* rc_last_error(void);
RC_API int rc_abi_version(void);
/* Release all cached device workspace of `prog` (also done by rc_free_program). */
RC_API int rc_release_workspace(rc_program* prog);


/* ---- interleaving explorer -------------------------
 * Every interleaving of ONE barrier interval under the paper's global
 * semantics: one work-item steps at a time on the shared
 * heap with immediate visibility; the interval ends when no work-item is
 * RUNNING (all suspended at a barrier P:218, exited, or stopped by ⊥ / ⊤ as
 * readings L5 / L6).  The paper's race definition is
 * non-determinism of the end states: n_differ > 0.  The explorer is a witness
 * generator: `witness` is a schedule whose end heap differs from schedule 0's
 * (always run the lowest runnable tid), as a choice sequence of tids.
 *
 * Schedules are numbered: index i decodes in mixed radix over the runnable
 * work-items of each state (d = i mod r, i /= r, step the d-th runnable);
 * an index is a schedule of its own when the quotient left at the end is 0,
 * otherwise it repeats a lower one and is not counted.  `complete` = every
 * schedule has an index in [0, index_end) (proved from max_product <=
 * index_end, explore.cu); else call again with a larger index_end.
 * RC_EXPLORE_REDUCED steps only the shared accesses (LD/ST) and runs the
 * private instructions between them eagerly: the same terminal states (they
 * commute with every other work-item's steps) and far fewer schedules.      */
#define RC_EXPLORE_REDUCED 1u

typedef struct {
  uint64_t n_schedules; /* schedules (own indices) among [index_begin, index_end) */
  uint64_t n_differ;    /* of them, end heap != schedule 0's end heap         */
  uint64_t witness;     /* smallest such index, UINT64_MAX if none            */
  uint64_t max_product; /* max radix product over the examined indices        */
  uint64_t n_terminal;  /* rows written to `terminals` (<= cap)               */
  uint32_t witness_len; /* choices in the witness schedule (may exceed max_len) */
  uint32_t complete;    /* 1: index_begin == 0 and every schedule was examined */
} rc_explore_result;

/* Explore the interval of `prog` that starts in the given state, n work-items
 * (1..32).  sizes: HOST, n_arrays element counts.  heap (all arrays
 * concatenated, sum(sizes) int32), regs [n][n_regs] int32, pc [n] u32, status
 * [n] u8 (0 RUNNING 1 WAITING 2 EXITED 3 PRUNED 4 OOB 5 ASSERT 6 DIV0 7 FUEL;
 * only RUNNING work-items step): device or host pointers, borrowed, read
 * once.  fuel: per work-item instruction budget for the interval (0 = 2^20;
 * reading L17: the work-item whose budget is spent stops with status FUEL).
 * terminals (DEVICE, nullable when cap == 0): receives up to `cap` end states,
 * one row of sum(sizes) + n*(4+n_regs) int32 per counted schedule, in no
 * particular order: the heap, then per work-item pc, status, 0, 0, registers.
 * witness_sched (DEVICE, nullable when max_len == 0): the witness's first
 * max_len choices (tids).  out (HOST) is always written.  Synchronises
 * `cuda_stream` (cudaStream_t, NULL = legacy default) on the current device.
 * Device buffers are cached on `prog` (freed by rc_release_workspace /
 * rc_free_program); like rc_run, not re-entrant on one program object.
 * RC_EINVAL for bad arguments, RC_ELIMIT when the state row exceeds 4096
 * words, RC_ENOMEM / RC_ECUDA for device failures.                         */
RC_API int rc_explore(const rc_program* prog, uint32_t n, const uint32_t* sizes, const int32_t* heap,
               const int32_t* regs, const uint32_t* pc, const uint8_t* status, uint64_t fuel,
               uint64_t index_begin, uint64_t index_end, uint32_t flags, int32_t* terminals,
               uint64_t cap, uint32_t* witness_sched, uint32_t max_len, void* cuda_stream,
               rc_explore_result* out);

/* ---- symbolic NoRace pre-pass ----
 * The paper's symbolic execution (Table 1): one generic work-item
 * whose tid is universally quantified, sets of symbolic heaps, and at every
 * barrier the NoRace check for two renamed instances i != j, with
 * a prover the paper leaves open — here a decision procedure
 * over the concrete shape: work_group_size work-items (one work-group), the
 * given array sizes, any input values.  Host only; no device work.
 * verdict: RC_PROVE_NO_CONFLICT — in every interval no two work-items touch
 *   one cell with a write, and no ⊥ (OOB / ASSERT / DIV0 / FUEL) and no
 *   barrier divergence is possible: rc_run reports nothing, for any input;
 * RC_PROVE_NORACE — as above except that write-write conflicts are possible,
 *   each provably benign (equal values): rc_run can report only WW_BENIGN
 *   (the paper's NoRace: the shared state at every barrier is deterministic);
 * RC_PROVE_UNKNOWN — not proved (the checker must run); `reason` / `pc` say
 *   where the proof stopped.  Sound, not complete.
 * sizes: HOST, n_arrays element counts.  fuel_per_interval: as rc_options (0
 * = 2^20).  budget: prover work units (~ tid evaluations; 0 = 2^32).  out
 * (HOST) is always written.  RC_EINVAL for bad arguments.                  */
#define RC_PROVE_UNKNOWN 0u
#define RC_PROVE_NO_CONFLICT 1u
#define RC_PROVE_NORACE 2u
/* reasons (RC_PROVE_UNKNOWN) */
#define RC_PROVE_R_RW 1u           /* a read and another work-item's write may meet */
#define RC_PROVE_R_WW 2u           /* two writes may meet with values not provably equal */
#define RC_PROVE_R_OOB 3u          /* an index may leave its array */
#define RC_PROVE_R_DATA_INDEX 4u   /* an index depends on loaded values */
#define RC_PROVE_R_ASSERT 5u       /* an assert may fail */
#define RC_PROVE_R_DIV0 6u         /* a divisor may be 0 */
#define RC_PROVE_R_DIVERGENCE 7u   /* work-items may reach different barriers */
#define RC_PROVE_R_OWN_ALIAS 8u    /* a work-item's own writes may alias */
#define RC_PROVE_R_FUEL 9u         /* fuel or the interval limit may run out */
#define RC_PROVE_R_BUDGET 10u      /* the prover's budget (paths, work) ran out */
#define RC_PROVE_R_UNSUPPORTED 11u
typedef struct {
  uint32_t verdict;   /* RC_PROVE_*                                     */
  uint32_t reason;    /* RC_PROVE_R_* when UNKNOWN                        */
  uint32_t pc;        /* instruction where the proof stopped (0: at a barrier check) */
  uint32_t intervals; /* barrier intervals checked                       */
  uint64_t terms;     /* symbolic terms built                             */
  uint64_t work;      /* prover work units spent                          */
} rc_prove_result;
RC_API int rc_prove(const rc_program* prog, uint32_t work_group_size, const uint32_t* sizes, uint32_t n_arrays,
             uint64_t fuel_per_interval, uint64_t budget, rc_prove_result* out);

#ifdef __cplusplus
}
#endif
#endif /* RC_H */
