/*
 * oracle.c — TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU
 * definition of what the race-checking hot path computes.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.  It shares no code, header, table or constant with the
 * CUDA path (paper_1308_3203_b200/): it has its own bytecode decoder, its own
 * opcode numbers (re-typed from the RCB1 format description in DESIGN.md §2)
 * and its own report layout.
 *
 * Two independent parts:
 *
 *  (1) oracle_run: the canonical algorithm of DESIGN.md §3 / SURVEY.md §8(c),
 *      step by step: thread-local rules of PAPER.md:168-201 under delayed
 *      visibility inside each barrier interval, the race rule of
 *      PAPER.md:224-229 read as per-cell access conflicts (reading L1), the
 *      benign test of PAPER.md:23, 229 on final per-thread values (L3), the
 *      barrier release PAPER.md:220-222 as "max-tid writer wins" (I4), the
 *      implicit final barrier PAPER.md:233.
 *
 *  (2) oracle_enumerate: the paper's own global semantics:
 *      one thread steps at a time on a SHARED heap with immediate visibility,
 *      every interleaving of one barrier interval is explored, and the set of
 *      reachable end-of-interval states is returned.  Tests use it to check
 *      invariants I1-I4 that tie (1) to the paper's race definition
 *      (PAPER.md:230-232).
 *
 * Arithmetic is int32 two's complement with wrap (reading L7), done through
 * uint32_t so C's signed-overflow UB is avoided.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* ---- bytecode (RCB1) --------------------------------------- */
enum {
  O_CONST = 1, O_MOV, O_TID, O_SIZE, O_ADD, O_SUB, O_MUL, O_DIV, O_MOD, O_MIN,
  O_MAX, O_AND, O_OR, O_XOR, O_LT, O_EQ, O_LAND, O_LNOT, O_LD, O_ST, O_BAR,
  O_ASSUME, O_ASSERT, O_BR, O_JMP, O_EXIT, O_ADDI,
  O_GID, O_LID, O_LSIZE  /* work-group id, local id, work-group size (reading L20) */
};

typedef struct { uint8_t op, a, b, c; int32_t imm; } oins;
typedef struct { uint32_t n_regs, n_arrays, n_instr; oins* code; } oprog;

static uint32_t rd_u32(const uint8_t* p) { return (uint32_t)p[0] | (uint32_t)p[1] << 8 | (uint32_t)p[2] << 16 | (uint32_t)p[3] << 24; }
static uint16_t rd_u16(const uint8_t* p) { return (uint16_t)(p[0] | p[1] << 8); }

static int decode(const uint8_t* bc, size_t nbytes, oprog* P) {
  if (nbytes < 16 || rd_u32(bc) != 0x31424352u) return -1;
  P->n_regs = rd_u16(bc + 8);
  P->n_arrays = rd_u16(bc + 10);
  P->n_instr = rd_u32(bc + 12);
  if (nbytes != 16 + 8 * (size_t)P->n_instr || P->n_regs == 0) return -1;
  P->code = (oins*)malloc(sizeof(oins) * (P->n_instr ? P->n_instr : 1));
  for (uint32_t i = 0; i < P->n_instr; i++) {
    const uint8_t* q = bc + 16 + 8 * i;
    P->code[i].op = q[0]; P->code[i].a = q[1]; P->code[i].b = q[2]; P->code[i].c = q[3];
    P->code[i].imm = (int32_t)rd_u32(q + 4);
  }
  return 0;
}

/* ---- reports (own layout; 32 bytes, field order of DESIGN.md §2) --------- */
typedef struct {
  uint32_t instance, interval;
  int32_t array, index;
  uint32_t tid1, tid2;
  uint16_t kind, flags;
  uint32_t reserved;
} orep;

enum { K_RW = 1, K_WWB = 2, K_WWN = 3, K_OOB = 4, K_ASSERT = 5, K_DIV0 = 6, K_FUEL = 7, K_DIV = 8,
       K_IG_RW = 9, K_IG_WWB = 10, K_IG_WWN = 11 /* inter-group races (reading L20) */ };
#define IG_INTERVAL 0xFFFFFFFFu /* inter-group reports concern the whole kernel */

/* the work-group a work-item belongs to (reading L20): tids base .. base+lsize-1 */
typedef struct { uint32_t base, gid, lsize; } ogroup;
#define NOTID 0xFFFFFFFFu

typedef struct { orep* v; size_t n, cap; } replist;
static void rep_push(replist* L, orep r) {
  if (L->n == L->cap) { L->cap = L->cap ? 2 * L->cap : 64; L->v = (orep*)realloc(L->v, L->cap * sizeof(orep)); }
  L->v[L->n++] = r;
}
static orep mkrep(uint32_t inst, uint32_t k, int32_t arr, int32_t idx, uint32_t t1, uint32_t t2, int kind, int flags) {
  orep r; memset(&r, 0, sizeof r);
  r.instance = inst; r.interval = k; r.array = arr; r.index = idx; r.tid1 = t1; r.tid2 = t2;
  r.kind = (uint16_t)kind; r.flags = (uint16_t)flags;
  return r;
}
/* canonical order: (instance, interval, array, index, kind, tid1, tid2) */
static int rep_cmp(const void* x, const void* y) {
  const orep* a = (const orep*)x; const orep* b = (const orep*)y;
#define C(f) if (a->f != b->f) return a->f < b->f ? -1 : 1;
  C(instance) C(interval) C(array) C(index) C(kind) C(tid1) C(tid2)
#undef C
  return 0;
}

/* ---- lane (work-item) state ----------------------------------------------- */
enum { S_RUNNING = 0, S_WAITING, S_EXITED, S_PRUNED, S_OOB, S_ASSERT, S_DIV0, S_FUEL };

/* int32 semantics (reading L7) */
static int32_t w_add(int32_t x, int32_t y) { return (int32_t)((uint32_t)x + (uint32_t)y); }
static int32_t w_sub(int32_t x, int32_t y) { return (int32_t)((uint32_t)x - (uint32_t)y); }
static int32_t w_mul(int32_t x, int32_t y) { return (int32_t)((uint32_t)x * (uint32_t)y); }
static int32_t w_div(int32_t x, int32_t y) { /* y != 0; C99 truncation; INT_MIN/-1 = INT_MIN */
  if (y == -1) return (int32_t)(0u - (uint32_t)x);
  return x / y;
}
static int32_t w_mod(int32_t x, int32_t y) { if (y == -1) return 0; return x % y; }

/* Outcome of one ALU/control instruction that does not touch shared memory.
 * Returns 1 if handled (regs/pc updated), 0 if the instruction is a memory,
 * barrier or termination instruction the caller must handle. */
static int step_private(const oprog* P, const oins* I, int32_t* r, uint32_t t, const ogroup* G,
                        const uint32_t* sizes, uint32_t* pc, int* fault) {
  *fault = 0;
  switch (I->op) {
    case O_CONST: r[I->a] = I->imm; break;
    case O_MOV: r[I->a] = r[I->b]; break;
    case O_TID: r[I->a] = (int32_t)(G->base + t); break; /* global id = gid * lsize + lid */
    case O_GID: r[I->a] = (int32_t)G->gid; break;
    case O_LID: r[I->a] = (int32_t)t; break;
    case O_LSIZE: r[I->a] = (int32_t)G->lsize; break;
    case O_SIZE: r[I->a] = (int32_t)sizes[I->b]; break;
    case O_ADD: r[I->a] = w_add(r[I->b], r[I->c]); break;
    case O_SUB: r[I->a] = w_sub(r[I->b], r[I->c]); break;
    case O_MUL: r[I->a] = w_mul(r[I->b], r[I->c]); break;
    case O_DIV: if (r[I->c] == 0) { *fault = S_DIV0; return 1; } r[I->a] = w_div(r[I->b], r[I->c]); break;
    case O_MOD: if (r[I->c] == 0) { *fault = S_DIV0; return 1; } r[I->a] = w_mod(r[I->b], r[I->c]); break;
    case O_MIN: r[I->a] = r[I->b] < r[I->c] ? r[I->b] : r[I->c]; break;
    case O_MAX: r[I->a] = r[I->b] > r[I->c] ? r[I->b] : r[I->c]; break;
    case O_AND: r[I->a] = r[I->b] & r[I->c]; break;
    case O_OR: r[I->a] = r[I->b] | r[I->c]; break;
    case O_XOR: r[I->a] = r[I->b] ^ r[I->c]; break;
    case O_LT: r[I->a] = r[I->b] < r[I->c]; break;
    case O_EQ: r[I->a] = r[I->b] == r[I->c]; break;
    case O_LAND: r[I->a] = (r[I->b] != 0) && (r[I->c] != 0); break;
    case O_LNOT: r[I->a] = r[I->b] == 0; break;
    case O_ADDI: r[I->a] = w_add(r[I->b], I->imm); break;
    case O_BR: *pc = r[I->a] != 0 ? (uint32_t)I->imm : (uint32_t)I->b + 256u * I->c; return 1;
    case O_JMP: *pc = (uint32_t)I->imm; return 1;
    default: return 0;
  }
  (void)P;
  *pc += 1;
  return 1;
}

/* ---- (1) the canonical algorithm ---------------------------------------- */

typedef struct { uint32_t cell_arr; int32_t idx; uint32_t tid; uint8_t w; int32_t val; } acc; /* one access record */
typedef struct { acc* v; size_t n, cap; } acclist;
static void acc_push(acclist* L, acc a) {
  if (L->n == L->cap) { L->cap = L->cap ? 2 * L->cap : 1024; L->v = (acc*)realloc(L->v, L->cap * sizeof(acc)); }
  L->v[L->n++] = a;
}
static int acc_cmp(const void* x, const void* y) {
  const acc* a = (const acc*)x; const acc* b = (const acc*)y;
  if (a->cell_arr != b->cell_arr) return a->cell_arr < b->cell_arr ? -1 : 1;
  if (a->idx != b->idx) return a->idx < b->idx ? -1 : 1;
  if (a->tid != b->tid) return a->tid < b->tid ? -1 : 1;
  if (a->w != b->w) return a->w < b->w ? -1 : 1;
  return 0;
}

typedef struct { uint32_t arr; int32_t idx; int32_t val; } ownw; /* own-write overlay entry */

typedef struct {
  uint64_t checked, loads, stores, instructions, intervals_max, lanes_final[8];
  uint64_t op_count[32]; /* executed instructions per opcode (test coverage only; no semantics) */
} ostats;

typedef struct {
  const oprog* P; uint32_t n; const uint32_t* sizes;
  const int32_t* const* inputs; uint32_t n_instances; uint32_t instance_offset;
  uint64_t fuel; uint32_t max_intervals;
  int32_t* const* final_heaps;
  int classify;
  uint32_t n_groups; /* work-groups per instance, each of n work-items (reading L20) */
  /* per-thread results */
  int next_instance; pthread_mutex_t mu;
} runctx;

typedef struct { replist reps; ostats st; } thread_out;

/* One work-item's part of interval k (PAPER.md:168-201 under delayed
 * visibility, reading L2): it runs from pc[t] until it suspends, exits or
 * halts, logging one read record per performed LD and, at the end, one write
 * record per distinct cell with its final value (reading L3).  A read of cell
 * c sees the work-item's own earlier write, else snap[c] — or alt[c] when
 * altmask[c] is set (the second visibility of the RW value classification,
 * DESIGN.md §3; NULL in the canonical run). */
static void exec_thread(const oprog* P, uint32_t t, const ogroup* G, const uint32_t* sizes, int32_t* r, uint32_t* pc,
                        uint8_t* status, int32_t* node, uint8_t* arrived, int32_t* const* snap,
                        int32_t* const* alt, uint8_t* const* altmask, uint64_t fuel, uint32_t inst_global,
                        uint32_t k, replist* reps, ostats* st, acclist* log, ownw** ownp, size_t* own_cap) {
  ownw* own = *ownp;
  size_t n_own = 0;
  uint64_t steps = 0;
  const uint32_t tg = G->base + t; /* the work-item's (global) tid in reports and the log */
  for (;;) {
    if (steps == fuel) { /* fuel exhausted (reading L17) */
      rep_push(reps, mkrep(inst_global, k, -1, (int32_t)pc[t], tg, NOTID, K_FUEL, 0));
      status[t] = S_FUEL; break;
    }
    steps++;
    st->instructions++;
    const oins* I = &P->code[pc[t]];
    st->op_count[I->op & 31]++;
    int fault;
    if (step_private(P, I, r, t, G, sizes, &pc[t], &fault)) {
      if (fault == S_DIV0) {
        rep_push(reps, mkrep(inst_global, k, -1, (int32_t)pc[t], tg, NOTID, K_DIV0, 0));
        status[t] = S_DIV0; break;
      }
      continue;
    }
    if (I->op == O_LD) { /* v := a[w]   (reading L11) */
      int32_t idx = r[I->c];
      if (idx < 0 || (uint32_t)idx >= sizes[I->b]) { /* ⊥: not performed, not logged (L5) */
        rep_push(reps, mkrep(inst_global, k, I->b, idx, tg, NOTID, K_OOB, 0));
        status[t] = S_OOB; break;
      }
      int32_t v = (altmask && altmask[I->b][idx]) ? alt[I->b][idx] : snap[I->b][idx];
      for (size_t j = 0; j < n_own; j++)
        if (own[j].arr == I->b && own[j].idx == idx) v = own[j].val; /* own earlier write */
      acc a = {I->b, idx, tg, 0, 0};
      acc_push(log, a);
      st->checked++; st->loads++;
      r[I->a] = v;
      pc[t]++;
    } else if (I->op == O_ST) { /* a[v] := e */
      int32_t idx = r[I->b];
      if (idx < 0 || (uint32_t)idx >= sizes[I->a]) {
        rep_push(reps, mkrep(inst_global, k, I->a, idx, tg, NOTID, K_OOB, 0));
        status[t] = S_OOB; break;
      }
      size_t j;
      for (j = 0; j < n_own; j++)
        if (own[j].arr == I->a && own[j].idx == idx) break;
      if (j == n_own) {
        if (n_own == *own_cap) { *own_cap *= 2; own = (ownw*)realloc(own, *own_cap * sizeof(ownw)); *ownp = own; }
        own[n_own].arr = I->a; own[n_own].idx = idx; n_own++;
      }
      own[j].val = r[I->c];
      st->checked++; st->stores++;
      pc[t]++;
    } else if (I->op == O_BAR) { /* τ ⊡ σ */
      status[t] = S_WAITING; node[t] = (int32_t)pc[t]; arrived[t] = 1; pc[t]++; break;
    } else if (I->op == O_EXIT) { /* exit node = implicit final barrier */
      status[t] = S_EXITED; node[t] = -1; arrived[t] = 1; break;
    } else if (I->op == O_ASSUME) { /* false -> ⊤, reading L6 */
      if (r[I->a] == 0) { status[t] = S_PRUNED; break; }
      pc[t]++;
    } else if (I->op == O_ASSERT) { /* false -> ⊥ */
      if (r[I->a] == 0) {
        rep_push(reps, mkrep(inst_global, k, -1, (int32_t)pc[t], tg, NOTID, K_ASSERT, 0));
        status[t] = S_ASSERT; break;
      }
      pc[t]++;
    } else {
      fprintf(stderr, "oracle: bad opcode %d\n", I->op); abort();
    }
  }
  /* the work-item's writes of this interval, one per cell, final value (L3) */
  for (size_t j = 0; j < n_own; j++) {
    acc a = {own[j].arr, own[j].idx, tg, 1, own[j].val};
    acc_push(log, a);
  }
}

/* Run one instance exactly as DESIGN.md §3 describes.  If stop_at >= 0 the
 * run stops at the START of interval stop_at and the lane state + heap are
 * copied out (used to seed the enumerator); returns 1 if that interval is
 * reached, 0 otherwise.  classify: RW value classification of every interval
 * with an RW report. */
static int run_instance(const oprog* P, uint32_t n, const ogroup* G, const uint32_t* sizes, int32_t** heap,
                        uint32_t inst_global, uint64_t fuel, uint32_t max_intervals,
                        replist* reps, ostats* st, int stop_at,
                        int32_t* out_regs, uint32_t* out_pc, uint8_t* out_status, uint64_t* out_intervals,
                        int classify, acclist* glog) {
  uint32_t A = P->n_arrays, R = P->n_regs;
  int32_t* regs = (int32_t*)calloc((size_t)n * R + 1, sizeof(int32_t)); /* registers start at 0 (L18) */
  uint32_t* pc = (uint32_t*)calloc(n + 1, sizeof(uint32_t));              /* start = pc 0 */
  uint8_t* status = (uint8_t*)calloc(n + 1, 1);                           /* RUNNING */
  int32_t* node = (int32_t*)malloc((n + 1) * sizeof(int32_t));
  uint8_t* arrived = (uint8_t*)malloc(n + 1);
  int32_t** snap = (int32_t**)malloc((A + 1) * sizeof(int32_t*));
  for (uint32_t a = 0; a < A; a++) snap[a] = (int32_t*)malloc(((size_t)sizes[a] + 1) * sizeof(int32_t));
  /* classification: the lane state at the interval start, a second heap, the flagged-cell masks */
  int32_t* regs0 = classify ? (int32_t*)malloc(((size_t)n * R + 1) * sizeof(int32_t)) : NULL;
  uint32_t* pc0 = classify ? (uint32_t*)malloc((n + 1) * sizeof(uint32_t)) : NULL;
  uint8_t* status0 = classify ? (uint8_t*)malloc(n + 1) : NULL;
  int32_t** heapB = classify ? (int32_t**)malloc((A + 1) * sizeof(int32_t*)) : NULL;
  uint8_t** mask = classify ? (uint8_t**)malloc((A + 1) * sizeof(uint8_t*)) : NULL;
  for (uint32_t a = 0; classify && a < A; a++) {
    heapB[a] = (int32_t*)malloc(((size_t)sizes[a] + 1) * sizeof(int32_t));
    mask[a] = (uint8_t*)malloc((size_t)sizes[a] + 1);
  }
  acclist log = {0};
  size_t own_cap = 16; ownw* own = (ownw*)malloc(own_cap * sizeof(ownw));
  uint32_t k = 0;
  int reached = 0;

  for (;;) {
    if (stop_at >= 0 && k == (uint32_t)stop_at) { reached = 1; break; }
    /* interval k: snap <- heap (the shared state every read of this interval sees) */
    for (uint32_t a = 0; a < A; a++) memcpy(snap[a], heap[a], (size_t)sizes[a] * sizeof(int32_t));
    if (classify) {
      memcpy(regs0, regs, (size_t)n * R * sizeof(int32_t));
      memcpy(pc0, pc, n * sizeof(uint32_t));
      memcpy(status0, status, n);
    }
    log.n = 0;
    memset(arrived, 0, n);
    for (uint32_t t = 0; t < n; t++) {
      if (status[t] != S_RUNNING) continue;
      exec_thread(P, t, G, sizes, regs + (size_t)t * R, pc, status, node, arrived, snap, NULL, NULL, fuel,
                  inst_global, k, reps, st, &log, &own, &own_cap);
    }

    const size_t rep_mark = reps->n;  /* reports of this interval start here */
    if (glog) /* every access of the group, all intervals (inter-group races, reading L20) */
      for (size_t i = 0; i < log.n; i++) acc_push(glog, log.v[i]);
    /* race rule per cell (PAPER.md:224-229 as reading L1), in (array,index) order */
    qsort(log.v, log.n, sizeof(acc), acc_cmp);
    size_t g = 0;
    uint32_t* rt = NULL; uint32_t* wt = NULL; int32_t* wv = NULL; size_t cap = 0;
    while (g < log.n) {
      size_t e = g;
      while (e < log.n && log.v[e].cell_arr == log.v[g].cell_arr && log.v[e].idx == log.v[g].idx) e++;
      if (e - g > cap) { cap = e - g; rt = (uint32_t*)realloc(rt, cap * 4); wt = (uint32_t*)realloc(wt, cap * 4); wv = (int32_t*)realloc(wv, cap * 4); }
      size_t nr = 0, nw = 0;  /* R(c): distinct readers ascending; W(c): writers ascending */
      for (size_t i = g; i < e; i++) {
        if (log.v[i].w) { wt[nw] = log.v[i].tid; wv[nw] = log.v[i].val; nw++; }
        else if (nr == 0 || rt[nr - 1] != log.v[i].tid) rt[nr++] = log.v[i].tid;
      }
      uint32_t arr = log.v[g].cell_arr; int32_t idx = log.v[g].idx;
      /* membership helpers (linear, plain) */
#define IN_R(x) ({ int f_ = 0; for (size_t q_ = 0; q_ < nr; q_++) if (rt[q_] == (x)) f_ = 1; f_; })
#define IN_W(x) ({ int f_ = 0; for (size_t q_ = 0; q_ < nw; q_++) if (wt[q_] == (x)) f_ = 1; f_; })
#define FLAGS(a_, b_) ((IN_R(a_) ? 1 : 0) | (IN_W(a_) ? 2 : 0) | (IN_R(b_) ? 4 : 0) | (IN_W(b_) ? 8 : 0))
      /* RW: lexicographically smallest (t1<t2), one reads and the other writes */
      int have_rw = 0; uint32_t p1 = 0, p2 = 0;
      if (nr > 0 && nw > 0) {
        /* candidates in ascending order: the sorted union of R and W */
        size_t nu = 0; uint32_t* u = (uint32_t*)malloc((nr + nw) * 4);
        size_t i = 0, j = 0;
        while (i < nr || j < nw) {
          uint32_t x;
          if (j >= nw || (i < nr && rt[i] < wt[j])) x = rt[i++];
          else if (i >= nr || wt[j] < rt[i]) x = wt[j++];
          else { x = rt[i]; i++; j++; }
          u[nu++] = x;
        }
        for (size_t a1 = 0; a1 < nu && !have_rw; a1++)
          for (size_t a2 = a1 + 1; a2 < nu; a2++)
            if ((IN_R(u[a1]) && IN_W(u[a2])) || (IN_W(u[a1]) && IN_R(u[a2]))) {
              have_rw = 1; p1 = u[a1]; p2 = u[a2]; break;
            }
        free(u);
      }
      if (have_rw) rep_push(reps, mkrep(inst_global, k, (int32_t)arr, idx, p1, p2, K_RW, FLAGS(p1, p2)));
      /* WW: |W(c)| >= 2; non-benign iff two writers' final values differ */
      if (nw >= 2) {
        size_t d = 0;
        for (size_t q = 1; q < nw; q++) if (wv[q] != wv[0]) { d = q; break; }
        if (d) rep_push(reps, mkrep(inst_global, k, (int32_t)arr, idx, wt[0], wt[d], K_WWN, FLAGS(wt[0], wt[d])));
        else rep_push(reps, mkrep(inst_global, k, (int32_t)arr, idx, wt[0], wt[1], K_WWB, FLAGS(wt[0], wt[1])));
      }
#undef IN_R
#undef IN_W
#undef FLAGS
      /* barrier release: the max-tid writer's value is committed (I4) */
      if (nw > 0) heap[arr][idx] = wv[nw - 1];
      g = e;
    }
    free(rt); free(wt); free(wv);

    /* RW value classification (reading L19): re-run interval k
     * from its start state with reads of the RW-flagged cells seeing the value
     * the canonical run committed (writers first); commit the second run's
     * writes (max-tid writer) onto the interval-start heap and compare the two
     * committed heaps.  Every RW report of the interval gets flag bit 4 (equal:
     * the RW races of this interval do not change the state, for this input)
     * or bit 5 (the committed state depends on the read values). */
    if (classify && reps->n > rep_mark) {
      int any_rw = 0;
      for (uint32_t a = 0; a < A; a++) memset(mask[a], 0, sizes[a]);
      for (size_t i = rep_mark; i < reps->n; i++)
        if (reps->v[i].kind == K_RW) { mask[reps->v[i].array][reps->v[i].index] = 1; any_rw = 1; }
      if (any_rw) {
        int32_t* rB = (int32_t*)malloc(((size_t)n * R + 1) * sizeof(int32_t));
        uint32_t* pB = (uint32_t*)malloc((n + 1) * sizeof(uint32_t));
        uint8_t* sB = (uint8_t*)malloc(n + 1);
        int32_t* nodeB = (int32_t*)malloc((n + 1) * sizeof(int32_t));
        uint8_t* arrB = (uint8_t*)calloc(n + 1, 1);
        memcpy(rB, regs0, (size_t)n * R * sizeof(int32_t));
        memcpy(pB, pc0, n * sizeof(uint32_t));
        memcpy(sB, status0, n);
        replist junk = {0};
        ostats junk_st; memset(&junk_st, 0, sizeof junk_st);
        acclist logB = {0};
        for (uint32_t t = 0; t < n; t++) {
          if (sB[t] != S_RUNNING) continue;
          exec_thread(P, t, G, sizes, rB + (size_t)t * R, pB, sB, nodeB, arrB, snap, heap, mask, fuel,
                      inst_global, k, &junk, &junk_st, &logB, &own, &own_cap);
        }
        for (uint32_t a = 0; a < A; a++) memcpy(heapB[a], snap[a], (size_t)sizes[a] * sizeof(int32_t));
        /* barrier release of the second run: write records are in ascending tid
         * order, so the last assignment to a cell is its max-tid writer's (I4) */
        for (size_t i = 0; i < logB.n; i++)
          if (logB.v[i].w) heapB[logB.v[i].cell_arr][logB.v[i].idx] = logB.v[i].val;
        int diff = 0;
        for (uint32_t a = 0; a < A && !diff; a++)
          if (memcmp(heapB[a], heap[a], (size_t)sizes[a] * sizeof(int32_t))) diff = 1;
        for (size_t i = rep_mark; i < reps->n; i++)
          if (reps->v[i].kind == K_RW) reps->v[i].flags |= diff ? 0x20 : 0x10;
        free(rB); free(pB); free(sB); free(nodeB); free(arrB); free(junk.v); free(logB.v);
      }
    }

    /* barrier divergence among the work-items that arrived in this interval (L9) */
    {
      int64_t t1 = -1;
      for (uint32_t t = 0; t < n; t++) if (arrived[t]) { t1 = t; break; }
      if (t1 >= 0) {
        for (uint32_t t = (uint32_t)t1 + 1; t < n; t++)
          if (arrived[t] && node[t] != node[t1]) {
            rep_push(reps, mkrep(inst_global, k, -1, node[t1], G->base + (uint32_t)t1, G->base + t, K_DIV, 0));
            break;
          }
      }
    }

    int any_waiting = 0;
    for (uint32_t t = 0; t < n; t++) if (status[t] == S_WAITING) { status[t] = S_RUNNING; any_waiting = 1; }
    if (!any_waiting) break;
    k++;
    if (k >= max_intervals) {
      rep_push(reps, mkrep(inst_global, k, -1, -1, NOTID, NOTID, K_FUEL, 0));
      for (uint32_t t = 0; t < n; t++) if (status[t] == S_RUNNING) status[t] = S_WAITING;
      k--; /* intervals executed = max_intervals */
      break;
    }
  }
  if (stop_at >= 0) { /* lane state at the start of interval stop_at (or at the end) */
    memcpy(out_regs, regs, (size_t)n * R * sizeof(int32_t));
    memcpy(out_pc, pc, n * sizeof(uint32_t));
    memcpy(out_status, status, n);
  }
  if (!reached) {
    for (uint32_t t = 0; t < n; t++) {
      int s = status[t];
      int slot = s == S_EXITED ? 0 : s == S_PRUNED ? 1 : s == S_OOB ? 2 : s == S_ASSERT ? 3 :
                 s == S_DIV0 ? 4 : s == S_FUEL ? 5 : 6;
      st->lanes_final[slot]++;
    }
    if ((uint64_t)k + 1 > st->intervals_max) st->intervals_max = (uint64_t)k + 1;
    if (out_intervals) *out_intervals = (uint64_t)k + 1;
  }
  free(regs); free(pc); free(status); free(node); free(arrived);
  for (uint32_t a = 0; a < A; a++) free(snap[a]);
  free(snap); free(log.v); free(own);
  if (classify) {
    for (uint32_t a = 0; a < A; a++) { free(heapB[a]); free(mask[a]); }
    free(heapB); free(mask); free(regs0); free(pc0); free(status0);
  }
  return reached;
}

typedef struct { runctx* ctx; thread_out out; } worker_arg;

/* one group's last written value of a cell (reading L20) */
typedef struct { uint32_t arr; int32_t idx; uint32_t g; int32_t val; } lastv;
static int lastv_cmp(const void* x, const void* y) {
  const lastv* a = (const lastv*)x; const lastv* b = (const lastv*)y;
  if (a->arr != b->arr) return a->arr < b->arr ? -1 : 1;
  if (a->idx != b->idx) return a->idx < b->idx ? -1 : 1;
  if (a->g != b->g) return a->g < b->g ? -1 : 1;
  return 0;
}

/* Inter-group races of one instance (reading L20): no barrier orders two
 * work-groups, so two work-items of different groups that touch the same cell
 * anywhere in the kernel, at least one writing, race.  Per cell, plainly:
 *   IG_RW: lexicographically smallest (t1 < t2), different groups, one reads
 *          and the other writes;
 *   IG_WW: smallest (t1 < t2), different groups, both write; non-benign iff
 *          two groups' last written values differ (the final value of a
 *          write-only cell is the last value of whichever group writes last);
 * interval = IG_INTERVAL, flags 0.  log: every access of every group (tids
 * global); lv: per group and written cell its last value. */
static void inter_group_reports(acclist* log, lastv* lv, size_t nlv, uint32_t lsize, uint32_t inst_global,
                                replist* reps) {
  qsort(log->v, log->n, sizeof(acc), acc_cmp);
  qsort(lv, nlv, sizeof(lastv), lastv_cmp);
  size_t g = 0, q = 0;
  while (g < log->n) {
    size_t e = g;
    while (e < log->n && log->v[e].cell_arr == log->v[g].cell_arr && log->v[e].idx == log->v[g].idx) e++;
    const uint32_t arr = log->v[g].cell_arr; const int32_t idx = log->v[g].idx;
    /* every access pair (x, y) of the cell, plain O(m^2) */
    uint32_t rw1 = NOTID, rw2 = NOTID, ww1 = NOTID, ww2 = NOTID;
    for (size_t x = g; x < e; x++)
      for (size_t y = g; y < e; y++) {
        const acc* A = &log->v[x]; const acc* B = &log->v[y];
        if (!(A->tid < B->tid) || A->tid / lsize == B->tid / lsize) continue;
        if (A->w != B->w && (A->tid < rw1 || (A->tid == rw1 && B->tid < rw2))) { rw1 = A->tid; rw2 = B->tid; }
        if (A->w && B->w && (A->tid < ww1 || (A->tid == ww1 && B->tid < ww2))) { ww1 = A->tid; ww2 = B->tid; }
      }
    if (rw1 != NOTID) rep_push(reps, mkrep(inst_global, IG_INTERVAL, (int32_t)arr, idx, rw1, rw2, K_IG_RW, 0));
    if (ww1 != NOTID) {
      while (q < nlv && (lv[q].arr < arr || (lv[q].arr == arr && lv[q].idx < idx))) q++;
      int differ = 0;
      for (size_t j = q; j < nlv && lv[j].arr == arr && lv[j].idx == idx; j++)
        if (lv[j].val != lv[q].val) differ = 1;
      rep_push(reps, mkrep(inst_global, IG_INTERVAL, (int32_t)arr, idx, ww1, ww2, differ ? K_IG_WWN : K_IG_WWB, 0));
    }
    g = e;
  }
}

static void* worker(void* p) {
  worker_arg* W = (worker_arg*)p;
  runctx* c = W->ctx;
  const oprog* P = c->P;
  int32_t** heap = (int32_t**)malloc((P->n_arrays + 1) * sizeof(int32_t*));
  for (uint32_t a = 0; a < P->n_arrays; a++) heap[a] = (int32_t*)malloc(((size_t)c->sizes[a] + 1) * sizeof(int32_t));
  for (;;) {
    pthread_mutex_lock(&c->mu);
    int i = c->next_instance++;
    pthread_mutex_unlock(&c->mu);
    if (i >= (int)c->n_instances) break;
    for (uint32_t a = 0; a < P->n_arrays; a++)  /* heap <- copy(inputs[inst]) */
      memcpy(heap[a], c->inputs[a] + (size_t)i * c->sizes[a], (size_t)c->sizes[a] * sizeof(int32_t));
    /* the work-groups one after another in ascending order (reading L20):
     * each runs the paper's semantics on the heap the previous ones left */
    acclist glog = {0}, gone = {0};
    lastv* lv = NULL; size_t nlv = 0, lvcap = 0;
    for (uint32_t gi = 0; gi < c->n_groups; gi++) {
      const ogroup G = {gi * c->n, gi, c->n};
      gone.n = 0;
      run_instance(P, c->n, &G, c->sizes, heap, c->instance_offset + (uint32_t)i, c->fuel, c->max_intervals,
                   &W->out.reps, &W->out.st, -1, NULL, NULL, NULL, NULL, c->classify,
                   c->n_groups > 1 ? &gone : NULL);
      for (size_t j = 0; j < gone.n; j++) {
        acc_push(&glog, gone.v[j]);
        if (!gone.v[j].w) continue;
        /* a cell this group wrote: its value now is the group's last (committed) one */
        if (nlv == lvcap) { lvcap = lvcap ? 2 * lvcap : 256; lv = (lastv*)realloc(lv, lvcap * sizeof(lastv)); }
        lv[nlv].arr = gone.v[j].cell_arr; lv[nlv].idx = gone.v[j].idx; lv[nlv].g = gi;
        lv[nlv].val = heap[gone.v[j].cell_arr][gone.v[j].idx];
        nlv++;
      }
    }
    if (c->n_groups > 1) inter_group_reports(&glog, lv, nlv, c->n, c->instance_offset + (uint32_t)i, &W->out.reps);
    free(glog.v); free(gone.v); free(lv);
    if (c->final_heaps)
      for (uint32_t a = 0; a < P->n_arrays; a++)
        if (c->final_heaps[a])
          memcpy(c->final_heaps[a] + (size_t)i * c->sizes[a], heap[a], (size_t)c->sizes[a] * sizeof(int32_t));
  }
  for (uint32_t a = 0; a < P->n_arrays; a++) free(heap[a]);
  free(heap);
  return NULL;
}

/* Public: run the canonical algorithm on n_instances instances.
 * inputs[a] = n_instances * sizes[a] int32 (instance-major).  Reports are
 * returned malloc'd in canonical order (free with oracle_free).  stats[45] =
 * checked, loads, stores, instructions, intervals_max, lanes_final[8],
 * op_count[32] (executed instructions per opcode; a coverage counter).
 * classify != 0: RW value classification flags on the RW reports. */
int oracle_run(const uint8_t* bc, size_t nbytes, uint32_t n, const uint32_t* sizes,
               const int32_t* const* inputs, uint32_t n_instances, uint32_t instance_offset,
               uint64_t fuel, uint32_t max_intervals, int n_threads,
               orep** reports, uint64_t* n_reports, int32_t* const* final_heaps, uint64_t* stats, int classify,
               uint32_t n_groups) {
  oprog P;
  if (decode(bc, nbytes, &P)) return -1;
  runctx c;
  memset(&c, 0, sizeof c);
  c.P = &P; c.n = n; c.sizes = sizes; c.inputs = inputs; c.n_instances = n_instances;
  c.instance_offset = instance_offset; c.fuel = fuel; c.max_intervals = max_intervals;
  c.final_heaps = final_heaps;
  c.classify = classify;
  c.n_groups = n_groups ? n_groups : 1;
  pthread_mutex_init(&c.mu, NULL);
  if (n_threads < 1) n_threads = 1;
  worker_arg* W = (worker_arg*)calloc((size_t)n_threads, sizeof(worker_arg));
  pthread_t* th = (pthread_t*)calloc((size_t)n_threads, sizeof(pthread_t));
  for (int i = 0; i < n_threads; i++) { W[i].ctx = &c; pthread_create(&th[i], NULL, worker, &W[i]); }
  for (int i = 0; i < n_threads; i++) pthread_join(th[i], NULL);
  replist all = {0};
  ostats S; memset(&S, 0, sizeof S);
  for (int i = 0; i < n_threads; i++) {
    for (size_t j = 0; j < W[i].out.reps.n; j++) rep_push(&all, W[i].out.reps.v[j]);
    free(W[i].out.reps.v);
    S.checked += W[i].out.st.checked; S.loads += W[i].out.st.loads; S.stores += W[i].out.st.stores;
    S.instructions += W[i].out.st.instructions;
    if (W[i].out.st.intervals_max > S.intervals_max) S.intervals_max = W[i].out.st.intervals_max;
    for (int q = 0; q < 8; q++) S.lanes_final[q] += W[i].out.st.lanes_final[q];
    for (int q = 0; q < 32; q++) S.op_count[q] += W[i].out.st.op_count[q];
  }
  if (all.n) qsort(all.v, all.n, sizeof(orep), rep_cmp);
  *reports = all.v; *n_reports = all.n;
  if (stats) {
    stats[0] = S.checked; stats[1] = S.loads; stats[2] = S.stores; stats[3] = S.instructions;
    stats[4] = S.intervals_max;
    for (int q = 0; q < 8; q++) stats[5 + q] = S.lanes_final[q];
    for (int q = 0; q < 32; q++) stats[13 + q] = S.op_count[q];
  }
  free(W); free(th); free(P.code);
  pthread_mutex_destroy(&c.mu);
  return 0;
}

void oracle_free(void* p) { free(p); }

/* Public: canonical state at the START of interval k of ONE instance
 * (heap per array concatenated into heap_out, lane regs/pc/status).
 * Returns 1 if interval k is reached, 0 if the instance ended earlier, -1 on
 * a decode error. */
int oracle_state_at(const uint8_t* bc, size_t nbytes, uint32_t n, const uint32_t* sizes,
                    const int32_t* const* inputs, uint64_t fuel, uint32_t k,
                    int32_t* heap_out, int32_t* regs_out, uint32_t* pc_out, uint8_t* status_out) {
  oprog P;
  if (decode(bc, nbytes, &P)) return -1;
  int32_t** heap = (int32_t**)malloc((P.n_arrays + 1) * sizeof(int32_t*));
  for (uint32_t a = 0; a < P.n_arrays; a++) {
    heap[a] = (int32_t*)malloc(((size_t)sizes[a] + 1) * sizeof(int32_t));
    memcpy(heap[a], inputs[a], (size_t)sizes[a] * sizeof(int32_t));
  }
  replist reps = {0}; ostats st; memset(&st, 0, sizeof st);
  const ogroup G = {0, 0, n}; /* (work-group 0) */
  int reached = run_instance(&P, n, &G, sizes, heap, 0, fuel, 0xFFFFFFFFu, &reps, &st, (int)k,
                             regs_out, pc_out, status_out, NULL, 0, NULL);
  size_t off = 0;
  for (uint32_t a = 0; a < P.n_arrays; a++) {
    memcpy(heap_out + off, heap[a], (size_t)sizes[a] * sizeof(int32_t));
    off += sizes[a];
    free(heap[a]);
  }
  free(heap); free(reps.v); free(P.code);
  return reached;
}

/* ---- (2) the brute-force interleaving enumerator ------
 * State = every thread's (pc, registers, status, steps) + ONE shared heap.
 * A global step picks any RUNNING thread and applies one thread-local rule
 * to the shared heap with immediate visibility
 * (PAPER.md:212).  The interval ends when no thread is RUNNING (all
 * suspended at a barrier, exited, or stopped by ⊥/⊤ as readings
 * L5/L6).  Explores every interleaving; with memo != 0 identical states are
 * merged (schedule counts are summed), without memo every schedule is walked
 * (used for the C(a+b,a) count check). */

typedef struct {
  const oprog* P; uint32_t n; const uint32_t* sizes; uint32_t cells; uint64_t fuel;
  size_t state_words;                  /* int32 words per state */
  /* memo table: open addressing over state blobs */
  int32_t* keys; uint64_t* counts; uint8_t* used; size_t tcap, tn;
  /* terminal set */
  int32_t* terms; uint8_t* tused; size_t ttcap, ttn;
  uint64_t n_schedules; int memo; int reduced; uint64_t budget; int over_budget;
} enumctx;

/* state layout (int32 words): heap[cells] | per thread: pc, status, steps_lo, steps_hi, regs[R] */
static size_t lane_words(const oprog* P) { return 4 + P->n_regs; }

static uint64_t hash_words(const int32_t* w, size_t n) {
  uint64_t h = 1469598103934665603ull;
  for (size_t i = 0; i < n; i++) { h ^= (uint32_t)w[i]; h *= 1099511628211ull; h ^= h >> 29; }
  return h;
}

static int set_insert(int32_t** keys, uint8_t** used, size_t* cap, size_t* cnt, size_t words,
                      const int32_t* s, size_t* slot_out, uint64_t** counts) {
  if ((*cnt + 1) * 2 > *cap) { /* grow */
    size_t ncap = *cap ? *cap * 2 : 1024;
    int32_t* nk = (int32_t*)malloc(ncap * words * sizeof(int32_t));
    uint8_t* nu = (uint8_t*)calloc(ncap, 1);
    uint64_t* nc = counts ? (uint64_t*)calloc(ncap, sizeof(uint64_t)) : NULL;
    for (size_t i = 0; i < *cap; i++) if ((*used)[i]) {
      size_t h = hash_words(*keys + i * words, words) & (ncap - 1);
      while (nu[h]) h = (h + 1) & (ncap - 1);
      nu[h] = 1; memcpy(nk + h * words, *keys + i * words, words * sizeof(int32_t));
      if (counts) nc[h] = (*counts)[i];
    }
    free(*keys); free(*used); *keys = nk; *used = nu; *cap = ncap;
    if (counts) { free(*counts); *counts = nc; }
  }
  size_t h = hash_words(s, words) & (*cap - 1);
  while ((*used)[h]) {
    if (!memcmp(*keys + h * words, s, words * sizeof(int32_t))) { *slot_out = h; return 0; }
    h = (h + 1) & (*cap - 1);
  }
  (*used)[h] = 1; memcpy(*keys + h * words, s, words * sizeof(int32_t)); (*cnt)++;
  *slot_out = h;
  return 1;
}

/* apply one step of thread t to state s (in place). */
static void enum_step(enumctx* E, int32_t* s, uint32_t t) {
  const oprog* P = E->P;
  int32_t* heap = s;
  int32_t* L = s + E->cells + (size_t)t * lane_words(P);
  uint32_t* pc = (uint32_t*)&L[0];
  int32_t* st = &L[1];
  uint64_t steps = (uint32_t)L[2] | ((uint64_t)(uint32_t)L[3] << 32);
  int32_t* r = L + 4;
  if (steps == E->fuel) { *st = S_FUEL; return; }
  steps++;
  L[2] = (int32_t)(uint32_t)steps; L[3] = (int32_t)(uint32_t)(steps >> 32);
  const oins* I = &P->code[*pc];
  int fault;
  const ogroup G = {0, 0, E->n}; /* the enumerator explores one work-group (group 0) */
  if (step_private(P, I, r, t, &G, E->sizes, pc, &fault)) { if (fault) *st = fault; return; }
  size_t base = 0;
  switch (I->op) {
    case O_LD: {
      for (uint32_t a = 0; a < I->b; a++) base += E->sizes[a];
      int32_t idx = r[I->c];
      if (idx < 0 || (uint32_t)idx >= E->sizes[I->b]) { *st = S_OOB; return; }
      r[I->a] = heap[base + (uint32_t)idx]; (*pc)++; return;
    }
    case O_ST: {
      for (uint32_t a = 0; a < I->a; a++) base += E->sizes[a];
      int32_t idx = r[I->b];
      if (idx < 0 || (uint32_t)idx >= E->sizes[I->a]) { *st = S_OOB; return; }
      heap[base + (uint32_t)idx] = r[I->c]; (*pc)++; return;
    }
    case O_BAR: *st = S_WAITING; (*pc)++; return;
    case O_EXIT: *st = S_EXITED; return;
    case O_ASSUME: if (r[I->a] == 0) *st = S_PRUNED; else (*pc)++; return;
    case O_ASSERT: if (r[I->a] == 0) *st = S_ASSERT; else (*pc)++; return;
    default: abort();
  }
}

static uint64_t enum_dfs(enumctx* E, int32_t* s) {
  if (E->over_budget) return 0;
  size_t W = E->state_words, LW = lane_words(E->P);
  int any = 0;
  for (uint32_t t = 0; t < E->n; t++) if (s[E->cells + (size_t)t * LW + 1] == S_RUNNING) { any = 1; break; }
  if (!any) { /* end of interval: record the terminal state (steps zeroed: not observable) */
    int32_t* c = (int32_t*)malloc(W * sizeof(int32_t));
    memcpy(c, s, W * sizeof(int32_t));
    for (uint32_t t = 0; t < E->n; t++) { c[E->cells + (size_t)t * LW + 2] = 0; c[E->cells + (size_t)t * LW + 3] = 0; }
    size_t slot;
    set_insert(&E->terms, &E->tused, &E->ttcap, &E->ttn, W, c, &slot, NULL);
    free(c);
    return 1;
  }
  size_t slot = 0;
  if (E->memo) {
    if (!set_insert(&E->keys, &E->used, &E->tcap, &E->tn, W, s, &slot, &E->counts))
      return E->counts[slot];
    if (E->tn > E->budget) { E->over_budget = 1; return 0; }
  } else {
    if (++E->tn > E->budget) { E->over_budget = 1; return 0; }
  }
  uint64_t total = 0;
  int32_t* nxt = (int32_t*)malloc(W * sizeof(int32_t));
  /* reduced: a step that touches no shared cell (everything but LD / ST:
   * it reads and writes only the thread's own τ — pc, status, registers,
   * fuel — PAPER.md:168-201) commutes with every step of every other
   * thread, so running the lowest such thread first reaches the same set of
   * terminal states; only LD / ST remain scheduling points. */
  int32_t eager = -1;
  for (uint32_t t = 0; E->reduced && t < E->n && eager < 0; t++) {
    const int32_t* L = s + E->cells + (size_t)t * LW;
    if (L[1] != S_RUNNING) continue;
    const uint8_t op = E->P->code[(uint32_t)L[0]].op;
    if (op != O_LD && op != O_ST) eager = (int32_t)t;
  }
  for (uint32_t t = 0; t < E->n; t++) {
    if (s[E->cells + (size_t)t * LW + 1] != S_RUNNING) continue;
    if (eager >= 0 && t != (uint32_t)eager) continue;
    memcpy(nxt, s, W * sizeof(int32_t));
    enum_step(E, nxt, t);
    total += enum_dfs(E, nxt);
  }
  free(nxt);
  if (E->memo) {
    /* re-find the slot (the table may have grown) */
    size_t h = hash_words(s, W) & (E->tcap - 1);
    while (memcmp(E->keys + h * W, s, W * sizeof(int32_t))) h = (h + 1) & (E->tcap - 1);
    E->counts[h] = total;
  }
  return total;
}

/* Public: explore all interleavings of one interval.
 * heap0: all arrays concatenated (cells words); regs0 [n][n_regs]; pc0[n];
 * status0[n] (0 = RUNNING, others are left as they are).
 * Outputs: *n_schedules (saturating), terminal states malloc'd into *terms as
 * *n_terms rows of (cells + n*(4+n_regs)) int32 words (heap, then per thread
 * pc, status, 0, 0, regs).  Returns 0, or 1 if `budget` states/schedules were
 * exceeded (results incomplete), -1 on decode error.
 * memo: bit 0 = merge equal states (counts summed); bit 1 = reduced
 * scheduling (only LD / ST are interleaving points; the same terminal set,
 * fewer schedules — see enum_dfs). */
int oracle_enumerate(const uint8_t* bc, size_t nbytes, uint32_t n, const uint32_t* sizes,
                     const int32_t* heap0, const int32_t* regs0, const uint32_t* pc0,
                     const uint8_t* status0, uint64_t fuel, int memo, uint64_t budget,
                     uint64_t* n_schedules, int32_t** terms, uint64_t* n_terms, uint64_t* row_words) {
  oprog P;
  if (decode(bc, nbytes, &P)) return -1;
  enumctx E;
  memset(&E, 0, sizeof E);
  E.P = &P; E.n = n; E.sizes = sizes; E.fuel = fuel; E.memo = memo & 1; E.reduced = (memo >> 1) & 1;
  E.budget = budget;
  for (uint32_t a = 0; a < P.n_arrays; a++) E.cells += sizes[a];
  size_t LW = lane_words(&P);
  E.state_words = E.cells + (size_t)n * LW;
  int32_t* s = (int32_t*)calloc(E.state_words, sizeof(int32_t));
  memcpy(s, heap0, E.cells * sizeof(int32_t));
  for (uint32_t t = 0; t < n; t++) {
    int32_t* L = s + E.cells + (size_t)t * LW;
    L[0] = (int32_t)pc0[t]; L[1] = status0[t]; L[2] = 0; L[3] = 0;
    memcpy(L + 4, regs0 + (size_t)t * P.n_regs, P.n_regs * sizeof(int32_t));
  }
  uint64_t cnt = enum_dfs(&E, s);
  *n_schedules = cnt;
  *row_words = E.state_words;
  *n_terms = E.ttn;
  int32_t* out = (int32_t*)malloc((E.ttn ? E.ttn : 1) * E.state_words * sizeof(int32_t));
  size_t o = 0;
  for (size_t i = 0; i < E.ttcap; i++)
    if (E.tused[i]) { memcpy(out + o * E.state_words, E.terms + i * E.state_words, E.state_words * sizeof(int32_t)); o++; }
  *terms = out;
  free(s); free(E.keys); free(E.counts); free(E.used); free(E.terms); free(E.tused); free(P.code);
  return E.over_budget ? 1 : 0;
}
