/*
 * bitrev_oracle.c -- TEST INFRASTRUCTURE ONLY (CPU oracle and CPU baseline).
 *
 * A plain-C restatement of the reference package's algorithms for the
 * bit-reversed permutation path (/root/reference/pkg/src/bitrev, "src/" below).
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
 * arm load it (through oracle/oracle.py); the product library never does.
 *
 *   oracle_gather                 src/verify.py:19-39   (rev table + gather)
 *   oracle_cobra_oop              src/permutations.py:225-249, 293-308
 *   oracle_cobra_inplace          src/permutations.py:252-285, 311-321
 *   oracle_recursive              src/recursive.py:27-228 with the swap
 *                                 schedules of src/schedule.py:23-121
 *   oracle_parallel_semi_recursive src/parallel.py:60-156 (pthreads)
 *   oracle_bitwise_inplace        src/permutations.py:66-88 (paper Listing 1)
 *
 * Elements are moved as opaque E-byte words (E in {1,2,4,8,16}); every
 * function returns 0 on success, negative on a bad argument.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define SCHEDULE_MAX_BITS 26 /* src/schedule.py:17-19 */
#define TRANSPOSE_LEAF 8     /* src/recursive.py:27 */

typedef struct {
  uint64_t lo, hi;
} w128;

static uint64_t rev_bits(uint64_t v, int w) { /* src/bits.py:31-47 */
  uint64_t r = 0;
  for (int k = 0; k < w; ++k) {
    r = (r << 1) | (v & 1);
    v >>= 1;
  }
  return r;
}

/* ------------------------------------------------------------------------ */
/* swap schedules (src/schedule.py:23-97)                                   */

static int64_t swap_count(int b) { /* closed form of the recurrence, :23-37 */
  return (int64_t)(((uint64_t)1 << b) - ((uint64_t)1 << ((b + 1) / 2))) / 2;
}

static int64_t fill_pairs(int64_t base, int depth, int b, int64_t* out, int64_t pos) {
  /* src/schedule.py:53-75: fix one (top, bottom) bit pair per level */
  const int rem = b - 2 * depth;
  if (rem < 2) return pos;
  pos = fill_pairs(base, depth + 1, b, out, pos);
  const int mid = rem - 2;
  const int64_t lo_bit = (int64_t)1 << depth;
  const int64_t hi_bit = (int64_t)1 << (b - 1 - depth);
  for (int64_t x = 0; x < ((int64_t)1 << mid); ++x) {
    const int64_t rx = (int64_t)rev_bits((uint64_t)x, mid);
    out[2 * pos] = base | (x << (depth + 1)) | lo_bit;
    out[2 * pos + 1] = base | (rx << (depth + 1)) | hi_bit;
    ++pos;
  }
  return fill_pairs(base | lo_bit | hi_bit, depth + 1, b, out, pos);
}

static int64_t* g_sched[SCHEDULE_MAX_BITS + 1];
static pthread_mutex_t g_sched_mu = PTHREAD_MUTEX_INITIALIZER;

static const int64_t* cached_schedule(int b) { /* src/schedule.py:94-97 */
  pthread_mutex_lock(&g_sched_mu);
  if (!g_sched[b]) {
    const int64_t cnt = swap_count(b);
    int64_t* p = (int64_t*)malloc((size_t)(cnt > 0 ? cnt : 1) * 2 * sizeof(int64_t));
    fill_pairs(0, 0, b, p, 0);
    g_sched[b] = p;
  }
  pthread_mutex_unlock(&g_sched_mu);
  return g_sched[b];
}

int64_t oracle_swap_count(int b) { return (b >= 1 && b <= 62) ? swap_count(b) : -1; }

int oracle_schedule(int b, int64_t* out) {
  if (b < 1 || b > SCHEDULE_MAX_BITS) return -1;
  fill_pairs(0, 0, b, out, 0);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* element-typed kernels, instantiated per word type                        */

#define DEFINE_KERNELS(T, SFX)                                                                  \
  static void gather_##SFX(const T* src, T* dst, int b) {                                       \
    const int64_t n = (int64_t)1 << b;                                                          \
    for (int64_t i = 0; i < n; ++i) dst[i] = src[rev_bits((uint64_t)i, b)];                     \
  }                                                                                             \
  static void cobra_copy_##SFX(const T* src, T* dst, T* buf, int b, int q, const int64_t* rq) { \
    const int64_t side = (int64_t)1 << q;                                                       \
    const int mid = b - 2 * q, hi_shift = b - q;                                                \
    for (int64_t y = 0; y < ((int64_t)1 << mid); ++y) {                                         \
      const int64_t ry = (int64_t)rev_bits((uint64_t)y, mid);                                   \
      const int64_t y_base = y << q, ry_base = ry << q;                                         \
      for (int64_t x = 0; x < side; ++x) {                                                      \
        const int64_t sb = (x << hi_shift) | y_base, bb = rq[x] << q;                           \
        for (int64_t z = 0; z < side; ++z) buf[bb + z] = src[sb + z];                           \
      }                                                                                         \
      for (int64_t z = 0; z < side; ++z) {                                                      \
        const int64_t db = (rq[z] << hi_shift) | ry_base;                                       \
        for (int64_t x = 0; x < side; ++x) dst[db + x] = buf[(x << q) + z];                     \
      }                                                                                         \
    }                                                                                           \
  }                                                                                             \
  static void cobra_swap_##SFX(T* a, T* buf, int b, int q, const int64_t* rq) {                 \
    const int64_t side = (int64_t)1 << q;                                                       \
    const int mid = b - 2 * q, hi_shift = b - q;                                                \
    for (int64_t y = 0; y < ((int64_t)1 << mid); ++y) {                                         \
      const int64_t ry = (int64_t)rev_bits((uint64_t)y, mid);                                   \
      if (ry < y) continue;                                                                     \
      const int64_t y_base = y << q, ry_base = ry << q;                                         \
      for (int64_t x = 0; x < side; ++x) {                                                      \
        const int64_t sb = (x << hi_shift) | y_base, bb = rq[x] << q;                           \
        for (int64_t z = 0; z < side; ++z) buf[bb + z] = a[sb + z];                             \
      }                                                                                         \
      for (int64_t z = 0; z < side; ++z) {                                                      \
        const int64_t db = (rq[z] << hi_shift) | ry_base;                                       \
        for (int64_t x = 0; x < side; ++x) {                                                    \
          const T t = a[db + x];                                                                \
          a[db + x] = buf[(x << q) + z];                                                        \
          buf[(x << q) + z] = t;                                                                \
        }                                                                                       \
      }                                                                                         \
      for (int64_t x = 0; x < side; ++x) {                                                      \
        const int64_t sb = (x << hi_shift) | y_base, bb = rq[x] << q;                           \
        for (int64_t z = 0; z < side; ++z) a[sb + z] = buf[bb + z];                             \
      }                                                                                         \
    }                                                                                           \
  }                                                                                             \
  static void apply_pairs_##SFX(T* a, const int64_t* p, int64_t cnt) {                          \
    for (int64_t k = 0; k < cnt; ++k) {                                                         \
      const int64_t i = p[2 * k], j = p[2 * k + 1];                                             \
      const T t = a[i];                                                                         \
      a[i] = a[j];                                                                              \
      a[j] = t;                                                                                 \
    }                                                                                           \
  }                                                                                             \
  static void apply_pairs_blocks_##SFX(T* a, const int64_t* p, int64_t cnt, int64_t blen,       \
                                       int64_t lo, int64_t hi) {                                \
    for (int64_t blk = lo; blk < hi; ++blk) apply_pairs_##SFX(a + blk * blen, p, cnt);          \
  }                                                                                             \
  static void transpose_offdiag_##SFX(T* a, int64_t rl, int64_t r0, int64_t c0, int64_t sz) {   \
    if (sz <= TRANSPOSE_LEAF) {                                                                 \
      for (int64_t i = 0; i < sz; ++i)                                                          \
        for (int64_t j = 0; j < sz; ++j) {                                                      \
          const int64_t p = (r0 + i) * rl + c0 + j, s = (c0 + j) * rl + r0 + i;                 \
          const T t = a[p];                                                                     \
          a[p] = a[s];                                                                          \
          a[s] = t;                                                                             \
        }                                                                                       \
      return;                                                                                   \
    }                                                                                           \
    const int64_t h = sz >> 1;                                                                  \
    transpose_offdiag_##SFX(a, rl, r0, c0, h);                                                  \
    transpose_offdiag_##SFX(a, rl, r0, c0 + h, h);                                              \
    transpose_offdiag_##SFX(a, rl, r0 + h, c0, h);                                              \
    transpose_offdiag_##SFX(a, rl, r0 + h, c0 + h, h);                                          \
  }                                                                                             \
  static void transpose_diag_##SFX(T* a, int64_t rl, int64_t r0, int64_t sz) {                  \
    if (sz <= TRANSPOSE_LEAF) {                                                                 \
      for (int64_t i = 0; i < sz; ++i)                                                          \
        for (int64_t j = i + 1; j < sz; ++j) {                                                  \
          const int64_t p = (r0 + i) * rl + r0 + j, s = (r0 + j) * rl + r0 + i;                 \
          const T t = a[p];                                                                     \
          a[p] = a[s];                                                                          \
          a[s] = t;                                                                             \
        }                                                                                       \
      return;                                                                                   \
    }                                                                                           \
    const int64_t h = sz >> 1;                                                                  \
    transpose_diag_##SFX(a, rl, r0, h);                                                         \
    transpose_diag_##SFX(a, rl, r0 + h, h);                                                     \
    transpose_offdiag_##SFX(a, rl, r0, r0 + h, h);                                              \
  }                                                                                             \
  static void even_odd_##SFX(T* a, int64_t n, T* scratch) {                                     \
    const int64_t half = n >> 1;                                                                \
    for (int64_t j = 0; j < half; ++j) scratch[j] = a[2 * j + 1];                               \
    for (int64_t j = 0; j < half; ++j) a[j] = a[2 * j];                                         \
    for (int64_t j = 0; j < half; ++j) a[half + j] = scratch[j];                                \
  }                                                                                             \
  static void bitwise_##SFX(T* a, int b) {                                                      \
    const int64_t n = (int64_t)1 << b;                                                          \
    for (int64_t i = 1; i < n - 1; ++i) {                                                       \
      const int64_t r = (int64_t)rev_bits((uint64_t)i, b);                                      \
      if (i < r) {                                                                              \
        const T t = a[i];                                                                       \
        a[i] = a[r];                                                                            \
        a[r] = t;                                                                               \
      }                                                                                         \
    }                                                                                           \
  }

DEFINE_KERNELS(uint8_t, 1)
DEFINE_KERNELS(uint16_t, 2)
DEFINE_KERNELS(uint32_t, 4)
DEFINE_KERNELS(uint64_t, 8)
DEFINE_KERNELS(w128, 16)

/* Dispatch a call on element size E to the typed instance. */
#define DISPATCH(E, NAME, ...)                         \
  switch (E) {                                         \
    case 1: NAME##_1(__VA_ARGS__); break;              \
    case 2: NAME##_2(__VA_ARGS__); break;              \
    case 4: NAME##_4(__VA_ARGS__); break;              \
    case 8: NAME##_8(__VA_ARGS__); break;              \
    case 16: NAME##_16(__VA_ARGS__); break;            \
    default: return -2;                                \
  }

static int valid(int b, int E) {
  if (b < 1 || b > 48) return -1;
  if (E != 1 && E != 2 && E != 4 && E != 8 && E != 16) return -2;
  return 0;
}

/* ------------------------------------------------------------------------ */

int oracle_gather(const void* src, void* dst, int b, int E, int64_t batch) {
  int rc = valid(b, E);
  if (rc) return rc;
  const int64_t row = ((int64_t)1 << b) * E;
  for (int64_t r = 0; r < batch; ++r) {
    const char* s = (const char*)src + r * row;
    char* d = (char*)dst + r * row;
    DISPATCH(E, gather, (const void*)s, (void*)d, b)
  }
  return 0;
}

static int64_t* rev_table(int q) { /* src/permutations.py:219-222 */
  int64_t* t = (int64_t*)malloc(sizeof(int64_t) << q);
  for (int64_t x = 0; x < ((int64_t)1 << q); ++x) t[x] = (int64_t)rev_bits((uint64_t)x, q);
  return t;
}

int oracle_cobra_oop(const void* src, void* dst, int b, int E, int q) {
  int rc = valid(b, E);
  if (rc) return rc;
  if (q < 0 || 2 * q > b) return -3;
  void* buf = malloc((size_t)E << (2 * q));
  int64_t* rq = rev_table(q);
  switch (E) {
    case 1: cobra_copy_1(src, dst, buf, b, q, rq); break;
    case 2: cobra_copy_2(src, dst, buf, b, q, rq); break;
    case 4: cobra_copy_4(src, dst, buf, b, q, rq); break;
    case 8: cobra_copy_8(src, dst, buf, b, q, rq); break;
    case 16: cobra_copy_16(src, dst, buf, b, q, rq); break;
  }
  free(rq);
  free(buf);
  return 0;
}

int oracle_cobra_inplace(void* a, int b, int E, int q) {
  int rc = valid(b, E);
  if (rc) return rc;
  if (q < 0 || 2 * q > b) return -3;
  void* buf = malloc((size_t)E << (2 * q));
  int64_t* rq = rev_table(q);
  switch (E) {
    case 1: cobra_swap_1(a, buf, b, q, rq); break;
    case 2: cobra_swap_2(a, buf, b, q, rq); break;
    case 4: cobra_swap_4(a, buf, b, q, rq); break;
    case 8: cobra_swap_8(a, buf, b, q, rq); break;
    case 16: cobra_swap_16(a, buf, b, q, rq); break;
  }
  free(rq);
  free(buf);
  return 0;
}

int oracle_bitwise_inplace(void* a, int b, int E) {
  int rc = valid(b, E);
  if (rc) return rc;
  DISPATCH(E, bitwise, a, b)
  return 0;
}

/* ------------------------------------------------------------------------ */
/* recursive / semi-recursive driver (src/recursive.py:139-213)             */

typedef struct {
  int base_bits;
  int depth_limit; /* 0 = None */
} policy_t;

static int hits_base(int bb, int depth, const policy_t* p) { /* :139-149 */
  if (bb <= p->base_bits) return 1;
  return p->depth_limit > 0 && depth >= p->depth_limit && bb <= SCHEDULE_MAX_BITS;
}

static void apply_pairs_any(int E, void* a, const int64_t* p, int64_t cnt) {
  switch (E) {
    case 1: apply_pairs_1(a, p, cnt); break;
    case 2: apply_pairs_2(a, p, cnt); break;
    case 4: apply_pairs_4(a, p, cnt); break;
    case 8: apply_pairs_8(a, p, cnt); break;
    case 16: apply_pairs_16(a, p, cnt); break;
  }
}

static void apply_blocks_any(int E, void* a, const int64_t* p, int64_t cnt, int64_t blen, int64_t lo,
                             int64_t hi) {
  switch (E) {
    case 1: apply_pairs_blocks_1(a, p, cnt, blen, lo, hi); break;
    case 2: apply_pairs_blocks_2(a, p, cnt, blen, lo, hi); break;
    case 4: apply_pairs_blocks_4(a, p, cnt, blen, lo, hi); break;
    case 8: apply_pairs_blocks_8(a, p, cnt, blen, lo, hi); break;
    case 16: apply_pairs_blocks_16(a, p, cnt, blen, lo, hi); break;
  }
}

static void transpose_diag_any(int E, void* a, int64_t rl, int64_t r0, int64_t sz) {
  switch (E) {
    case 1: transpose_diag_1(a, rl, r0, sz); break;
    case 2: transpose_diag_2(a, rl, r0, sz); break;
    case 4: transpose_diag_4(a, rl, r0, sz); break;
    case 8: transpose_diag_8(a, rl, r0, sz); break;
    case 16: transpose_diag_16(a, rl, r0, sz); break;
  }
}

static void transpose_offdiag_any(int E, void* a, int64_t rl, int64_t r0, int64_t c0, int64_t sz) {
  switch (E) {
    case 1: transpose_offdiag_1(a, rl, r0, c0, sz); break;
    case 2: transpose_offdiag_2(a, rl, r0, c0, sz); break;
    case 4: transpose_offdiag_4(a, rl, r0, c0, sz); break;
    case 8: transpose_offdiag_8(a, rl, r0, c0, sz); break;
    case 16: transpose_offdiag_16(a, rl, r0, c0, sz); break;
  }
}

static void even_odd_any(int E, void* a, int64_t n, void* scratch) {
  switch (E) {
    case 1: even_odd_1(a, n, scratch); break;
    case 2: even_odd_2(a, n, scratch); break;
    case 4: even_odd_4(a, n, scratch); break;
    case 8: even_odd_8(a, n, scratch); break;
    case 16: even_odd_16(a, n, scratch); break;
  }
}

static void run_rec(int E, char* a, int64_t off, int bb, int depth, const policy_t* p,
                    char* scratch) { /* src/recursive.py:152-186 (trace-free path) */
  const int64_t n = (int64_t)1 << bb;
  if (hits_base(bb, depth, p)) {
    apply_pairs_any(E, a + off * E, cached_schedule(bb), swap_count(bb));
    return;
  }
  const int nxt = depth + 1;
  if (bb & 1) {
    const int64_t half = n >> 1;
    even_odd_any(E, a + off * E, n, scratch);
    run_rec(E, a, off, bb - 1, nxt, p, scratch);
    run_rec(E, a, off + half, bb - 1, nxt, p, scratch);
    return;
  }
  const int h = bb >> 1;
  const int64_t m = (int64_t)1 << h;
  char* view = a + off * E;
  if (hits_base(h, nxt, p)) {
    const int64_t* pairs = cached_schedule(h);
    apply_blocks_any(E, view, pairs, swap_count(h), m, 0, m);
    transpose_diag_any(E, view, m, 0, m);
    apply_blocks_any(E, view, pairs, swap_count(h), m, 0, m);
    return;
  }
  for (int64_t blk = 0; blk < m; ++blk) run_rec(E, a, off + blk * m, h, nxt, p, scratch);
  transpose_diag_any(E, view, m, 0, m);
  for (int64_t blk = 0; blk < m; ++blk) run_rec(E, a, off + blk * m, h, nxt, p, scratch);
}

int oracle_recursive(void* a, int b, int E, int base_bits, int depth_limit) {
  int rc = valid(b, E);
  if (rc) return rc;
  if (base_bits < 1 || base_bits > SCHEDULE_MAX_BITS || depth_limit < 0) return -3;
  policy_t p = {base_bits, depth_limit};
  char* scratch = (char*)malloc((size_t)E << (b - 1 > 0 ? b - 1 : 0));
  run_rec(E, (char*)a, 0, b, 0, &p, scratch);
  free(scratch);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* threaded semi-recursive variant (src/parallel.py:60-156)                 */

typedef struct {
  int kind; /* 0 diag, 1 offdiag */
  int64_t r0, c0, size;
} tile_item;

typedef struct {
  int E;
  char* a;
  int phase; /* 0 blocks, 1 tiles */
  const int64_t* pairs;
  int64_t npairs, m;
  const int64_t (*chunks)[2];
  int nchunks;
  const tile_item* tiles;
  int ntiles;
  volatile int next; /* dynamic work counter (like pool.submit order) */
  pthread_mutex_t mu;
} phase_ctx;

static int take(phase_ctx* c) {
  pthread_mutex_lock(&c->mu);
  const int k = c->next++;
  pthread_mutex_unlock(&c->mu);
  return k;
}

static void* worker(void* arg) {
  phase_ctx* c = (phase_ctx*)arg;
  for (;;) {
    const int k = take(c);
    if (c->phase == 0) {
      if (k >= c->nchunks) break;
      apply_blocks_any(c->E, c->a, c->pairs, c->npairs, c->m, c->chunks[k][0], c->chunks[k][1]);
    } else {
      if (k >= c->ntiles) break;
      const tile_item* t = &c->tiles[k];
      if (t->kind == 0)
        transpose_diag_any(c->E, c->a, c->m, t->r0, t->size);
      else
        transpose_offdiag_any(c->E, c->a, c->m, t->r0, t->c0, t->size);
    }
  }
  return NULL;
}

typedef struct {
  int E;
  char* a;
  int bb;
  const policy_t* p;
  char* scratch;
} half_job;

static void* half_worker(void* arg) {
  half_job* j = (half_job*)arg;
  run_rec(j->E, j->a, 0, j->bb, 1, j->p, j->scratch);
  return NULL;
}

static void run_phase(phase_ctx* c, int workers) {
  pthread_t th[256];
  if (workers > 256) workers = 256;
  c->next = 0;
  for (int t = 0; t < workers; ++t) pthread_create(&th[t], NULL, worker, c);
  for (int t = 0; t < workers; ++t) pthread_join(th[t], NULL);
}

int oracle_parallel_semi_recursive(void* a, int b, int E, int base_bits, int threads) {
  int rc = valid(b, E);
  if (rc) return rc;
  if (threads < 1 || base_bits < 1 || base_bits > SCHEDULE_MAX_BITS) return -3;
  policy_t p = {base_bits, 1};
  const int64_t n = (int64_t)1 << b;
  if (b <= base_bits) { /* :116-118 */
    run_rec(E, (char*)a, 0, b, 0, &p, NULL);
    return 0;
  }
  if (b & 1) { /* :121-137 */
    const int64_t half = n >> 1, quarter = half >> 1;
    char* scratch = (char*)malloc((size_t)half * E);
    even_odd_any(E, a, n, scratch);
    half_job jobs[2] = {{E, (char*)a, b - 1, &p, scratch},
                        {E, (char*)a + half * E, b - 1, &p, scratch + quarter * E}};
    if (threads >= 2) {
      pthread_t th[2];
      for (int t = 0; t < 2; ++t) pthread_create(&th[t], NULL, half_worker, &jobs[t]);
      for (int t = 0; t < 2; ++t) pthread_join(th[t], NULL);
    } else {
      half_worker(&jobs[0]);
      half_worker(&jobs[1]);
    }
    free(scratch);
    return 0;
  }
  const int h = b >> 1;
  const int64_t m = (int64_t)1 << h;
  /* chunk_ranges(m, workers), :60-66 */
  int workers = threads < m ? threads : (int)m;
  const int64_t step = (m + workers - 1) / workers;
  int64_t(*chunks)[2] = malloc(sizeof(int64_t[2]) * (size_t)workers);
  int nchunks = 0;
  for (int64_t lo = 0; lo < m; lo += step) {
    chunks[nchunks][0] = lo;
    chunks[nchunks][1] = lo + step < m ? lo + step : m;
    ++nchunks;
  }
  /* transpose_tiles(h, bands=8), :69-84 */
  const int bands = 8;
  tile_item tiles[64];
  int ntiles = 0;
  if (m <= TRANSPOSE_LEAF || m < bands) {
    tiles[ntiles++] = (tile_item){0, 0, 0, m};
  } else {
    const int64_t tile = m / bands;
    for (int i = 0; i < bands; ++i) {
      tiles[ntiles++] = (tile_item){0, i * tile, i * tile, tile};
      for (int j = i + 1; j < bands; ++j) tiles[ntiles++] = (tile_item){1, i * tile, j * tile, tile};
    }
  }
  phase_ctx c;
  memset(&c, 0, sizeof c);
  pthread_mutex_init(&c.mu, NULL);
  c.E = E;
  c.a = (char*)a;
  c.pairs = cached_schedule(h);
  c.npairs = swap_count(h);
  c.m = m;
  c.chunks = (const int64_t(*)[2])chunks;
  c.nchunks = nchunks;
  c.tiles = tiles;
  c.ntiles = ntiles;
  for (int ph = 0; ph < 3; ++ph) { /* blocks, tiles, blocks; join = barrier */
    c.phase = (ph == 1);
    run_phase(&c, threads);
  }
  pthread_mutex_destroy(&c.mu);
  free(chunks);
  return 0;
}
