/*
 * dsk_oracle.c -- CPU restatement of the dartsketch hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path (paper_2005_11547_b200/csrc).  Only tests/, the smoke() check in
 * __graft_entry__.py and bench.py's cpu_baseline / --impl reference leg may load
 * it.  It is never part of the product path.
 *
 * It restates, scalar and single-threaded per set, the reference algorithm of
 * the Python package `dartsketch` (read-only at /root/reference/pkg/src):
 *   ref/ = /root/reference/pkg/src/dartsketch/
 *   - tabulation hash + splitmix64 finalizer   ref/randomness.py:58-63, 121-131
 *   - uniform / poisson1 / fingerprint / bucket ref/randomness.py:140-158
 *   - Poisson(1) CDF table                      ref/randomness.py:66-85
 *   - mix64 (LSH key fold)                      ref/randomness.py:160-166
 *   - l1 = np.sum(weights) (numpy pairwise)     ref/core.py:44
 *   - minhash_density                           ref/core.py:150-156
 *   - DartHasher.dart_batch (Algorithm 1)       ref/darthash.py:80-95, 142-295
 *   - _minhash_values / _bucket_minima          ref/sketching.py:93-112
 *   - lsh_key                                   ref/annindex.py:64-82
 *   - weight_class / scale_pow2                 ref/annindex.py:39-44, ref/core.py:57-60
 * It is pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py) and the reference's known answers.
 *
 * Compile with -ffp-contract=off: every floating-point expression of the
 * reference is a sequence of separately rounded IEEE operations.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "dsk_oracle.h"

#define MIX_MUL1 0xBF58476D1CE4E5B9ULL
#define MIX_MUL2 0x94D049BB133111EBULL
#define MAX_PHI_STEPS 64                      /* ref/sketching.py:22, ref/annindex.py:21 */
#define MAX_AREAS_PER_CALL ((double)(1 << 27)) /* ref/darthash.py:32 */
#define CAND_CLIP 1099511627776.0             /* 2^40, ref/darthash.py:36 */

/* ---------------------------------------------------------------- hashing */

/* ref/randomness.py:58-63 */
uint64_t or_finalize(uint64_t h) {
  h ^= h >> 30;
  h *= MIX_MUL1;
  h ^= h >> 27;
  h *= MIX_MUL2;
  return h ^ (h >> 31);
}

/* ref/randomness.py:121-131: key = pack("<QBBIIHH", element, nu&0xFF,
 * rho&0xFF, w&0xFFFFFFFF, r&0xFFFFFFFF, j&0xFFFF, stream&0xFFFF); XOR of one
 * table entry per key byte; splitmix64 finalizer. */
uint64_t or_hash64(const uint64_t *tab, uint64_t element, uint64_t nu, uint64_t rho,
                   uint64_t w, uint64_t r, uint64_t j, uint64_t stream) {
  uint8_t key[22];
  for (int p = 0; p < 8; p++) key[p] = (uint8_t)(element >> (8 * p));
  key[8] = (uint8_t)nu;
  key[9] = (uint8_t)rho;
  for (int p = 0; p < 4; p++) key[10 + p] = (uint8_t)(w >> (8 * p));
  for (int p = 0; p < 4; p++) key[14 + p] = (uint8_t)(r >> (8 * p));
  key[18] = (uint8_t)j;
  key[19] = (uint8_t)(j >> 8);
  key[20] = (uint8_t)stream;
  key[21] = (uint8_t)(stream >> 8);
  uint64_t h = 0;
  for (int p = 0; p < 22; p++) h ^= tab[p * 256 + key[p]];
  return or_finalize(h);
}

/* ref/randomness.py:140-143 */
static double or_uniform(const uint64_t *tab, uint64_t e, int nu, int rho, uint64_t w,
                         uint64_t r, uint64_t j, int stream) {
  return (double)(or_hash64(tab, e, nu, rho, w, r, j, stream) >> 11) * 0x1p-53;
}

/* ref/randomness.py:145-147 (bisect_right over the CDF list) */
static int or_poisson1(const uint64_t *tab, const double *cdf, uint64_t e, int nu, int rho,
                       uint64_t w, uint64_t r) {
  double u = or_uniform(tab, e, nu, rho, w, r, 0, OR_STREAM_POISSON);
  int lo = 0, hi = 64;
  while (lo < hi) { /* first index with cdf[idx] > u */
    int mid = (lo + hi) / 2;
    if (u < cdf[mid]) hi = mid; else lo = mid + 1;
  }
  return lo;
}

/* ref/randomness.py:66-82 */
void or_poisson1_cdf(double *cdf) {
  double term = exp(-1.0);
  double total = term;
  cdf[0] = total;
  for (int n = 1; n < 64; n++) {
    term /= (double)n;
    total += term;
    cdf[n] = total;
  }
  cdf[63] = 1.0;
}

/* ref/randomness.py:160-166 */
uint64_t or_mix64(const uint64_t *tab, const uint64_t *values, int64_t n) {
  uint64_t mixed = 0;
  for (int64_t pos = 0; pos < n; pos++)
    mixed = or_hash64(tab, values[pos] ^ mixed, 0, 0, (uint64_t)pos, 0, 0, OR_STREAM_KEY_MIX);
  return mixed;
}

/* ------------------------------------------------------------ set helpers */

/* numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
 * pairwise_sum_DOUBLE, PW_BLOCKSIZE 128), which is what
 * `float(np.sum(weights))` computes for a contiguous float64 vector
 * (ref/core.py:44). */
double or_pairwise_sum(const double *a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; i++) res += a[i];
    return res;
  } else if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; j++) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return or_pairwise_sum(a, n2) + or_pairwise_sum(a + n2, n - n2);
  }
}

/* ref/core.py:150-156 */
int64_t or_minhash_density(int64_t k) {
  if (k < 1) return -1;
  if (k == 1) return 1;
  return (int64_t)ceil((double)k * log((double)k)) + k;
}

/* ref/annindex.py:39-44 */
int or_weight_class(double l1) {
  int e;
  frexp(l1, &e);
  return e - 1;
}

/* floor(math.log2(y)) as an int; returns INT32_MAX for inf/NaN (the
 * reference raises OverflowError there, mapped to OR_OVERFLOW). */
static int floor_log2(double y) {
  double l = log2(y);
  if (!isfinite(l)) return INT32_MAX;
  return (int)floor(l);
}

/* ---------------------------------------------------------- dart vectors */

static int dv_push(or_dart_vec *v, const or_dart *d) {
  if (v->size == v->cap) {
    int64_t nc = v->cap ? v->cap * 2 : 1024;
    or_dart *nd = (or_dart *)realloc(v->data, (size_t)nc * sizeof(or_dart));
    if (!nd) return -1;
    v->data = nd;
    v->cap = nc;
  }
  v->data[v->size++] = *d;
  return 0;
}

void or_dart_vec_free(or_dart_vec *v) {
  free(v->data);
  v->data = NULL;
  v->size = v->cap = 0;
}

/* ref/darthash.py:80-95 */
static int64_t largest_passing(double quotient, int nu_bits, double origin, double step,
                               double bound) {
  /* limit_idx = 2^nu_bits - 1 as an exact integer (saturated; candidates are
   * at most 2^40 + 2 so saturation never changes a comparison) */
  int64_t limit_idx = nu_bits >= 62 ? INT64_MAX : (((int64_t)1 << nu_bits) - 1);
  double capf = nu_bits <= 40 ? (double)limit_idx : CAND_CLIP;
  double q = quotient < capf ? quotient : capf; /* Python min(quotient, capf) */
  int64_t base = (int64_t)floor(q);
  for (int delta = 2; delta >= -2; delta--) {
    int64_t c = base + delta;
    if (c < 0 || c > limit_idx) continue;
    if (origin + (double)c * step <= bound) return c;
  }
  return -1;
}

typedef struct {
  uint64_t elem;
  double xi;
  int nu, rho;
  int64_t w_hi, r_hi;
  double w0, dnu, r0, drho;
} region_t;

/* ref/darthash.py:142-295, scalar form.  Appends every dart hitting the set
 * with rank <= limit.  Returns OR_OK or an OR_* error status. */
int or_dart_batch(const uint64_t *tab, const double *cdf, int64_t t, const uint64_t *ids,
                  const double *x, int64_t n, double limit, or_dart_vec *out) {
  if (n == 0) return OR_EMPTY;                        /* :144 (_check_set) */
  if (!(limit > 0) || isinf(limit)) return OR_LIMIT;  /* :145 (_check_limit) */
  double tf = (double)t;
  int max_depth = -1;
  int *depth = (int *)malloc((size_t)n * sizeof(int));
  if (!depth) return OR_NOMEM;
  for (int64_t i = 0; i < n; i++) { /* :154-156 */
    depth[i] = floor_log2(1.0 + tf * x[i]);
    if (depth[i] > max_depth) max_depth = depth[i];
  }
  if (max_depth == INT32_MAX) { /* :154-156: math.floor(math.log2(inf)) raises OverflowError */
    free(depth);
    return OR_OVERFLOW;
  }
  int rank_depth = floor_log2(1.0 + limit); /* :157 */
  if (max_depth > 255 || rank_depth > 255) { /* :159-160 */
    free(depth);
    return OR_DEPTH;
  }
  /* regions (:180-225); the reference groups elements by depth, the set of
   * (element, nu, rho) regions and their rectangles are identical */
  int64_t nreg = 0, creg = 0;
  region_t *regs = NULL;
  double total_areas = 0.0;
  for (int nu = 0; nu <= max_depth; nu++) {
    double p2nu = ldexp(1.0, nu);
    for (int rho = 0; rho <= rank_depth; rho++) {
      double p2rho = ldexp(1.0, rho);
      double w0 = (p2nu - 1.0) / tf;
      double r0 = p2rho - 1.0;
      double dnu = p2nu / (tf * p2rho);
      double drho = p2rho / p2nu;
      int64_t r_hi = largest_passing(limit >= r0 ? (limit - r0) / drho : -1.0, nu, r0, drho,
                                     limit);
      if (r_hi < 0) continue;
      double wmax = ldexp(1.0, rho) - 1.0; /* float(wmax) as numpy compares it */
      double capw = wmax < CAND_CLIP ? wmax : CAND_CLIP;
      for (int64_t i = 0; i < n; i++) {
        if (depth[i] < nu) continue;
        double xi = x[i];
        double base = floor((xi - w0) / dnu); /* :201-203 */
        base = base < capw ? base : capw;      /* np.minimum */
        base = base > 0.0 ? base : 0.0;        /* np.maximum */
        double w_hi = -1.0;
        for (int delta = 2; delta >= -2; delta--) { /* :205-209 */
          double cand = base + (double)delta;
          if (cand >= 0.0 && cand <= wmax && w0 + cand * dnu <= xi) {
            w_hi = cand;
            break;
          }
        }
        if (w_hi < 0.0) continue;
        if (nreg == creg) {
          creg = creg ? creg * 2 : 256;
          region_t *nr = (region_t *)realloc(regs, (size_t)creg * sizeof(region_t));
          if (!nr) { free(regs); free(depth); return OR_NOMEM; }
          regs = nr;
        }
        region_t *g = &regs[nreg++];
        g->elem = ids[i]; g->xi = xi; g->nu = nu; g->rho = rho;
        g->w_hi = (int64_t)w_hi; g->r_hi = r_hi;
        g->w0 = w0; g->dnu = dnu; g->r0 = r0; g->drho = drho;
        total_areas += (w_hi + 1.0) * ((double)r_hi + 1.0); /* :242 */
      }
    }
  }
  free(depth);
  if (total_areas > MAX_AREAS_PER_CALL) { /* :243-244 */
    free(regs);
    return OR_AREAS;
  }
  /* areas w-major, r-minor (:248-256); Poisson counts (:258-262); darts
   * (:264-282); hit filter (:284); fingerprints (:293) */
  for (int64_t g = 0; g < nreg; g++) {
    const region_t *R = &regs[g];
    for (int64_t w = 0; w <= R->w_hi; w++) {
      for (int64_t r = 0; r <= R->r_hi; r++) {
        int cnt = or_poisson1(tab, cdf, R->elem, R->nu, R->rho, (uint64_t)w, (uint64_t)r);
        for (int j = 0; j < cnt; j++) {
          double v = or_uniform(tab, R->elem, R->nu, R->rho, w, r, j, OR_STREAM_V);
          double u = or_uniform(tab, R->elem, R->nu, R->rho, w, r, j, OR_STREAM_U);
          double weight = R->w0 + ((double)w + v) * R->dnu;
          double rank = R->r0 + ((double)r + u) * R->drho;
          if (weight <= R->xi && rank <= limit) {
            or_dart d;
            d.element = R->elem; d.nu = (uint16_t)R->nu; d.rho = (uint16_t)R->rho;
            d.w = (uint32_t)w; d.r = (uint32_t)r; d.j = (uint16_t)j;
            d.weight = weight; d.rank = rank;
            d.fingerprint = or_hash64(tab, R->elem, R->nu, R->rho, w, r, j, OR_STREAM_FINGERPRINT);
            if (dv_push(out, &d)) { free(regs); return OR_NOMEM; }
          }
        }
      }
    }
  }
  free(regs);
  return OR_OK;
}

/* ----------------------------------------------------------- sketches */

/* total order of ref/sketching.py:96 / ref/darthash.py:69-71 within a
 * bucket: (rank, element, nu, rho, w, r, j) */
static int dart_less(const or_dart *a, const or_dart *b) {
  if (a->rank != b->rank) return a->rank < b->rank;
  if (a->element != b->element) return a->element < b->element;
  if (a->nu != b->nu) return a->nu < b->nu;
  if (a->rho != b->rho) return a->rho < b->rho;
  if (a->w != b->w) return a->w < b->w;
  if (a->r != b->r) return a->r < b->r;
  return a->j < b->j;
}

uint64_t or_bucket_hash(const uint64_t *tab, uint64_t fp) {
  return or_hash64(tab, fp, 0, 0, 0, 0, 0, OR_STREAM_BUCKET); /* ref/randomness.py:154-158 */
}

/* ref/sketching.py:102-112 (+ _bucket_minima :93-99).  values[k]; phi_out =
 * the reference's final step; hits_out = darts hitting x at that step. */
int or_minhash(const uint64_t *tab, const double *cdf, const uint64_t *ids, const double *x,
               int64_t n, double l1, int64_t k, uint64_t *values, int32_t *phi_out,
               int64_t *hits_out) {
  if (n == 0) return OR_EMPTY; /* :86-90 */
  if (k < 1) return OR_BADARG;
  int64_t t = or_minhash_density(k);
  or_dart_vec dv = {0};
  int64_t *best = (int64_t *)malloc((size_t)k * sizeof(int64_t));
  if (!best) return OR_NOMEM;
  int status = OR_NOCONV;
  for (int phi = 1; phi <= MAX_PHI_STEPS; phi++) {
    dv.size = 0;
    int st = or_dart_batch(tab, cdf, t, ids, x, n, (double)phi / l1, &dv);
    if (st != OR_OK) { status = st; break; }
    if (dv.size < k) continue; /* :107-108 */
    for (int64_t b = 0; b < k; b++) best[b] = -1;
    for (int64_t i = 0; i < dv.size; i++) {
      int64_t b = (int64_t)(or_bucket_hash(tab, dv.data[i].fingerprint) % (uint64_t)k);
      if (best[b] < 0 || dart_less(&dv.data[i], &dv.data[best[b]])) best[b] = i;
    }
    int filled = 1;
    for (int64_t b = 0; b < k; b++) if (best[b] < 0) { filled = 0; break; }
    if (!filled) continue; /* :110 */
    for (int64_t b = 0; b < k; b++) values[b] = dv.data[best[b]].fingerprint;
    if (phi_out) *phi_out = phi;
    if (hits_out) *hits_out = dv.size;
    status = OR_OK;
    break;
  }
  free(best);
  or_dart_vec_free(&dv);
  return status;
}

/* ref/sketching.py:146-156: density t = k; at the first phi with >= k darts,
 * the k smallest darts by (rank, index) (_bottom_indices :126-143), ascending. */
static __thread const or_dart *t_bk_darts;
static int bk_cmp(const void *pa, const void *pb) {
  const or_dart *a = &t_bk_darts[*(const int64_t *)pa], *b = &t_bk_darts[*(const int64_t *)pb];
  if (dart_less(a, b)) return -1;
  if (dart_less(b, a)) return 1;
  return 0;
}

int or_bottom_k(const uint64_t *tab, const double *cdf, const uint64_t *ids, const double *x,
                int64_t n, double l1, int64_t k, or_dart *out, int32_t *phi_out) {
  if (n == 0) return OR_EMPTY;
  if (k < 1) return OR_BADARG;
  or_dart_vec dv = {0};
  int status = OR_NOCONV;
  for (int phi = 1; phi <= MAX_PHI_STEPS; phi++) {
    dv.size = 0;
    int st = or_dart_batch(tab, cdf, k, ids, x, n, (double)phi / l1, &dv);
    if (st != OR_OK) { status = st; break; }
    if (dv.size < k) continue;
    int64_t *idx = (int64_t *)malloc((size_t)dv.size * sizeof(int64_t));
    if (!idx) { status = OR_NOMEM; break; }
    for (int64_t i = 0; i < dv.size; i++) idx[i] = i;
    t_bk_darts = dv.data;
    qsort(idx, (size_t)dv.size, sizeof(int64_t), bk_cmp);
    for (int64_t i = 0; i < k; i++) out[i] = dv.data[idx[i]];
    free(idx);
    if (phi_out) *phi_out = phi;
    status = OR_OK;
    break;
  }
  or_dart_vec_free(&dv);
  return status;
}

typedef struct {
  int64_t idx;
  int64_t bucket;
} keyed_t;

static const or_dart *g_sort_darts; /* qsort context (per-thread copy below) */
static __thread const or_dart *t_sort_darts;

static int keyed_cmp(const void *pa, const void *pb) {
  const keyed_t *a = (const keyed_t *)pa, *b = (const keyed_t *)pb;
  if (a->bucket != b->bucket) return a->bucket < b->bucket ? -1 : 1;
  const or_dart *da = &t_sort_darts[a->idx], *db = &t_sort_darts[b->idx];
  if (dart_less(da, db)) return -1;
  if (dart_less(db, da)) return 1;
  return 0;
}

/* ref/annindex.py:64-82; out_fp[L*K] rank-ordered fingerprints per table. */
int or_lsh_key(const uint64_t *tab, const double *cdf, const uint64_t *ids, const double *x,
               int64_t n, double l1, int64_t L, int64_t K, uint64_t *out_fp, int32_t *phi_out,
               int64_t *hits_out) {
  (void)g_sort_darts;
  if (n == 0) return OR_EMPTY;
  if (L < 1 || K < 1) return OR_BADARG;
  int64_t t = L * K;
  or_dart_vec dv = {0};
  int64_t *cnt = (int64_t *)calloc((size_t)L, sizeof(int64_t));
  if (!cnt) return OR_NOMEM;
  int status = OR_NOCONV;
  for (int phi = 1; phi <= MAX_PHI_STEPS; phi++) {
    dv.size = 0;
    int st = or_dart_batch(tab, cdf, t, ids, x, n, (double)phi / l1, &dv);
    if (st != OR_OK) { status = st; break; }
    if (dv.size < t) continue; /* :72-73 */
    keyed_t *kv = (keyed_t *)malloc((size_t)dv.size * sizeof(keyed_t));
    if (!kv) { status = OR_NOMEM; break; }
    memset(cnt, 0, (size_t)L * sizeof(int64_t));
    for (int64_t i = 0; i < dv.size; i++) {
      kv[i].idx = i;
      kv[i].bucket = (int64_t)(or_bucket_hash(tab, dv.data[i].fingerprint) % (uint64_t)L);
      cnt[kv[i].bucket]++;
    }
    int ok = 1;
    for (int64_t b = 0; b < L; b++) if (cnt[b] < K) { ok = 0; break; } /* :75-76 */
    if (!ok) { free(kv); continue; }
    t_sort_darts = dv.data;
    qsort(kv, (size_t)dv.size, sizeof(keyed_t), keyed_cmp); /* :77 lexsort */
    int64_t pos = 0;
    for (int64_t b = 0; b < L; b++) { /* :78-81 */
      for (int64_t q = 0; q < K; q++) out_fp[b * K + q] = dv.data[kv[pos + q].idx].fingerprint;
      pos += cnt[b];
    }
    free(kv);
    if (phi_out) *phi_out = phi;
    if (hits_out) *hits_out = dv.size;
    status = OR_OK;
    break;
  }
  free(cnt);
  or_dart_vec_free(&dv);
  return status;
}

/* ------------------------------------------------------- batch drivers */

typedef struct {
  const uint64_t *tab;
  const double *cdf;
  const int64_t *indptr;
  const uint64_t *ids;
  const double *w;
  int64_t n, k, L, K;
  int normalize;
  uint64_t *out;     /* minhash: n*k values; lsh: n*L keys */
  uint64_t *out_fp;  /* lsh only: n*L*K fingerprints, may be NULL */
  int32_t *status;
  int32_t *phi;
  int64_t *hits;
  int64_t next;
  pthread_mutex_t mu;
} batch_job;

static int64_t job_take(batch_job *j, int64_t chunk) {
  pthread_mutex_lock(&j->mu);
  int64_t s = j->next;
  j->next += chunk;
  pthread_mutex_unlock(&j->mu);
  return s;
}

static void *minhash_worker(void *arg) {
  batch_job *j = (batch_job *)arg;
  for (;;) {
    int64_t s0 = job_take(j, 4);
    if (s0 >= j->n) break;
    int64_t s1 = s0 + 4 < j->n ? s0 + 4 : j->n;
    for (int64_t s = s0; s < s1; s++) {
      int64_t lo = j->indptr[s], hi = j->indptr[s + 1];
      const double *x = j->w + lo;
      double l1 = or_pairwise_sum(x, hi - lo);
      int32_t phi = 0;
      int64_t hits = 0;
      int st = or_minhash(j->tab, j->cdf, j->ids + lo, x, hi - lo, l1, j->k, j->out + s * j->k,
                          &phi, &hits);
      j->status[s] = st;
      if (j->phi) j->phi[s] = phi;
      if (j->hits) j->hits[s] = hits;
    }
  }
  return NULL;
}

static void *lsh_worker(void *arg) {
  batch_job *j = (batch_job *)arg;
  uint64_t *fps = (uint64_t *)malloc((size_t)(j->L * j->K) * sizeof(uint64_t));
  double *scaled = NULL;
  int64_t scap = 0;
  for (;;) {
    int64_t s0 = job_take(j, 2);
    if (s0 >= j->n) break;
    int64_t s1 = s0 + 2 < j->n ? s0 + 2 : j->n;
    for (int64_t s = s0; s < s1; s++) {
      int64_t lo = j->indptr[s], hi = j->indptr[s + 1], nn = hi - lo;
      const double *x = j->w + lo;
      double l1 = or_pairwise_sum(x, nn);
      if (j->normalize && nn > 0) {
        /* LshIndex.insert: c = weight_class(l1); x.scale_pow2(-c)
         * (ref/annindex.py:130-131, ref/core.py:57-60) */
        if (nn > scap) {
          scap = nn;
          free(scaled);
          scaled = (double *)malloc((size_t)scap * sizeof(double));
        }
        int c = or_weight_class(l1);
        for (int64_t i = 0; i < nn; i++) scaled[i] = ldexp(x[i], -c);
        x = scaled;
        l1 = or_pairwise_sum(x, nn);
      }
      int32_t phi = 0;
      int64_t hits = 0;
      int st = or_lsh_key(j->tab, j->cdf, j->ids + lo, x, nn, l1, j->L, j->K, fps, &phi, &hits);
      j->status[s] = st;
      if (j->phi) j->phi[s] = phi;
      if (j->hits) j->hits[s] = hits;
      if (st == OR_OK) {
        for (int64_t b = 0; b < j->L; b++) {
          j->out[s * j->L + b] = or_mix64(j->tab, fps + b * j->K, j->K);
          if (j->out_fp)
            memcpy(j->out_fp + (s * j->L + b) * j->K, fps + b * j->K,
                   (size_t)j->K * sizeof(uint64_t));
        }
      }
    }
  }
  free(fps);
  free(scaled);
  return NULL;
}

static int run_pool(batch_job *j, int nthreads, void *(*fn)(void *)) {
  if (nthreads < 1) nthreads = 1;
  pthread_t *th = (pthread_t *)malloc((size_t)nthreads * sizeof(pthread_t));
  if (!th) return OR_NOMEM;
  pthread_mutex_init(&j->mu, NULL);
  j->next = 0;
  for (int i = 0; i < nthreads; i++) pthread_create(&th[i], NULL, fn, j);
  for (int i = 0; i < nthreads; i++) pthread_join(th[i], NULL);
  pthread_mutex_destroy(&j->mu);
  free(th);
  return OR_OK;
}

int or_minhash_csr(const uint64_t *tab, const double *cdf, const int64_t *indptr,
                   const uint64_t *ids, const double *w, int64_t n, int64_t k, uint64_t *out,
                   int32_t *status, int32_t *phi, int64_t *hits, int nthreads) {
  batch_job j;
  memset(&j, 0, sizeof(j));
  j.tab = tab; j.cdf = cdf; j.indptr = indptr; j.ids = ids; j.w = w; j.n = n; j.k = k;
  j.out = out; j.status = status; j.phi = phi; j.hits = hits;
  return run_pool(&j, nthreads, minhash_worker);
}

int or_lsh_csr(const uint64_t *tab, const double *cdf, const int64_t *indptr,
               const uint64_t *ids, const double *w, int64_t n, int64_t L, int64_t K,
               int normalize, uint64_t *out_keys, uint64_t *out_fp, int32_t *status,
               int32_t *phi, int64_t *hits, int nthreads) {
  batch_job j;
  memset(&j, 0, sizeof(j));
  j.tab = tab; j.cdf = cdf; j.indptr = indptr; j.ids = ids; j.w = w; j.n = n;
  j.L = L; j.K = K; j.normalize = normalize;
  j.out = out_keys; j.out_fp = out_fp; j.status = status; j.phi = phi; j.hits = hits;
  return run_pool(&j, nthreads, lsh_worker);
}

/* flat-array form of or_dart_batch for ctypes callers: returns the dart
 * count (>= 0) or -status; columns are allocated with malloc and must be
 * released with or_free. */
int64_t or_darts_flat(const uint64_t *tab, const double *cdf, int64_t t, const uint64_t *ids,
                      const double *x, int64_t n, double limit, or_dart **out) {
  or_dart_vec dv = {0};
  int st = or_dart_batch(tab, cdf, t, ids, x, n, limit, &dv);
  if (st != OR_OK) {
    or_dart_vec_free(&dv);
    *out = NULL;
    return -(int64_t)st;
  }
  *out = dv.data;
  return dv.size;
}

void or_free(void *p) { free(p); }

void or_hash64_batch(const uint64_t *tab, const uint64_t *element, const uint64_t *nu,
                     const uint64_t *rho, const uint64_t *w, const uint64_t *r,
                     const uint64_t *j, const uint64_t *stream, int64_t n, uint64_t *out) {
  for (int64_t i = 0; i < n; i++)
    out[i] = or_hash64(tab, element[i], nu[i], rho[i], w[i], r[i], j[i], stream[i]);
}
