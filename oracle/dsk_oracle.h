/* dsk_oracle.h -- TEST INFRASTRUCTURE ONLY (see dsk_oracle.c). */
#ifndef DSK_ORACLE_H
#define DSK_ORACLE_H
#include <stdint.h>

/* stream tags, ref/randomness.py:28-39 */
#define OR_STREAM_V 1
#define OR_STREAM_U 2
#define OR_STREAM_POISSON 3
#define OR_STREAM_FINGERPRINT 4
#define OR_STREAM_BUCKET 5
#define OR_STREAM_KEY_MIX 12

/* per-set status codes; identical numbering to include/dsk_b200.h */
#define OR_OK 0
#define OR_EMPTY 1   /* ValidationError: empty set            ref/sketching.py:86-88 */
#define OR_WEIGHT 2  /* ValidationError: weight not finite>0  ref/core.py:38-41 */
#define OR_DEPTH 3   /* ValidationError: depth > 255          ref/darthash.py:158-160 */
#define OR_OVERFLOW 9 /* OverflowError: 1 + t*x is inf          ref/darthash.py:154-156 */
#define OR_AREAS 4   /* ValidationError: > 2^27 areas         ref/darthash.py:242-244 */
#define OR_NOCONV 5  /* RuntimeError: 64 phi steps            ref/sketching.py:112 */
#define OR_LIMIT 6   /* ValidationError: rank limit <=0 / inf ref/darthash.py:136-138 */
#define OR_BADARG 7
#define OR_NOMEM 8

typedef struct {
  uint64_t element;
  uint16_t nu, rho;
  uint32_t w, r;
  uint16_t j;
  uint16_t pad;
  double weight, rank;
  uint64_t fingerprint;
} or_dart; /* one row of DartBatch, ref/darthash.py:39-53 */

typedef struct {
  or_dart *data;
  int64_t size, cap;
} or_dart_vec;

uint64_t or_finalize(uint64_t h);
uint64_t or_hash64(const uint64_t *tab, uint64_t element, uint64_t nu, uint64_t rho, uint64_t w,
                   uint64_t r, uint64_t j, uint64_t stream);
void or_poisson1_cdf(double *cdf);
uint64_t or_mix64(const uint64_t *tab, const uint64_t *values, int64_t n);
double or_pairwise_sum(const double *a, int64_t n);
int64_t or_minhash_density(int64_t k);
int or_weight_class(double l1);
uint64_t or_bucket_hash(const uint64_t *tab, uint64_t fp);
int or_dart_batch(const uint64_t *tab, const double *cdf, int64_t t, const uint64_t *ids,
                  const double *x, int64_t n, double limit, or_dart_vec *out);
void or_dart_vec_free(or_dart_vec *v);
int or_minhash(const uint64_t *tab, const double *cdf, const uint64_t *ids, const double *x,
               int64_t n, double l1, int64_t k, uint64_t *values, int32_t *phi_out,
               int64_t *hits_out);
int or_lsh_key(const uint64_t *tab, const double *cdf, const uint64_t *ids, const double *x,
               int64_t n, double l1, int64_t L, int64_t K, uint64_t *out_fp, int32_t *phi_out,
               int64_t *hits_out);
int or_bottom_k(const uint64_t *tab, const double *cdf, const uint64_t *ids, const double *x,
                int64_t n, double l1, int64_t k, or_dart *out, int32_t *phi_out);
int or_minhash_csr(const uint64_t *tab, const double *cdf, const int64_t *indptr,
                   const uint64_t *ids, const double *w, int64_t n, int64_t k, uint64_t *out,
                   int32_t *status, int32_t *phi, int64_t *hits, int nthreads);
int or_lsh_csr(const uint64_t *tab, const double *cdf, const int64_t *indptr,
               const uint64_t *ids, const double *w, int64_t n, int64_t L, int64_t K,
               int normalize, uint64_t *out_keys, uint64_t *out_fp, int32_t *status,
               int32_t *phi, int64_t *hits, int nthreads);
int64_t or_darts_flat(const uint64_t *tab, const double *cdf, int64_t t, const uint64_t *ids,
                      const double *x, int64_t n, double limit, or_dart **out);
void or_free(void *p);
void or_hash64_batch(const uint64_t *tab, const uint64_t *element, const uint64_t *nu,
                     const uint64_t *rho, const uint64_t *w, const uint64_t *r,
                     const uint64_t *j, const uint64_t *stream, int64_t n, uint64_t *out);
#endif
