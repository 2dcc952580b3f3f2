/* pqkv_oracle.h -- TEST INFRASTRUCTURE ONLY (see pqkv_oracle.c header).
 * C restatement of the reference pqkv hot path; used by tests/, smoke() and
 * bench.py's CPU-baseline leg as the checker, never by the product path. */
#ifndef PQKV_ORACLE_H
#define PQKV_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_ERANGE = 2, ORC_ESTATE = 3 };
enum { ORC_GAUSSIAN = 0, ORC_POWERLAW = 1 };

typedef struct {
    uint64_t mt[312];
    int idx;
} orc_rng;

void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_u64(orc_rng* r);
double orc_rng_uniform(orc_rng* r);
double orc_rng_normal(orc_rng* r);
uint64_t orc_rng_index(orc_rng* r, uint64_t n);
uint64_t orc_rng_fork_seed(orc_rng* r);
uint64_t orc_rng_stream(uint64_t seed, uint64_t* out, size_t n, int kind);

int orc_gen_workload(size_t s, size_t d_h, size_t h_kv, size_t g, int kind,
                     size_t n_components, double spread, double zipf, uint64_t seed,
                     float* keys, float* values, float* queries);

int orc_kmeans_fit(const float* points, size_t n, size_t dim, size_t n_clusters,
                   size_t max_iter, uint64_t seed, float* centroids_out,
                   uint64_t* assign_out, double* inertia_trace, size_t* iterations_run);
int orc_assign_nearest(const float* points, size_t n, size_t dim, const float* centroids,
                       size_t k, uint64_t* assign_out);

int orc_pq_config(size_t m, size_t b, size_t d_h, size_t* d_m, size_t* n_clusters);
int orc_pq_construct(const float* keys, size_t s, size_t d_h, size_t m, size_t b,
                     size_t max_iter, uint64_t seed, float* centroids_out,
                     uint16_t* codes_out);
int orc_pq_encode_one(const float* key, const float* centroids, size_t m, size_t C,
                      size_t d_m, uint16_t* code_out);
int orc_pq_score_gqa(const float* queries, size_t g, size_t d_h, const float* centroids,
                     size_t m, size_t C, const uint16_t* codes, size_t s, float* scores_out);

int orc_top_k_desc(const float* scores, size_t n, size_t k, const uint8_t* excluded,
                   uint64_t* ids_out);

int orc_exact_scores(const float* query, const float* keys, size_t t, size_t d_h,
                     float* scores_out);
int orc_softmax_rows(const float* query, const float* keys, const float* values, size_t d_h,
                     const uint64_t* rows, size_t t, float* out);
int orc_selective_attention(const float* query, const float* keys, const float* values,
                            size_t d_h, size_t total, size_t n_init, size_t n_local,
                            const uint64_t* middle_ids, size_t n_ids, float* out);

#ifdef __cplusplus
}
#endif

#endif
