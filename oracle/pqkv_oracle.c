/*
 * pqkv_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded CPU restatement of the reference `pqkv` hot path
 * (PQCache, arxiv 2407.12820; reference checkout /root/reference/proj).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library, and only as the CHECKER.  The product
 * path (paper_2407_12820_b200/lib/libpqkv.so) never links or calls it.
 *
 * Pinning: every function below is checked against the reference itself --
 * the reference sources compiled unmodified into oracle/_ref/libpqkv_ref.so
 * (oracle/Makefile) and the golden fixtures in tests/golden/ generated from
 * that library by tests/golden/make_golden.py (see tests/test_oracle.py).
 *
 * Arithmetic contract: IEEE binary64 with no contraction (compile with
 * -ffp-contract=off and no -march, exactly like the reference's CMake build),
 * glibc libm for exp/log/cos/sqrt/pow, identical operation order.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "pqkv_oracle.h"

/* ------------------------------------------------------------------------ */
/* mt19937_64 + the reference's draw math (rng.hpp:11-37)                    */
/* ------------------------------------------------------------------------ */

#define MT_N 312
#define MT_M 156

void orc_rng_seed(orc_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = MT_N;
}

uint64_t orc_rng_u64(orc_rng* r) {
    static const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    if (r->idx >= MT_N) {
        for (int i = 0; i < MT_N; ++i) {
            uint64_t y = (r->mt[i] & upper) | (r->mt[(i + 1) % MT_N] & lower);
            uint64_t v = r->mt[(i + MT_M) % MT_N] ^ (y >> 1);
            if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
            r->mt[i] = v;
        }
        r->idx = 0;
    }
    uint64_t x = r->mt[r->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* uniform() rng.hpp:18-20 */
double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_u64(r) >> 11) * 0x1.0p-53; }

/* normal() rng.hpp:23-27: Box-Muller, redraw u1 while zero, no cached spare */
double orc_rng_normal(orc_rng* r) {
    double u1 = orc_rng_uniform(r), u2 = orc_rng_uniform(r);
    while (u1 == 0.0) u1 = orc_rng_uniform(r);
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

/* index(n) rng.hpp:30 */
uint64_t orc_rng_index(orc_rng* r, uint64_t n) { return orc_rng_u64(r) % n; }

/* fork_seed() rng.hpp:33 */
uint64_t orc_rng_fork_seed(orc_rng* r) { return orc_rng_u64(r) ^ 0x9e3779b97f4a7c15ULL; }

/* ------------------------------------------------------------------------ */
/* Synthetic workload (workload.cpp:16-117)                                 */
/* ------------------------------------------------------------------------ */

static void unit_vector(orc_rng* r, double* v, size_t d) {
    double norm2;
    do {
        norm2 = 0.0;
        for (size_t j = 0; j < d; ++j) {
            v[j] = orc_rng_normal(r);
            norm2 += v[j] * v[j];
        }
    } while (norm2 == 0.0);
    double inv = 1.0 / sqrt(norm2);
    for (size_t j = 0; j < d; ++j) v[j] *= inv;
}

static void fill_normal(orc_rng* r, float* out, size_t n) {
    for (size_t i = 0; i < n; ++i) out[i] = (float)(1.0 * orc_rng_normal(r));
}

int orc_gen_workload(size_t s, size_t d_h, size_t h_kv, size_t g, int kind,
                     size_t n_components, double spread, double zipf, uint64_t seed,
                     float* keys, float* values, float* queries) {
    if (s < 1 || d_h < 1 || h_kv < 1 || g < 1) return ORC_EINVAL;
    if (kind == ORC_GAUSSIAN && n_components < 1) return ORC_EINVAL;
    if (spread < 0.0 || zipf <= 0.0) return ORC_EINVAL;
    orc_rng rng;
    orc_rng_seed(&rng, seed);
    size_t d = d_h;
    for (size_t h = 0; h < h_kv; ++h) {
        float* k = keys + h * s * d;
        float* v = values + h * s * d;
        float* q = queries + h * g * d;
        if (kind == ORC_GAUSSIAN) { /* gen_gaussian_head workload.cpp:39-51 */
            double* means = (double*)malloc(n_components * d * sizeof(double));
            for (size_t i = 0; i < n_components * d; ++i) means[i] = orc_rng_normal(&rng);
            for (size_t i = 0; i < s; ++i) {
                const double* mean = means + orc_rng_index(&rng, n_components) * d;
                for (size_t j = 0; j < d; ++j)
                    k[i * d + j] = (float)(mean[j] + spread * orc_rng_normal(&rng));
            }
            fill_normal(&rng, v, s * d);
            fill_normal(&rng, q, g * d);
            free(means);
        } else { /* gen_powerlaw_head workload.cpp:53-79 */
            double* qd = (double*)malloc(d * sizeof(double));
            double* u = (double*)malloc(d * sizeof(double));
            size_t* rank_of = (size_t*)malloc(s * sizeof(size_t));
            unit_vector(&rng, qd, d);
            for (size_t i = 0; i < s; ++i) rank_of[i] = i;
            for (size_t i = s; i > 1; --i) {
                size_t j = (size_t)orc_rng_index(&rng, i);
                size_t t = rank_of[i - 1];
                rank_of[i - 1] = rank_of[j];
                rank_of[j] = t;
            }
            double top = 8.0 * sqrt((double)d);
            for (size_t i = 0; i < s; ++i) {
                unit_vector(&rng, u, d);
                double target = top / pow((double)(rank_of[i] + 1), zipf);
                double along = 0.0;
                for (size_t j = 0; j < d; ++j) along += u[j] * qd[j];
                for (size_t j = 0; j < d; ++j)
                    k[i * d + j] = (float)(u[j] + (target - along) * qd[j]);
            }
            fill_normal(&rng, v, s * d);
            for (size_t r = 0; r < g; ++r)
                for (size_t j = 0; j < d; ++j) q[r * d + j] = (float)qd[j];
            free(qd);
            free(u);
            free(rank_of);
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* k-means (kmeans.cpp:14-220)                                               */
/* ------------------------------------------------------------------------ */

/* dist2 kmeans.cpp:14-21: acc from 0.0, ascending t, separate sub/mul/add */
static double dist2(const float* a, const double* b, size_t dim) {
    double acc = 0.0;
    for (size_t t = 0; t < dim; ++t) {
        double diff = (double)a[t] - b[t];
        acc += diff * diff;
    }
    return acc;
}

typedef struct {
    const float* pts;
    size_t n, dim, k;
    double* cen; /* [k][dim] fp64 centroids */
} fitter;

static const float* fpoint(const fitter* f, size_t i) { return f->pts + i * f->dim; }

static void set_centroid(fitter* f, size_t c, const float* p) {
    for (size_t t = 0; t < f->dim; ++t) f->cen[c * f->dim + t] = (double)p[t];
}

/* seed_from_distinct kmeans.cpp:44-57 (n <= k only) */
static void seed_from_distinct(fitter* f) {
    size_t* distinct = (size_t*)malloc(f->n * sizeof(size_t));
    size_t nd = 0;
    for (size_t i = 0; i < f->n; ++i) {
        int seen = 0;
        for (size_t q = 0; q < nd; ++q)
            if (memcmp(fpoint(f, i), fpoint(f, distinct[q]), f->dim * sizeof(float)) == 0) {
                seen = 1;
                break;
            }
        if (!seen) distinct[nd++] = i;
    }
    for (size_t c = 0; c < f->k; ++c) set_centroid(f, c, fpoint(f, distinct[c < nd - 1 ? c : nd - 1]));
    free(distinct);
}

/* seed_plus_plus kmeans.cpp:59-84: two serial fp64 running sums per centroid */
static void seed_plus_plus(fitter* f, orc_rng* rng) {
    size_t n = f->n;
    set_centroid(f, 0, fpoint(f, (size_t)orc_rng_index(rng, n)));
    double* min_d2 = (double*)malloc(n * sizeof(double));
    for (size_t i = 0; i < n; ++i) min_d2[i] = dist2(fpoint(f, i), f->cen, f->dim);
    for (size_t c = 1; c < f->k; ++c) {
        double total = 0.0;
        for (size_t i = 0; i < n; ++i) total += min_d2[i];
        size_t chosen;
        if (total > 0.0) {
            double target = orc_rng_uniform(rng) * total, cum = 0.0;
            chosen = n - 1;
            for (size_t i = 0; i < n; ++i) {
                cum += min_d2[i];
                if (cum >= target) {
                    chosen = i;
                    break;
                }
            }
        } else {
            chosen = (size_t)orc_rng_index(rng, n);
        }
        set_centroid(f, c, fpoint(f, chosen));
        const double* cc = f->cen + c * f->dim;
        for (size_t i = 0; i < n; ++i) {
            double d = dist2(fpoint(f, i), cc, f->dim);
            if (d < min_d2[i]) min_d2[i] = d; /* std::min(a, b) keeps a unless b < a */
        }
    }
    free(min_d2);
}

/* nearest kmeans.cpp:86-97: strict < from c=0, ties to the lower index */
static size_t nearest(const fitter* f, size_t i) {
    size_t best = 0;
    double best_d = dist2(fpoint(f, i), f->cen, f->dim);
    for (size_t c = 1; c < f->k; ++c) {
        double d = dist2(fpoint(f, i), f->cen + c * f->dim, f->dim);
        if (d < best_d) {
            best_d = d;
            best = c;
        }
    }
    return best;
}

/* assign_with_repair kmeans.cpp:103-130 */
static void assign_with_repair(const fitter* f, size_t* assign, size_t* count) {
    memset(count, 0, f->k * sizeof(size_t));
    for (size_t i = 0; i < f->n; ++i) {
        assign[i] = nearest(f, i);
        ++count[assign[i]];
    }
    if (f->n >= f->k) {
        for (size_t c = 0; c < f->k; ++c) {
            if (count[c] != 0) continue;
            size_t donor = f->n;
            double worst = -1.0;
            for (size_t i = 0; i < f->n; ++i) {
                if (count[assign[i]] < 2) continue;
                double d = dist2(fpoint(f, i), f->cen + assign[i] * f->dim, f->dim);
                if (d > worst) {
                    worst = d;
                    donor = i;
                }
            }
            if (donor == f->n) break;
            --count[assign[donor]];
            assign[donor] = c;
            ++count[c];
        }
    }
}

/* update_means kmeans.cpp:133-147: sums in ascending point order */
static void update_means(fitter* f, const size_t* assign) {
    double* sums = (double*)calloc(f->k * f->dim, sizeof(double));
    size_t* count = (size_t*)calloc(f->k, sizeof(size_t));
    for (size_t i = 0; i < f->n; ++i) {
        double* s = sums + assign[i] * f->dim;
        const float* p = fpoint(f, i);
        for (size_t t = 0; t < f->dim; ++t) s[t] += (double)p[t];
        ++count[assign[i]];
    }
    for (size_t c = 0; c < f->k; ++c) {
        if (count[c] == 0) continue;
        for (size_t t = 0; t < f->dim; ++t)
            f->cen[c * f->dim + t] = sums[c * f->dim + t] / (double)count[c];
    }
    free(sums);
    free(count);
}

/* inertia kmeans.cpp:149-154 */
static double inertia(const fitter* f, const size_t* assign) {
    double total = 0.0;
    for (size_t i = 0; i < f->n; ++i) total += dist2(fpoint(f, i), f->cen + assign[i] * f->dim, f->dim);
    return total;
}

/* kmeans_fit kmeans.cpp:159-190 */
int orc_kmeans_fit(const float* points, size_t n, size_t dim, size_t n_clusters,
                   size_t max_iter, uint64_t seed, float* centroids_out,
                   uint64_t* assign_out, double* inertia_trace, size_t* iterations_run) {
    if (n < 1 || dim < 1) return ORC_EINVAL;
    if (n_clusters < 1 || max_iter < 1) return ORC_EINVAL;
    for (size_t i = 0; i < n * dim; ++i)
        if (!isfinite(points[i])) return ORC_EINVAL;
    fitter f = {points, n, dim, n_clusters, (double*)calloc(n_clusters * dim, sizeof(double))};
    if (n <= n_clusters) {
        seed_from_distinct(&f);
    } else {
        orc_rng rng;
        orc_rng_seed(&rng, seed);
        seed_plus_plus(&f, &rng);
    }
    size_t* assign = (size_t*)malloc(n * sizeof(size_t));
    size_t* next = (size_t*)malloc(n * sizeof(size_t));
    size_t* count = (size_t*)malloc(n_clusters * sizeof(size_t));
    assign_with_repair(&f, assign, count);
    size_t iters = 0;
    for (size_t iter = 1; iter <= max_iter; ++iter) {
        update_means(&f, assign);
        if (inertia_trace) inertia_trace[iter - 1] = inertia(&f, assign);
        iters = iter;
        assign_with_repair(&f, next, count);
        if (memcmp(next, assign, n * sizeof(size_t)) == 0) break;
        size_t* t = assign;
        assign = next;
        next = t;
    }
    for (size_t i = 0; i < n_clusters * dim; ++i) centroids_out[i] = (float)f.cen[i];
    for (size_t i = 0; i < n; ++i) assign_out[i] = assign[i];
    if (iterations_run) *iterations_run = iters;
    free(f.cen);
    free(assign);
    free(next);
    free(count);
    return ORC_OK;
}

/* assign_nearest kmeans.cpp:192-220: f32 centroids widened, best_d = +inf */
int orc_assign_nearest(const float* points, size_t n, size_t dim, const float* centroids,
                       size_t k, uint64_t* assign_out) {
    for (size_t i = 0; i < n; ++i) {
        const float* p = points + i * dim;
        size_t best = 0;
        double best_d = INFINITY;
        for (size_t c = 0; c < k; ++c) {
            const float* q = centroids + c * dim;
            double acc = 0.0;
            for (size_t t = 0; t < dim; ++t) {
                double diff = (double)p[t] - (double)q[t];
                acc += diff * diff;
            }
            if (acc < best_d) {
                best_d = acc;
                best = c;
            }
        }
        assign_out[i] = best;
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Product quantization (pq.cpp:13-177)                                     */
/* ------------------------------------------------------------------------ */

/* PqConfig::create pq.cpp:13-25 */
int orc_pq_config(size_t m, size_t b, size_t d_h, size_t* d_m, size_t* n_clusters) {
    if (m < 1) return ORC_EINVAL;
    if (b < 1 || b > 16) return ORC_EINVAL;
    if (d_h < 1 || d_h % m != 0) return ORC_EINVAL;
    *d_m = d_h / m;
    *n_clusters = (size_t)1 << b;
    return ORC_OK;
}

/* pq_construct pq.cpp:42-72: per partition j, kmeans_fit with
 * seed + 0x9e3779b97f4a7c15 * (j + 1) (mod 2^64); codes[i*m+j] = assign */
int orc_pq_construct(const float* keys, size_t s, size_t d_h, size_t m, size_t b,
                     size_t max_iter, uint64_t seed, float* centroids_out,
                     uint16_t* codes_out) {
    size_t d_m, C;
    if (orc_pq_config(m, b, d_h, &d_m, &C) != ORC_OK) return ORC_EINVAL;
    if (s < 1) return ORC_EINVAL;
    float* sub = (float*)malloc(s * d_m * sizeof(float));
    uint64_t* assign = (uint64_t*)malloc(s * sizeof(uint64_t));
    int rc = ORC_OK;
    for (size_t j = 0; j < m && rc == ORC_OK; ++j) {
        for (size_t i = 0; i < s; ++i)
            for (size_t t = 0; t < d_m; ++t) sub[i * d_m + t] = keys[i * d_h + j * d_m + t];
        rc = orc_kmeans_fit(sub, s, d_m, C, max_iter, seed + 0x9e3779b97f4a7c15ULL * (uint64_t)(j + 1),
                            centroids_out + j * C * d_m, assign, NULL, NULL);
        for (size_t i = 0; i < s; ++i) codes_out[i * m + j] = (uint16_t)assign[i];
    }
    free(sub);
    free(assign);
    return rc;
}

/* pq_encode_one pq.cpp:74-99: f32 centroids, best_d = +inf, strict < */
int orc_pq_encode_one(const float* key, const float* centroids, size_t m, size_t C,
                      size_t d_m, uint16_t* code_out) {
    for (size_t j = 0; j < m; ++j) {
        size_t best = 0;
        double best_d = INFINITY;
        for (size_t c = 0; c < C; ++c) {
            const float* cen = centroids + (j * C + c) * d_m;
            double acc = 0.0;
            for (size_t t = 0; t < d_m; ++t) {
                double diff = (double)key[j * d_m + t] - (double)cen[t];
                acc += diff * diff;
            }
            if (acc < best_d) {
                best_d = acc;
                best = c;
            }
        }
        code_out[j] = (uint16_t)best;
    }
    return ORC_OK;
}

/* add_score_table pq.cpp:113-126 accumulated over the g query rows
 * (pq_score_gqa pq.cpp:152-161), then gather_scores pq.cpp:128-140 */
int orc_pq_score_gqa(const float* queries, size_t g, size_t d_h, const float* centroids,
                     size_t m, size_t C, const uint16_t* codes, size_t s, float* scores_out) {
    if (g < 1 || d_h % m != 0) return ORC_EINVAL;
    size_t d_m = d_h / m;
    double* table = (double*)calloc(m * C, sizeof(double));
    for (size_t r = 0; r < g; ++r) {
        const float* query = queries + r * d_h;
        for (size_t j = 0; j < m; ++j) {
            const float* q = query + j * d_m;
            for (size_t c = 0; c < C; ++c) {
                const float* cen = centroids + (j * C + c) * d_m;
                double acc = 0.0;
                for (size_t t = 0; t < d_m; ++t) acc += (double)q[t] * (double)cen[t];
                table[j * C + c] += acc;
            }
        }
    }
    for (size_t i = 0; i < s; ++i) {
        const uint16_t* code = codes + i * m;
        double acc = 0.0;
        for (size_t j = 0; j < m; ++j) acc += table[j * C + code[j]];
        scores_out[i] = (float)acc;
    }
    free(table);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* top_k_desc topk.cpp:8-25: (score desc, id asc), float compare            */
/* ------------------------------------------------------------------------ */

static const float* g_sort_scores;
static int cmp_desc(const void* pa, const void* pb) {
    uint64_t a = *(const uint64_t*)pa, b = *(const uint64_t*)pb;
    float sa = g_sort_scores[a], sb = g_sort_scores[b];
    if (sa != sb) return sa > sb ? -1 : 1;
    return a < b ? -1 : (a > b ? 1 : 0);
}

int orc_top_k_desc(const float* scores, size_t n, size_t k, const uint8_t* excluded,
                   uint64_t* ids_out) {
    uint64_t* ids = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    size_t cnt = 0;
    for (size_t i = 0; i < n; ++i)
        if (!excluded || !excluded[i]) ids[cnt++] = i;
    if (k > cnt) {
        free(ids);
        return ORC_EINVAL;
    }
    /* a strict total order, so a full sort then truncation equals partial_sort */
    g_sort_scores = scores;
    qsort(ids, cnt, sizeof(uint64_t), cmp_desc);
    memcpy(ids_out, ids, k * sizeof(uint64_t));
    free(ids);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Attention (attention.cpp:11-104)                                         */
/* ------------------------------------------------------------------------ */

/* exact_scores attention.cpp:11-26 over an explicit row list */
static float exact_score_row(const float* query, const float* k, size_t d_h, double scale) {
    double acc = 0.0;
    for (size_t j = 0; j < d_h; ++j) acc += (double)query[j] * (double)k[j];
    return (float)(acc * scale);
}

int orc_exact_scores(const float* query, const float* keys, size_t t, size_t d_h,
                     float* scores_out) {
    double scale = 1.0 / sqrt((double)d_h);
    for (size_t i = 0; i < t; ++i) scores_out[i] = exact_score_row(query, keys + i * d_h, d_h, scale);
    return ORC_OK;
}

/* softmax_attention attention.cpp:35-60 over rows[0..t) of keys/values
 * (row indices given, NULL = identity) */
int orc_softmax_rows(const float* query, const float* keys, const float* values, size_t d_h,
                     const uint64_t* rows, size_t t, float* out) {
    if (t < 1) return ORC_EINVAL;
    double scale = 1.0 / sqrt((double)d_h);
    float* scores = (float*)malloc(t * sizeof(float));
    double* w = (double*)malloc(t * sizeof(double));
    double* acc = (double*)calloc(d_h, sizeof(double));
    for (size_t i = 0; i < t; ++i) {
        size_t r = rows ? (size_t)rows[i] : i;
        scores[i] = exact_score_row(query, keys + r * d_h, d_h, scale);
    }
    float mx = scores[0]; /* std::max_element: first maximal element */
    for (size_t i = 1; i < t; ++i)
        if (mx < scores[i]) mx = scores[i];
    double max_score = (double)mx, total = 0.0;
    for (size_t i = 0; i < t; ++i) {
        w[i] = exp((double)scores[i] - max_score);
        total += w[i];
    }
    for (size_t i = 0; i < t; ++i) {
        double wi = w[i] / total;
        size_t r = rows ? (size_t)rows[i] : i;
        const float* v = values + r * d_h;
        for (size_t j = 0; j < d_h; ++j) acc[j] += wi * (double)v[j];
    }
    for (size_t j = 0; j < d_h; ++j) out[j] = (float)acc[j];
    free(scores);
    free(w);
    free(acc);
    return ORC_OK;
}

static int cmp_u64(const void* pa, const void* pb) {
    uint64_t a = *(const uint64_t*)pa, b = *(const uint64_t*)pb;
    return a < b ? -1 : (a > b ? 1 : 0);
}

/* selective_attention attention.cpp:62-91 on the flat token-id layout:
 * rows = init [0,n_init) ++ sorted middle ids ++ local [total-n_local, total).
 * Middle ids must lie in [n_init, total-n_local) (out_of_range otherwise) and
 * be distinct (invalid_argument). */
int orc_selective_attention(const float* query, const float* keys, const float* values,
                            size_t d_h, size_t total, size_t n_init, size_t n_local,
                            const uint64_t* middle_ids, size_t n_ids, float* out) {
    if (n_init + n_local > total) return ORC_EINVAL;
    uint64_t* ids = (uint64_t*)malloc((n_ids ? n_ids : 1) * sizeof(uint64_t));
    memcpy(ids, middle_ids, n_ids * sizeof(uint64_t));
    qsort(ids, n_ids, sizeof(uint64_t), cmp_u64);
    for (size_t i = 1; i < n_ids; ++i)
        if (ids[i] == ids[i - 1]) {
            free(ids);
            return ORC_EINVAL;
        }
    for (size_t i = 0; i < n_ids; ++i)
        if (ids[i] < n_init || ids[i] >= total - n_local) {
            free(ids);
            return ORC_ERANGE;
        }
    size_t t = n_init + n_ids + n_local;
    uint64_t* rows = (uint64_t*)malloc((t ? t : 1) * sizeof(uint64_t));
    size_t r = 0;
    for (size_t i = 0; i < n_init; ++i) rows[r++] = i;
    for (size_t i = 0; i < n_ids; ++i) rows[r++] = ids[i];
    for (size_t i = total - n_local; i < total; ++i) rows[r++] = i;
    int rc = orc_softmax_rows(query, keys, values, d_h, rows, t, out);
    free(ids);
    free(rows);
    return rc;
}

/* Raw draw streams for pinning the RNG restatement against the reference:
 * kind 0 = next_u64, 1 = uniform, 2 = normal, 3 = fork_seed (doubles are
 * returned bit-cast into the u64 slots). */
uint64_t orc_rng_stream(uint64_t seed, uint64_t* out, size_t n, int kind) {
    orc_rng r;
    orc_rng_seed(&r, seed);
    for (size_t i = 0; i < n; ++i) {
        if (kind == 0) {
            out[i] = orc_rng_u64(&r);
        } else if (kind == 1) {
            double u = orc_rng_uniform(&r);
            memcpy(&out[i], &u, 8);
        } else if (kind == 2) {
            double u = orc_rng_normal(&r);
            memcpy(&out[i], &u, 8);
        } else {
            out[i] = orc_rng_fork_seed(&r);
        }
    }
    return 0;
}
