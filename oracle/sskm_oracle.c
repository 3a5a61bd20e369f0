/* TEST INFRASTRUCTURE ONLY — the CPU oracle (a restatement, "port").
 *
 * Plain-C restatement of the reference's hot path (sparse spherical k-means,
 * /root/reference/proj). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it, and only as the checker or
 * the timed CPU baseline; the product (paper_2108_00895_b200) never does.
 *
 * Parity is PINNED: tests/test_oracle.py checks this port bit-for-bit against
 * the compiled reference (oracle/_ref/libsskm_ref.so, built from the read-only
 * sources by oracle/Makefile) and against the golden vectors in tests/golden/
 * that tests/golden/make_golden.py generated from that reference.
 *
 * Every function cites the reference file:line it restates. Differences:
 *  - ncc+index runs the NCC path (the Lemma-1 index is out of scope, SURVEY §2
 *    row 5); its assignments are identical by mode equivalence,
 *    only the index_* counters differ.
 *  - normalize() caps the Brent cycle search (finding 4 in SURVEY §0: some
 *    orbits do not close in 2e6 passes); when the cap hits, the single-division
 *    state is returned and o_normalize_capped() counts it.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define OK 0
#define EINVAL_ 1

static __thread char g_err[256];
const char* o_last_error(void) { return g_err; }
static int fail(const char* m) {
    strncpy(g_err, m, sizeof g_err - 1);
    return EINVAL_;
}

/* ------------------------------------------------------------ mt19937_64 */
/* std::mt19937_64 as used by the pinned helpers (random.hpp:11-19). */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt_seed(mt64* g, uint64_t s) {
    g->mt[0] = s;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt_next(mt64* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* random.hpp:11-13 */
static double uniform_unit(mt64* g) { return (double)(mt_next(g) >> 11) * 0x1.0p-53; }
/* random.hpp:16-19 */
static size_t uniform_index(mt64* g, size_t n) {
    size_t i = (size_t)(uniform_unit(g) * (double)n);
    return i < n ? i : n - 1;
}

uint64_t o_mt64_draw(uint64_t seed, uint64_t skip) {
    mt64 g;
    mt_seed(&g, seed);
    for (uint64_t i = 0; i < skip; ++i) mt_next(&g);
    return mt_next(&g);
}

/* ------------------------------------------------------------------ dot */
/* gallop_to, sparse_vector.cpp:45-68 */
static size_t gallop_to(const uint32_t* dims, size_t n, size_t lo, uint32_t dim) {
    size_t step = 1, hi = lo;
    while (hi < n && dims[hi] < dim) {
        lo = hi + 1;
        hi += step;
        step <<= 1;
    }
    if (hi > n) hi = n;
    while (lo < n && dims[lo] < dim) {
        size_t mid = lo + (hi - lo) / 2;
        if (mid == lo) break;
        if (dims[mid] < dim) lo = mid;
        else hi = mid;
    }
    while (lo < n && dims[lo] < dim) ++lo;
    return lo;
}

/* dot_impl, sparse_vector.cpp:72-101: shared dims in ascending order. */
static double dot_impl(size_t ns, const uint32_t* is, const double* vs, size_t nb,
                       const uint32_t* ib, const double* vb) {
    double s = 0.0;
    if (ns == 0 || nb == 0) return 0.0;
    if (nb / (ns + 1) >= 16) {
        size_t pos = 0;
        for (size_t e = 0; e < ns; ++e) {
            pos = gallop_to(ib, nb, pos, is[e]);
            if (pos == nb) break;
            if (ib[pos] == is[e]) {
                s += vs[e] * vb[pos];
                ++pos;
            }
        }
        return s;
    }
    size_t i = 0, j = 0;
    while (i < ns && j < nb) {
        uint32_t di = is[i], dj = ib[j];
        if (di == dj) {
            s += vs[i] * vb[j];
            ++i;
            ++j;
        } else if (di < dj) ++i;
        else ++j;
    }
    return s;
}

/* dot, sparse_vector.cpp:105-108 */
double o_dot(int64_t na, const uint32_t* ia, const double* va, int64_t nb, const uint32_t* ib,
             const double* vb) {
    if (na <= nb) return dot_impl((size_t)na, ia, va, (size_t)nb, ib, vb);
    return dot_impl((size_t)nb, ib, vb, (size_t)na, ia, va);
}

/* ------------------------------------------------------------ normalize */
typedef struct {
    size_t n, cap;
    uint32_t* d;
    double* w;
} vec;

static void vec_reserve(vec* v, size_t n) {
    if (v->cap < n) {
        v->cap = n < 4 ? 4 : n;
        v->d = (uint32_t*)realloc(v->d, v->cap * sizeof(uint32_t));
        v->w = (double*)realloc(v->w, v->cap * sizeof(double));
    }
}
static void vec_free(vec* v) {
    free(v->d);
    free(v->w);
    memset(v, 0, sizeof *v);
}
static void vec_copy(vec* dst, const vec* src) {
    vec_reserve(dst, src->n);
    dst->n = src->n;
    memcpy(dst->d, src->d, src->n * sizeof(uint32_t));
    memcpy(dst->w, src->w, src->n * sizeof(double));
}
/* Entry operator== over the whole vector (sparse_vector.hpp:15-17, 48-50). */
static int vec_eq(const vec* a, const vec* b) {
    if (a->n != b->n) return 0;
    for (size_t i = 0; i < a->n; ++i)
        if (a->d[i] != b->d[i] || a->w[i] != b->w[i]) return 0;
    return 1;
}
/* lex_less, sparse_vector.cpp:112-117 */
static int lex_less(const vec* a, const vec* b) {
    for (size_t i = 0; i < a->n && i < b->n; ++i)
        if (a->w[i] != b->w[i]) return a->w[i] < b->w[i];
    return a->n < b->n;
}

/* unit_step, sparse_vector.cpp:122-149 (in: cur, out: next; may alias-free swap) */
static int unit_step(const vec* cur_in, vec* next) {
    vec cur = {0};
    vec_copy(&cur, cur_in);
    for (;;) {
        double s = 0.0;
        for (size_t i = 0; i < cur.n; ++i) s += cur.w[i] * cur.w[i];
        double nrm = sqrt(s);
        if (nrm == 0.0 || isinf(nrm)) {
            double scale = nrm == 0.0 ? 0x1p538 : 0x1p-538;
            size_t q = 0;
            for (size_t i = 0; i < cur.n; ++i) {
                double w = cur.w[i] * scale;
                if (w != 0.0) {
                    cur.d[q] = cur.d[i];
                    cur.w[q] = w;
                    ++q;
                }
            }
            if (q == 0) {
                vec_free(&cur);
                return fail("cannot normalize zero vector");
            }
            cur.n = q;
            continue;
        }
        if (nrm == 1.0) {
            vec_copy(next, &cur);
            vec_free(&cur);
            return OK;
        }
        vec_reserve(next, cur.n);
        size_t q = 0;
        for (size_t i = 0; i < cur.n; ++i) {
            double w = cur.w[i] / nrm;
            if (w != 0.0) {
                next->d[q] = cur.d[i];
                next->w[q] = w;
                ++q;
            }
        }
        next->n = q;
        vec_free(&cur);
        return OK;
    }
}

static uint64_t g_normalize_capped = 0;
uint64_t o_normalize_capped(void) { return g_normalize_capped; }
#define BRENT_CAP 4000000

/* normalize, sparse_vector.cpp:160-209. Result into `out`. */
static int normalize_vec(const vec* v, vec* out) {
    if (v->n == 0) return fail("cannot normalize zero vector");
    if (v->n == 1) {
        vec_reserve(out, 1);
        out->n = 1;
        out->d[0] = v->d[0];
        out->w[0] = v->w[0] > 0.0 ? 1.0 : -1.0;
        return OK;
    }
    vec cur = {0}, prev = {0}, next = {0};
    vec_copy(&cur, v);
    int rc = OK;
    for (int pass = 0; pass < 8; ++pass) {
        if ((rc = unit_step(&cur, &next)) != OK) goto done;
        if (vec_eq(&next, &cur)) {
            vec_copy(out, &next);
            goto done;
        }
        if (prev.d && vec_eq(&next, &prev)) {
            vec_copy(out, lex_less(&cur, &next) ? &cur : &next);
            goto done;
        }
        vec t = prev;
        prev = cur;
        cur = next;
        next = t;
    }
    {
        /* Brent's cycle detection on the orbit of unit_step (sparse_vector.cpp:187-199). */
        size_t power = 1, lam = 1, guard_ = 0;
        vec tort = {0}, hare = {0}, tmp = {0};
        vec_copy(&tort, &cur);
        if ((rc = unit_step(&cur, &hare)) != OK) goto brent_done;
        while (!vec_eq(&tort, &hare)) {
            if (++guard_ > BRENT_CAP) {
                ++g_normalize_capped;
                break;
            }
            if (power == lam) {
                vec_copy(&tort, &hare);
                power *= 2;
                lam = 0;
            }
            if ((rc = unit_step(&hare, &tmp)) != OK) goto brent_done;
            vec_copy(&hare, &tmp);
            ++lam;
        }
        if (guard_ > BRENT_CAP) {
            vec_copy(out, &hare);
            goto brent_done;
        }
        {
            /* smallest state on the terminal cycle (sparse_vector.cpp:200-207) */
            vec best = {0}, walk = {0};
            vec_copy(&best, &hare);
            if ((rc = unit_step(&hare, &walk)) == OK) {
                for (size_t i = 1; i < lam; ++i) {
                    if (lex_less(&walk, &best)) vec_copy(&best, &walk);
                    if ((rc = unit_step(&walk, &tmp)) != OK) break;
                    vec_copy(&walk, &tmp);
                }
                vec_copy(out, &best);
            }
            vec_free(&best);
            vec_free(&walk);
        }
    brent_done:
        vec_free(&tort);
        vec_free(&hare);
        vec_free(&tmp);
    }
done:
    vec_free(&cur);
    vec_free(&prev);
    vec_free(&next);
    return rc;
}

int o_normalize(int64_t n, uint32_t* idx, double* val, int64_t* n_out) {
    vec v = {0}, out = {0};
    vec_reserve(&v, (size_t)(n > 0 ? n : 1));
    v.n = (size_t)n;
    if (n) {
        memcpy(v.d, idx, (size_t)n * 4);
        memcpy(v.w, val, (size_t)n * 8);
    }
    int rc = normalize_vec(&v, &out);
    if (rc == OK) {
        memcpy(idx, out.d, out.n * 4);
        memcpy(val, out.w, out.n * 8);
        *n_out = (int64_t)out.n;
    }
    vec_free(&v);
    vec_free(&out);
    return rc;
}

/* sq_euclidean, sparse_vector.cpp:211-235 */
static double sq_euclidean(const vec* a, const vec* b) {
    double s = 0.0;
    size_t i = 0, j = 0;
    while (i < a->n && j < b->n) {
        uint32_t di = a->d[i], dj = b->d[j];
        double d;
        if (di == dj) {
            d = a->w[i] - b->w[j];
            ++i;
            ++j;
        } else if (di < dj) {
            d = a->w[i];
            ++i;
        } else {
            d = -b->w[j];
            ++j;
        }
        s += d * d;
    }
    for (; i < a->n; ++i) s += a->w[i] * a->w[i];
    for (; j < b->n; ++j) s += b->w[j] * b->w[j];
    return s;
}

/* --------------------------------------------------------------- state */
typedef struct {
    uint32_t iteration, n_unchanged_centroids;
    uint64_t n_reassigned, dot_products, index_queries, candidates_total;
    double wall_seconds, index_build_seconds, max_sq_drift, objective;
    int32_t index_active, n_repaired;
} ostats; /* field order = ref_shim.cpp CStats = engine.hpp:43-57 */

enum { M_BASELINE = 0, M_NCC = 1, M_NCC_INDEX = 2 };

typedef struct {
    /* corpus (borrowed, CSR; values widened fp32 -> double by the caller) */
    int64_t n;
    uint32_t dims;
    const int64_t* ptr;
    const int32_t* idx;
    const double* val;
    /* config (engine.hpp:20-41) */
    uint32_t k, max_iters, threads;
    int mode;
    double eps, conv;
    /* ClusteringState (engine.hpp:110-117) */
    uint32_t* a;
    double* sims;
    uint8_t* unchanged;
    uint32_t iteration;
    vec* cent; /* k sparse centroids */
    vec* prev;
    uint32_t* repaired;
    uint32_t n_repaired;
} ostate;

int o_parse_mode(const char* m) {
    if (!strcmp(m, "baseline")) return M_BASELINE;
    if (!strcmp(m, "ncc")) return M_NCC;
    if (!strcmp(m, "ncc+index")) return M_NCC_INDEX;
    return -1;
}

/* RunConfig::validate, engine.cpp:47-64 */
int o_validate(uint64_t n_docs, uint32_t k, double conv, double eps, uint32_t max_iters,
               const double* lambdas, uint32_t n_lambdas) {
    if (k < 2) return fail("k must be at least 2");
    if (k > n_docs) return fail("k exceeds the number of documents");
    for (uint32_t i = 0; i < n_lambdas; ++i) {
        if (!(lambdas[i] > 0.0 && lambdas[i] < 1.0)) return fail("lambda must be in (0, 1)");
        if (i > 0 && !(lambdas[i] > lambdas[i - 1])) return fail("lambdas must be strictly ascending");
    }
    if (!(conv > 0.0)) return fail("conv_sq_dist must be positive");
    if (eps < 0.0) return fail("ncc_epsilon must be nonnegative");
    if (max_iters < 1) return fail("max_iters must be at least 1");
    return OK;
}

void* o_state_new(int64_t n, uint32_t dims, const int64_t* ptr, const int32_t* idx,
                  const double* val, uint32_t k, const char* mode, double eps, double conv,
                  uint32_t max_iters, uint32_t threads) {
    int m = o_parse_mode(mode);
    if (m < 0) {
        fail("unknown mode (expected baseline, ncc, or ncc+index)");
        return NULL;
    }
    if (o_validate((uint64_t)n, k, conv, eps, max_iters, NULL, 0) != OK) return NULL;
    ostate* s = (ostate*)calloc(1, sizeof(ostate));
    s->n = n;
    s->dims = dims;
    s->ptr = ptr;
    s->idx = idx;
    s->val = val;
    s->k = k;
    s->mode = m;
    s->eps = eps;
    s->conv = conv;
    s->max_iters = max_iters;
    s->threads = threads;
    s->a = (uint32_t*)calloc((size_t)n, 4);
    s->sims = (double*)malloc((size_t)n * 8);
    for (int64_t i = 0; i < n; ++i) s->sims[i] = -2.0;
    s->unchanged = (uint8_t*)calloc(k, 1);
    s->cent = (vec*)calloc(k, sizeof(vec));
    s->prev = (vec*)calloc(k, sizeof(vec));
    s->repaired = (uint32_t*)calloc(k, 4);
    return s;
}

void o_state_free(void* h) {
    ostate* s = (ostate*)h;
    if (!s) return;
    for (uint32_t j = 0; j < s->k; ++j) {
        vec_free(&s->cent[j]);
        vec_free(&s->prev[j]);
    }
    free(s->cent);
    free(s->prev);
    free(s->a);
    free(s->sims);
    free(s->unchanged);
    free(s->repaired);
    free(s);
}

static double doc_dot(const ostate* s, int64_t i, const vec* c) {
    int64_t b = s->ptr[i], e = s->ptr[i + 1];
    return o_dot(e - b, (const uint32_t*)(s->idx + b), s->val + b, (int64_t)c->n, c->d, c->w);
}

/* ------------------------------------------------------------- assign */
typedef struct {
    ostate* s;
    int full_scan;
    const uint32_t* changed_ids;
    uint32_t n_changed;
    const uint32_t* unchanged_ids;
    uint32_t n_unch;
    int64_t begin, end;
    uint64_t dots, reassigned;
} assign_job;

/* The per-document loop of assign, engine.cpp:249-312 (index branch elided). */
static void* assign_worker(void* arg) {
    assign_job* J = (assign_job*)arg;
    ostate* s = J->s;
    for (int64_t i = J->begin; i < J->end; ++i) {
        const uint32_t old_a = s->a[i];
        const double old_sim = s->sims[i];
        uint32_t arg_ = 0;
        double best = -2.0;
#define EVAL(j_)                                                   \
    do {                                                           \
        uint32_t jj = (j_);                                        \
        double sv = doc_dot(s, i, &s->cent[jj]);                   \
        ++J->dots;                                                 \
        if (sv > best || (sv == best && jj < arg_)) {              \
            best = sv;                                             \
            arg_ = jj;                                             \
        }                                                          \
    } while (0)
        if (J->full_scan) {
            for (uint32_t j = 0; j < s->k; ++j) EVAL(j);
        } else {
            const int a_unchanged = s->unchanged[old_a] != 0;
            if (a_unchanged) {
                best = old_sim;
            } else {
                best = doc_dot(s, i, &s->cent[old_a]);
                ++J->dots;
            }
            arg_ = old_a;
            for (uint32_t c = 0; c < J->n_changed; ++c)
                if (J->changed_ids[c] != old_a) EVAL(J->changed_ids[c]);
            if (!a_unchanged && !(best > old_sim))
                for (uint32_t c = 0; c < J->n_unch; ++c) EVAL(J->unchanged_ids[c]);
        }
#undef EVAL
        if (arg_ != old_a) ++J->reassigned;
        s->a[i] = arg_;
        s->sims[i] = best;
    }
    return NULL;
}

static unsigned resolve_threads(unsigned t, size_t n) {
    if (t == 0) {
        long h = 8;
#ifdef _SC_NPROCESSORS_ONLN
        h = sysconf(_SC_NPROCESSORS_ONLN);
#endif
        t = h > 0 ? (unsigned)h : 1;
    }
    if (n == 0) return 1;
    if ((size_t)t > n) t = (unsigned)n;
    return t;
}

/* assign, engine.cpp:218-322 */
int o_assign(void* h, ostats* st) {
    ostate* s = (ostate*)h;
    memset(st, 0, sizeof *st);
    const int full_scan = s->iteration <= 1 || s->mode == M_BASELINE;
    st->iteration = s->iteration;
    uint32_t* ch = (uint32_t*)malloc((size_t)s->k * 4);
    uint32_t* un = (uint32_t*)malloc((size_t)s->k * 4);
    uint32_t nc = 0, nu = 0;
    for (uint32_t j = 0; j < s->k; ++j) {
        if (s->unchanged[j]) un[nu++] = j;
        else ch[nc++] = j;
    }
    st->n_unchanged_centroids = nu;
    unsigned t = resolve_threads(s->threads, (size_t)s->n);
    int64_t chunk = (s->n + t - 1) / t;
    assign_job* jobs = (assign_job*)calloc(t, sizeof(assign_job));
    pthread_t* th = (pthread_t*)calloc(t, sizeof(pthread_t));
    for (unsigned w = 0; w < t; ++w) {
        jobs[w] = (assign_job){s, full_scan, ch, nc, un, nu, (int64_t)w * chunk, 0, 0, 0};
        jobs[w].end = jobs[w].begin + chunk < s->n ? jobs[w].begin + chunk : s->n;
        if (jobs[w].begin > jobs[w].end) jobs[w].begin = jobs[w].end;
    }
    for (unsigned w = 1; w < t; ++w) pthread_create(&th[w], NULL, assign_worker, &jobs[w]);
    assign_worker(&jobs[0]);
    for (unsigned w = 1; w < t; ++w) pthread_join(th[w], NULL);
    for (unsigned w = 0; w < t; ++w) { /* fixed-order merge, engine.cpp:315-320 */
        st->dot_products += jobs[w].dots;
        st->n_reassigned += jobs[w].reassigned;
    }
    double obj = 0.0; /* run(): objective = sum of cached sims, engine.cpp:403-405 */
    for (int64_t i = 0; i < s->n; ++i) obj += s->sims[i];
    st->objective = obj;
    free(jobs);
    free(th);
    free(ch);
    free(un);
    return OK;
}

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : x > y;
}
void o_sort_u32(uint32_t* p, size_t n) { qsort(p, n, 4, cmp_u32); }

/* ---------------------------------------------------- compute_centroids */
/* engine.cpp:137-195: sizes, ascending empty repair, ascending-doc sums
 * (DenseAccumulator, sparse_vector.cpp:237-274), normalize. */
static int compute_centroids(ostate* s, vec* out) {
    const int64_t n = s->n;
    const uint32_t k = s->k;
    size_t* sizes = (size_t*)calloc(k, sizeof(size_t));
    for (int64_t i = 0; i < n; ++i) {
        if (s->a[i] >= k) {
            free(sizes);
            return fail("assignment out of range");
        }
        ++sizes[s->a[i]];
    }
    s->n_repaired = 0;
    for (uint32_t j = 0; j < k; ++j) {
        if (sizes[j] != 0) continue;
        int64_t donor = n;
        for (int64_t i = 0; i < n; ++i) {
            if (sizes[s->a[i]] < 2) continue;
            if (donor == n || s->sims[i] < s->sims[donor]) donor = i;
        }
        --sizes[s->a[donor]];
        s->a[donor] = j;
        sizes[j] = 1;
        s->repaired[s->n_repaired++] = j;
    }
    /* members in ascending doc order per cluster (engine.cpp:169-177) */
    int64_t* off = (int64_t*)calloc((size_t)k + 1, 8);
    for (int64_t i = 0; i < n; ++i) ++off[s->a[i] + 1];
    for (uint32_t j = 0; j < k; ++j) off[j + 1] += off[j];
    int64_t* fill = (int64_t*)malloc((size_t)k * 8);
    memcpy(fill, off, (size_t)k * 8);
    uint32_t* members = (uint32_t*)malloc((size_t)(n > 0 ? n : 1) * 4);
    for (int64_t i = 0; i < n; ++i) members[fill[s->a[i]]++] = (uint32_t)i;

    double* acc = (double*)calloc(s->dims ? s->dims : 1, 8);
    uint8_t* touched = (uint8_t*)calloc(s->dims ? s->dims : 1, 1);
    uint32_t* tl = (uint32_t*)malloc((size_t)(s->dims ? s->dims : 1) * 4);
    int rc = OK;
    for (uint32_t j = 0; j < k && rc == OK; ++j) {
        size_t nt = 0;
        for (int64_t m = off[j]; m < off[j + 1]; ++m) {
            int64_t i = members[m];
            for (int64_t p = s->ptr[i]; p < s->ptr[i + 1]; ++p) {
                uint32_t d = (uint32_t)s->idx[p];
                if (!touched[d]) {
                    touched[d] = 1;
                    acc[d] = 0.0;
                    tl[nt++] = d;
                }
                acc[d] += s->val[p];
            }
        }
        /* extract: touched dims ascending, exact zeros dropped (sparse_vector.cpp:264-274) */
        vec sum = {0};
        vec_reserve(&sum, nt ? nt : 1);
        size_t q = 0;
        o_sort_u32(tl, nt); /* touched dims ascending (std::sort in extract) */
        for (size_t x = 0; x < nt; ++x) {
            uint32_t d = tl[x];
            touched[d] = 0;
            if (acc[d] != 0.0) {
                sum.d[q] = d;
                sum.w[q] = acc[d];
                ++q;
            }
        }
        sum.n = q;
        rc = normalize_vec(&sum, &out[j]);
        vec_free(&sum);
    }
    free(acc);
    free(touched);
    free(tl);
    free(members);
    free(fill);
    free(off);
    free(sizes);
    return rc;
}

/* --------------------------------------------------------------- steps */
/* First half of the Stepper body (test_engine.cpp:65-84; run() engine.cpp:361-378). */
int o_update(void* h, uint32_t* n_unchanged_out, double* drift_out) {
    ostate* s = (ostate*)h;
    s->iteration += 1;
    vec* next = (vec*)calloc(s->k, sizeof(vec));
    int rc = compute_centroids(s, next);
    if (rc != OK) {
        for (uint32_t j = 0; j < s->k; ++j) vec_free(&next[j]);
        free(next);
        return rc;
    }
    uint32_t nu = 0;
    double drift = 0.0;
    if (s->iteration == 1) {
        memset(s->unchanged, 0, s->k);
    } else {
        /* detect_unchanged, engine.cpp:197-216 */
        for (uint32_t j = 0; j < s->k; ++j) {
            double dj = sq_euclidean(&s->cent[j], &next[j]);
            s->unchanged[j] = dj <= s->eps ? 1 : 0;
            if (dj > drift) drift = dj;
        }
        for (uint32_t r = 0; r < s->n_repaired; ++r) s->unchanged[s->repaired[r]] = 0;
        for (uint32_t j = 0; j < s->k; ++j) nu += s->unchanged[j];
    }
    for (uint32_t j = 0; j < s->k; ++j) {
        vec_free(&s->prev[j]);
        s->prev[j] = s->cent[j];
        s->cent[j] = next[j];
    }
    free(next);
    *n_unchanged_out = nu;
    *drift_out = drift;
    return OK;
}

int o_step(void* h, ostats* st) {
    uint32_t nu;
    double drift;
    int rc = o_update(h, &nu, &drift);
    if (rc != OK) return rc;
    o_assign(h, st);
    st->max_sq_drift = drift;
    st->n_repaired = (int32_t)((ostate*)h)->n_repaired;
    return OK;
}

/* BASELINE init: centroid j = doc seeds[j]; full-scan assign (engine.cpp:82-97). */
int o_init_seeds(void* h, const uint32_t* seeds, ostats* st) {
    ostate* s = (ostate*)h;
    for (uint32_t j = 0; j < s->k; ++j) {
        if ((int64_t)seeds[j] >= s->n) return fail("seed out of range");
        int64_t b = s->ptr[seeds[j]], e = s->ptr[seeds[j] + 1];
        vec* c = &s->cent[j];
        vec_reserve(c, (size_t)(e - b) + 1);
        c->n = (size_t)(e - b);
        for (int64_t p = b; p < e; ++p) {
            c->d[p - b] = (uint32_t)s->idx[p];
            c->w[p - b] = s->val[p];
        }
    }
    for (int64_t i = 0; i < s->n; ++i) {
        s->a[i] = 0;
        s->sims[i] = -2.0;
    }
    memset(s->unchanged, 0, s->k);
    s->iteration = 0;
    ostats tmp;
    o_assign(h, st ? st : &tmp);
    return OK;
}

/* seed_kmeanspp, engine.cpp:66-130 */
int o_seed_kmeanspp(void* h, uint64_t seed, uint32_t* seeds_out) {
    ostate* s = (ostate*)h;
    const int64_t n = s->n;
    mt64 g;
    mt_seed(&g, seed);
    uint8_t* chosen = (uint8_t*)calloc((size_t)n, 1);
    double* cum = (double*)malloc((size_t)n * 8);
    for (int64_t i = 0; i < n; ++i) {
        s->a[i] = 0;
        s->sims[i] = -2.0;
    }
    int64_t pick = (int64_t)uniform_index(&g, (size_t)n);
    for (uint32_t c = 0; c < s->k; ++c) {
        if (c > 0) {
            double total = 0.0;
            for (int64_t i = 0; i < n; ++i) {
                double w = 0.0;
                if (!chosen[i]) {
                    double d = 1.0 - s->sims[i];
                    if (d > 0.0) w = d * d;
                }
                total += w;
                cum[i] = total;
            }
            if (total > 0.0) {
                double target = uniform_unit(&g) * total;
                int64_t lo = 0, hi = n; /* upper_bound */
                while (lo < hi) {
                    int64_t mid = lo + (hi - lo) / 2;
                    if (!(target < cum[mid])) lo = mid + 1;
                    else hi = mid;
                }
                pick = lo;
                if (pick >= n) {
                    pick = n - 1;
                    while (chosen[pick]) --pick;
                }
            } else {
                pick = 0;
                while (chosen[pick]) ++pick;
            }
        }
        chosen[pick] = 1;
        seeds_out[c] = (uint32_t)pick;
        int64_t b = s->ptr[pick], e = s->ptr[pick + 1];
        for (int64_t i = 0; i < n; ++i) {
            int64_t bi = s->ptr[i], ei = s->ptr[i + 1];
            double sim = o_dot(ei - bi, (const uint32_t*)(s->idx + bi), s->val + bi, e - b,
                               (const uint32_t*)(s->idx + b), s->val + b);
            if (sim > s->sims[i]) {
                s->sims[i] = sim;
                s->a[i] = c;
            }
        }
    }
    memset(s->unchanged, 0, s->k);
    s->iteration = 0;
    free(chosen);
    free(cum);
    return OK;
}

/* run loop after seeding, engine.cpp:357-424. Returns stop reason. */
int o_run(void* h, ostats* stats, uint32_t cap, uint32_t* n_iters, int32_t* stop_reason) {
    ostate* s = (ostate*)h;
    int32_t stop = 2; /* kMaxIterations */
    uint32_t t = 0;
    for (uint32_t iter = 1; iter <= s->max_iters; ++iter) {
        ostats st;
        int rc = o_step(h, &st);
        if (rc != OK) return rc;
        if (t < cap) stats[t] = st;
        ++t;
        if (st.n_reassigned == 0) {
            stop = 0;
            break;
        }
        if (iter > 1 && st.max_sq_drift < s->conv) {
            stop = 1;
            break;
        }
    }
    *n_iters = t;
    *stop_reason = stop;
    return OK;
}

/* ------------------------------------------------------------- access */
uint32_t o_iteration(void* h) { return ((ostate*)h)->iteration; }

void o_get_state(void* h, uint32_t* a, double* sims, uint8_t* unchanged) {
    ostate* s = (ostate*)h;
    if (a) memcpy(a, s->a, (size_t)s->n * 4);
    if (sims) memcpy(sims, s->sims, (size_t)s->n * 8);
    if (unchanged) memcpy(unchanged, s->unchanged, s->k);
}

void o_set_state(void* h, const uint32_t* a, const double* sims, const uint8_t* unchanged,
                 uint32_t iteration) {
    ostate* s = (ostate*)h;
    if (a) memcpy(s->a, a, (size_t)s->n * 4);
    if (sims) memcpy(s->sims, sims, (size_t)s->n * 8);
    if (unchanged) memcpy(s->unchanged, unchanged, s->k);
    s->iteration = iteration;
}

int64_t o_centroids_nnz(void* h) {
    ostate* s = (ostate*)h;
    int64_t t = 0;
    for (uint32_t j = 0; j < s->k; ++j) t += (int64_t)s->cent[j].n;
    return t;
}

void o_get_centroids(void* h, int64_t* ptr, uint32_t* idx, double* val) {
    ostate* s = (ostate*)h;
    int64_t p = 0;
    ptr[0] = 0;
    for (uint32_t j = 0; j < s->k; ++j) {
        memcpy(idx + p, s->cent[j].d, s->cent[j].n * 4);
        memcpy(val + p, s->cent[j].w, s->cent[j].n * 8);
        p += (int64_t)s->cent[j].n;
        ptr[j + 1] = p;
    }
}

void o_set_centroids(void* h, const int64_t* ptr, const uint32_t* idx, const double* val) {
    ostate* s = (ostate*)h;
    for (uint32_t j = 0; j < s->k; ++j) {
        size_t n = (size_t)(ptr[j + 1] - ptr[j]);
        vec_reserve(&s->cent[j], n ? n : 1);
        s->cent[j].n = n;
        memcpy(s->cent[j].d, idx + ptr[j], n * 4);
        memcpy(s->cent[j].w, val + ptr[j], n * 8);
    }
}

uint32_t o_repaired(void* h, uint32_t* out) {
    ostate* s = (ostate*)h;
    if (out) memcpy(out, s->repaired, s->n_repaired * 4);
    return s->n_repaired;
}

/* standalone compute_centroids on the state's own a/sims (teacher forcing) */
int o_compute_centroids(void* h) {
    ostate* s = (ostate*)h;
    vec* next = (vec*)calloc(s->k, sizeof(vec));
    int rc = compute_centroids(s, next);
    for (uint32_t j = 0; j < s->k; ++j) {
        vec_free(&s->cent[j]);
        s->cent[j] = next[j];
    }
    free(next);
    return rc;
}
