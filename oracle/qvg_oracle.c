/*
 * TEST INFRASTRUCTURE ONLY — the parity checker, never the product.
 *
 * Plain-C restatement of the reference's BQ-native query path (QuIVer `qivr`,
 * /root/reference/proj/core).  Only tests/, __graft_entry__.smoke() and the
 * CPU-baseline leg of bench.py may load this (oracle/liboracle.so).  The
 * product (paper_2605_02171_b200/) never links or calls it.
 *
 * Parity is PINNED: tests/test_oracle_pins.py checks every function below
 * against the compiled reference library (oracle/_ref/libqivr_ref.so, built
 * from the reference's own sources by oracle/Makefile) and against the
 * committed golden vectors in tests/golden/.
 *
 * Functions and the reference code they restate:
 *   orc_encode_query     search.cpp:128-136 (finite check), vec_math.hpp:28-44
 *                        (l2_norm / normalize_l2), encoding.cpp:23-45
 *                        (compute_threshold, encode_sm2_into)
 *   orc_sm2_distance     encoding.hpp:169-176 (scalar sm2_distance_words)
 *   orc_dot4             vec_math.hpp:13-26 (dot_f32, 4 strided double chains)
 *   orc_beam_search_heap search.cpp:27-81 (dual-heap best-first search)
 *   orc_beam_search_list SURVEY §8.A.3 sorted-list formulation (the GPU
 *                        kernel's state machine: sorted pool, tie stack,
 *                        prefix admission, lossy visited table)
 *   orc_rerank           search.cpp:96-120
 *   orc_query_batch      search.cpp:122-143 + eval.cpp:225-247 (1 thread)
 *   orc_float_topk       eval.cpp:17-57, 86-97 (float_cosine brute force)
 *   orc_robust_prune     graph.hpp:162-183
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_NONFINITE_COORD 1
#define ORC_BAD_NORM 2
#define ORC_NONFINITE_ENCODE 3
#define ORC_BAD_PARAMS 4
#define ORC_DIM_MISMATCH 5
#define ORC_OVERFLOW 6

static size_t words_for_dim(size_t d) { return (d + 63) / 64; }

/* ---- encode (query path) ------------------------------------------------ */

int orc_encode_query(const float* x, uint32_t dim, float* out_norm, uint64_t* out_code,
                     float* out_tau) {
    const size_t w = words_for_dim(dim);
    for (uint32_t i = 0; i < dim; ++i)
        if (!isfinite(x[i])) return ORC_NONFINITE_COORD;
    double acc = 0.0;
    for (uint32_t i = 0; i < dim; ++i) acc += (double)x[i] * (double)x[i];
    const double norm = sqrt(acc);
    if (!(norm > 0.0) || !isfinite(norm)) return ORC_BAD_NORM;
    const float inv = (float)(1.0 / norm);
    for (uint32_t i = 0; i < dim; ++i) out_norm[i] = x[i] * inv;
    for (uint32_t i = 0; i < dim; ++i)
        if (!isfinite(out_norm[i])) return ORC_NONFINITE_ENCODE;
    double s = 0.0;
    for (uint32_t i = 0; i < dim; ++i) s += fabs((double)out_norm[i]);
    const float tau = (float)(s / (double)dim);
    memset(out_code, 0, 2 * w * sizeof(uint64_t));
    for (uint32_t i = 0; i < dim; ++i) {
        const uint64_t bit = 1ULL << (i % 64);
        if (out_norm[i] > 0.0f) out_code[i / 64] |= bit;
        if (fabsf(out_norm[i]) > tau) out_code[w + i / 64] |= bit;
    }
    if (out_tau) *out_tau = tau;
    return ORC_OK;
}

/* ---- distances ------------------------------------------------------------ */

/* a, b: reference layout (W pos words then W strong words). */
uint32_t orc_sm2_distance(const uint64_t* a, const uint64_t* b, uint64_t w) {
    uint64_t t = 0;
    for (uint64_t i = 0; i < w; ++i) {
        const uint64_t x = a[i] ^ b[i];
        const uint64_t so = a[w + i] | b[w + i];
        const uint64_t sa = a[w + i] & b[w + i];
        t += (uint64_t)__builtin_popcountll(x) + (uint64_t)__builtin_popcountll(x & so) +
             2ULL * (uint64_t)__builtin_popcountll(x & sa);
    }
    return (uint32_t)t;
}

float orc_dot4(const float* a, const float* b, uint64_t n) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    uint64_t i = 0;
    for (; i + 4 <= n; i += 4) {
        s0 += (double)a[i] * (double)b[i];
        s1 += (double)a[i + 1] * (double)b[i + 1];
        s2 += (double)a[i + 2] * (double)b[i + 2];
        s3 += (double)a[i + 3] * (double)b[i + 3];
    }
    for (; i < n; ++i) s0 += (double)a[i] * (double)b[i];
    return (float)((s0 + s1) + (s2 + s3));
}

/* ---- index view ----------------------------------------------------------- */

typedef struct {
    const uint64_t* codes; /* n x 2W, reference SignatureStore layout */
    const uint32_t* adj;   /* n x (R+1), reference AdjacencyTable slot layout */
    const float* cold;     /* n x dim, unit-normalised */
    uint64_t n;
    uint32_t dim;
    uint32_t R;
    uint32_t entry;
} orc_index;

static inline uint32_t node_dist(const orc_index* ix, const uint64_t* q, uint32_t v) {
    const uint64_t w = words_for_dim(ix->dim);
    return orc_sm2_distance(q, ix->codes + (uint64_t)v * 2 * w, w);
}

static inline uint64_t mkkey(uint32_t dist, uint32_t id) { return ((uint64_t)dist << 32) | id; }

/* ---- binary heaps on (dist<<32|id) keys ----------------------------------- */

typedef struct {
    uint64_t* a;
    uint64_t n, cap;
    int max; /* 1: max-heap, 0: min-heap */
} heap;

static int heap_before(const heap* h, uint64_t x, uint64_t y) { return h->max ? x > y : x < y; }

static int heap_push(heap* h, uint64_t k) {
    if (h->n == h->cap) {
        uint64_t nc = h->cap ? 2 * h->cap : 64;
        uint64_t* na = (uint64_t*)realloc(h->a, nc * sizeof(uint64_t));
        if (!na) return -1;
        h->a = na;
        h->cap = nc;
    }
    uint64_t i = h->n++;
    h->a[i] = k;
    while (i > 0) {
        uint64_t p = (i - 1) / 2;
        if (!heap_before(h, h->a[i], h->a[p])) break;
        uint64_t t = h->a[i];
        h->a[i] = h->a[p];
        h->a[p] = t;
        i = p;
    }
    return 0;
}

static uint64_t heap_pop(heap* h) {
    uint64_t top = h->a[0];
    h->a[0] = h->a[--h->n];
    uint64_t i = 0;
    for (;;) {
        uint64_t l = 2 * i + 1, r = l + 1, b = i;
        if (l < h->n && heap_before(h, h->a[l], h->a[b])) b = l;
        if (r < h->n && heap_before(h, h->a[r], h->a[b])) b = r;
        if (b == i) break;
        uint64_t t = h->a[i];
        h->a[i] = h->a[b];
        h->a[b] = t;
        i = b;
    }
    return top;
}

/* ---- search context -------------------------------------------------------- */

typedef struct {
    uint32_t* stamp; /* exact visited set (epoch stamps), search.hpp:31-60 */
    uint32_t* inpool;
    uint32_t epoch;
    uint64_t n;
    heap frontier, pool;
} orc_ctx;

orc_ctx* orc_ctx_new(uint64_t n) {
    orc_ctx* c = (orc_ctx*)calloc(1, sizeof(orc_ctx));
    c->stamp = (uint32_t*)calloc(n, sizeof(uint32_t));
    c->inpool = (uint32_t*)calloc(n, sizeof(uint32_t));
    c->n = n;
    c->pool.max = 1;
    return c;
}

void orc_ctx_free(orc_ctx* c) {
    if (!c) return;
    free(c->stamp);
    free(c->inpool);
    free(c->frontier.a);
    free(c->pool.a);
    free(c);
}

static void ctx_next(orc_ctx* c) {
    if (++c->epoch == 0) {
        memset(c->stamp, 0, c->n * sizeof(uint32_t));
        memset(c->inpool, 0, c->n * sizeof(uint32_t));
        c->epoch = 1;
    }
}

/* stats[0] expansions, [1] tie expansions (node popped from the frontier after
 * eviction from the pool), [2] distance evaluations incl. the entry, [3]
 * adjacency bytes (4 + 4*deg per expansion, reference slot layout). */
int orc_beam_search_heap(const orc_index* ix, orc_ctx* c, const uint64_t* q, uint32_t ef,
                         uint32_t entry, uint32_t* out_ids, uint32_t* out_dists,
                         uint32_t* out_n, uint64_t* stats) {
    ctx_next(c);
    const uint32_t ep = c->epoch;
    c->frontier.n = 0;
    c->pool.n = 0;
    uint64_t st[4] = {0, 0, 0, 0};
    const uint64_t start = mkkey(node_dist(ix, q, entry), entry);
    st[2]++;
    c->stamp[entry] = ep;
    heap_push(&c->frontier, start);
    heap_push(&c->pool, start);
    c->inpool[entry] = ep;
    while (c->frontier.n > 0) {
        const uint64_t cur = c->frontier.a[0];
        if (c->pool.n == ef && (cur >> 32) > (c->pool.a[0] >> 32)) break;
        heap_pop(&c->frontier);
        const uint32_t cid = (uint32_t)cur;
        st[0]++;
        if (c->inpool[cid] != ep) st[1]++;
        const uint32_t* slot = ix->adj + (uint64_t)cid * (ix->R + 1);
        const uint32_t deg = slot[0];
        st[3] += 4 + 4ull * deg;
        for (uint32_t i = 0; i < deg; ++i) {
            const uint32_t v = slot[1 + i];
            if (c->stamp[v] == ep) continue;
            c->stamp[v] = ep;
            const uint64_t k = mkkey(node_dist(ix, q, v), v);
            st[2]++;
            if (c->pool.n < ef || k < c->pool.a[0]) {
                heap_push(&c->frontier, k);
                heap_push(&c->pool, k);
                c->inpool[v] = ep;
                if (c->pool.n > ef) {
                    const uint64_t ev = heap_pop(&c->pool);
                    c->inpool[(uint32_t)ev] = 0;
                }
            }
        }
    }
    const uint64_t np = c->pool.n;
    for (uint64_t i = np; i-- > 0;) {
        const uint64_t k = heap_pop(&c->pool);
        out_ids[i] = (uint32_t)k;
        out_dists[i] = (uint32_t)(k >> 32);
    }
    *out_n = (uint32_t)np;
    if (stats)
        for (int i = 0; i < 4; ++i) stats[i] += st[i];
    return ORC_OK;
}

/* ---- sorted-list formulation (the GPU kernel's state machine) ---------------
 * pool P: ascending keys + expanded flags, |P| <= ef.
 * tie stack T: evicted, unexpanded keys whose dist equals the worst pool dist;
 *   all live entries share one dist (tdist) and are pushed smallest-on-top.
 * visited: exact stamps (vslots == 0) or a direct-mapped lossy table of
 *   vslots ids (power of two), slot = (id * 0x9E3779B1) >> (32 - log2 vslots).
 * Every scored key already present in P is dropped (exact membership), which
 * makes the lossy table result-preserving.
 * stats: [0] expansions [1] tie expansions [2] evals [3] adj bytes
 *        [4] in-pool drops [5] tie-stack overflows [6] max tie depth      */

static uint32_t vhash(uint32_t id, uint32_t lg) { return (id * 0x9E3779B1u) >> (32 - lg); }

static uint64_t lower_bound_u64(const uint64_t* a, uint32_t n, uint64_t x) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        uint32_t mid = (lo + hi) / 2;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

int orc_beam_search_list(const orc_index* ix, orc_ctx* c, const uint64_t* q, uint32_t ef,
                         uint32_t entry, uint32_t vslots, uint32_t tie_cap, uint32_t* out_ids,
                         uint32_t* out_dists, uint32_t* out_n, uint64_t* stats) {
    const uint32_t R = ix->R;
    uint64_t* P = (uint64_t*)malloc((size_t)(ef + R + 1) * sizeof(uint64_t));
    uint8_t* Pf = (uint8_t*)malloc((size_t)(ef + R + 1));
    uint64_t* NP = (uint64_t*)malloc((size_t)(ef + R + 1) * sizeof(uint64_t));
    uint8_t* NPf = (uint8_t*)malloc((size_t)(ef + R + 1));
    uint64_t* C = (uint64_t*)malloc((size_t)(R + 1) * sizeof(uint64_t));
    uint32_t* T = (uint32_t*)malloc((size_t)(tie_cap + 1) * sizeof(uint32_t));
    uint32_t* vt = NULL;
    uint32_t lg = 0;
    if (vslots) {
        while ((1u << lg) < vslots) ++lg;
        vt = (uint32_t*)malloc((size_t)vslots * sizeof(uint32_t));
        memset(vt, 0xFF, (size_t)vslots * sizeof(uint32_t));
    } else {
        ctx_next(c);
    }
    const uint32_t ep = c ? c->epoch : 0;
    uint64_t st[7] = {0, 0, 0, 0, 0, 0, 0};
    uint32_t np = 0, tn = 0, tdist = 0;
    int rc = ORC_OK;

#define VISITED_TEST_SET(v, hit)                          \
    do {                                                  \
        if (vt) {                                         \
            uint32_t s_ = vhash((v), lg);                 \
            hit = vt[s_] == (v);                          \
            vt[s_] = (v);                                 \
        } else {                                          \
            hit = c->stamp[(v)] == ep;                    \
            c->stamp[(v)] = ep;                           \
        }                                                 \
    } while (0)

    {
        int hit;
        VISITED_TEST_SET(entry, hit);
        (void)hit;
        P[0] = mkkey(node_dist(ix, q, entry), entry);
        Pf[0] = 0;
        np = 1;
        st[2]++;
    }
    for (;;) {
        /* 1. pick */
        uint32_t u;
        uint32_t pi = 0;
        while (pi < np && Pf[pi]) ++pi;
        if (pi < np) {
            Pf[pi] = 1;
            u = (uint32_t)P[pi];
        } else if (tn > 0) {
            u = T[--tn];
            st[1]++;
        } else {
            break;
        }
        st[0]++;
        /* 2. score the row (stored order) */
        const uint32_t* slot = ix->adj + (uint64_t)u * (R + 1);
        const uint32_t deg = slot[0];
        st[3] += 4 + 4ull * deg;
        uint32_t m = 0;
        for (uint32_t i = 0; i < deg; ++i) {
            const uint32_t v = slot[1 + i];
            int dup = 0;
            for (uint32_t j = 0; j < i; ++j) dup |= slot[1 + j] == v; /* first slot wins */
            if (dup) continue;
            int hit;
            VISITED_TEST_SET(v, hit);
            if (hit) continue;
            const uint64_t k = mkkey(node_dist(ix, q, v), v);
            st[2]++;
            const uint64_t r = lower_bound_u64(P, np, k);
            if (r < np && P[r] == k) { /* already in the pool */
                st[4]++;
                continue;
            }
            C[m++] = k;
        }
        /* 3./4. prefix admission + merge: positions in the sorted union */
        uint32_t total = np + m;
        uint32_t newnp = total < ef ? total : ef;
        /* rank of each candidate among candidates */
        uint64_t worst = 0;
        /* build merged array */
        {
            uint32_t a = 0, b = 0, o = 0;
            /* sorted copy of C */
            uint64_t* Cs = (uint64_t*)malloc((size_t)(m + 1) * sizeof(uint64_t));
            memcpy(Cs, C, m * sizeof(uint64_t));
            for (uint32_t i = 1; i < m; ++i) { /* insertion sort, m <= R */
                uint64_t x = Cs[i];
                uint32_t j = i;
                while (j > 0 && Cs[j - 1] > x) {
                    Cs[j] = Cs[j - 1];
                    --j;
                }
                Cs[j] = x;
            }
            while (a < np || b < m) {
                if (b >= m || (a < np && P[a] < Cs[b])) {
                    NP[o] = P[a];
                    NPf[o] = Pf[a];
                    ++a;
                } else {
                    NP[o] = Cs[b];
                    NPf[o] = 2; /* candidate, unexpanded */
                    ++b;
                }
                ++o;
            }
            free(Cs);
        }
        if (total >= ef) worst = NP[ef - 1];
        if (total > ef) {
            const uint32_t wd = (uint32_t)(worst >> 32);
            if (tn == 0 || wd < tdist) {
                tn = 0;
                tdist = wd;
            }
            /* evicted unexpanded entries with dist == wd, ascending keys */
            uint32_t adds = 0;
            uint32_t* add = (uint32_t*)malloc((size_t)(total - ef) * sizeof(uint32_t));
            for (uint32_t o = ef; o < total; ++o) {
                const uint64_t k = NP[o];
                if ((uint32_t)(k >> 32) != wd) continue;
                if (NPf[o] == 1) continue; /* expanded: dropped */
                if (NPf[o] == 2) {         /* candidate: admitted by prefix rule? */
                    uint32_t idx = 0;
                    while (C[idx] != k) ++idx;
                    uint32_t cnt = (uint32_t)lower_bound_u64(P, np, k);
                    for (uint32_t j = 0; j < idx; ++j) cnt += C[j] < k;
                    if (cnt >= ef) continue;
                }
                add[adds++] = (uint32_t)k;
            }
            if (tn + adds > tie_cap) {
                st[5]++;
                rc = ORC_OVERFLOW;
                adds = tie_cap > tn ? tie_cap - tn : 0; /* keep the smallest */
            }
            for (uint32_t j = adds; j-- > 0;) T[tn++] = add[j];
            if (tn > st[6]) st[6] = tn;
            free(add);
        }
        for (uint32_t o = 0; o < newnp; ++o) {
            P[o] = NP[o];
            Pf[o] = NPf[o] == 1;
        }
        np = newnp;
    }
#undef VISITED_TEST_SET
    for (uint32_t i = 0; i < np; ++i) {
        out_ids[i] = (uint32_t)P[i];
        out_dists[i] = (uint32_t)(P[i] >> 32);
    }
    *out_n = np;
    if (stats) {
        for (int i = 0; i < 6; ++i) stats[i] += st[i];
        if (st[6] > stats[6]) stats[6] = st[6];
    }
    free(P);
    free(Pf);
    free(NP);
    free(NPf);
    free(C);
    free(T);
    free(vt);
    return rc;
}

/* ---- rerank ---------------------------------------------------------------- */

typedef struct {
    uint32_t id;
    float score;
} scored;

static int scored_cmp(const void* pa, const void* pb) {
    const scored* a = (const scored*)pa;
    const scored* b = (const scored*)pb;
    if (a->score != b->score) return a->score > b->score ? -1 : 1;
    return a->id < b->id ? -1 : (a->id > b->id ? 1 : 0);
}

uint32_t orc_rerank(const orc_index* ix, const uint32_t* ids, uint32_t n, const float* qn,
                    uint32_t k, uint32_t* out_ids, float* out_scores) {
    scored* s = (scored*)malloc((size_t)(n + 1) * sizeof(scored));
    for (uint32_t i = 0; i < n; ++i) {
        s[i].id = ids[i];
        s[i].score = orc_dot4(qn, ix->cold + (uint64_t)ids[i] * ix->dim, ix->dim);
    }
    qsort(s, n, sizeof(scored), scored_cmp);
    const uint32_t take = n < k ? n : k;
    for (uint32_t i = 0; i < take; ++i) {
        out_ids[i] = s[i].id;
        out_scores[i] = s[i].score;
    }
    free(s);
    return take;
}

/* ---- batch query (1 thread) ----------------------------------------------
 * mode 0: dual-heap search; mode 1: sorted-list search (exact visited);
 * mode 2: sorted-list with a lossy visited table of `vslots` entries.
 * Rows of out_ids/out_scores are padded with UINT32_MAX / NaN.
 * out_pool (optional): nq x ef ids, out_pool_dists, out_pool_n.
 * stats: 7 u64 accumulators (see orc_beam_search_list) + [7] pool sizes.   */
int orc_query_batch(const orc_index* ix, const float* queries, uint64_t nq, uint32_t ef,
                    uint32_t k, int mode, uint32_t vslots, uint32_t tie_cap, uint32_t* out_ids,
                    float* out_scores, uint32_t* out_count, int32_t* out_status,
                    uint32_t* out_pool_ids, uint32_t* out_pool_dists, uint32_t* out_pool_n,
                    uint64_t* stats) {
    if (k < 1 || ef < k) return ORC_BAD_PARAMS;
    const uint32_t dim = ix->dim;
    const size_t w = words_for_dim(dim);
    orc_ctx* c = orc_ctx_new(ix->n);
    float* qn = (float*)malloc(dim * sizeof(float));
    uint64_t* code = (uint64_t*)malloc(2 * w * sizeof(uint64_t));
    uint32_t* pid = (uint32_t*)malloc((size_t)(ef + 1) * sizeof(uint32_t));
    uint32_t* pd = (uint32_t*)malloc((size_t)(ef + 1) * sizeof(uint32_t));
    int worst_rc = ORC_OK;
    for (uint64_t qi = 0; qi < nq; ++qi) {
        for (uint32_t j = 0; j < k; ++j) {
            out_ids[qi * k + j] = UINT32_MAX;
            out_scores[qi * k + j] = NAN;
        }
        out_count[qi] = 0;
        int rc = orc_encode_query(queries + qi * dim, dim, qn, code, NULL);
        if (out_status) out_status[qi] = rc;
        if (rc != ORC_OK) {
            worst_rc = rc;
            continue;
        }
        uint32_t np = 0;
        if (mode == 0)
            rc = orc_beam_search_heap(ix, c, code, ef, ix->entry, pid, pd, &np, stats);
        else
            rc = orc_beam_search_list(ix, c, code, ef, ix->entry, mode == 2 ? vslots : 0,
                                      tie_cap, pid, pd, &np, stats);
        if (rc != ORC_OK) {
            if (out_status) out_status[qi] = rc;
            worst_rc = rc;
        }
        if (stats) stats[7] += np;
        if (out_pool_ids) {
            for (uint32_t j = 0; j < ef; ++j) {
                out_pool_ids[qi * ef + j] = j < np ? pid[j] : UINT32_MAX;
                out_pool_dists[qi * ef + j] = j < np ? pd[j] : UINT32_MAX;
            }
            out_pool_n[qi] = np;
        }
        out_count[qi] = orc_rerank(ix, pid, np, qn, k, out_ids + qi * k, out_scores + qi * k);
    }
    free(qn);
    free(code);
    free(pid);
    free(pd);
    orc_ctx_free(c);
    return worst_rc;
}

/* ---- rerank depth (GPU-only knob, BASELINE config 4; no reference oracle) ----
 * Definition: rerank the `depth` smallest (dist, id) keys among every node the
 * search scored.  The final pool is exactly the ef smallest scored keys (a key
 * left out of it was rejected or evicted while above the then-worst pool key,
 * and the worst only falls), so depth <= ef reranks a pool prefix and
 * depth == ef is the reference's query (search.cpp:138-142).  The dual-heap
 * search runs with exact visited stamps, so the scored set is the stamped set. */
static int u64_cmp(const void* pa, const void* pb) {
    const uint64_t a = *(const uint64_t*)pa, b = *(const uint64_t*)pb;
    return a < b ? -1 : (a > b ? 1 : 0);
}

int orc_query_depth(const orc_index* ix, const float* queries, uint64_t nq, uint32_t ef,
                    uint32_t k, uint32_t depth, uint32_t* out_ids, float* out_scores,
                    uint32_t* out_count) {
    if (k < 1 || ef < k || depth < k) return ORC_BAD_PARAMS;
    const uint32_t dim = ix->dim;
    const size_t w = words_for_dim(dim);
    orc_ctx* c = orc_ctx_new(ix->n);
    float* qn = (float*)malloc(dim * sizeof(float));
    uint64_t* code = (uint64_t*)malloc(2 * w * sizeof(uint64_t));
    uint32_t* pid = (uint32_t*)malloc((size_t)(ef + 1) * sizeof(uint32_t));
    uint32_t* pd = (uint32_t*)malloc((size_t)(ef + 1) * sizeof(uint32_t));
    uint64_t* keys = (uint64_t*)malloc((size_t)ix->n * sizeof(uint64_t));
    uint32_t* ids = (uint32_t*)malloc((size_t)ix->n * sizeof(uint32_t));
    int worst_rc = ORC_OK;
    for (uint64_t qi = 0; qi < nq; ++qi) {
        for (uint32_t j = 0; j < k; ++j) {
            out_ids[qi * k + j] = UINT32_MAX;
            out_scores[qi * k + j] = NAN;
        }
        out_count[qi] = 0;
        int rc = orc_encode_query(queries + qi * dim, dim, qn, code, NULL);
        if (rc != ORC_OK) {
            worst_rc = rc;
            continue;
        }
        uint32_t np = 0;
        orc_beam_search_heap(ix, c, code, ef, ix->entry, pid, pd, &np, NULL);
        uint64_t ns = 0;
        for (uint64_t v = 0; v < ix->n; ++v)
            if (c->stamp[v] == c->epoch) keys[ns++] = mkkey(node_dist(ix, code, (uint32_t)v), (uint32_t)v);
        qsort(keys, ns, sizeof(uint64_t), u64_cmp);
        const uint64_t take = ns < depth ? ns : depth;
        for (uint64_t i = 0; i < take; ++i) ids[i] = (uint32_t)keys[i];
        for (uint32_t i = 0; i < np && i < take; ++i)
            if (ids[i] != pid[i]) worst_rc = ORC_OVERFLOW; /* pool != scored prefix: bug */
        out_count[qi] = orc_rerank(ix, ids, (uint32_t)take, qn, k, out_ids + qi * k, out_scores + qi * k);
    }
    free(qn);
    free(code);
    free(pid);
    free(pd);
    free(keys);
    free(ids);
    orc_ctx_free(c);
    return worst_rc;
}

/* ---- exact float top-k (ground truth) ------------------------------------- */

int orc_float_topk(const float* base, uint64_t n, const float* queries, uint64_t nq,
                   uint32_t dim, uint32_t k, uint32_t* out) {
    scored* best = (scored*)malloc((size_t)(k + 1) * sizeof(scored));
    for (uint64_t qi = 0; qi < nq; ++qi) {
        uint32_t cnt = 0;
        const float* q = queries + qi * dim;
        for (uint64_t j = 0; j < n; ++j) {
            scored s = {(uint32_t)j, orc_dot4(q, base + j * dim, dim)};
            /* insert into ascending-by-rank list of at most k */
            if (cnt == k && scored_cmp(&s, &best[k - 1]) >= 0) continue;
            uint32_t pos = cnt < k ? cnt : k - 1;
            while (pos > 0 && scored_cmp(&s, &best[pos - 1]) < 0) {
                best[pos] = best[pos - 1];
                --pos;
            }
            best[pos] = s;
            if (cnt < k) ++cnt;
        }
        for (uint32_t j = 0; j < k; ++j) out[qi * k + j] = j < cnt ? best[j].id : UINT32_MAX;
    }
    free(best);
    return ORC_OK;
}

/* ---- robust prune ------------------------------------------------------------ */

int orc_robust_prune(const orc_index* ix, const uint32_t* ids, const uint32_t* dists,
                     uint32_t n, uint32_t max_degree, float alpha, uint32_t* out,
                     uint32_t* out_n) {
    const uint64_t w = words_for_dim(ix->dim);
    uint64_t* keys = (uint64_t*)malloc((size_t)(n + 1) * sizeof(uint64_t));
    for (uint32_t i = 0; i < n; ++i) keys[i] = mkkey(dists[i], ids[i]);
    for (uint32_t i = 1; i < n; ++i) {
        uint64_t x = keys[i];
        uint32_t j = i;
        while (j > 0 && keys[j - 1] > x) {
            keys[j] = keys[j - 1];
            --j;
        }
        keys[j] = x;
    }
    uint32_t sel = 0;
    for (uint32_t i = 0; i < n && sel < max_degree; ++i) {
        const uint32_t cid = (uint32_t)keys[i];
        const float cd = (float)(uint32_t)(keys[i] >> 32);
        int keep = 1;
        for (uint32_t s = 0; s < sel; ++s) {
            const uint32_t d = orc_sm2_distance(ix->codes + (uint64_t)cid * 2 * w,
                                                ix->codes + (uint64_t)out[s] * 2 * w, w);
            const float covered = alpha * (float)d;
            if (cd > covered) {
                keep = 0;
                break;
            }
        }
        if (keep) out[sel++] = cid;
    }
    *out_n = sel;
    free(keys);
    return ORC_OK;
}
