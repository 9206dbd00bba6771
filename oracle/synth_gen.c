/* TEST INFRASTRUCTURE — plain-C restatement of the synthetic graph generators of the
 * BASELINE configs 2-5 (R-MAT and Chung-Lu).  Not product code.
 *
 * The reference ships only ring / star / regular / gnp generators
 * (/root/reference/proj/src/generate.cpp:11-87); BASELINE.json's configs 2-5 name R-MAT
 * and Chung-Lu graphs that it does not generate, so the product defines them as
 * counter-based generators (paper_2112_01743_b200/csrc/generate.cu, gen::rmat_edge,
 * gen::chung_lu_cdf, k_chung_lu, rewire_partner).  This file restates that definition
 * independently so that the CPU legs (bench.py --impl reference, the full-size parity
 * tests) build the reference's graph from an edge list without loading the product
 * library.  tests/test_oracle.py pins it: identical edge arrays to the product's host and
 * device generators on small and medium sizes.
 *
 * Definition (every edge an independent function of (seed, edge index)):
 *   mix64        splitmix64 finaliser
 *   draw(s, i)   mix64(mix64(seed ^ s * 0xD1B54A32D192ED03) + i * 0x9E3779B97F4A7C15)
 *   R-MAT edge i: `scale` quadrant choices, two per 64-bit draw (low then high 32 bits)
 *                of stream 1 at counter i*64 + level/2, against the thresholds
 *                floor(a 2^32), floor((a+b) 2^32), floor((a+b+c) 2^32); ids relabelled by
 *                a Fisher-Yates permutation (std::mt19937_64 seeded with seed ^ 0x5EED, the
 *                reference's bias-free rejection draw, generate.cpp:11-19); self-loops
 *                dropped; edge order = draw order.
 *   Chung-Lu:    weights w_v = (lo + u_v (hi - lo))^(1/(1-gamma)), lo/hi = wmin/wmax^(1-gamma),
 *                u_v from stream 0; integer CDF of llround(w_v 2^20); endpoints of draw i
 *                picked by mulhi(draw(2|3, i), total) through the CDF; self-loops dropped;
 *                then every vertex no kept edge touches, ascending, gets (v, partner) with
 *                partner = the first mulhi(draw(4, v | t << 40), n) != v, t = 0, 1, ...
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include "cpaa_oracle.h"

int or_set_error(int code, const char* msg); /* cpaa_oracle.c */

static uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static uint64_t draw(uint64_t seed, uint64_t s, uint64_t i) {
    return mix64(mix64(seed ^ (s * 0xD1B54A32D192ED03ull)) + i * 0x9E3779B97F4A7C15ull);
}

static uint64_t mulhi(uint64_t a, uint64_t b) { return (uint64_t)(((unsigned __int128)a * b) >> 64); }

/* ---- std::mt19937_64 (for the relabelling permutation) ---- */
typedef struct {
    uint64_t mt[312];
    int i;
} mt64s;

static void mt_seed(mt64s* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int k = 1; k < 312; ++k)
        s->mt[k] = 6364136223846793005ull * (s->mt[k - 1] ^ (s->mt[k - 1] >> 62)) + (uint64_t)k;
    s->i = 312;
}

static uint64_t mt_next(mt64s* s) {
    if (s->i >= 312) {
        for (int k = 0; k < 312; ++k) {
            const uint64_t y = (s->mt[k] & 0xFFFFFFFF80000000ull) | (s->mt[(k + 1) % 312] & 0x7FFFFFFFull);
            uint64_t v = s->mt[(k + 156) % 312] ^ (y >> 1);
            if (y & 1) v ^= 0xB5026F5AA96619E9ull;
            s->mt[k] = v;
        }
        s->i = 0;
    }
    uint64_t x = s->mt[s->i++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= x >> 43;
    return x;
}

/* ---- worker pool over contiguous draw ranges; outputs concatenated in range order ---- */
typedef struct {
    int kind; /* 0 rmat, 1 chung-lu */
    int64_t b, e;
    /* rmat */
    int scale;
    uint64_t ta, tb, tc, seed;
    const int32_t* perm;
    /* chung-lu */
    const uint64_t* cum;
    int64_t n;
    /* out: int64 pairs */
    int64_t* out;
    int64_t cnt;
} job_t;

static uint32_t cdf_pick(const uint64_t* cum, int64_t n, uint64_t x) {
    int64_t lo = 0, hi = n - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (cum[mid] > x) hi = mid;
        else lo = mid + 1;
    }
    return (uint32_t)lo;
}

static void* run_job(void* arg) {
    job_t* j = (job_t*)arg;
    int64_t c = 0;
    if (j->kind == 0) {
        for (int64_t i = j->b; i < j->e; ++i) {
            uint32_t a = 0, bb = 0;
            uint64_t r = 0;
            for (int l = 0; l < j->scale; ++l) {
                if ((l & 1) == 0) r = draw(j->seed, 1, (uint64_t)i * 64 + (uint64_t)(l >> 1));
                const uint64_t q = (l & 1) ? (r >> 32) : (r & 0xffffffffull);
                const uint32_t bu = q >= j->tb ? 1u : 0u;
                const uint32_t bv = ((q >= j->ta && q < j->tb) || q >= j->tc) ? 1u : 0u;
                a = (a << 1) | bu;
                bb = (bb << 1) | bv;
            }
            if (a == bb) continue;
            j->out[2 * c] = j->perm[a];
            j->out[2 * c + 1] = j->perm[bb];
            ++c;
        }
    } else {
        const uint64_t T = j->cum[j->n - 1];
        for (int64_t i = j->b; i < j->e; ++i) {
            const uint32_t u = cdf_pick(j->cum, j->n, mulhi(draw(j->seed, 2, (uint64_t)i), T));
            const uint32_t v = cdf_pick(j->cum, j->n, mulhi(draw(j->seed, 3, (uint64_t)i), T));
            if (u == v) continue;
            j->out[2 * c] = u;
            j->out[2 * c + 1] = v;
            ++c;
        }
    }
    j->cnt = c;
    return NULL;
}

static int nthreads(int64_t work) {
    long t = sysconf(_SC_NPROCESSORS_ONLN);
    if (t < 1) t = 1;
    if (t > 64) t = 64;
    if (work < 1 << 16) t = 1;
    return (int)t;
}

/* Runs the jobs over [0, draws) and compacts into one malloc'ed int64 pair array with
 * room for `extra` more pairs. */
static int64_t* run_all(job_t proto, int64_t draws, int64_t extra, int64_t* count) {
    const int T = nthreads(draws);
    job_t jobs[64];
    pthread_t th[64];
    int64_t* out = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)(draws + extra + 1));
    if (!out) return NULL;
    for (int t = 0; t < T; ++t) {
        jobs[t] = proto;
        jobs[t].b = draws * t / T;
        jobs[t].e = draws * (t + 1) / T;
        jobs[t].out = out + 2 * jobs[t].b; /* in place: a range only shrinks */
        pthread_create(&th[t], NULL, run_job, &jobs[t]);
    }
    int64_t pos = 0;
    for (int t = 0; t < T; ++t) {
        pthread_join(th[t], NULL);
        if (out + 2 * pos != jobs[t].out)
            memmove(out + 2 * pos, jobs[t].out, sizeof(int64_t) * 2 * (size_t)jobs[t].cnt);
        pos += jobs[t].cnt;
    }
    *count = pos;
    return out;
}

int or_rmat_edges(int scale, int64_t edge_factor, double a, double b, double c, uint64_t seed,
                  int64_t** edges, int64_t* count) {
    if (scale < 1 || scale > 30) return or_set_error(2, "rmat scale must be in [1,30]");
    const int64_t n = (int64_t)1 << scale;
    const int64_t draws = edge_factor * n;
    int32_t* perm = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    if (!perm) return or_set_error(5, "out of host memory");
    for (int64_t i = 0; i < n; ++i) perm[i] = (int32_t)i;
    mt64s* eng = (mt64s*)malloc(sizeof(mt64s));
    mt_seed(eng, seed ^ 0x5EEDull);
    for (int64_t i = n - 1; i > 0; --i) {
        const uint64_t bound = (uint64_t)i + 1;
        const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
        uint64_t r;
        do r = mt_next(eng);
        while (r >= limit);
        const int64_t k = (int64_t)(r % bound);
        const int32_t t = perm[i];
        perm[i] = perm[k];
        perm[k] = t;
    }
    free(eng);
    const double two32 = 4294967296.0;
    job_t p;
    memset(&p, 0, sizeof p);
    p.kind = 0;
    p.scale = scale;
    p.ta = (uint64_t)floor(a * two32);
    p.tb = (uint64_t)floor((a + b) * two32);
    p.tc = (uint64_t)floor((a + b + c) * two32);
    p.seed = seed;
    p.perm = perm;
    int64_t* out = run_all(p, draws, 0, count);
    free(perm);
    if (!out) return or_set_error(5, "out of host memory");
    *edges = out;
    return 0;
}

int or_chung_lu_edges(int64_t n, double gamma, double wmin, double wmax, int64_t draws, uint64_t seed,
                      int64_t** edges, int64_t* count) {
    if (n < 2 || n > INT32_MAX) return or_set_error(2, "chung_lu needs 2 <= n < 2^31");
    if (!(gamma > 1.0) || !(wmin > 0.0) || !(wmax >= wmin))
        return or_set_error(2, "chung_lu needs gamma > 1 and 0 < wmin <= wmax");
    uint64_t* cum = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n);
    if (!cum) return or_set_error(5, "out of host memory");
    const double e = 1.0 - gamma;
    const double lo = pow(wmin, e), hi = pow(wmax, e);
    uint64_t acc = 0;
    for (int64_t v = 0; v < n; ++v) {
        const double u = (double)(draw(seed, 0, (uint64_t)v) >> 11) * 0x1.0p-53;
        const double w = pow(lo + u * (hi - lo), 1.0 / e);
        acc += (uint64_t)llround(w * 1048576.0);
        cum[v] = acc;
    }
    job_t p;
    memset(&p, 0, sizeof p);
    p.kind = 1;
    p.seed = seed;
    p.cum = cum;
    p.n = n;
    int64_t kept = 0;
    int64_t* out = run_all(p, draws, n, &kept);
    free(cum);
    if (!out) return or_set_error(5, "out of host memory");
    unsigned char* touched = (unsigned char*)calloc((size_t)n, 1);
    if (!touched) {
        free(out);
        return or_set_error(5, "out of host memory");
    }
    for (int64_t i = 0; i < 2 * kept; ++i) touched[out[i]] = 1;
    int64_t pos = kept;
    for (int64_t v = 0; v < n; ++v) {
        if (touched[v]) continue;
        uint64_t u = 0;
        for (uint64_t t = 0;; ++t) {
            u = mulhi(draw(seed, 4, (uint64_t)v | (t << 40)), (uint64_t)n);
            if (u != (uint64_t)v) break;
        }
        out[2 * pos] = v;
        out[2 * pos + 1] = (int64_t)u;
        ++pos;
    }
    free(touched);
    *edges = out;
    *count = pos;
    return 0;
}
