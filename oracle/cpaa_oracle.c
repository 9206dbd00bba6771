/* TEST INFRASTRUCTURE — CPU oracle for the CPAA hot path.  See cpaa_oracle.h.
 *
 * Plain-C restatement of the reference algorithms (paths relative to
 * /root/reference/proj).  Compiled with -ffp-contract=off so that no
 * multiply-add is fused: the reference is built without -march on x86-64 and
 * therefore never emits FMA, and bit-identity with it is the point.
 */
#include "cpaa_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[512];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* or_last_error(void) { return g_err; }
int or_set_error(int code, const char* msg) { return fail(code, "%s", msg); }
void or_free(void* p) { free(p); }

/* ---- src/graph.cpp:10-19 ------------------------------------------------ */
double or_kahan_sum(const double* x, int64_t n) {
    double sum = 0.0, comp = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double y = x[i] - comp;
        double t = sum + y;
        comp = (t - sum) - y;
        sum = t;
    }
    return sum;
}

/* ---- src/coefficients.cpp ----------------------------------------------- */
static int check_c(double c) { /* coefficients.cpp:13-16 */
    if (!(c > 0.0 && c < 1.0))
        return fail(2, "damping factor must lie in (0,1), got %f", c);
    return 0;
}

int or_beta(double c, double* out) { /* coefficients.cpp:20-23 */
    int s = check_c(c);
    if (s) return s;
    *out = (1.0 - sqrt(1.0 - c * c)) / c;
    return 0;
}

int or_err_bound(double c, int M, double* out) { /* coefficients.cpp:33-38 */
    int s = check_c(c);
    if (s) return s;
    if (M < 0) return fail(2, "iteration bound must be non-negative");
    double b;
    or_beta(c, &b);
    *out = 2.0 * pow(b, M + 1) / (1.0 + b);
    return 0;
}

int or_plan_iterations(double c, double eps, int* M_out, double* predicted) {
    /* coefficients.cpp:40-55 */
    int s = check_c(c);
    if (s) return s;
    if (!(eps > 0.0 && eps < 1.0)) return fail(2, "target error must lie in (0,1), got %f", eps);
    int M = 0;
    double e;
    for (;;) {
        or_err_bound(c, M, &e);
        if (!(e > eps)) break;
        if (++M > 1000000) return fail(3, "iteration planning did not terminate");
    }
    *M_out = M;
    or_err_bound(c, M, predicted);
    return 0;
}

int or_coefficients(double c, int M, double* coeffs, double* beta_out, double* c0_out) {
    /* coefficients.cpp:57-71: c_k by repeated multiplication c0*beta*beta... */
    int s = check_c(c);
    if (s) return s;
    if (M < 0) return fail(2, "coefficient count must be non-negative");
    double b;
    or_beta(c, &b);
    double c0 = 2.0 / sqrt(1.0 - c * c);
    double ck = c0;
    for (int k = 0; k <= M; ++k) {
        if (coeffs) coeffs[k] = ck;
        ck *= b;
    }
    if (beta_out) *beta_out = b;
    if (c0_out) *c0_out = c0;
    return 0;
}

/* ---- std::mt19937_64 (Matsumoto & Nishimura 64-bit MT; the parameters the
 * C++ standard fixes for mt19937_64) and the reference's Rng helpers
 * (include/chebpr/generate.hpp:18-25, src/generate.cpp:11-19). ------------ */
typedef struct {
    uint64_t mt[312];
    int mti;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->mti = 312;
}

static uint64_t mt64_next(mt64* s) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
    if (s->mti >= 312) {
        int i;
        uint64_t x;
        for (i = 0; i < 312 - 156; ++i) {
            x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
            s->mt[i] = s->mt[i + 156] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
        }
        for (; i < 311; ++i) {
            x = (s->mt[i] & UM) | (s->mt[i + 1] & LM);
            s->mt[i] = s->mt[i + (156 - 312)] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
        }
        x = (s->mt[311] & UM) | (s->mt[0] & LM);
        s->mt[311] = s->mt[155] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
        s->mti = 0;
    }
    uint64_t x = s->mt[s->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

static double mt64_uniform01(mt64* s) { return (double)(mt64_next(s) >> 11) * 0x1.0p-53; }

static int64_t mt64_below(mt64* s, int64_t bound) {
    uint64_t b = (uint64_t)bound;
    uint64_t limit = UINT64_MAX - UINT64_MAX % b;
    for (;;) {
        uint64_t r = mt64_next(s);
        if (r < limit) return (int64_t)(r % b);
    }
}

typedef struct {
    int64_t* e;
    int64_t n, cap;
} edgevec;

static void ev_push(edgevec* v, int64_t a, int64_t b) {
    if (v->n == v->cap) {
        v->cap = v->cap ? 2 * v->cap : 1024;
        v->e = (int64_t*)realloc(v->e, sizeof(int64_t) * 2 * (size_t)v->cap);
    }
    v->e[2 * v->n] = a;
    v->e[2 * v->n + 1] = b;
    v->n++;
}

int or_gnp_edges(int64_t n, double p, uint64_t seed, int64_t** edges, int64_t* count) {
    /* src/generate.cpp:51-87 */
    if (n < 2) return fail(2, "gnp needs n >= 2");
    if (!(p >= 0.0 && p <= 1.0)) return fail(2, "gnp needs p in [0,1]");
    mt64 rng;
    mt64_seed(&rng, seed);
    edgevec ev = {0, 0, 0};
    if (p > 0.0 && p < 1.0) {
        double logq = log1p(-p);
        int64_t v = 1, w = -1;
        while (v < n) {
            double skip = floor(log1p(-mt64_uniform01(&rng)) / logq);
            w += 1 + (int64_t)skip;
            while (w >= v && v < n) {
                w -= v;
                ++v;
            }
            if (v < n) ev_push(&ev, v, w);
        }
    } else if (p == 1.0) {
        for (int64_t v = 1; v < n; ++v)
            for (int64_t w = 0; w < v; ++w) ev_push(&ev, v, w);
    }
    char* touched = (char*)calloc((size_t)n, 1);
    for (int64_t i = 0; i < ev.n; ++i) {
        touched[ev.e[2 * i]] = 1;
        touched[ev.e[2 * i + 1]] = 1;
    }
    for (int64_t v = 0; v < n; ++v) {
        if (touched[v]) continue;
        int64_t u = v;
        while (u == v) u = mt64_below(&rng, n);
        ev_push(&ev, v, u);
        touched[u] = 1;
    }
    free(touched);
    if (!ev.e) ev.e = (int64_t*)malloc(16);
    *edges = ev.e;
    *count = ev.n;
    return 0;
}

/* ---- src/graph.cpp:23-102 ----------------------------------------------- */
static int cmp_pair(const void* a, const void* b) {
    const int64_t* x = (const int64_t*)a;
    const int64_t* y = (const int64_t*)b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    if (x[1] != y[1]) return x[1] < y[1] ? -1 : 1;
    return 0;
}

static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

int or_build_graph(const int64_t* edges, int64_t E, int dedup, int drop_isolated,
                   int64_t n_hint, int64_t* n_out, int64_t* m_out, int64_t** offsets_out,
                   int64_t** neighbors_out, int64_t** degrees_out, double** inv_out,
                   int64_t* duplicates_removed, int64_t* isolated_dropped) {
    int64_t n = n_hint > 0 ? n_hint : 0; /* graph.cpp:25-29 */
    for (int64_t i = 0; i < E; ++i) {
        int64_t a = edges[2 * i], b = edges[2 * i + 1];
        if (a < 0 || b < 0) return fail(1, "negative vertex id in edge list");
        int64_t mx = (a > b ? a : b) + 1;
        if (mx > n) n = mx;
    }
    /* canonical (min,max), sorted: graph.cpp:31-36 */
    int64_t* canon = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)(E + 1));
    for (int64_t i = 0; i < E; ++i) {
        int64_t a = edges[2 * i], b = edges[2 * i + 1];
        canon[2 * i] = a < b ? a : b;
        canon[2 * i + 1] = a < b ? b : a;
    }
    qsort(canon, (size_t)E, 2 * sizeof(int64_t), cmp_pair);
    int64_t m = E;
    *duplicates_removed = 0;
    if (dedup) { /* graph.cpp:39-43 */
        int64_t w = 0;
        for (int64_t i = 0; i < E; ++i) {
            if (w > 0 && canon[2 * (w - 1)] == canon[2 * i] &&
                canon[2 * (w - 1) + 1] == canon[2 * i + 1])
                continue;
            canon[2 * w] = canon[2 * i];
            canon[2 * w + 1] = canon[2 * i + 1];
            ++w;
        }
        *duplicates_removed = E - w;
        m = w;
    }
    int64_t* deg = (int64_t*)calloc((size_t)(n + 1), sizeof(int64_t)); /* graph.cpp:45-49 */
    for (int64_t i = 0; i < m; ++i) {
        deg[canon[2 * i]]++;
        if (canon[2 * i + 1] != canon[2 * i]) deg[canon[2 * i + 1]]++;
    }
    *isolated_dropped = 0;
    if (drop_isolated) { /* graph.cpp:51-69: order-preserving renumbering */
        int64_t* remap = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
        int64_t next = 0;
        for (int64_t v = 0; v < n; ++v) remap[v] = deg[v] > 0 ? next++ : -1;
        *isolated_dropped = n - next;
        if (*isolated_dropped > 0) {
            for (int64_t i = 0; i < 2 * m; ++i) canon[i] = remap[canon[i]];
            n = next;
            memset(deg, 0, sizeof(int64_t) * (size_t)(n + 1));
            for (int64_t i = 0; i < m; ++i) {
                deg[canon[2 * i]]++;
                if (canon[2 * i + 1] != canon[2 * i]) deg[canon[2 * i + 1]]++;
            }
        }
        free(remap);
    } else { /* graph.cpp:70-75 */
        for (int64_t v = 0; v < n; ++v)
            if (deg[v] == 0) {
                free(canon);
                free(deg);
                return fail(1, "vertex %lld is isolated (degree 0)", (long long)v);
            }
    }
    /* CSR fill: graph.cpp:77-95 */
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
    off[0] = 0;
    for (int64_t v = 0; v < n; ++v) off[v + 1] = off[v] + deg[v];
    int64_t nnz = off[n];
    int64_t* nb = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nnz + 1));
    int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
    memcpy(cur, off, sizeof(int64_t) * (size_t)n);
    for (int64_t i = 0; i < m; ++i) {
        int64_t a = canon[2 * i], b = canon[2 * i + 1];
        nb[cur[a]++] = b;
        if (b != a) nb[cur[b]++] = a;
    }
    for (int64_t v = 0; v < n; ++v)
        qsort(nb + off[v], (size_t)(off[v + 1] - off[v]), sizeof(int64_t), cmp_i64);
    double* inv = (double*)malloc(sizeof(double) * (size_t)(n + 1)); /* graph.cpp:97-99 */
    for (int64_t v = 0; v < n; ++v) inv[v] = 1.0 / (double)deg[v];
    free(cur);
    free(canon);
    *n_out = n;
    *m_out = m;
    *offsets_out = off;
    *neighbors_out = nb;
    *degrees_out = deg;
    *inv_out = inv;
    return 0;
}

/* ---- src/graph.cpp:104-121 ---------------------------------------------- */
void or_transition_apply(int64_t n, const int64_t* off, const int64_t* nb, const double* inv,
                         const double* x, double* y) {
    double* ctb = (double*)malloc(sizeof(double) * (size_t)(n + 1));
    for (int64_t v = 0; v < n; ++v) ctb[v] = x[v] * inv[v];
    for (int64_t u = 0; u < n; ++u) {
        double s = 0.0;
        for (int64_t i = off[u]; i < off[u + 1]; ++i) s += ctb[nb[i]];
        y[u] = s;
    }
    free(ctb);
}

/* ---- src/cpaa.cpp:40-68 ------------------------------------------------- */
int or_partition_vertices(int64_t n, const int64_t* degrees, int K, int64_t* cuts) {
    if (K < 1) return fail(2, "parallelism must be >= 1");
    int64_t* prefix = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
    prefix[0] = 0;
    for (int64_t v = 0; v < n; ++v) prefix[v + 1] = prefix[v] + degrees[v];
    const double total = (double)prefix[n];
    cuts[0] = 0;
    cuts[K] = n;
    for (int j = 1; j < K; ++j) {
        double ideal = total * j / K;
        int64_t lo = 0, hi = n + 1; /* lower_bound: first prefix[idx] >= ideal */
        while (lo < hi) {
            int64_t mid = lo + (hi - lo) / 2;
            if ((double)prefix[mid] < ideal) lo = mid + 1;
            else hi = mid;
        }
        int64_t idx = lo;
        if (idx > n) idx = n;
        if (idx > 0 && (idx == n + 1 || (double)prefix[idx] - ideal > ideal - (double)prefix[idx - 1]))
            --idx;
        if (idx < cuts[j - 1]) idx = cuts[j - 1];
        if (idx > n) idx = n;
        cuts[j] = idx;
    }
    free(prefix);
    return 0;
}

/* ---- src/cpaa.cpp:79-165 ------------------------------------------------ */
int or_run_cpaa(int64_t n, const int64_t* off, const int64_t* nb, const double* invdeg,
                double c, int M, const double* p, double* ranks, double* trace_out,
                double* total_mass) {
    if (n < 1) return fail(1, "graph has no vertices");
    if (M < 0) return fail(2, "coefficient count must be non-negative");
    double* coeffs = (double*)malloc(sizeof(double) * (size_t)(M + 1));
    double beta, c0;
    int s = or_coefficients(c, M, coeffs, &beta, &c0);
    if (s) {
        free(coeffs);
        return s;
    }
    double* T_prev = (double*)malloc(sizeof(double) * (size_t)n);
    double* T_curr = (double*)malloc(sizeof(double) * (size_t)n);
    double* T_next = (double*)malloc(sizeof(double) * (size_t)n);
    double* ctb = (double*)malloc(sizeof(double) * (size_t)n);
    double* acc = (double*)malloc(sizeof(double) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) { /* cpaa.cpp:88-92 (T0 = ones unless p given) */
        double t0 = p ? p[i] : 1.0;
        T_prev[i] = t0;
        T_curr[i] = t0;
        acc[i] = p ? (c0 / 2.0) * t0 : c0 / 2.0;
    }
    double residual = (double)n * c0 * beta / (1.0 - beta); /* cpaa.cpp:99 */
    double last_S = 0.0;
    int rc = 0;
    for (int k = 1; k <= M; ++k) { /* cpaa.cpp:109-156 */
        const double ck = coeffs[k];
        for (int64_t v = 0; v < n; ++v) ctb[v] = T_curr[v] * invdeg[v]; /* :116 */
        const int first = k == 1;
        for (int64_t u = 0; u < n; ++u) { /* :126-132 */
            double sum = 0.0;
            for (int64_t i = off[u]; i < off[u + 1]; ++i) sum += ctb[nb[i]];
            double t = first ? sum : 2.0 * sum - T_prev[u];
            T_next[u] = t;
            acc[u] += ck * t;
        }
        double* tmp = T_prev; /* :136-137 */
        T_prev = T_curr;
        T_curr = T_next;
        T_next = tmp;
        double mass_T = or_kahan_sum(T_curr, n); /* :142-145 */
        double S_k = or_kahan_sum(acc, n);
        residual *= beta;
        if (trace_out) {
            double* r = trace_out + 10 * (k - 1);
            r[0] = k;
            r[1] = ck;
            r[2] = S_k;
            r[3] = residual;
            r[4] = r[5] = r[7] = r[8] = r[9] = 0.0;
            r[6] = mass_T;
        }
        if (!isfinite(mass_T) || !isfinite(S_k)) { /* :147-148 */
            rc = fail(3, "non-finite value at round %d", k);
            goto done;
        }
        last_S = S_k;
    }
    {
        double total = M == 0 ? or_kahan_sum(acc, n) : last_S; /* :158-163 */
        if (!isfinite(total) || total <= 0.0) {
            rc = fail(3, "normalization total is not positive and finite");
            goto done;
        }
        for (int64_t i = 0; i < n; ++i) ranks[i] = acc[i] / total;
        *total_mass = total;
    }
done:
    free(coeffs);
    free(T_prev);
    free(T_curr);
    free(T_next);
    free(ctb);
    free(acc);
    return rc;
}

/* ---- src/power.cpp:28-109 ----------------------------------------------- */
int or_run_power(int64_t n, const int64_t* off, const int64_t* nb, const double* invdeg,
                 double c, int rounds, double tol, int max_rounds, double* ranks,
                 double* trace_out, int* rounds_out, double* total_mass) {
    if (n < 1) return fail(1, "graph has no vertices");
    if (!(c > 0.0 && c < 1.0)) return fail(2, "damping factor must lie in (0,1)");
    const int fixed = rounds >= 0;
    const int by_tol = tol > 0.0;
    if (fixed == by_tol) return fail(4, "set exactly one of rounds and tol");
    const int budget = fixed ? rounds : max_rounds;
    if (budget < 0) return fail(4, "round budget must be non-negative");
    const double base = (1.0 - c) / (double)n;
    double* x = (double*)malloc(sizeof(double) * (size_t)n);
    double* y = (double*)malloc(sizeof(double) * (size_t)n);
    double* ctb = (double*)malloc(sizeof(double) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) x[i] = 1.0 / (double)n;
    int k = 0, rc = 0;
    while (k < budget) {
        ++k;
        for (int64_t v = 0; v < n; ++v) ctb[v] = x[v] * invdeg[v];
        for (int64_t u = 0; u < n; ++u) {
            double s = 0.0;
            for (int64_t i = off[u]; i < off[u + 1]; ++i) s += ctb[nb[i]];
            y[u] = c * s + base;
        }
        double l1 = 0.0, comp = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            double d = fabs(y[i] - x[i]) - comp;
            double t = l1 + d;
            comp = (t - l1) - d;
            l1 = t;
        }
        double* tmp = x;
        x = y;
        y = tmp;
        if (trace_out) {
            double* r = trace_out + 10 * (k - 1);
            memset(r, 0, 10 * sizeof(double));
            r[0] = k;
            r[4] = l1;
            r[6] = or_kahan_sum(x, n);
        }
        if (!isfinite(l1)) {
            rc = fail(3, "non-finite value at round %d", k);
            goto done;
        }
        if (by_tol && l1 < tol) break;
    }
    memcpy(ranks, x, sizeof(double) * (size_t)n);
    *rounds_out = k;
    *total_mass = or_kahan_sum(ranks, n);
done:
    free(x);
    free(y);
    free(ctb);
    return rc;
}
