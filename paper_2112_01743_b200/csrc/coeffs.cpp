// Host coefficient kit of the CPAA path.  Restates the reference's closed forms
// (/root/reference/proj/src/coefficients.cpp:13-71, cpaa.cpp:28-36) with the same
// floating-point operation order: the table c_0..c_M feeds every term kernel, so
// its bits must match the reference's exactly.
#include <cmath>
#include <string>
#include <vector>

#include "common.cuh"

namespace chebgpu {

namespace {
void require_damping(double c) {
    // coefficients.cpp:13-16
    if (!(c > 0.0 && c < 1.0))
        fail(CHEB_DOMAIN, "damping factor must lie in (0,1), got " + std::to_string(c));
}
}  // namespace

double beta(double c) {  // coefficients.cpp:20-23, (1 - sqrt(1-c^2)) / c
    require_damping(c);
    const double root = std::sqrt(1.0 - c * c);
    return (1.0 - root) / c;
}

double sigma(double c) {  // coefficients.cpp:25-31, evaluated independently of beta
    require_damping(c);
    const double s = std::sqrt(1.0 - c * c);
    const double numer = c * c - (2.0 - c) * (1.0 - s);
    const double denom = c * c - c * (1.0 - s);
    return numer / denom;
}

double err_bound(double c, int M) {  // coefficients.cpp:33-38, 2 beta^(M+1) / (1+beta)
    require_damping(c);
    if (M < 0) fail(CHEB_DOMAIN, "iteration bound must be non-negative");
    const double b = beta(c);
    return 2.0 * std::pow(b, M + 1) / (1.0 + b);
}

int plan_iterations(double c, double eps, double* predicted) {  // coefficients.cpp:40-55
    require_damping(c);
    if (!(eps > 0.0 && eps < 1.0))
        fail(CHEB_DOMAIN, "target error must lie in (0,1), got " + std::to_string(eps));
    int M = 0;
    while (err_bound(c, M) > eps)
        if (++M > 1000000) fail(CHEB_NUMERIC, "iteration planning did not terminate");
    if (predicted) *predicted = err_bound(c, M);
    return M;
}

void coefficients(double c, int M, std::vector<double>& out, double* beta_out, double* c0_out) {
    // coefficients.cpp:57-71: c_k = c0 * beta^k by REPEATED multiplication.
    require_damping(c);
    if (M < 0) fail(CHEB_DOMAIN, "coefficient count must be non-negative");
    const double b = beta(c);
    const double c0 = 2.0 / std::sqrt(1.0 - c * c);
    out.assign(static_cast<size_t>(M) + 1, 0.0);
    double ck = c0;
    for (auto& v : out) {
        v = ck;
        ck *= b;
    }
    if (beta_out) *beta_out = b;
    if (c0_out) *c0_out = c0;
}

int resolve_rounds(double c, int rounds, double eps, int max_rounds) {
    // cpaa.cpp:28-36 — an explicit round count is clamped to max_rounds too.
    const bool by_rounds = rounds >= 0;
    const bool by_eps = eps > 0.0;
    if (by_rounds == by_eps) fail(CHEB_INVALID_ARG, "set exactly one of rounds and eps");
    if (max_rounds < 0) fail(CHEB_INVALID_ARG, "max_rounds must be non-negative");
    const int M = by_rounds ? rounds : plan_iterations(c, eps, nullptr);
    return M < max_rounds ? M : max_rounds;
}

void partition_cuts(const int64_t* degrees, int64_t n, int K, int64_t* cuts) {
    // cpaa.cpp:40-68: the j-th cut at the degree prefix nearest j/K of the total.
    if (K < 1) fail(CHEB_DOMAIN, "parallelism must be >= 1");
    std::vector<int64_t> prefix(static_cast<size_t>(n) + 1, 0);
    for (int64_t v = 0; v < n; ++v) prefix[v + 1] = prefix[v] + degrees[v];
    const double total = static_cast<double>(prefix[n]);
    cuts[0] = 0;
    cuts[K] = n;
    for (int j = 1; j < K; ++j) {
        const double ideal = total * j / K;
        int64_t lo = 0, hi = n + 1;  // first prefix >= ideal (as doubles)
        while (lo < hi) {
            const int64_t mid = lo + (hi - lo) / 2;
            if (static_cast<double>(prefix[mid]) < ideal) lo = mid + 1;
            else hi = mid;
        }
        int64_t idx = lo > n ? n : lo;
        if (idx > 0 && static_cast<double>(prefix[idx]) - ideal > ideal - static_cast<double>(prefix[idx - 1]))
            --idx;
        if (idx < cuts[j - 1]) idx = cuts[j - 1];
        if (idx > n) idx = n;
        cuts[j] = idx;
    }
}

double kahan_sum(const double* x, int64_t n) {  // graph.cpp:10-19, compensated serial sum
    double total = 0.0, lost = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double y = x[i] - lost;
        const double t = total + y;
        lost = (t - total) - y;
        total = t;
    }
    return total;
}

}  // namespace chebgpu
