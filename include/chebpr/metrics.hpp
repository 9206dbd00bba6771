// Drop-in for /root/reference/proj/include/chebpr/metrics.hpp (host test-oracle helpers).
#pragma once

#include "chebpr/graph.hpp"

namespace chebpr {

struct ErrorReport {
    double max_rel_err = 0.0;  // max |est - ref| / ref
    double l1_err = 0.0;       // sum |est - ref| (compensated)
    double mass_gap = 0.0;     // |sum(est) - 1|
};

ErrorReport max_relative_error(const Vector& est, const Vector& ref);
Vector dense_direct_solve(const UndirectedGraph& g, double c);  // n <= 512
double symmetry_similarity_check(const UndirectedGraph& g);     // n <= 2048
double mass_check(const Vector& vec, double expected);

}  // namespace chebpr
