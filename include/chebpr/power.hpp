// Drop-in for /root/reference/proj/include/chebpr/power.hpp: the Power comparator on the
// B200 (C-ABI cheb_power).
#pragma once

#include "chebpr/cpaa.hpp"
#include "chebpr/graph.hpp"

namespace chebpr {

struct PowerConfig {
    double c = 0.85;
    int rounds = -1;  // exactly one of rounds / tol; rounds ignores max_rounds
    double tol = -1.0;
    int max_rounds = 60;
    int parallelism = 1;
    Mode mode = Mode::Auto;  // new
    int device = 0;          // new
};

PageRankResult run_power(const UndirectedGraph& g, const PowerConfig& cfg,
                         const Vector* reference = nullptr);
Vector reference_pagerank(const UndirectedGraph& g, double c);

}  // namespace chebpr
