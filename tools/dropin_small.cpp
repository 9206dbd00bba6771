// Per-call latency of the drop-in on config 1 (gnp(10000, 0.001, seed 1)): a stateless
// chebpr::run_cpaa(g, cfg) as a reference user calls it, median of 20 calls, Auto mode
// (bit-exact for this size) and Fast mode.
// Build: g++ -std=c++20 -O2 -Iinclude tools/dropin_small.cpp -Lpaper_2112_01743_b200/lib \
//        -lchebpr_dropin -lchebpr_b200 -Wl,-rpath,$PWD/paper_2112_01743_b200/lib -o build/dropin_small
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>

#include "chebpr/cpaa.hpp"
#include "chebpr/generate.hpp"
#include "chebpr/graph.hpp"

int main() {
    using clk = std::chrono::steady_clock;
    chebpr::UndirectedGraph g = chebpr::build_graph(chebpr::gnp_edges(10000, 0.001, 1)).graph;
    for (int mode = 0; mode < 2; ++mode) {
        chebpr::SolverConfig cfg;
        cfg.eps = 1e-10;
        cfg.mode = mode == 0 ? chebpr::Mode::Auto : chebpr::Mode::Fast;
        std::vector<double> ms;
        for (int i = 0; i < 21; ++i) {
            auto t = clk::now();
            chebpr::PageRankResult r = chebpr::run_cpaa(g, cfg);
            ms.push_back(std::chrono::duration<double, std::milli>(clk::now() - t).count());
            (void)r;
        }
        std::sort(ms.begin() + 1, ms.end());
        std::printf("config 1, %s: median %.2f ms per call (first %.1f)\n", mode == 0 ? "Auto (bit-exact)" : "Fast",
                    ms[10], ms[0]);
    }
    return 0;
}
