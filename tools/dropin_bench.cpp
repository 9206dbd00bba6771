// The drop-in as a C++ reference user calls it: build_graph on host edges, then
// chebpr::run_cpaa(g, cfg) (stateless: each call uploads the host CSR, solves, returns host
// ranks).  Prints the per-call wall time on a config-2-sized Chung-Lu graph.
// Build: g++ -std=c++20 -O2 -Iinclude tools/dropin_bench.cpp -Lpaper_2112_01743_b200/lib \
//        -lchebpr_dropin -lchebpr_b200 -Wl,-rpath,$PWD/paper_2112_01743_b200/lib -o build/dropin_bench
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>

#include "chebpr/cpaa.hpp"
#include "chebpr/generate.hpp"
#include "chebpr/graph.hpp"

int main() {
    using clk = std::chrono::steady_clock;
    auto t0 = clk::now();
    chebpr::EdgeList e = chebpr::chung_lu_edges(1 << 20, 2.1, 2.0, 50000.0, 10485760, 2);
    const double gen_ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
    double build_ms = 0;
    chebpr::BuildResult b;
    for (int i = 0; i < 3; ++i) {  // build_graph: host edges -> K1 on the device -> host CSR
        auto t = clk::now();
        b = chebpr::build_graph(e);
        build_ms = std::chrono::duration<double, std::milli>(clk::now() - t).count();
    }
    const auto& g = b.graph;
    std::printf("graph: n=%lld nnz=%zu; generate %.0f ms, build_graph %.1f ms (3rd call)\n", (long long)g.n,
                g.neighbors.size(), gen_ms, build_ms);
    chebpr::SolverConfig cfg;
    cfg.eps = 1e-10;
    std::vector<double> ms;
    double total = 0;
    for (int i = 0; i < 6; ++i) {
        auto t = clk::now();
        chebpr::PageRankResult r = chebpr::run_cpaa(g, cfg);
        ms.push_back(std::chrono::duration<double, std::milli>(clk::now() - t).count());
        total = r.total_mass;
    }
    std::sort(ms.begin() + 1, ms.end());
    std::printf("run_cpaa(UndirectedGraph) per call: first %.1f ms, median of next 5 %.2f ms (total mass %.6g)\n",
                ms[0], ms[3], total);
    return 0;
}
