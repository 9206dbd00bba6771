// Drop-in for /root/reference/proj/include/chebpr/cpaa.hpp: run_cpaa and its staged pieces
// on the B200 (C-ABI cheb_cpaa / cheb_state_*).  Additive SolverConfig fields select the
// schedule: Mode::Auto runs the bit-exact storage-order schedule for graphs up to
// kAutoExactNnz CSR entries (results bitwise equal to the reference, trace included) and
// the degree-binned FAST schedule above it (<= 1e-12 from the reference).
#pragma once

#include <cstdint>
#include <vector>

#include "chebpr/graph.hpp"

namespace chebpr {

enum class Mode { Auto = -1, Fast = 0, BitExact = 1 };
constexpr int64_t kAutoExactNnz = int64_t(1) << 20;

struct SolverConfig {
    double c = 0.85;
    int rounds = -1;      // exactly one of rounds / eps
    double eps = -1.0;
    int max_rounds = 60;  // clamp for either
    int parallelism = 1;  // accepted; results never depend on it
    // new (additive)
    Mode mode = Mode::Auto;
    int precision = 64;   // 64 or 32
    int device = 0;
};

struct TraceRow {
    int k = 0;
    double c_k = 0.0;
    double S_k = 0.0;
    double residual_mass = 0.0;
    double l1_change = 0.0;
    double elapsed_ms = 0.0;
    double mass_T = 0.0;
    double err = 0.0;
    double err_l1 = 0.0;
};

struct PageRankResult {
    Vector ranks;
    std::vector<TraceRow> trace;
    int rounds = 0;
    bool has_err = false;
    double total_mass = 0.0;
};

struct VertexRange {
    int64_t begin = 0;
    int64_t end = 0;
};
std::vector<VertexRange> partition_vertices(const UndirectedGraph& g, int K);

Vector normalize(const Vector& v);

PageRankResult run_cpaa(const UndirectedGraph& g, const SolverConfig& cfg,
                        const Vector* reference = nullptr);

struct IterationState {
    Vector T_prev, T_curr, T_next, acc;
    int k = 1;
};
IterationState init_state(const UndirectedGraph& g, double c0);
void generate_stage(const UndirectedGraph& g, IterationState& state);
void accumulate_stage(IterationState& state, double c_k);

}  // namespace chebpr
