// Drop-in for /root/reference/proj/include/chebpr/generate.hpp: the reference's synthetic
// generators (host, std::mt19937_64 — byte-identical edge sequences; C-ABI cheb_gen_*).
#pragma once

#include <cstdint>
#include <random>
#include <string>
#include <utility>
#include <vector>

namespace chebpr {

using EdgeList = std::vector<std::pair<int64_t, int64_t>>;

// 64-bit Mersenne Twister with hand-rolled draws (the standard distributions are not
// bit-stable across library implementations).
struct Rng {
    std::mt19937_64 eng;
    explicit Rng(uint64_t seed) : eng(seed) {}
    double uniform01() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; }  // 53 bits
    int64_t below(int64_t bound);                                                // rejection
};

EdgeList ring_edges(int64_t n);
EdgeList star_edges(int64_t n);
EdgeList regular_edges(int64_t n, int64_t k);
EdgeList gnp_edges(int64_t n, double p, uint64_t seed);
void write_edge_list(const std::string& path, const EdgeList& edges, const std::string& comment);

// new: the configs' generators (counter-based, host == device bit for bit)
EdgeList rmat_edges(int scale, int64_t edge_factor, double a, double b, double c, uint64_t seed);
EdgeList chung_lu_edges(int64_t n, double gamma, double wmin, double wmax, int64_t draws, uint64_t seed);

}  // namespace chebpr
