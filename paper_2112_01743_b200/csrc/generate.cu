// Synthetic inputs.
//
// * ring / star / regular / gnp: the reference's generators
//   (/root/reference/proj/include/chebpr/generate.hpp:27-40, src/generate.cpp:11-87),
//   restated on the host with std::mt19937_64 (a standard-fixed engine, so the edge
//   sequence is byte-identical to the reference's; config 1 is gnp_edges(10000,0.001,1)).
// * R-MAT (configs 3/4) and Chung-Lu (configs 2/5): new, counter-based so that every
//   edge is an independent function of (seed, edge index).  All sampling decisions are
//   integer comparisons (quadrant thresholds out of 2^32, an integer CDF of the
//   Chung-Lu weights), so the host path (used by the CPU reference arm) and the device
//   path (used by the GPU arm) produce the SAME edge list bit for bit.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "common.cuh"

namespace chebgpu {
namespace gen {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Counter-based draw: stream s, index i.
__host__ __device__ __forceinline__ uint64_t draw(uint64_t seed, uint64_t s, uint64_t i) {
    return mix64(mix64(seed ^ (s * 0xD1B54A32D192ED03ull)) + i * 0x9E3779B97F4A7C15ull);
}

__host__ __device__ __forceinline__ uint64_t mulhi(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

struct RmatParams {
    int scale;
    uint64_t ta, tb, tc;  // cumulative thresholds out of 2^32
    uint64_t seed;
};

// Edge i of an R-MAT graph before relabelling.
__host__ __device__ __forceinline__ void rmat_edge(const RmatParams& p, uint64_t i, uint32_t& u,
                                                   uint32_t& v) {
    uint32_t a = 0, b = 0;
    uint64_t r = 0;
    for (int l = 0; l < p.scale; ++l) {
        if ((l & 1) == 0) r = draw(p.seed, 1, i * 64 + (uint64_t)(l >> 1));
        const uint64_t q = (l & 1) ? (r >> 32) : (r & 0xffffffffull);
        const uint32_t bu = q >= p.tb ? 1u : 0u;                 // quadrants c,d: u bit set
        const uint32_t bv = (q >= p.ta && q < p.tb) || q >= p.tc ? 1u : 0u;  // b,d: v bit set
        a = (a << 1) | bu;
        b = (b << 1) | bv;
    }
    u = a;
    v = b;
}

// first index v with cum[v] > x
__host__ __device__ __forceinline__ uint32_t cdf_pick(const uint64_t* cum, int64_t n, uint64_t x) {
    int64_t lo = 0, hi = n - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (cum[mid] > x) hi = mid;
        else lo = mid + 1;
    }
    return (uint32_t)lo;
}

__global__ void k_rmat(RmatParams p, const int* __restrict__ perm, int64_t E,
                       uint64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t u, v;
        rmat_edge(p, (uint64_t)i, u, v);
        const uint64_t pu = (uint32_t)perm[u], pv = (uint32_t)perm[v];
        out[i] = (u == v) ? ~0ull : ((pv << 32) | pu);  // memory order (u, v) as int32 pair
    }
}

__global__ void k_chung_lu(uint64_t seed, const uint64_t* __restrict__ cum, int64_t n, int64_t E,
                           uint64_t* __restrict__ out) {
    const uint64_t T = cum[n - 1];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t u = cdf_pick(cum, n, mulhi(draw(seed, 2, i), T));
        const uint64_t v = cdf_pick(cum, n, mulhi(draw(seed, 3, i), T));
        out[i] = (u == v) ? ~0ull : ((v << 32) | u);
    }
}

__global__ void k_touch(const uint64_t* __restrict__ e, int64_t E, unsigned char* __restrict__ t) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = e[i];
        t[k & 0xffffffffull] = 1;
        t[k >> 32] = 1;
    }
}

__host__ __device__ __forceinline__ uint64_t rewire_partner(uint64_t seed, uint64_t v, int64_t n) {
    for (uint64_t t = 0;; ++t) {
        const uint64_t u = mulhi(draw(seed, 4, v | (t << 40)), (uint64_t)n);
        if (u != v) return u;
    }
}

__global__ void k_rewire(const int* __restrict__ iso, int64_t cnt, uint64_t seed, int64_t n,
                         uint64_t* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t v = (uint64_t)iso[i];
        out[i] = (rewire_partner(seed, v, n) << 32) | v;
    }
}

__global__ void k_invert(unsigned char* __restrict__ t, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        t[i] = t[i] ? 0 : 1;
}

struct NotSentinel {
    __host__ __device__ bool operator()(const uint64_t& k) const { return k != ~0ull; }
};

RmatParams rmat_params(int scale, double a, double b, double c, uint64_t seed) {
    RmatParams p;
    p.scale = scale;
    const double two32 = 4294967296.0;
    p.ta = (uint64_t)std::floor(a * two32);
    p.tb = (uint64_t)std::floor((a + b) * two32);
    p.tc = (uint64_t)std::floor((a + b + c) * two32);
    p.seed = seed;
    return p;
}

// Seeded Fisher-Yates relabelling (host; std::mt19937_64 + the reference's bias-free
// rejection draw, generate.cpp:11-19).
std::vector<int> relabel_perm(int64_t n, uint64_t seed) {
    std::vector<int> perm(n);
    for (int64_t i = 0; i < n; ++i) perm[i] = (int)i;
    std::mt19937_64 eng(seed);
    for (int64_t i = n - 1; i > 0; --i) {
        const uint64_t bound = (uint64_t)i + 1;
        const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
        uint64_t r;
        do r = eng();
        while (r >= limit);
        std::swap(perm[i], perm[(int64_t)(r % bound)]);
    }
    return perm;
}

// Truncated power-law expected degrees (inverse CDF) -> integer CDF (host only).
std::vector<uint64_t> chung_lu_cdf(int64_t n, double gamma, double wmin, double wmax, uint64_t seed) {
    std::vector<uint64_t> cum(n);
    const double e = 1.0 - gamma;
    const double lo = std::pow(wmin, e), hi = std::pow(wmax, e);
    uint64_t acc = 0;
    for (int64_t v = 0; v < n; ++v) {
        const double u = (double)(draw(seed, 0, (uint64_t)v) >> 11) * 0x1.0p-53;
        const double w = std::pow(lo + u * (hi - lo), 1.0 / e);
        acc += (uint64_t)std::llround(w * 1048576.0);  // 2^20 fixed point
        cum[v] = acc;
    }
    return cum;
}

template <class F>
void parallel_chunks(int64_t N, F&& f) {
    const int T = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) th.emplace_back([&, t] { f(N * t / T, N * (t + 1) / T, t); });
    for (auto& x : th) x.join();
}

// Host versions (identical output to the device versions).
std::vector<uint64_t> host_compact_fix(std::vector<std::vector<uint64_t>>& parts, int64_t n,
                                       uint64_t seed, bool rewire) {
    std::vector<uint64_t> all;
    size_t tot = 0;
    for (auto& p : parts) tot += p.size();
    all.reserve(tot);
    for (auto& p : parts) {
        all.insert(all.end(), p.begin(), p.end());
        std::vector<uint64_t>().swap(p);
    }
    if (rewire) {
        std::vector<unsigned char> touched(n, 0);
        for (uint64_t k : all) {
            touched[k & 0xffffffffull] = 1;
            touched[k >> 32] = 1;
        }
        for (int64_t v = 0; v < n; ++v)
            if (!touched[v]) all.push_back((rewire_partner(seed, (uint64_t)v, n) << 32) | (uint64_t)v);
    }
    return all;
}

}  // namespace gen

// -------------------------------------------------------------------------------------
// Output: E pairs of int32 (u,v) either on the host (malloc) or the device (cudaMalloc).
// -------------------------------------------------------------------------------------
namespace {

void* device_compact(cheb_graph* dummy_unused, uint64_t* d_raw, int64_t E, int64_t n, uint64_t seed,
                     bool rewire, int64_t* out_E, cudaStream_t st) {
    (void)dummy_unused;
    DevMem cnt(sizeof(int64_t));
    DevMem tmpb;
    uint64_t* d_out = nullptr;
    CHEB_CUDA_CHECK(cudaMalloc(&d_out, sizeof(uint64_t) * (size_t)std::max<int64_t>(E + n, 1)));
    size_t bytes = 0;
    CHEB_CUDA_CHECK(cub::DeviceSelect::If(nullptr, bytes, d_raw, d_out, cnt.ptr<int64_t>(), E,
                                          gen::NotSentinel(), st));
    tmpb.ensure(bytes);
    CHEB_CUDA_CHECK(cub::DeviceSelect::If(tmpb.get(), bytes, d_raw, d_out, cnt.ptr<int64_t>(), E,
                                          gen::NotSentinel(), st));
    int64_t kept = 0;
    CHEB_CUDA_CHECK(cudaMemcpyAsync(&kept, cnt.get(), sizeof kept, cudaMemcpyDeviceToHost, st));
    CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
    if (rewire) {
        DevMem touched(n), iso(sizeof(int) * n);
        CHEB_CUDA_CHECK(cudaMemsetAsync(touched.get(), 0, n, st));
        gen::k_touch<<<1184, 256, 0, st>>>(d_out, kept, touched.ptr<unsigned char>());
        CHEB_CUDA_CHECK(cudaGetLastError());
        gen::k_invert<<<1184, 256, 0, st>>>(touched.ptr<unsigned char>(), n);
        CHEB_CUDA_CHECK(cudaGetLastError());
        cub::CountingInputIterator<int> it(0);
        bytes = 0;
        CHEB_CUDA_CHECK(cub::DeviceSelect::Flagged(nullptr, bytes, it, touched.ptr<unsigned char>(),
                                                   iso.ptr<int>(), cnt.ptr<int64_t>(), n, st));
        tmpb.ensure(bytes);
        CHEB_CUDA_CHECK(cub::DeviceSelect::Flagged(tmpb.get(), bytes, it, touched.ptr<unsigned char>(),
                                                   iso.ptr<int>(), cnt.ptr<int64_t>(), n, st));
        int64_t niso = 0;
        CHEB_CUDA_CHECK(cudaMemcpyAsync(&niso, cnt.get(), sizeof niso, cudaMemcpyDeviceToHost, st));
        CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
        if (niso > 0) {
            gen::k_rewire<<<std::max<int64_t>(1, std::min<int64_t>((niso + 255) / 256, 1184)), 256, 0, st>>>(
                iso.ptr<int>(), niso, seed, n, d_out + kept);
            CHEB_CUDA_CHECK(cudaGetLastError());
        }
        kept += niso;
    }
    CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
    *out_E = kept;
    return d_out;
}

}  // namespace
}  // namespace chebgpu

using namespace chebgpu;

namespace {
thread_local std::string g_gen_err;
template <class F>
cheb_status gen_guard(F&& f) {
    try {
        f();
        return CHEB_OK;
    } catch (const Error& e) {
        g_gen_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_gen_err = e.what();
        return CHEB_CUDA;
    }
}

int64_t* pack_host(const std::vector<std::pair<int64_t, int64_t>>& el, int64_t* E) {
    *E = (int64_t)el.size();
    auto* out = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * 2 * (el.size() + 1)));
    for (size_t i = 0; i < el.size(); ++i) {
        out[2 * i] = el[i].first;
        out[2 * i + 1] = el[i].second;
    }
    return out;
}
}  // namespace

extern "C" {

const char* cheb_gen_last_error(void) { return g_gen_err.c_str(); }
void cheb_free(void* p) { std::free(p); }
void cheb_device_free(void* p, int device) {
    if (!p) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    cudaFree(p);
    cudaSetDevice(prev);
}

// generate.cpp:21-28
cheb_status cheb_gen_ring(int64_t n, int64_t** edges, int64_t* E) {
    return gen_guard([&] {
        if (n < 2) fail(CHEB_DOMAIN, "ring needs n >= 2");
        std::vector<std::pair<int64_t, int64_t>> el;
        for (int64_t i = 0; i < n; ++i) el.emplace_back(i, (i + 1) % n);
        if (n == 2) el.pop_back();
        *edges = pack_host(el, E);
    });
}

// generate.cpp:30-36
cheb_status cheb_gen_star(int64_t n, int64_t** edges, int64_t* E) {
    return gen_guard([&] {
        if (n < 2) fail(CHEB_DOMAIN, "star needs n >= 2");
        std::vector<std::pair<int64_t, int64_t>> el;
        for (int64_t i = 1; i < n; ++i) el.emplace_back(0, i);
        *edges = pack_host(el, E);
    });
}

// generate.cpp:38-49
cheb_status cheb_gen_regular(int64_t n, int64_t k, int64_t** edges, int64_t* E) {
    return gen_guard([&] {
        if (n < 2) fail(CHEB_DOMAIN, "regular needs n >= 2");
        if (k < 1 || k >= n) fail(CHEB_DOMAIN, "regular needs 1 <= k < n");
        if (k % 2 == 1 && n % 2 == 1) fail(CHEB_DOMAIN, "odd k requires even n (k*n must be even)");
        std::vector<std::pair<int64_t, int64_t>> el;
        for (int64_t j = 1; j <= k / 2; ++j)
            for (int64_t i = 0; i < n; ++i) el.emplace_back(i, (i + j) % n);
        if (k % 2 == 1)
            for (int64_t i = 0; i < n / 2; ++i) el.emplace_back(i, i + n / 2);
        *edges = pack_host(el, E);
    });
}

// generate.cpp:51-87 — geometric skipping over the strictly-lower-triangular pairs,
// then one random edge for every vertex the draw left isolated.
cheb_status cheb_gen_gnp(int64_t n, double p, uint64_t seed, int64_t** edges, int64_t* E) {
    return gen_guard([&] {
        if (n < 2) fail(CHEB_DOMAIN, "gnp needs n >= 2");
        if (!(p >= 0.0 && p <= 1.0)) fail(CHEB_DOMAIN, "gnp needs p in [0,1]");
        std::mt19937_64 eng(seed);
        auto unit = [&] { return static_cast<double>(eng() >> 11) * 0x1.0p-53; };
        auto below = [&](int64_t bound) {
            const uint64_t b = (uint64_t)bound;
            const uint64_t limit = UINT64_MAX - UINT64_MAX % b;
            for (;;) {
                const uint64_t r = eng();
                if (r < limit) return (int64_t)(r % b);
            }
        };
        std::vector<std::pair<int64_t, int64_t>> el;
        if (p > 0.0 && p < 1.0) {
            const double logq = std::log1p(-p);
            int64_t row = 1, colm = -1;
            while (row < n) {
                const double gap = std::floor(std::log1p(-unit()) / logq);
                colm += 1 + (int64_t)gap;
                while (colm >= row && row < n) {
                    colm -= row;
                    ++row;
                }
                if (row < n) el.emplace_back(row, colm);
            }
        } else if (p == 1.0) {
            for (int64_t a = 1; a < n; ++a)
                for (int64_t b = 0; b < a; ++b) el.emplace_back(a, b);
        }
        std::vector<char> seen(n, 0);
        for (const auto& e : el) seen[e.first] = seen[e.second] = 1;
        for (int64_t v = 0; v < n; ++v) {
            if (seen[v]) continue;
            int64_t u = v;
            while (u == v) u = below(n);
            el.emplace_back(v, u);
            seen[u] = 1;
        }
        *edges = pack_host(el, E);
    });
}

// R-MAT (scale, edge_factor, a,b,c), relabelled by a seeded Fisher-Yates permutation,
// self-loops removed.  Output: E int32 pairs, on the device (cudaMalloc on `device`)
// when on_device, else on the host (malloc).  Host and device outputs are identical.
cheb_status cheb_gen_rmat(int scale, int64_t edge_factor, double a, double b, double c,
                          uint64_t seed, int on_device, int device, void** edges, int64_t* E) {
    return gen_guard([&] {
        if (scale < 1 || scale > 30) fail(CHEB_DOMAIN, "rmat scale must be in [1,30]");
        const int64_t n = int64_t(1) << scale;
        const int64_t draws = edge_factor * n;
        const gen::RmatParams p = gen::rmat_params(scale, a, b, c, seed);
        const std::vector<int> perm = gen::relabel_perm(n, seed ^ 0x5EEDull);
        if (on_device) {
            DeviceGuard dg(device);
            cudaStream_t st;
            CHEB_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            DevMem dperm(sizeof(int) * n), raw(sizeof(uint64_t) * draws);
            CHEB_CUDA_CHECK(cudaMemcpyAsync(dperm.get(), perm.data(), sizeof(int) * n, cudaMemcpyHostToDevice, st));
            gen::k_rmat<<<148 * 16, 256, 0, st>>>(p, dperm.ptr<int>(), draws, raw.ptr<uint64_t>());
            CHEB_CUDA_CHECK(cudaGetLastError());
            *edges = device_compact(nullptr, raw.ptr<uint64_t>(), draws, n, seed, false, E, st);
            cudaStreamDestroy(st);
        } else {
            std::vector<std::vector<uint64_t>> parts(64);
            gen::parallel_chunks(draws, [&](int64_t b0, int64_t e0, int t) {
                auto& out = parts[t];
                out.reserve(e0 - b0);
                for (int64_t i = b0; i < e0; ++i) {
                    uint32_t u, v;
                    gen::rmat_edge(p, (uint64_t)i, u, v);
                    if (u == v) continue;
                    out.push_back(((uint64_t)(uint32_t)perm[v] << 32) | (uint32_t)perm[u]);
                }
            });
            std::vector<uint64_t> all = gen::host_compact_fix(parts, n, seed, false);
            *E = (int64_t)all.size();
            void* out = std::malloc(sizeof(uint64_t) * std::max<size_t>(all.size(), 1));
            std::memcpy(out, all.data(), sizeof(uint64_t) * all.size());
            *edges = out;
        }
    });
}

// Chung-Lu: expected degrees ~ truncated power law (exponent gamma on [wmin,wmax]);
// `draws` endpoint pairs drawn proportional to weight; self-loops removed; every
// vertex the draw left isolated gets one edge to a uniform other vertex (so n is kept).
cheb_status cheb_gen_chung_lu(int64_t n, double gamma, double wmin, double wmax, int64_t draws,
                              uint64_t seed, int on_device, int device, void** edges, int64_t* E) {
    return gen_guard([&] {
        if (n < 2 || n > INT32_MAX) fail(CHEB_DOMAIN, "chung_lu needs 2 <= n < 2^31");
        if (!(gamma > 1.0) || !(wmin > 0.0) || !(wmax >= wmin))
            fail(CHEB_DOMAIN, "chung_lu needs gamma > 1 and 0 < wmin <= wmax");
        const std::vector<uint64_t> cum = gen::chung_lu_cdf(n, gamma, wmin, wmax, seed);
        if (on_device) {
            DeviceGuard dg(device);
            cudaStream_t st;
            CHEB_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            DevMem dcum(sizeof(uint64_t) * n), raw(sizeof(uint64_t) * std::max<int64_t>(draws, 1));
            CHEB_CUDA_CHECK(cudaMemcpyAsync(dcum.get(), cum.data(), sizeof(uint64_t) * n, cudaMemcpyHostToDevice, st));
            gen::k_chung_lu<<<148 * 16, 256, 0, st>>>(seed, dcum.ptr<uint64_t>(), n, draws, raw.ptr<uint64_t>());
            CHEB_CUDA_CHECK(cudaGetLastError());
            *edges = device_compact(nullptr, raw.ptr<uint64_t>(), draws, n, seed, true, E, st);
            cudaStreamDestroy(st);
        } else {
            std::vector<std::vector<uint64_t>> parts(64);
            const uint64_t T = cum[n - 1];
            gen::parallel_chunks(draws, [&](int64_t b0, int64_t e0, int t) {
                auto& out = parts[t];
                out.reserve(e0 - b0);
                for (int64_t i = b0; i < e0; ++i) {
                    const uint64_t u = gen::cdf_pick(cum.data(), n, gen::mulhi(gen::draw(seed, 2, i), T));
                    const uint64_t v = gen::cdf_pick(cum.data(), n, gen::mulhi(gen::draw(seed, 3, i), T));
                    if (u == v) continue;
                    out.push_back((v << 32) | u);
                }
            });
            std::vector<uint64_t> all = gen::host_compact_fix(parts, n, seed, true);
            *E = (int64_t)all.size();
            void* out = std::malloc(sizeof(uint64_t) * std::max<size_t>(all.size(), 1));
            std::memcpy(out, all.data(), sizeof(uint64_t) * all.size());
            *edges = out;
        }
    });
}

}  // extern "C"
