// K6 Power comparator (run_power, power.cpp:28-117), K7 transition_apply (graph.cpp:104-121)
// and the staged API (init_state / generate_stage / accumulate_stage, cpaa.cpp:167-196) on
// the term kernel with their own epilogues.
#include "term.cuh"

namespace chebgpu {

// ---------------- Power method (power.cpp:28-109) -------------------------------------
namespace {
__global__ void k_fill(double* __restrict__ x, int64_t n, double v) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
        x[u] = v;
}

template <class RP>
void power_t(cheb_graph* g, double c, int budget, bool by_tol, double tol, int mode,
             const double* h_ref, double* ranks, cheb_trace_row* trace, int cap, int* rounds_out,
             double* total) {
    cudaStream_t st = g->stream;
    const Layout L = layout_of(g, mode);
    const int64_t n = g->n;
    ensure_workspace<double>(g, std::max(budget, 1), 1);
    Workspace& w = g->ws;
    double* X = w.T0.ptr<double>();                 // x (in place)
    double* C[2] = {w.X0.ptr<double>(), w.X1.ptr<double>()};
    const double base = (1.0 - c) / (double)n;
    const double x0 = 1.0 / (double)n;
    {   // x = e/n, contrib = x D^-1
        k_fill<<<grid1d(n), kThreads, 0, st>>>(X, n, x0);
        k_prescale<RP, double><<<grid1d(n), kThreads, 0, st>>>(static_cast<const RP*>(L.rp), L.inv, X, n, C[0]);
        CHEB_CUDA_CHECK(cudaGetLastError());
    }
    DevMem d_ref, d_err;
    if (h_ref) {
        d_ref.alloc(sizeof(double) * n);
        DevMem tmp(sizeof(double) * n);
        CHEB_CUDA_CHECK(cudaMemcpyAsync(tmp.get(), h_ref, sizeof(double) * n, cudaMemcpyHostToDevice, st));
        k_permute_in<double><<<grid1d(n), kThreads, 0, st>>>(tmp.ptr<double>(), L.order, n, d_ref.ptr<double>());
        d_err.alloc(sizeof(double) * (2 * (size_t)grid1d(n) + 8));
    }
    double* dtr = w.trace.ptr<double>();
    const int grid = L.fast ? g->view.grid : 0;
    int k = 0;
    // Speculative batches of rounds (no reference tracking): round j of a batch reads x from
    // snapshot j-1 and writes snapshot j, the batch's L1 changes and masses are read back once,
    // and the solve stops at the first round that meets tol — its x is in the snapshots, so
    // the result is the per-round one.
    const int B = h_ref ? 0 : (int)std::min<int64_t>(16, std::max(budget, 1));
    DevMem snaps;
    if (B > 0) {
        size_t free_b = 0, total_b = 0;
        cudaMemGetInfo(&free_b, &total_b);
        if (sizeof(double) * (size_t)(B + 1) * (size_t)n <= free_b / 4)
            snaps.alloc(sizeof(double) * (size_t)(B + 1) * (size_t)n);
    }
    // per-round kernel time for the trace's elapsed_ms (power.cpp:92: the round's kernel)
    std::vector<cudaEvent_t> rev(2 * (size_t)std::max(B, 1));
    for (auto& e : rev) CHEB_CUDA_CHECK(cudaEventCreate(&e));
    struct EvFree {
        std::vector<cudaEvent_t>& v;
        ~EvFree() {
            for (auto e : v) cudaEventDestroy(e);
        }
    } ev_free{rev};
    auto round_ms = [&](int j) {
        float ms = 0.f;
        CHEB_CUDA_CHECK(cudaEventElapsedTime(&ms, rev[2 * j], rev[2 * j + 1]));
        return (double)ms;
    };
    double final_mass = -1.0;  // FAST: the last round's device mass (fixed-order sum of x)
    if (snaps) {
        double* S = snaps.ptr<double>();
        CHEB_CUDA_CHECK(cudaMemcpyAsync(S, X, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
        const double* final_x = S;
        bool done = budget == 0;
        while (!done) {
            const int nb = std::min(B, budget - k);
            for (int j = 1; j <= nb; ++j) {
                const int kk = k + j;
                double* Sj = S + (size_t)j * n;
                TermArgs<RP, double> a = base_args<RP, double>(g, L);
                a.x_in = C[(kk - 1) & 1];
                a.x_out = C[kk & 1];
                a.T = Sj - n;  // x_{k-1}
                a.out = Sj;    // y = x_k
                a.ck = c;
                a.base = base;
                a.first = 0;
                if (L.fast) {  // per-round partial slots: one trace reduction per batch
                    a.part = w.part.ptr<double>() + (size_t)(j - 1) * grid * 2;
                    a.hub_part = w.hub_part.ptr<double>();
                    a.hub_ts = g->view.n_hub ? w.hub_ts.ptr<double>() + (size_t)(j - 1) * g->view.n_hub * 2 : nullptr;
                }
                CHEB_CUDA_CHECK(cudaEventRecord(rev[2 * (j - 1)], st));
                launch_pass<EPI_POWER>(g, L, a);
                CHEB_CUDA_CHECK(cudaEventRecord(rev[2 * (j - 1) + 1], st));
            }
            if (L.fast) {
                k_trace_reduce<<<nb, kTraceThreads, 0, st>>>(w.part.ptr<double>(), grid, w.hub_ts.ptr<double>(),
                                                        (int)g->view.n_hub, 0, dtr);
                CHEB_CUDA_CHECK(cudaGetLastError());
            }
            if (!L.fast) {
                k_power_many<<<(2 * nb + 31) / 32, 32, 0, st>>>(S, n, nb, dtr);
                CHEB_CUDA_CHECK(cudaGetLastError());
            }
            std::vector<double> h(2 * (size_t)nb);
            CHEB_CUDA_CHECK(cudaMemcpyAsync(h.data(), dtr, sizeof(double) * 2 * nb, cudaMemcpyDeviceToHost, st));
            CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
            int stop = 0;
            for (int j = 1; j <= nb && !stop; ++j) {
                const int kk = k + j;
                if (trace && kk <= cap) {
                    cheb_trace_row& r = trace[kk - 1];
                    std::memset(&r, 0, sizeof r);
                    r.k = kk;
                    r.l1_change = h[2 * (j - 1)];
                    r.mass_T = h[2 * (j - 1) + 1];
                    r.elapsed_ms = round_ms(j - 1);
                }
                if (!std::isfinite(h[2 * (j - 1)])) fail(CHEB_NUMERIC, "non-finite value at round " + std::to_string(kk));
                if (by_tol && h[2 * (j - 1)] < tol) stop = j;
            }
            if (stop) {
                k += stop;
                final_x = S + (size_t)stop * n;
                final_mass = h[2 * (stop - 1) + 1];
                done = true;
            } else {
                k += nb;
                final_x = S + (size_t)nb * n;
                final_mass = h[2 * (nb - 1) + 1];
                done = k >= budget;
                if (!done)  // next batch starts from this batch's last x
                    CHEB_CUDA_CHECK(cudaMemcpyAsync(S, final_x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
                if (!done) final_x = S;
            }
        }
        CHEB_CUDA_CHECK(cudaMemcpyAsync(X, final_x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    }
    while (!snaps && k < budget) {
        ++k;
        TermArgs<RP, double> a = base_args<RP, double>(g, L);
        a.x_in = C[(k - 1) & 1];
        a.x_out = C[k & 1];
        a.T = X;
        a.ck = c;
        a.base = base;
        a.first = 0;
        if (L.fast) {
            a.part = w.part.ptr<double>();
            a.hub_part = w.hub_part.ptr<double>();
            a.hub_ts = g->view.n_hub ? w.hub_ts.ptr<double>() : nullptr;
        }
        CHEB_CUDA_CHECK(cudaEventRecord(rev[0], st));
        if (!L.fast) {
            // y goes to a separate buffer so the Kahan L1 sees old and new x (power.cpp:80-86)
            a.T = w.acc.ptr<double>();
            CHEB_CUDA_CHECK(cudaMemcpyAsync(a.T, X, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
            CHEB_CUDA_CHECK(cudaEventRecord(rev[0], st));
            launch_pass<EPI_POWER>(g, L, a);
            CHEB_CUDA_CHECK(cudaEventRecord(rev[1], st));
            k_serial_sums<1><<<1, 256, 0, st>>>(a.T, X, n, dtr);
            CHEB_CUDA_CHECK(cudaMemcpyAsync(X, a.T, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
        } else {
            launch_pass<EPI_POWER>(g, L, a);
            CHEB_CUDA_CHECK(cudaEventRecord(rev[1], st));
            k_trace_reduce<<<1, kTraceThreads, 0, st>>>(w.part.ptr<double>(), grid, a.hub_ts, (int)g->view.n_hub, 0, dtr);
        }
        CHEB_CUDA_CHECK(cudaGetLastError());
        double err2[2] = {0.0, 0.0};
        if (h_ref) {
            const int eg = grid1d(n);
            k_err<double><<<eg, kThreads, 0, st>>>(X, d_ref.ptr<double>(), n, nullptr, 0, d_err.ptr<double>() + 4);
            k_err_final<<<1, kThreads, 0, st>>>(d_err.ptr<double>() + 4, eg, d_err.ptr<double>());
            CHEB_CUDA_CHECK(cudaMemcpyAsync(err2, d_err.get(), sizeof err2, cudaMemcpyDeviceToHost, st));
        }
        double h[2];
        CHEB_CUDA_CHECK(cudaMemcpyAsync(h, dtr, sizeof h, cudaMemcpyDeviceToHost, st));
        CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
        if (trace && k <= cap) {
            cheb_trace_row& r = trace[k - 1];
            std::memset(&r, 0, sizeof r);
            r.k = k;
            r.l1_change = h[0];
            r.mass_T = h[1];
            r.elapsed_ms = round_ms(0);
            r.err = err2[0];
            r.err_l1 = err2[1];
        }
        if (!std::isfinite(h[0])) fail(CHEB_NUMERIC, "non-finite value at round " + std::to_string(k));
        if (by_tol && h[0] < tol) break;
    }
    // ranks = x (original order); total = Kahan(x) on the host (power.cpp:105-107)
    std::vector<double> xs(n);
    DevMem o(sizeof(double) * n);
    k_permute_out<double><<<grid1d(n), kThreads, 0, st>>>(X, L.order, L.rank, n, o.ptr<double>());
    CHEB_CUDA_CHECK(cudaMemcpyAsync(ranks, o.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
    *rounds_out = k;
    // FAST: the device's fixed-order mass of the final x (a host Kahan pass over n entries
    // costs milliseconds); BITEXACT and unbatched runs: Kahan(x) as the reference
    *total = L.fast && final_mass >= 0.0 ? final_mass : kahan_sum(ranks, n);
}
}  // namespace

void power_solve(cheb_graph* g, double c, int rounds, double tol, int max_rounds, int mode,
                 const double* reference, double* ranks, cheb_trace_row* trace, int cap,
                 int* rounds_out, double* total) {
    GraphScope gs(g);
    const bool fixed = rounds >= 0;
    const int budget = fixed ? rounds : max_rounds;
    const bool rp64 = mode == CHEB_MODE_FAST ? (ensure_view(g), g->view.rp64) : g->rp64;
    if (rp64) power_t<int64_t>(g, c, budget, !fixed, tol, mode, reference, ranks, trace, cap, rounds_out, total);
    else power_t<int>(g, c, budget, !fixed, tol, mode, reference, ranks, trace, cap, rounds_out, total);
}

// ---------------- transition_apply (graph.cpp:104-121) --------------------------------
namespace {
template <class RP>
void transition_t(cheb_graph* g, const double* x, double* y, int mode) {
    cudaStream_t st = g->stream;
    const Layout L = layout_of(g, mode);
    const int64_t n = g->n;
    ensure_workspace<double>(g, 1, 1);
    Workspace& w = g->ws;
    DevMem dx(sizeof(double) * n);
    CHEB_CUDA_CHECK(cudaMemcpyAsync(dx.get(), x, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    k_permute_in<double><<<grid1d(n), kThreads, 0, st>>>(dx.ptr<double>(), L.order, n, w.T0.ptr<double>());
    k_prescale<RP, double><<<grid1d(n), kThreads, 0, st>>>(static_cast<const RP*>(L.rp), L.inv,
                                                          w.T0.ptr<double>(), n, w.X0.ptr<double>());
    TermArgs<RP, double> a = base_args<RP, double>(g, L);
    a.x_in = w.X0.ptr<double>();
    a.out = w.T1.ptr<double>();
    if (L.fast) {
        a.hub_part = w.hub_part.ptr<double>();
    }
    launch_pass<EPI_PLAIN>(g, L, a);
    k_permute_out<double><<<grid1d(n), kThreads, 0, st>>>(w.T1.ptr<double>(), L.order, L.rank, n, dx.ptr<double>());
    CHEB_CUDA_CHECK(cudaGetLastError());
    CHEB_CUDA_CHECK(cudaMemcpyAsync(y, dx.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
}
}  // namespace

void transition_apply(cheb_graph* g, const double* x, double* y, int mode) {
    GraphScope gs(g);
    const bool rp64 = mode == CHEB_MODE_FAST ? (ensure_view(g), g->view.rp64) : g->rp64;
    if (rp64) transition_t<int64_t>(g, x, y, mode);
    else transition_t<int>(g, x, y, mode);
}

// ---------------- staged API (cpaa.cpp:167-196) ---------------------------------------
void staged_init(cheb_graph* g, double c0, int mode) {
    GraphScope gs(g);
    StagedState& S = g->staged;
    const int64_t n = g->n;
    const size_t vb = sizeof(double) * std::max<int64_t>(n, 1);
    S.T_prev.ensure(vb);
    S.T_curr.ensure(vb);
    S.T_next.ensure(vb);
    S.acc.ensure(vb);
    S.x.ensure(vb);
    S.mode = mode;
    S.k = 1;
    S.active = true;
    std::vector<double> ones(n, 1.0), half(n, c0 / 2.0), zero(n, 0.0);
    staged_set(g, ones.data(), ones.data(), half.data(), 1);
    CHEB_CUDA_CHECK(cudaMemcpy(S.T_next.get(), zero.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
}

void staged_set(cheb_graph* g, const double* Tp, const double* Tc, const double* acc, int k) {
    GraphScope gs(g);
    StagedState& S = g->staged;
    if (!S.active) fail(CHEB_INVALID_ARG, "staged state not initialised");
    const Layout L = layout_of(g, S.mode);
    const int64_t n = g->n;
    DevMem tmp(sizeof(double) * std::max<int64_t>(n, 1));
    auto put = [&](const double* h, DevMem& d) {
        if (!h) return;
        CHEB_CUDA_CHECK(cudaMemcpyAsync(tmp.get(), h, sizeof(double) * n, cudaMemcpyHostToDevice, g->stream));
        k_permute_in<double><<<grid1d(n), kThreads, 0, g->stream>>>(tmp.ptr<double>(), L.order, n, d.ptr<double>());
        CHEB_CUDA_CHECK(cudaGetLastError());
        CHEB_CUDA_CHECK(cudaStreamSynchronize(g->stream));
    };
    put(Tp, S.T_prev);
    put(Tc, S.T_curr);
    put(acc, S.acc);
    if (k > 0) S.k = k;
}

namespace {
template <class RP>
void staged_generate_t(cheb_graph* g) {
    StagedState& S = g->staged;
    const Layout L = layout_of(g, S.mode);
    const int64_t n = g->n;
    ensure_workspace<double>(g, 1, 1);
    cudaStream_t st = g->stream;
    // contrib = T_curr D^-1 (cpaa.cpp:180-182), then gather + recurrence (:183-189)
    k_prescale<RP, double><<<grid1d(n), kThreads, 0, st>>>(static_cast<const RP*>(L.rp), L.inv,
                                                          S.T_curr.ptr<double>(), n, S.x.ptr<double>());
    TermArgs<RP, double> a = base_args<RP, double>(g, L);
    a.x_in = S.x.ptr<double>();
    a.T_prev = S.T_prev.ptr<double>();
    a.out = S.T_next.ptr<double>();
    a.first = S.k == 1;
    if (L.fast) {
        a.hub_part = g->ws.hub_part.ptr<double>();
    }
    launch_pass<EPI_GEN>(g, L, a);
    CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
}
}  // namespace

void staged_generate(cheb_graph* g) {
    GraphScope gs(g);
    if (!g->staged.active) fail(CHEB_INVALID_ARG, "staged state not initialised");
    const bool rp64 = g->staged.mode == CHEB_MODE_FAST ? (ensure_view(g), g->view.rp64) : g->rp64;
    if (rp64) staged_generate_t<int64_t>(g);
    else staged_generate_t<int>(g);
}

void staged_accumulate(cheb_graph* g, double ck) {
    GraphScope gs(g);
    StagedState& S = g->staged;
    if (!S.active) fail(CHEB_INVALID_ARG, "staged state not initialised");
    k_accumulate<double><<<grid1d(g->n), kThreads, 0, g->stream>>>(S.acc.ptr<double>(), S.T_next.ptr<double>(), g->n, ck);
    CHEB_CUDA_CHECK(cudaGetLastError());
    CHEB_CUDA_CHECK(cudaStreamSynchronize(g->stream));
}

void staged_rotate(cheb_graph* g) {
    StagedState& S = g->staged;
    if (!S.active) fail(CHEB_INVALID_ARG, "staged state not initialised");
    std::swap(S.T_prev, S.T_curr);
    std::swap(S.T_curr, S.T_next);
    S.k += 1;
}

void staged_get(cheb_graph* g, double* Tp, double* Tc, double* Tn, double* acc, int* k) {
    GraphScope gs(g);
    StagedState& S = g->staged;
    if (!S.active) fail(CHEB_INVALID_ARG, "staged state not initialised");
    const Layout L = layout_of(g, S.mode);
    const int64_t n = g->n;
    DevMem tmp(sizeof(double) * std::max<int64_t>(n, 1));
    auto get = [&](double* h, DevMem& d) {
        if (!h) return;
        k_permute_out<double><<<grid1d(n), kThreads, 0, g->stream>>>(d.ptr<double>(), L.order, L.rank, n, tmp.ptr<double>());
        CHEB_CUDA_CHECK(cudaMemcpyAsync(h, tmp.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, g->stream));
        CHEB_CUDA_CHECK(cudaStreamSynchronize(g->stream));
    };
    get(Tp, S.T_prev);
    get(Tc, S.T_curr);
    get(Tn, S.T_next);
    get(acc, S.acc);
    if (k) *k = S.k;
}

}  // namespace chebgpu
