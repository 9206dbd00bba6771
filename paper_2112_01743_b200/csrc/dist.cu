// Row-partitioned CPAA over G GPUs: the block-cyclic partition's solve in phases with
// the fused push exchange (x_{k+1} stored by the term kernels into every rank's buffer,
// flag barrier per term) or the NCCL all-gather baseline; one process per GPU or all ranks
// in lockstep from one process.
#include "term.cuh"

namespace chebgpu {
namespace {

// ---------------- multi-GPU: row partition + NCCL all-gather of x per term ----------
template <class V>
ncclDataType_t nccl_type() { return sizeof(V) == 8 ? ncclDouble : ncclFloat; }

template <class V>
__global__ void k_normalize_slot(const V* __restrict__ acc, int64_t nl, const double* __restrict__ total,
                                 V* __restrict__ slot) {
    const double tot = *total;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < nl;
         u += (int64_t)gridDim.x * blockDim.x)
        slot[u] = (V)((double)acc[u] / tot);
}

// NCCL exchange: every rank's local values, all-gathered into G slots of max_rows, back to
// the global sorted order (block-cyclic partition, common.cuh)
template <class V>
__global__ void k_unshuffle(const V* __restrict__ slots, int64_t n, int G, int64_t max_rows, V* __restrict__ out) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
        out[u] = slots[(int64_t)part_owner(u, G) * max_rows + part_local(u, G)];
}

// ranks[order[u]] = v[u] for every sorted row u (global sorted order -> vertex order)
template <class V>
__global__ void k_unpermute_global(const V* __restrict__ v, int64_t n, const int* __restrict__ order,
                                   V* __restrict__ out) {
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
        out[order[u]] = v[u];
}

// ---------------- fused push exchange: barrier and copy kernels ------------------------
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Wait for slot r of this rank's flags to reach epoch; give up after 20 s and raise the
// group's timeout flag (slot G) instead of hanging the GPU if a peer never signals.
__device__ __forceinline__ void wait_epoch(const unsigned long long* flags, int r, int G, unsigned long long epoch) {
    const unsigned long long t0 = global_ns();
    while (ld_acquire_sys(flags + r) < epoch) {
        __nanosleep(100);
        if (global_ns() - t0 > 20000000000ull) {
            atomicExch(const_cast<unsigned long long*>(flags) + G, 1ull);
            return;
        }
    }
}

// This rank reached `epoch`: publish it in slot [rank] of every rank's flag array.  The
// system-scope fence orders every earlier store of this stream (the term's pushes) before it.
__global__ void k_peer_signal(unsigned long long* const* flags, int G, int rank, unsigned long long epoch) {
    const int r = threadIdx.x;
    if (r < G) {
        __threadfence_system();
        st_release_sys(flags[r] + rank, epoch);
    }
}

// Wait until every rank published `epoch` into this rank's flags (acquire: their pushes are
// visible to every later kernel of this stream).
__global__ void k_peer_wait(const unsigned long long* flags, int G, unsigned long long epoch) {
    const int r = threadIdx.x;
    if (r < G) wait_epoch(flags, r, G, epoch);
    __syncthreads();
}

// Term tail of a one-process-per-GPU push run, one launch instead of three: this rank's
// trace partials of term k (as k_trace_reduce), then the barrier (signal every rank, wait
// for every rank).  Launched with PDL; waits for the term kernels before reading anything.
__global__ void __launch_bounds__(kTraceThreads) k_term_tail(const double* __restrict__ part, int grid,
                                                             const double* __restrict__ hub_ts, int n_hub, int k,
                                                             double* __restrict__ trace, unsigned long long* const* flags,
                                                             const unsigned long long* my_flags, int G, int rank,
                                                             unsigned long long epoch) {
    __shared__ double sh[32];
    pdl_wait();
    double a, b;
    trace_sums(part, grid, hub_ts, n_hub, k, sh, a, b);
    if (threadIdx.x == 0) {
        trace[2 * k] = a;
        trace[2 * k + 1] = b;
    }
    const int r = threadIdx.x;
    if (r < G) {
        __threadfence_system();  // the term's pushes (earlier kernels of this stream) first
        st_release_sys(flags[r] + rank, epoch);
    }
    if (r < G) wait_epoch(my_flags, r, G, epoch);
    __syncthreads();
}

// dst[r][off + i] = src[i] for every rank r (trace partials).
template <class T>
__global__ void k_push_copy(const T* __restrict__ src, int64_t n, T* const* dst, int G, int64_t off) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const T v = src[i];
        for (int r = 0; r < G; ++r) dst[r][off + i] = v;
    }
}

// Local rows' values to every rank's global-order buffer (x_0; block-cyclic positions).
template <class V>
__global__ void k_push_local(const V* __restrict__ src, int64_t nl, V* const* dst, int G, int rank) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nl; i += (int64_t)gridDim.x * blockDim.x) {
        const V v = src[i];
        const int64_t u = part_global(i, rank, G);
        for (int r = 0; r < G; ++r) dst[r][u] = v;
    }
}

// ranks of the local rows, normalised, pushed into every rank's global-order result buffer
template <class V>
__global__ void k_normalize_push(const V* __restrict__ acc, int64_t nl, const double* __restrict__ total,
                                 V* const* dst, int G, int rank) {
    const double tot = *total;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nl; i += (int64_t)gridDim.x * blockDim.x) {
        const V v = (V)((double)acc[i] / tot);
        const int64_t u = part_global(i, rank, G);
        for (int r = 0; r < G; ++r) dst[r][u] = v;
    }
}

// out[i] = sum over ranks r (in rank order: deterministic) of all[r * stride + i]
__global__ void k_sum_ranks_strided(const double* __restrict__ all, int G, int len, int64_t stride,
                                    double* __restrict__ out) {
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < G; ++r) s += all[(size_t)r * stride + i];
        out[i] = s;
    }
}

// One partitioned solve on one rank, in phases, so that a single process can also drive
// every rank of a group in lockstep.  Exchange: NCCL all-gathers (part.comm) or the fused
// push (g->peer): pushes inside the kernels + a flag barrier between phases.
template <class RP, class V>
struct DistSolve {
    cheb_graph* g;
    SolveSpec s;
    Layout L;
    PeerGroup* pg;  // null: NCCL
    std::vector<double> coeffs;
    double c0 = 0.0, beta_v = 0.0;
    DevMem d_p, trace_all, tglob, rbuf, slots, xloc;
    V* T[2];
    V* X[2];
    V* acc;
    int launches = 0;
    int64_t nl = 0, mr = 0, stride = 0;
    int M = 0, G = 1;
    std::vector<cudaEvent_t>* tev = nullptr;
    const double* d_total = nullptr;
    bool fused_tail = false;  // push, one process per GPU: trace reduce + barrier in one kernel

    DistSolve(cheb_graph* g_, const SolveSpec& s_, std::vector<cudaEvent_t>* ev) : g(g_), s(s_), tev(ev) {
        L = layout_of(g, CHEB_MODE_FAST);
        pg = g->peer;
        fused_tail = pg && !pg->lockstep;
        ensure_workspace<V>(g, s.M, 1);
        Workspace& w = g->ws;
        const SolverView& Vw = g->view;
        const Partition& P = g->part;
        nl = Vw.n_local;
        mr = P.max_rows;
        M = s.M;
        G = P.G;
        if (pg && M > kMaxPushTerms) fail(CHEB_CAPACITY, "push exchange supports at most 1024 terms");
        coefficients(s.c, M, coeffs, &beta_v, &c0);
        cudaStream_t st = g->stream;
        if (s.p) {
            d_p.alloc(sizeof(double) * g->n);
            CHEB_CUDA_CHECK(cudaMemcpyAsync(d_p.get(), s.p, sizeof(double) * g->n, cudaMemcpyHostToDevice, st));
        }
        tglob.alloc(sizeof(double) * 2 * std::max(M, 1));
        T[0] = w.T0.ptr<V>();
        T[1] = w.T1.ptr<V>();
        acc = w.acc.ptr<V>();
        xloc.alloc(sizeof(V) * (size_t)std::max<int64_t>(nl, 1));
        if (pg) {
            X[0] = static_cast<V*>(pg->X[0]);
            X[1] = static_cast<V*>(pg->X[1]);
            stride = 2 * (int64_t)kMaxPushTerms;
        } else {
            X[0] = w.X0.ptr<V>();
            X[1] = w.X1.ptr<V>();
            trace_all.alloc(sizeof(double) * 2 * (size_t)std::max(M, 1) * G);
            rbuf.alloc(sizeof(V) * (size_t)std::max<int64_t>(Vw.x_len, 1));
            slots.alloc(sizeof(V) * (size_t)std::max<int64_t>((int64_t)G * mr, 1));
            stride = 2 * (int64_t)std::max(M, 1);
        }
    }
    ncclComm_t comm() const { return static_cast<ncclComm_t>(g->part.comm); }
    // NCCL exchange: all-gather every rank's slot (in place, equal counts), then back to the
    // global sorted order in `dst`
    void gather_slots(V* dst) {
        cudaStream_t st = g->stream;
        V* my = slots.ptr<V>() + (int64_t)g->part.rank * mr;
        CHEB_NCCL_CHECK(ncclAllGather(my, slots.ptr<V>(), (size_t)mr, nccl_type<V>(), comm(), st));
        k_unshuffle<V><<<grid1d(g->n), kThreads, 0, st>>>(slots.ptr<V>(), g->n, G, mr, dst);
        CHEB_CUDA_CHECK(cudaGetLastError());
        ++launches;
    }
    V* const* push_table(int which) const {  // device pointer table of every rank's X[which]
        return reinterpret_cast<V* const*>(pg->table.ptr<void*>() + (size_t)which * G);
    }
    double* const* trace_table() const { return reinterpret_cast<double* const*>(pg->table.ptr<void*>() + 2 * (size_t)G); }
    V* const* rbuf_table() const { return reinterpret_cast<V* const*>(pg->table.ptr<void*>() + 3 * (size_t)G); }
    unsigned long long* const* flag_table() const {
        return reinterpret_cast<unsigned long long* const*>(pg->table.ptr<void*>() + 4 * (size_t)G);
    }

    // phase 0: T_{-1} = T_0, acc, x_0 of the local rows, then x_0 to every rank
    void begin() {
        cudaStream_t st = g->stream;
        const SolverView& Vw = g->view;
        CHEB_CUDA_CHECK(cudaEventRecord(g->ev0, st));
        V* x0 = pg ? xloc.ptr<V>() : slots.ptr<V>() + (int64_t)g->part.rank * mr;
        k_init<RP, V><<<grid1d(nl), kThreads, 0, st>>>(static_cast<const RP*>(L.rp), L.inv, d_p.ptr<double>(), L.order,
                                                       nl, c0 / 2.0, T[0], T[1], acc, x0);
        CHEB_CUDA_CHECK(cudaGetLastError());
        ++launches;
        (void)Vw;
        if (pg) {
            k_push_local<V><<<grid1d(nl), kThreads, 0, st>>>(x0, nl, push_table(0), G, g->part.rank);
            ++launches;
        } else {
            gather_slots(X[0]);
        }
        CHEB_CUDA_CHECK(cudaGetLastError());
    }

    // phase k: fused term k (pushes x_{k+1} to every rank) + this rank's trace partials
    void term(int k) {
        cudaStream_t st = g->stream;
        const SolverView& Vw = g->view;
        Workspace& w = g->ws;
        TermArgs<RP, V> a = base_args<RP, V>(g, L);
        a.x_in = X[(k - 1) & 1];
        if (pg) {
            a.x_out = X[k & 1];
            a.part_G = G;  // local row u -> global sorted position
            a.part_r = g->part.rank;
            a.push = push_table(k & 1);
            a.push_n = G;
            a.push_mask = tuning().halo ? Vw.push_mask.ptr<unsigned>() : nullptr;
        }
        if (!pg) a.x_out = slots.ptr<V>() + (int64_t)g->part.rank * mr;  // this rank's slot, local order
        a.T = T[(k - 1) & 1];
        a.acc = acc;
        a.ck = coeffs[k];
        a.first = k == 1;
        a.part = w.part.ptr<double>() + (size_t)(k - 1) * Vw.grid * 2;
        a.hub_part = w.hub_part.ptr<double>();
        a.hub_ts = Vw.n_hub ? w.hub_ts.ptr<double>() + (size_t)(k - 1) * Vw.n_hub * 2 : nullptr;
        if (tev) CHEB_CUDA_CHECK(cudaEventRecord((*tev)[2 * (k - 1)], st));
        launches += launch_pass<EPI_CPAA>(g, L, a);
        if (tev) CHEB_CUDA_CHECK(cudaEventRecord((*tev)[2 * (k - 1) + 1], st));
        if (fused_tail) {
            ++pg->epoch;
            cudaLaunchConfig_t tc = {};
            tc.gridDim = dim3(1);
            tc.blockDim = dim3(kTraceThreads);
            tc.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            tc.attrs = at;
            tc.numAttrs = tuning().pdl ? 1 : 0;
            CHEB_CUDA_CHECK(cudaLaunchKernelEx(&tc, k_term_tail, (const double*)w.part.ptr<double>(), Vw.grid,
                                               (const double*)w.hub_ts.ptr<double>(), (int)Vw.n_hub, k - 1,
                                               w.trace.ptr<double>(), flag_table(),
                                               (const unsigned long long*)pg->flags, G, pg->rank, pg->epoch));
        } else {
            k_trace_reduce<<<1, kTraceThreads, 0, st>>>(w.part.ptr<double>(), Vw.grid, w.hub_ts.ptr<double>(),
                                                   (int)Vw.n_hub, k - 1, w.trace.ptr<double>());
        }
        CHEB_CUDA_CHECK(cudaGetLastError());
        ++launches;
        if (!pg) gather_slots(X[k & 1]);  // x_{k+1}: every rank's slot -> global order on every rank
    }

    // phase M+1: every rank's trace (or, for M = 0, its acc total) to every rank
    void trace_out() {
        cudaStream_t st = g->stream;
        Workspace& w = g->ws;
        if (M == 0) {
            const int eg = grid1d(nl);
            k_sum_blocks<V><<<eg, kThreads, 0, st>>>(acc, nl, w.part.ptr<double>());
            k_sum_final<<<1, kThreads, 0, st>>>(w.part.ptr<double>(), eg, w.total.ptr<double>());
            launches += 2;
        }
        const double* src = M > 0 ? w.trace.ptr<double>() : w.total.ptr<double>();
        const int len = M > 0 ? 2 * M : 1;
        if (pg) {
            k_push_copy<double><<<1, kThreads, 0, st>>>(src, len, trace_table(), G, (int64_t)pg->rank * stride);
            ++launches;
        } else {
            CHEB_NCCL_CHECK(ncclAllGather(src, trace_all.ptr<double>(), (size_t)len, ncclDouble, comm(), st));
        }
        CHEB_CUDA_CHECK(cudaGetLastError());
    }

    // phase M+2: combine the traces in rank order, normalise the local rows, send them
    void normalize() {
        cudaStream_t st = g->stream;
        const SolverView& Vw = g->view;
        const double* all = pg ? static_cast<const double*>(pg->trace_all) : trace_all.ptr<double>();
        const int len = M > 0 ? 2 * M : 1;
        k_sum_ranks_strided<<<1, 256, 0, st>>>(all, G, len, pg ? stride : len, tglob.ptr<double>());
        d_total = M > 0 ? tglob.ptr<double>() + 2 * (M - 1) + 1 : tglob.ptr<double>();
        if (pg) {
            k_normalize_push<V><<<grid1d(nl), kThreads, 0, st>>>(acc, nl, d_total, rbuf_table(), G, g->part.rank);
        } else {
            k_normalize_slot<V><<<grid1d(nl), kThreads, 0, st>>>(acc, nl, d_total,
                                                                  slots.ptr<V>() + (int64_t)g->part.rank * mr);
            gather_slots(rbuf.ptr<V>());
        }
        (void)Vw;
        CHEB_CUDA_CHECK(cudaGetLastError());
        launches += 2;
    }

    // phase M+3: global-order ranks -> vertex order; read back the trace, check it
    void finish(std::vector<double>* tr, double* total) {
        cudaStream_t st = g->stream;
        const SolverView& Vw = g->view;
        Workspace& w = g->ws;
        const V* glob = pg ? static_cast<const V*>(pg->rbuf) : rbuf.ptr<V>();
        const int* order_g = Vw.order_full ? Vw.order_full.ptr<int>() : Vw.order.ptr<int>();  // (G = 1: same)
        k_unpermute_global<V><<<grid1d(g->n), kThreads, 0, st>>>(glob, g->n, order_g, w.out.ptr<V>());
        CHEB_CUDA_CHECK(cudaGetLastError());
        ++launches;
        CHEB_CUDA_CHECK(cudaEventRecord(g->ev1, st));
        g->last_terms = M;
        g->last_launches = launches;
        w.launches = launches;
        std::vector<double> t(2 * (size_t)std::max(M, 1));
        CHEB_CUDA_CHECK(cudaMemcpyAsync(t.data(), tglob.get(), sizeof(double) * (M > 0 ? 2 * M : 1),
                                        cudaMemcpyDeviceToHost, st));
        unsigned long long timed_out = 0;
        if (pg)
            CHEB_CUDA_CHECK(cudaMemcpyAsync(&timed_out, pg->flags + G, sizeof timed_out, cudaMemcpyDeviceToHost, st));
        CHEB_CUDA_CHECK(cudaStreamSynchronize(st));
        if (timed_out) fail(CHEB_CUDA, "push exchange barrier timed out (a peer stopped signalling)");
        float ms = 0.f;
        CHEB_CUDA_CHECK(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
        g->last_loop_ms = ms;
        for (int k = 1; k <= M; ++k)
            if (!std::isfinite(t[2 * (k - 1)]) || !std::isfinite(t[2 * (k - 1) + 1]))
                fail(CHEB_NUMERIC, "non-finite value at round " + std::to_string(k));
        const double tot = M > 0 ? t[2 * (M - 1) + 1] : t[0];
        if (!std::isfinite(tot) || tot <= 0.0) fail(CHEB_NUMERIC, "normalization total is not positive and finite");
        if (tr) *tr = t;
        if (total) *total = tot;
    }

    // push barrier, one rank per process: publish, then wait for every rank
    void signal() {
        ++pg->epoch;
        k_peer_signal<<<1, 32, 0, g->stream>>>(flag_table(), G, pg->rank, pg->epoch);
        CHEB_CUDA_CHECK(cudaGetLastError());
        if (pg->lockstep) CHEB_CUDA_CHECK(cudaEventRecord(pg->signalled, g->stream));
        ++launches;
    }
    void wait() {
        k_peer_wait<<<1, 32, 0, g->stream>>>(pg->flags, G, pg->epoch);
        CHEB_CUDA_CHECK(cudaGetLastError());
        ++launches;
    }
};

template <class RP, class V>
void run_solve_dist(cheb_graph* g, const SolveSpec& s, std::vector<double>* tr, double* total,
                    std::vector<double>* term_ms = nullptr) {
    std::vector<cudaEvent_t> tev;
    if (term_ms) {
        tev.resize(2 * (size_t)std::max(s.M, 1));
        for (auto& e : tev) CHEB_CUDA_CHECK(cudaEventCreate(&e));
    }
    DistSolve<RP, V> d(g, s, term_ms ? &tev : nullptr);
    const bool push = d.pg != nullptr;
    auto barrier = [&] {
        if (push) {
            d.signal();
            d.wait();
        }
    };
    d.begin();
    barrier();
    for (int k = 1; k <= s.M; ++k) {
        d.term(k);
        if (!d.fused_tail) barrier();  // (fused: the term's tail kernel was the barrier)
    }
    d.trace_out();
    barrier();
    d.normalize();
    barrier();
    d.finish(tr, total);
    if (term_ms) {
        term_ms->assign(s.M, 0.0);
        for (int k = 0; k < s.M; ++k) {
            float tk = 0.f;
            CHEB_CUDA_CHECK(cudaEventElapsedTime(&tk, tev[2 * k], tev[2 * k + 1]));
            (*term_ms)[k] = tk;
        }
        for (auto& e : tev) cudaEventDestroy(e);
    }
}

// One host thread drives every rank of a push group (one device or several): each phase is
// enqueued on every rank's stream, then every rank signals, and each rank's wait kernel is
// ordered (by events) after all signals — so no kernel ever spins on work that has not been
// enqueued, and ranks sharing one GPU cannot deadlock.
// rank_ms (profiling): the ranks' term kernels run one rank at a time (each rank's term waits
// for the previous rank's term on its own stream), so that every rank's per-term time is
// measured on the whole GPU with CUDA events — the per-rank load balance of the partition
// as one GPU per rank would see it (the exchange stores hit local memory here).
template <class RP, class V>
void run_group_lockstep(const std::vector<cheb_graph*>& gs, const SolveSpec& s, std::vector<double>* tr,
                        double* total, std::vector<double>* rank_ms = nullptr) {
    const int G = (int)gs.size();
    std::vector<std::unique_ptr<DistSolve<RP, V>>> d;
    std::vector<std::vector<cudaEvent_t>> tev(G);
    std::vector<cudaEvent_t> term_done(G, nullptr);
    for (int r = 0; r < G; ++r) {
        GraphScope sc(gs[r]);
        if (rank_ms) {
            tev[r].resize(2 * (size_t)std::max(s.M, 1));
            for (auto& e : tev[r]) CHEB_CUDA_CHECK(cudaEventCreate(&e));
            CHEB_CUDA_CHECK(cudaEventCreateWithFlags(&term_done[r], cudaEventDisableTiming));
        }
        d.emplace_back(new DistSolve<RP, V>(gs[r], s, rank_ms ? &tev[r] : nullptr));
    }
    auto each = [&](auto&& f) {
        for (int r = 0; r < G; ++r) {
            GraphScope sc(gs[r]);
            f(*d[r]);
        }
    };
    auto barrier = [&] {
        each([](DistSolve<RP, V>& x) { x.signal(); });
        for (int r = 0; r < G; ++r) {
            GraphScope sc(gs[r]);
            for (int q = 0; q < G; ++q)
                CHEB_CUDA_CHECK(cudaStreamWaitEvent(gs[r]->stream, gs[q]->peer->signalled, 0));
            d[r]->wait();
        }
    };
    each([](DistSolve<RP, V>& x) { x.begin(); });
    barrier();
    for (int k = 1; k <= s.M; ++k) {
        if (rank_ms) {  // serialised terms: rank r after rank r - 1
            for (int r = 0; r < G; ++r) {
                GraphScope sc(gs[r]);
                if (r > 0) CHEB_CUDA_CHECK(cudaStreamWaitEvent(gs[r]->stream, term_done[r - 1], 0));
                d[r]->term(k);
                CHEB_CUDA_CHECK(cudaEventRecord(term_done[r], gs[r]->stream));
            }
        } else {
            each([k](DistSolve<RP, V>& x) { x.term(k); });
        }
        barrier();
    }
    each([](DistSolve<RP, V>& x) { x.trace_out(); });
    barrier();
    each([](DistSolve<RP, V>& x) { x.normalize(); });
    barrier();
    for (int r = 0; r < G; ++r) {
        GraphScope sc(gs[r]);
        d[r]->finish(r == 0 ? tr : nullptr, r == 0 ? total : nullptr);
    }
    if (rank_ms) {
        rank_ms->assign(G, 0.0);
        for (int r = 0; r < G; ++r) {
            GraphScope sc(gs[r]);
            CHEB_CUDA_CHECK(cudaStreamSynchronize(gs[r]->stream));
            double sum = 0.0;
            for (int k = 0; k < s.M; ++k) {
                float t = 0.f;
                CHEB_CUDA_CHECK(cudaEventElapsedTime(&t, tev[r][2 * k], tev[r][2 * k + 1]));
                sum += t;
            }
            (*rank_ms)[r] = s.M > 0 ? sum / s.M : 0.0;
            for (auto& e : tev[r]) cudaEventDestroy(e);
            cudaEventDestroy(term_done[r]);
        }
    }
}

}  // namespace

// Partitioned solve of one rank (one process per GPU): precision / row-pointer dispatch.
void dist_solve(cheb_graph* g, const SolveSpec& s, std::vector<double>* tr, double* total,
                std::vector<double>* term_ms) {
    GraphScope gs(g);
    ensure_view(g);
    if (s.precision == CHEB_FP64) {
        if (g->view.rp64) run_solve_dist<int64_t, double>(g, s, tr, total, term_ms);
        else run_solve_dist<int, double>(g, s, tr, total, term_ms);
    } else {
        if (g->view.rp64) run_solve_dist<int64_t, float>(g, s, tr, total, term_ms);
        else run_solve_dist<int, float>(g, s, tr, total, term_ms);
    }
}

// Lockstep solve of a push group (every rank's handle driven by this thread).
void group_solve(const std::vector<cheb_graph*>& gs, const SolveSpec& s, std::vector<double>* tr, double* total,
                 std::vector<double>* rank_ms) {
    if (s.R != 1) fail(CHEB_INVALID_ARG, "R > 1 is served by the batched path");
    if (s.mode != CHEB_MODE_FAST) fail(CHEB_INVALID_ARG, "a partitioned handle runs the FAST schedule only");
    bool rp64 = false;
    for (cheb_graph* g : gs) {
        GraphScope sc(g);
        ensure_view(g);
        rp64 = rp64 || g->view.rp64;
    }
    for (cheb_graph* g : gs)
        if (g->view.rp64 != rp64) fail(CHEB_INVALID_ARG, "group members disagree on row-pointer width");
    if (s.precision == CHEB_FP64) {
        if (rp64) run_group_lockstep<int64_t, double>(gs, s, tr, total, rank_ms);
        else run_group_lockstep<int, double>(gs, s, tr, total, rank_ms);
    } else {
        if (rp64) run_group_lockstep<int64_t, float>(gs, s, tr, total, rank_ms);
        else run_group_lockstep<int, float>(gs, s, tr, total, rank_ms);
    }
}

}  // namespace chebgpu
