// api_multi.cuh -- C ABI of the many-triangulation engine (config C4).
// Included by tcg.cu inside its extern "C" block.

// ------------------------------------------------------------ many triangulations
struct tcg_multi {
    int device = 0, d = 0, K = 0, even = 0, ntri = 0;
    KParams *d_kp = nullptr;
    uint32_t *d_adj = nullptr, *d_edges = nullptr;
    size_t smem = 0;
    cudaStream_t stream = nullptr;
    int64_t cap = 0;
    uint64_t *d_sig = nullptr, *d_key = nullptr;
    uint8_t *d_ov = nullptr, *d_nr = nullptr;
    int32_t *d_st = nullptr;
    int4 *d_items = nullptr;
    int64_t items_cap = 0;
    float last_ms = 0.f;
    int64_t launches = 0;
    // host-buffer pipeline: two slots of pinned staging, one stream each
    cudaStream_t sst[2] = {nullptr, nullptr};
    cudaEvent_t ev[2][2] = {};       // kernel start / stop per slot
    uint8_t *h_stage[2] = {nullptr, nullptr};  // [MULTI_CHUNK] sig | key | st | ov | nr
};

// pairs per pipeline chunk (TCG_MULTI_CHUNK_LOG2, 18..26)
static int64_t multi_chunk() {
    static const int64_t c = [] {
        const char *e = std::getenv("TCG_MULTI_CHUNK_LOG2");
        return (int64_t)1 << (e ? std::max(18, std::min(26, std::atoi(e))) : 23);
    }();
    return c;
}

// Host copies of the pipeline split over a few threads (one memcpy stream is
// ~10 GB/s; the box has >= 16 cores).
static void par_for(int64_t n, const std::function<void(int64_t, int64_t)> &fn) {
    static const int nth = [] {
        const char *e = std::getenv("TCG_HOST_THREADS");
        const int hw = (int)std::thread::hardware_concurrency();
        return e ? std::max(1, std::atoi(e)) : std::max(1, std::min(8, hw / 2));
    }();
    const int t = (int)std::min<int64_t>(nth, std::max<int64_t>(1, n >> 16));
    if (t <= 1) {
        fn(0, n);
        return;
    }
    std::vector<std::thread> th;
    for (int i = 1; i < t; ++i) th.emplace_back(fn, n * i / t, n * (i + 1) / t);
    fn(0, n / t);
    for (auto &x : th) x.join();
}

static void *pick_multi(int K, bool even) {
    if (K == 2) return even ? (void *)k_multi<2, true> : (void *)k_multi<2, false>;
    if (K == 4) return even ? (void *)k_multi<4, true> : (void *)k_multi<4, false>;
    return even ? (void *)k_multi<6, true> : (void *)k_multi<6, false>;
}

int tcg_multi_destroy(tcg_multi *M) {
    if (!M) return TCG_OK;
    DeviceGuard guard(M->device);
    if (M->stream) cudaStreamSynchronize(M->stream);
    void *ptrs[] = {M->d_kp, M->d_adj, M->d_edges, M->d_sig, M->d_key, M->d_ov, M->d_nr,
                    M->d_st, M->d_items};
    for (void *q : ptrs)
        if (q) cudaFree(q);
    for (int i = 0; i < 2; ++i) {
        if (M->sst[i]) {
            cudaStreamSynchronize(M->sst[i]);
            cudaStreamDestroy(M->sst[i]);
        }
        for (int j = 0; j < 2; ++j)
            if (M->ev[i][j]) cudaEventDestroy(M->ev[i][j]);
        if (M->h_stage[i]) cudaFreeHost(M->h_stage[i]);
    }
    if (M->stream) cudaStreamDestroy(M->stream);
    delete M;
    return TCG_OK;
}

int tcg_multi_create(const tcg_desc *descs, int32_t ntri, int device, tcg_multi **out) {
    if (!descs || !out || ntri < 1) return fail(TCG_E_ARG, "bad arguments");
    *out = nullptr;
    std::vector<HostPlan> hps(ntri);
    for (int t = 0; t < ntri; ++t) {
        int rc = build_host_plan(descs + t, hps[t]);
        if (rc) return rc;
        if (hps[t].d != hps[0].d) return fail(TCG_E_ARG, "all triangulations must share one degree");
    }
    const int K = hps[0].K;
    const size_t arow = (size_t)32 * K * K;
    size_t ne_tot = 0;
    for (auto &h : hps) ne_tot += h.edges.size();
    if (device < 0 && cudaGetDevice(&device) != cudaSuccess) {
        cudaGetLastError();
        return fail(TCG_E_CUDA, "no CUDA device");
    }
    tcg_multi *M = new tcg_multi();
    M->device = device;
    M->d = hps[0].d;
    M->K = K;
    M->even = hps[0].even;
    M->ntri = ntri;
    DeviceGuard guard(device);
    auto bail = [&](cudaError_t e, const char *what) {
        std::string msg = std::string(what) + ": " + cudaGetErrorString(e);
        tcg_multi_destroy(M);
        return fail(TCG_E_CUDA, msg);
    };
    cudaError_t e;
    cudaDeviceProp prop;
    if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess) return bail(e, "props");
    if (prop.major < 10) {
        tcg_multi_destroy(M);
        return fail(TCG_E_UNSUPPORTED, "libtcg is built for sm_100a (Blackwell B200)");
    }
    if ((e = cudaStreamCreateWithFlags(&M->stream, cudaStreamNonBlocking)) != cudaSuccess)
        return bail(e, "stream");
    if ((e = cudaMalloc(&M->d_kp, sizeof(KParams) * ntri)) != cudaSuccess) return bail(e, "malloc");
    if ((e = cudaMalloc(&M->d_adj, 4 * arow * ntri)) != cudaSuccess) return bail(e, "malloc");
    if ((e = cudaMalloc(&M->d_edges, 4 * std::max<size_t>(1, ne_tot))) != cudaSuccess)
        return bail(e, "malloc");
    std::vector<KParams> kps(ntri);
    std::vector<uint32_t> adj(arow * ntri), edges(std::max<size_t>(1, ne_tot));
    size_t eo = 0;
    for (int t = 0; t < ntri; ++t) {
        kps[t] = hps[t].kp;
        kps[t].adj = M->d_adj + arow * t;
        kps[t].edges = M->d_edges + eo;
        std::copy(hps[t].adj.begin(), hps[t].adj.end(), adj.begin() + arow * t);
        std::copy(hps[t].edges.begin(), hps[t].edges.end(), edges.begin() + eo);
        eo += hps[t].edges.size();
    }
    cudaMemcpy(M->d_kp, kps.data(), sizeof(KParams) * ntri, cudaMemcpyHostToDevice);
    cudaMemcpy(M->d_adj, adj.data(), 4 * adj.size(), cudaMemcpyHostToDevice);
    if ((e = cudaMemcpy(M->d_edges, edges.data(), 4 * edges.size(), cudaMemcpyHostToDevice)) !=
        cudaSuccess)
        return bail(e, "upload");
    M->smem = 4 * arow;
    *out = M;
    return TCG_OK;
}

int tcg_multi_classify(tcg_multi *M, const int32_t *tri, const uint64_t *sig, int64_t n,
                       uint64_t *key, uint8_t *ov, uint8_t *nr, int32_t *st) {
    if (!M || (n > 0 && (!tri || !sig || !key || !ov || !nr || !st)))
        return fail(TCG_E_ARG, "null argument");
    if (n <= 0) return TCG_OK;
    if (n > INT32_MAX) return fail(TCG_E_RANGE, "at most 2^31-1 pairs per call");
    DeviceGuard guard(M->device);
    // pairs grouped by triangulation (a counting sort unless the caller's
    // triangulation ids are already non-decreasing, e.g. config C4's layout);
    // work items of <= 2048 pairs of one triangulation
    constexpr int ITEM = 2048;
    host_mark("multi start");
    std::vector<int64_t> cnt(M->ntri + 1, 0);
    {  // validate, count and test the order in parallel slices
        std::mutex mu;
        std::atomic<bool> bad{false}, unordered{false};
        par_for(n, [&](int64_t lo, int64_t hi) {
            std::vector<int64_t> c(M->ntri + 1, 0);
            bool ord = lo == 0 || (tri[lo] >= tri[lo - 1]);
            for (int64_t i = lo; i < hi; ++i) {
                const int32_t t = tri[i];
                if (t < 0 || t >= M->ntri) {
                    bad = true;
                    return;
                }
                c[t + 1]++;
                ord &= i == lo || t >= tri[i - 1];
            }
            if (!ord) unordered = true;
            std::lock_guard<std::mutex> g(mu);
            for (int t = 0; t <= M->ntri; ++t) cnt[t] += c[t];
        });
        if (bad) return fail(TCG_E_ARG, "triangulation index out of range");
        if (unordered) cnt[0] = -1;  // marker
    }
    const bool grouped = cnt[0] == 0;
    cnt[0] = 0;
    for (int t = 0; t < M->ntri; ++t) cnt[t + 1] += cnt[t];
    std::vector<int64_t> order;
    std::vector<uint64_t> ssig;
    if (!grouped) {
        std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
        order.resize(n);
        ssig.resize(n);
        for (int64_t i = 0; i < n; ++i) {
            const int64_t j = pos[tri[i]]++;
            order[j] = i;
            ssig[j] = sig[i];
        }
    }
    const uint64_t *gsig = grouped ? sig : ssig.data();
    std::vector<int4> items;
    for (int t = 0; t < M->ntri; ++t)
        for (int64_t a = cnt[t]; a < cnt[t + 1]; a += ITEM)
            items.push_back(make_int4(t, (int)a, (int)std::min<int64_t>(ITEM, cnt[t + 1] - a), 0));
    host_mark("multi grouped");
    if (n > M->cap) {
        void *ptrs[] = {M->d_sig, M->d_key, M->d_ov, M->d_nr, M->d_st};
        for (void *q : ptrs)
            if (q) cudaFree(q);
        M->cap = 0;
        const int64_t cap = std::max<int64_t>(n, 1 << 16);
        CUDA_TRY(cudaMalloc(&M->d_sig, cap * 8));
        CUDA_TRY(cudaMalloc(&M->d_key, cap * 8));
        CUDA_TRY(cudaMalloc(&M->d_ov, cap));
        CUDA_TRY(cudaMalloc(&M->d_nr, cap));
        CUDA_TRY(cudaMalloc(&M->d_st, cap * 4));
        M->cap = cap;
    }
    if ((int64_t)items.size() > M->items_cap) {
        if (M->d_items) cudaFree(M->d_items);
        M->d_items = nullptr;
        M->items_cap = 0;
        CUDA_TRY(cudaMalloc(&M->d_items, sizeof(int4) * items.size()));
        M->items_cap = (int64_t)items.size();
    }
    for (int i = 0; i < 2; ++i) {
        if (!M->sst[i]) CUDA_TRY(cudaStreamCreateWithFlags(&M->sst[i], cudaStreamNonBlocking));
        for (int j = 0; j < 2; ++j)
            if (!M->ev[i][j]) CUDA_TRY(cudaEventCreate(&M->ev[i][j]));
        if (!M->h_stage[i])
            CUDA_TRY(cudaHostAlloc((void **)&M->h_stage[i], (size_t)multi_chunk() * 22, cudaHostAllocDefault));
    }
    CUDA_TRY(cudaMemcpy(M->d_items, items.data(), sizeof(int4) * items.size(), cudaMemcpyHostToDevice));
    void *fn = pick_multi(M->K, M->even);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)M->smem);
    // Pipeline over chunks of whole items (<= MULTI_CHUNK pairs): slot c & 1
    // stages chunk c's signs into pinned memory (host threads), copies them up,
    // classifies, copies the results down on its stream; chunk c-2's results
    // leave the slot (host threads, scattered back if the input was regrouped)
    // before it is reused, so host copies, PCIe both ways and the kernel overlap.
    const int64_t MULTI_CHUNK = multi_chunk();
    struct Chunk { int64_t ib, ie, p0, p1; };
    std::vector<Chunk> chunks;
    for (int64_t ib = 0; ib < (int64_t)items.size();) {
        int64_t ie = ib, p0 = items[ib].y, p1 = p0;
        while (ie < (int64_t)items.size() && items[ie].y + items[ie].z - p0 <= MULTI_CHUNK) {
            p1 = items[ie].y + items[ie].z;
            ++ie;
        }
        chunks.push_back({ib, ie, p0, p1});
        ib = ie;
    }
    struct Stage {
        uint64_t *sig, *key;
        int32_t *st;
        uint8_t *ov, *nr;
    };
    auto stage = [&](int sl) {
        uint8_t *h = M->h_stage[sl];
        return Stage{reinterpret_cast<uint64_t *>(h), reinterpret_cast<uint64_t *>(h + 8 * MULTI_CHUNK),
                     reinterpret_cast<int32_t *>(h + 16 * MULTI_CHUNK), h + 20 * MULTI_CHUNK,
                     h + 21 * MULTI_CHUNK};
    };
    float kms = 0.f;
    auto drain = [&](size_t c) -> int {
        const int sl = (int)(c & 1);
        const Chunk &C = chunks[c];
        CUDA_TRY(cudaStreamSynchronize(M->sst[sl]));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, M->ev[sl][0], M->ev[sl][1]);
        kms += ms;
        const Stage S = stage(sl);
        const uint64_t *hk = S.key;
        const int32_t *hst = S.st;
        const uint8_t *hov = S.ov, *hnr = S.nr;
        const int64_t len = C.p1 - C.p0;
        par_for(len, [&](int64_t lo, int64_t hi) {
            if (grouped) {
                std::memcpy(key + C.p0 + lo, hk + lo, (hi - lo) * 8);
                std::memcpy(st + C.p0 + lo, hst + lo, (hi - lo) * 4);
                std::memcpy(ov + C.p0 + lo, hov + lo, hi - lo);
                std::memcpy(nr + C.p0 + lo, hnr + lo, hi - lo);
            } else {
                for (int64_t j = lo; j < hi; ++j) {
                    const int64_t i = order[C.p0 + j];
                    key[i] = hk[j];
                    st[i] = hst[j];
                    ov[i] = hov[j];
                    nr[i] = hnr[j];
                }
            }
        });
        return TCG_OK;
    };
    for (size_t c = 0; c < chunks.size() + 2; ++c) {
        if (c >= 2) {
            int rc = drain(c - 2);
            if (rc) return rc;
        }
        if (c >= chunks.size()) continue;
        const int sl = (int)(c & 1);
        const Chunk &C = chunks[c];
        const int64_t len = C.p1 - C.p0;
        cudaStream_t s = M->sst[sl];
        const Stage S = stage(sl);
        uint64_t *hs = S.sig, *hk = S.key;
        int32_t *hst = S.st;
        uint8_t *hov = S.ov, *hnr = S.nr;
        par_for(len, [&](int64_t lo, int64_t hi) { std::memcpy(hs + lo, gsig + C.p0 + lo, (hi - lo) * 8); });
        CUDA_TRY(cudaMemcpyAsync(M->d_sig + C.p0, hs, len * 8, cudaMemcpyHostToDevice, s));
        const int4 *it = M->d_items + C.ib;
        void *args[] = {&M->d_kp, &it, &M->d_sig, &M->d_key, &M->d_ov, &M->d_nr, &M->d_st};
        cudaEventRecord(M->ev[sl][0], s);
        CUDA_TRY(cudaLaunchKernel(fn, dim3((unsigned)(C.ie - C.ib)), dim3(THREADS), args, M->smem, s));
        cudaEventRecord(M->ev[sl][1], s);
        M->launches++;
        CUDA_TRY(cudaMemcpyAsync(hk, M->d_key + C.p0, len * 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(hst, M->d_st + C.p0, len * 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(hov, M->d_ov + C.p0, len, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(hnr, M->d_nr + C.p0, len, cudaMemcpyDeviceToHost, s));
    }
    host_mark("multi done");
    M->last_ms = kms;
    return TCG_OK;
}

double tcg_multi_last_ms(const tcg_multi *M) { return M ? (double)M->last_ms : -1.0; }
