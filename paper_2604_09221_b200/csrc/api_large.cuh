// api_large.cuh -- C ABI of the any-degree engine.  Included by tcg.cu
// inside its extern "C" block.

// ------------------------------------------------------------ any degree (host)
struct tcg_large {
    int device = 0;
    LargeParams lp{};
    int32_t *d_i32 = nullptr;  // eu, ev, src, apu, apv
    uint8_t *d_u8 = nullptr;   // par, used
    size_t smem = 0;
    cudaStream_t stream = nullptr;
    int blocks = 0;
    int64_t cap = 0;  // persistent batch buffers
    uint64_t *d_sig = nullptr;
    int32_t *d_st = nullptr, *d_nr = nullptr, *d_par = nullptr;
};

int tcg_large_destroy(tcg_large *G) {
    if (!G) return TCG_OK;
    DeviceGuard guard(G->device);
    if (G->stream) cudaStreamSynchronize(G->stream);
    if (G->d_i32) cudaFree(G->d_i32);
    if (G->d_u8) cudaFree(G->d_u8);
    void *bufs[] = {G->d_sig, G->d_st, G->d_nr, G->d_par};
    for (void *q : bufs)
        if (q) cudaFree(q);
    if (G->stream) cudaStreamDestroy(G->stream);
    delete G;
    return TCG_OK;
}

int tcg_large_create(const tcg_desc *D, int device, tcg_large **out) {
    if (!D || !out) return fail(TCG_E_ARG, "null argument");
    *out = nullptr;
    const int d = D->degree;
    if (d < 1 || D->nv != 2 * d * d + 2 * d + 1 || D->npts != (d + 1) * (d + 2) / 2)
        return fail(TCG_E_ARG, "descriptor sizes do not match the degree");
    if (D->maxreg < 1 || D->maxreg >= 65535) return fail(TCG_E_UNSUPPORTED, "maxreg out of range");
    if (D->ne < 1) return fail(TCG_E_ARG, "empty edge list");
    for (int e = 0; e < D->ne; ++e)
        if (D->edge_u[e] < 0 || D->edge_u[e] >= D->nv || D->edge_v[e] < 0 || D->edge_v[e] >= D->nv)
            return fail(TCG_E_ARG, "edge endpoint out of range");
    for (int v = 0; v < D->nv; ++v)
        if (D->src[v] < 0 || D->src[v] >= D->npts) return fail(TCG_E_ARG, "src out of range");
    for (int a = 0; a < D->nap; ++a)
        if (D->ap_u[a] < 0 || D->ap_u[a] >= D->nv || D->ap_v[a] < 0 || D->ap_v[a] >= D->nv)
            return fail(TCG_E_ARG, "antipodal pair out of range");
    if (device < 0 && cudaGetDevice(&device) != cudaSuccess) {
        cudaGetLastError();
        return fail(TCG_E_CUDA, "no CUDA device");
    }
    tcg_large *G = new tcg_large();
    G->device = device;
    DeviceGuard guard(device);
    auto bail = [&](cudaError_t e, const char *what) {
        std::string msg = std::string(what) + ": " + cudaGetErrorString(e);
        tcg_large_destroy(G);
        return fail(TCG_E_CUDA, msg);
    };
    cudaError_t e;
    cudaDeviceProp prop;
    if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess) return bail(e, "props");
    if (prop.major < 10) {
        tcg_large_destroy(G);
        return fail(TCG_E_UNSUPPORTED, "libtcg is built for sm_100a (Blackwell B200)");
    }
    if ((e = cudaStreamCreateWithFlags(&G->stream, cudaStreamNonBlocking)) != cudaSuccess)
        return bail(e, "stream");
    const size_t ni = 2 * (size_t)D->ne + D->nv + 2 * (size_t)D->nap;
    std::vector<int32_t> i32(ni);
    std::copy(D->edge_u, D->edge_u + D->ne, i32.begin());
    std::copy(D->edge_v, D->edge_v + D->ne, i32.begin() + D->ne);
    std::copy(D->src, D->src + D->nv, i32.begin() + 2 * D->ne);
    std::copy(D->ap_u, D->ap_u + D->nap, i32.begin() + 2 * D->ne + D->nv);
    std::copy(D->ap_v, D->ap_v + D->nap, i32.begin() + 2 * D->ne + D->nv + D->nap);
    std::vector<uint8_t> u8(2 * (size_t)D->nv);
    std::copy(D->par, D->par + D->nv, u8.begin());
    std::copy(D->used, D->used + D->nv, u8.begin() + D->nv);
    if ((e = cudaMalloc(&G->d_i32, 4 * ni)) != cudaSuccess) return bail(e, "malloc");
    if ((e = cudaMalloc(&G->d_u8, u8.size())) != cudaSuccess) return bail(e, "malloc");
    cudaMemcpy(G->d_i32, i32.data(), 4 * ni, cudaMemcpyHostToDevice);
    if ((e = cudaMemcpy(G->d_u8, u8.data(), u8.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
        return bail(e, "upload");
    LargeParams &L = G->lp;
    L.d = d;
    L.nv = D->nv;
    L.ne = D->ne;
    L.nap = D->nap;
    L.npts = D->npts;
    L.maxreg = D->maxreg;
    L.words = (D->npts + 63) / 64;
    L.eu = G->d_i32;
    L.ev = G->d_i32 + D->ne;
    L.src = G->d_i32 + 2 * D->ne;
    L.apu = G->d_i32 + 2 * D->ne + D->nv;
    L.apv = L.apu + D->nap;
    L.par = G->d_u8;
    L.used = G->d_u8 + D->nv;
    G->smem = 3 * 4 * (size_t)D->nv + 4 * (size_t)LHASH + 4 * (size_t)(5 * D->maxreg + 1) +
              3 * (size_t)D->nv + 16;
    if (G->smem > 200 * 1024) {
        tcg_large_destroy(G);
        return fail(TCG_E_UNSUPPORTED, "degree too large for one CTA's shared memory");
    }
    cudaFuncSetAttribute((void *)k_large, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)G->smem);
    int bps = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, (void *)k_large, THREADS, G->smem);
    G->blocks = std::max(1, bps) * prop.multiProcessorCount;
    *out = G;
    return TCG_OK;
}

int tcg_large_classify(tcg_large *G, const uint64_t *sigma_rows, int64_t n, int32_t *status,
                       int32_t *nreg, int32_t *parent) {
    if (!G || (n > 0 && (!sigma_rows || !status || !nreg || !parent)))
        return fail(TCG_E_ARG, "null argument");
    if (n <= 0) return TCG_OK;
    DeviceGuard guard(G->device);
    const LargeParams &L = G->lp;
    if (n > G->cap) {
        void *bufs[] = {G->d_sig, G->d_st, G->d_nr, G->d_par};
        for (void *q : bufs)
            if (q) cudaFree(q);
        G->d_sig = nullptr;
        G->d_st = G->d_nr = G->d_par = nullptr;
        G->cap = 0;
        const int64_t cap = std::max<int64_t>(n, 256);
        CUDA_TRY(cudaMalloc(&G->d_sig, 8 * (size_t)cap * L.words));
        CUDA_TRY(cudaMalloc(&G->d_st, 4 * (size_t)cap));
        CUDA_TRY(cudaMalloc(&G->d_nr, 4 * (size_t)cap));
        CUDA_TRY(cudaMalloc(&G->d_par, 4 * (size_t)cap * L.maxreg));
        G->cap = cap;
    }
    uint64_t *d_sig = G->d_sig;
    int32_t *d_st = G->d_st, *d_nr = G->d_nr, *d_par = G->d_par;
    CUDA_TRY(cudaMemcpyAsync(d_sig, sigma_rows, 8 * (size_t)n * L.words, cudaMemcpyHostToDevice,
                             G->stream));
    const unsigned blocks = (unsigned)std::min<int64_t>(G->blocks, n);
    LargeParams lp = L;
    void *args[] = {&lp, &d_sig, &n, &d_st, &d_nr, &d_par};
    CUDA_TRY(cudaLaunchKernel((void *)k_large, dim3(blocks), dim3(THREADS), args, G->smem,
                              G->stream));
    CUDA_TRY(cudaMemcpyAsync(status, d_st, 4 * (size_t)n, cudaMemcpyDeviceToHost, G->stream));
    CUDA_TRY(cudaMemcpyAsync(nreg, d_nr, 4 * (size_t)n, cudaMemcpyDeviceToHost, G->stream));
    CUDA_TRY(cudaMemcpyAsync(parent, d_par, 4 * (size_t)n * L.maxreg, cudaMemcpyDeviceToHost,
                             G->stream));
    CUDA_TRY(cudaStreamSynchronize(G->stream));
    return TCG_OK;
}
