// tcg.cu -- sm_100a real-scheme classifier for combinatorial patchworks.
//
// One thread classifies one (triangulation, sign vector) pair.  The whole
// per-patchwork state lives in registers as bitmasks over the diamond's
// vertices; the only memory traffic in the hot loop is one shared-memory
// adjacency row per visited vertex (a warp-divergent LDS.64/128).
//
// Algorithm (same outputs as the reference's classify_core,
// kernels.py:107-356, restructured for SIMT):
//   1. sign mask: sigma (bit k = point k) -> sign of every diamond vertex,
//      via the half-swap vertex layout (see build_layout): ~30 integer ops.
//   2. one breadth-first pass over all used vertices that labels REGIONS
//      directly: inside a layer it follows non-crossed edges (same-sign
//      neighbours, `adj & same & unvisited`); when the layer is exhausted it
//      jumps through the antipodal identification, which in this layout is a
//      swap of the two mask halves (free: register renaming).  Layers
//      alternate orientation parity, so the reference's parity union-find
//      (kernels.py:151-174) reduces to one check per region: an antipodal
//      pair whose ends sit in layers of equal parity closes an odd cycle.
//      Crossed-edge neighbours are OR-ed into XB on the fly.
//   3. region graph: regions r != r' are adjacent iff XB_r & R_r' != 0;
//      XB_r & R_r != 0 is a crossed edge inside r (pseudoline root in odd
//      degree, NONSEPARATING_OVAL in even degree).  Checks reproduce the
//      reference's status precedence; the two order-dependent collisions
//      (NOT_A_TREE racing NONSEPARATING_OVAL / ROOT_CONFLICT) fall back to
//      an exact replay of kernels.py:199-230 in edge order.
//   4. rooted tree -> AHU canonical code as a 64-bit key (sentinel bit).
//   5. sweep / sample kernels aggregate keys in a per-CTA shared-memory
//      hash table (warp-aggregated with __match_any_sync), flushed to a
//      global table: count sum, witness min (kernels.py:379-420).
//
// Source layout (one compilation unit; the .cuh files are included below):
//   classify.cuh     full-diamond classifier, batch / C4 / enumeration kernels,
//                    per-CTA scheme tables
//   tiles.cuh        sweep tiles: super-tiles, tile records, dedup, tile classify
//   level2.cuh       level-2 and two-stage records, their dedup and classifiers
//   large.cuh        any-degree kernel (d > 9)
//   split.cuh        separator-split sampler (C5) kernels
//   host_plan.cuh    plan-side host helpers: layout, tile tables, host plan
//   split_design.cuh the sampler's separator design and tables (host)
//   tcg.cu           plan lifetime, sweep / sample pipelines, aggregation fetch,
//                    multi-plan runs (the C ABI of include/tcg.h)
//   api_multi.cuh    C ABI of the many-triangulation engine
//   api_large.cuh    C ABI of the any-degree engine
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/tcg.h"

#define TCG_VERSION "tcg 0.1.0 sm_100a"

// Bounds-checked build (-DTCG_CHECKED, scripts/gpu_checked.sh): device
// asserts on the computed indices into lane-private shared memory, row slots,
// record pools and output lists.  compute-sanitizer is not available on this
// GPU pool; this build, run over the GPU test suite, stands in for memcheck.
#ifdef TCG_CHECKED
#include <cassert>
#define TCG_ASSERT(c) assert(c)
#else
#define TCG_ASSERT(c) ((void)0)
#endif

namespace {

constexpr int MAXK = 6;        // 32-bit words per vertex mask (d <= 9)
constexpr int MAXR = 32;       // regions representable (maxreg <= 31 for d <= 9)
constexpr int NQ4 = 8;         // compress runs for the mirrored quadrant
constexpr int THREADS = 256;   // threads per CTA
#ifndef TCG_TBL_BITS
#define TCG_TBL_BITS 9
#endif
constexpr int TBL_BITS = TCG_TBL_BITS;  // per-CTA scheme table slots (overflow goes to the global table)
constexpr int TBL = 1 << TBL_BITS;
constexpr int TBL_PROBES = 64;
constexpr int GCAP_BITS = 16;  // global scheme table: 65,536 slots (as the reference's agg)
constexpr int GCAP = 1 << GCAP_BITS;
constexpr int NHIST = 64;
constexpr uint64_t LAUNCH_MAX = 1ull << 33;  // indices per flat launch

enum Mode { MODE_RAW = 0, MODE_REP = 1, MODE_SAMPLE = 2 };

struct KParams {
    int d, npts, nused, maxreg, nq4, center, ne;
    uint32_t used[MAXK];
    uint32_t bd[MAXK];        // boundary vertices that have an antipodal partner
    uint32_t parP[MAXK / 2];  // P-half positions with |i|+|j| odd
    uint32_t jodd[MAXK / 2];  // mirrored-quadrant positions with j odd
    uint8_t q4src[NQ4], q4len[NQ4], q4dst[NQ4];
    const uint32_t *adj;    // [2H][K] adjacency rows (global; staged to smem)
    const uint32_t *edges;  // [ne] packed positions (u | v << 16), reference order
};

struct DevAgg {
    unsigned long long *keys;  // [GCAP]
    unsigned long long *cnt;   // [GCAP]
    unsigned long long *wit;   // [GCAP]
    unsigned long long *hist;  // [NHIST]
    unsigned long long *bad;   // [1] smallest failing index
    unsigned int *overflow;    // [1]
};

struct Result {
    int status;
    int nreg;
    uint64_t key;
};

#include "classify.cuh"

#include "tiles.cuh"

#include "level2.cuh"

#include "large.cuh"

__global__ void k_agg_clear(DevAgg g) {
    const int stride = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < GCAP; i += stride) {
        g.keys[i] = 0ull;
        g.cnt[i] = 0ull;
        g.wit[i] = ~0ull;
    }
    if (blockIdx.x == 0 && threadIdx.x < NHIST) g.hist[threadIdx.x] = 0ull;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *g.bad = ~0ull;
        *g.overflow = 0u;
    }
}

__global__ void k_agg_compact(DevAgg g, unsigned long long *okey, unsigned long long *ocnt,
                              unsigned long long *owit, unsigned int *on) {
    const int stride = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < GCAP; i += stride) {
        const unsigned long long k = g.keys[i];
        if (k) {
            const unsigned int j = atomicAdd(on, 1u);
            okey[j] = k;
            ocnt[j] = g.cnt[i];
            owit[j] = g.wit[i];
        }
    }
}

#include "split.cuh"

// ------------------------------------------------------------ error state
thread_local std::string g_last_error;

int fail(int code, const std::string &msg) {
    g_last_error = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                  \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess)                                                          \
            return fail(TCG_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

}  // namespace

// ------------------------------------------------------------------- plan
struct tcg_plan {
    int device = 0, d = 0, K = 0, even = 0, nused = 0, maxreg = 0, nsm = 0;
    int threads = THREADS;
    int blocks_enum = 0, blocks_batch = 0;
    size_t smem_enum = 0, smem_batch = 0;
    KParams kp{};
    uint32_t *d_adj = nullptr, *d_edges = nullptr;
    DevAgg agg{};
    unsigned long long *d_ckey = nullptr, *d_ccnt = nullptr, *d_cwit = nullptr;
    unsigned int *d_cn = nullptr;
    uint64_t *d_sig = nullptr, *d_key = nullptr;
    uint8_t *d_ov = nullptr, *d_nr = nullptr;
    int32_t *d_st = nullptr;
    int64_t batch_cap = 0;
    // pinned double-buffered staging for host-buffer batches
    bool stage_ok = false;
    uint64_t *h_in[2] = {}, *h_key[2] = {}, *sd_in[2] = {}, *sd_key[2] = {};
    uint8_t *h_ov[2] = {}, *h_nr[2] = {}, *sd_ov[2] = {}, *sd_nr[2] = {};
    int32_t *h_st[2] = {}, *sd_st[2] = {};
    cudaStream_t sst[2] = {nullptr, nullptr};
    cudaStream_t own = nullptr, stream = nullptr;
    int64_t launches = 0;
    // tile contraction (sweeps): per domain (raw, representative)
    TileTables *d_tiles = nullptr;   // [2]
    L15Lut *d_lut = nullptr;         // [2] stage-1 F-space tables
    TileRec *d_recs = nullptr;       // [chunk_cap]
    uint32_t chunk_cap = 0;          // tiles the record / dedup buffers hold
    uint32_t *d_dedup = nullptr;     // slots[2 pow2(C)] | mint[C] | dup[C] | count[1] | list[C]
    unsigned long long *d_tstats = nullptr;  // [0] level-1 reps classified, [1] level-2 reps
    int l2_ok[2] = {0, 0};           // level-2 contraction available per domain
    TileTables h_tiles[2];           // host copies of the tile tables
    int blocks_l2cls = 0;
    int l2 = -1;                     // -1: TCG_NO_L2 decides
    int l2_stride = 0;               // u64 words per level-2 record
    size_t l2_cap = 0;               // level-2 records the buffers hold
    size_t l2_sized_for = 0;         // largest request the pool was sized for
    size_t l15_sized_for = 0, chunk_sized_for = 0;
    unsigned long long *d_l2pool = nullptr, *d_l2hash = nullptr;
    uint32_t *d_l2u32 = nullptr;     // wts | poss | w2 | pos2 | list2 | count2
    unsigned long long *d_l2slots = nullptr;  // [2 pow2(l2_cap)] tag << 32 | record
    // two-stage level 2: stage-1 records and their dedup state
    size_t l15_cap = 0;
    unsigned long long *d_l15pool = nullptr, *d_l15hash = nullptr, *d_l15slots = nullptr;
    uint32_t *d_l15u32 = nullptr;    // wts | poss | w15 | pos15 | list15 | count15 | fail | saved
    int64_t l15_built = 0, l15_fallbacks = 0;
    uint32_t *d_oldlist = nullptr;   // [chunk_cap + 1]: count, then tiles for the level-1 path
    uint32_t *d_ovf = nullptr;       // [chunk_cap + 1]: count, then tiles of fallback super-tiles
    SuperRec *d_super = nullptr;     // [super_cap]
    uint32_t *d_srep = nullptr;      // [super_cap] super-tile twin (k_super_dedup)
    unsigned long long *d_sslots = nullptr;  // [2 pow2(super_cap)] super dedup table
    uint32_t *d_repof = nullptr;     // [chunk_cap] tile -> its dedup group's representative
    unsigned long long *d_hash = nullptr;   // [chunk_cap] record hashes (written by the builders)
    unsigned long long *d_slots = nullptr;  // [2 pow2(chunk_cap)] dedup table: tag << 32 | tile
    size_t super_cap = 0;
    int blocks_bgen = 0;             // grid of the list-driven k_tile_build_lanes
    int64_t reps1_host = 0, l2_built = 0;
    int dedup = -1;                  // -1: TCG_NO_DEDUP decides
    int64_t tiles_built = 0;
    int tiles_ok[2] = {0, 0};
    int tile_bits[2] = {0, 0};
    int blocks_build = 0, blocks_cls = 0;
    size_t smem_build = 0, smem_cls = 0;
    // optional per-kernel timing (CUDA events on the launching stream)
    int timing = 0;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> tev;  // kind, start, stop
    double t_ms[TCG_NKINDS] = {};    // per kernel kind, see tcg.h
    int64_t t_n[TCG_NKINDS] = {};
    // split-phase bookkeeping: how to map a failing index back to its sign word
    int pending_mode = -1;
    uint64_t pending_seed = 0, pending_mask = 0;
    // separator-split sampler (split.cuh), built at the first sample
    int split = -1;                  // -1: TCG_NO_SPLIT decides, 0 off, 1 on
    int split_state = 0;             // 0: not built, 1: ready, -1: unavailable
    std::vector<int32_t> h_eu, h_ev, h_src, h_apu, h_apv, h_pos;  // descriptor copy
    std::vector<uint8_t> h_par, h_used;
    int h_nv = 0, h_npts = 0;
    SplitParams split_sp{};
    uint32_t *d_splitA = nullptr, *d_splitB = nullptr, *d_fbl = nullptr;
    unsigned long long *d_pext = nullptr, *d_splitstats = nullptr;  // [0] list draws
    int blocks_split = 0, blocks_list = 0;
    int64_t split_draws = 0;
    size_t split_bytes = 0;
};

namespace {
#include "host_plan.cuh"

#include "split_design.cuh"

}  // namespace

extern "C" {

const char *tcg_last_error(void) { return g_last_error.c_str(); }
const char *tcg_version(void) { return TCG_VERSION; }

int tcg_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int64_t tcg_launch_count(const tcg_plan *plan) { return plan ? plan->launches : -1; }

int tcg_plan_create(const tcg_desc *D, int device, tcg_plan **out) {
    if (!D || !out) return fail(TCG_E_ARG, "null argument");
    *out = nullptr;
    HostPlan HP;
    int rc = build_host_plan(D, HP);
    if (rc) return rc;
    const Layout &L = HP.L;
    const int K = HP.K;
    tcg_plan *P = new tcg_plan();
    P->d = HP.d;
    P->K = K;
    P->even = HP.even;
    P->maxreg = D->maxreg;
    P->nused = HP.nused;
    P->h_nv = D->nv;
    P->h_npts = D->npts;
    P->h_eu.assign(D->edge_u, D->edge_u + D->ne);
    P->h_ev.assign(D->edge_v, D->edge_v + D->ne);
    P->h_src.assign(D->src, D->src + D->nv);
    P->h_par.assign(D->par, D->par + D->nv);
    P->h_used.assign(D->used, D->used + D->nv);
    P->h_apu.assign(D->ap_u, D->ap_u + D->nap);
    P->h_apv.assign(D->ap_v, D->ap_v + D->nap);
    P->h_pos = HP.L.pos;
    KParams &kp = P->kp;
    kp = HP.kp;
    std::vector<uint32_t> &adj = HP.adj;
    std::vector<uint32_t> &edges = HP.edges;
    if (device < 0) {
        if (cudaGetDevice(&device) != cudaSuccess) {
            delete P;
            cudaGetLastError();
            return fail(TCG_E_CUDA, "no CUDA device");
        }
    }
    P->device = device;
    DeviceGuard guard(device);
    auto bail = [&](cudaError_t e, const char *what) {
        std::string msg = std::string(what) + ": " + cudaGetErrorString(e);
        tcg_plan_destroy(P);
        return fail(TCG_E_CUDA, msg);
    };
    cudaError_t e;
    if ((e = cudaFree(nullptr)) != cudaSuccess) return bail(e, "context");
    cudaDeviceProp prop;
    if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess) return bail(e, "props");
    if (prop.major < 10) {
        tcg_plan_destroy(P);
        return fail(TCG_E_UNSUPPORTED, "libtcg is built for sm_100a (Blackwell B200)");
    }
    P->nsm = prop.multiProcessorCount;
    if ((e = cudaStreamCreateWithFlags(&P->own, cudaStreamNonBlocking)) != cudaSuccess)
        return bail(e, "stream");
    P->stream = P->own;
    if ((e = cudaMalloc(&P->d_adj, adj.size() * 4)) != cudaSuccess) return bail(e, "malloc adj");
    if ((e = cudaMalloc(&P->d_edges, std::max<size_t>(1, edges.size()) * 4)) != cudaSuccess)
        return bail(e, "malloc edges");
    cudaMemcpy(P->d_adj, adj.data(), adj.size() * 4, cudaMemcpyHostToDevice);
    if (!edges.empty())
        cudaMemcpy(P->d_edges, edges.data(), edges.size() * 4, cudaMemcpyHostToDevice);
    kp.adj = P->d_adj;
    kp.edges = P->d_edges;
    {
        TileTables tt[2];
        const char *no_tiles = std::getenv("TCG_NO_TILES");
        for (int mode = 0; mode < 2; ++mode) {
            P->tiles_ok[mode] = (!no_tiles || !*no_tiles || no_tiles[0] == '0') &&
                                build_tiles(D, L, mode, tt[mode]);
            P->tile_bits[mode] = P->tiles_ok[mode] ? tt[mode].bits : 0;
            P->l2_ok[mode] = P->tiles_ok[mode] && tt[mode].l2;
            P->h_tiles[mode] = tt[mode];
        }
        if ((e = cudaMalloc(&P->d_tiles, sizeof(tt))) != cudaSuccess) return bail(e, "malloc tiles");
        cudaMemcpy(P->d_tiles, tt, sizeof(tt), cudaMemcpyHostToDevice);
        L15Lut luts[2];
        for (int m = 0; m < 2; ++m)
            for (int byte = 0; byte < 4; ++byte)
                for (int v = 0; v < 256; ++v) {
                    uint32_t r = 0;
                    for (int bit = 0; bit < 8; ++bit) {
                        const int f = 8 * byte + bit;
                        if (((v >> bit) & 1) && f < MAXF && tt[m].ts && tt[m].l15F[f] >= 0)
                            r |= 1u << tt[m].l15F[f];
                    }
                    luts[m].b[byte][v] = r;
                }
        if ((e = cudaMalloc(&P->d_lut, sizeof(luts))) != cudaSuccess) return bail(e, "malloc lut");
        cudaMemcpy(P->d_lut, luts, sizeof(luts), cudaMemcpyHostToDevice);
    }
    DevAgg &g = P->agg;
    if ((e = cudaMalloc(&g.keys, GCAP * 8)) != cudaSuccess) return bail(e, "malloc agg");
    if ((e = cudaMalloc(&g.cnt, GCAP * 8)) != cudaSuccess) return bail(e, "malloc agg");
    if ((e = cudaMalloc(&g.wit, GCAP * 8)) != cudaSuccess) return bail(e, "malloc agg");
    if ((e = cudaMalloc(&g.hist, NHIST * 8)) != cudaSuccess) return bail(e, "malloc agg");
    if ((e = cudaMalloc(&g.bad, 8)) != cudaSuccess) return bail(e, "malloc agg");
    if ((e = cudaMalloc(&g.overflow, 4)) != cudaSuccess) return bail(e, "malloc agg");
    if ((e = cudaMalloc(&P->d_ckey, GCAP * 8)) != cudaSuccess) return bail(e, "malloc compact");
    if ((e = cudaMalloc(&P->d_ccnt, GCAP * 8)) != cudaSuccess) return bail(e, "malloc compact");
    if ((e = cudaMalloc(&P->d_cwit, GCAP * 8)) != cudaSuccess) return bail(e, "malloc compact");
    if ((e = cudaMalloc(&P->d_cn, 4)) != cudaSuccess) return bail(e, "malloc compact");

    // launch geometry: persistent grid = SMs x resident CTAs
    P->smem_enum = enum_smem(K);
    P->smem_batch = adj_bytes(K);
    int bps = 0;
    for (int mode = 0; mode < 3; ++mode) {
        void *fn = pick_enum(K, P->even, mode);
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smem_enum);
        if (const char *c = std::getenv("TCG_ENUM_CARVEOUT"))
            cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(c));
    }
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, pick_enum(K, P->even, MODE_RAW),
                                                           THREADS, P->smem_enum)) != cudaSuccess)
        return bail(e, "occupancy");
    if (const char *e = std::getenv("TCG_ENUM_BPS")) bps = std::min(bps, std::max(1, std::atoi(e)));
    P->blocks_enum = std::max(1, bps) * P->nsm;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, pick_batch(K, P->even), THREADS,
                                                           P->smem_batch)) != cudaSuccess)
        return bail(e, "occupancy");
    P->blocks_batch = std::max(1, bps) * P->nsm;
    P->smem_build = build_smem(K);
    for (int mode = 0; mode < 2; ++mode)
        if ((e = cudaFuncSetAttribute(pick_super(K, mode),
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)build_smem(K))) != cudaSuccess)
            return bail(e, "super smem");
    for (void *kb : {(void *)k_l2_build<false>, (void *)k_l2_build<true>})
        if ((e = cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)L2B_SMEM)) != cudaSuccess)
            return bail(e, "l2 build smem");
    if ((e = cudaFuncSetAttribute((void *)k_l2_from_l15<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)L2B_SMEM)) != cudaSuccess ||
        (e = cudaFuncSetAttribute((void *)k_l2_from_l15<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)L2B_SMEM)) != cudaSuccess ||
        (e = cudaFuncSetAttribute((void *)k_l15_build, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)L15_SMEM_MAX)) != cudaSuccess)
        return bail(e, "l15 smem");
    cudaFuncSetAttribute((void *)k_l2_classify_even, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)L2E_CLS_SMEM);
    cudaFuncSetAttribute((void *)k_l2_classify_even, cudaFuncAttributePreferredSharedMemoryCarveout,
                         std::getenv("TCG_CARVEOUT") ? std::atoi(std::getenv("TCG_CARVEOUT")) : 38);
    if ((e = cudaFuncSetAttribute((void *)k_tile_from_super,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)FROM_SUPER_SMEM)) != cudaSuccess)
        return bail(e, "from-super smem");
    P->smem_cls = cls_smem(K);
    for (int mode = 0; mode < 2; ++mode) {
        cudaFuncSetAttribute(pick_build(K, mode), cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)P->smem_build);
        cudaFuncSetAttribute(pick_cls(K, P->even, mode),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smem_cls);
        // 38 % of the unified L1/shared array as shared memory (the 100 KB config:
        // 4 resident CTAs), the rest stays L1
        // for the per-thread region arrays (measured: the driver's default
        // choice halves throughput with the 512-slot table)
        const char *c = std::getenv("TCG_CARVEOUT");
        cudaFuncSetAttribute(pick_cls(K, P->even, mode),
                             cudaFuncAttributePreferredSharedMemoryCarveout, c ? std::atoi(c) : 38);
    }
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, pick_cls(K, P->even, MODE_RAW),
                                                           THREADS, P->smem_cls)) != cudaSuccess)
        return bail(e, "occupancy");
    P->blocks_cls = std::max(1, bps) * P->nsm;
    cudaFuncSetAttribute((void *)k_l2_classify, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)L2_CLS_SMEM);
    cudaFuncSetAttribute((void *)k_l2_classify, cudaFuncAttributePreferredSharedMemoryCarveout,
                         std::getenv("TCG_CARVEOUT") ? std::atoi(std::getenv("TCG_CARVEOUT")) : 38);
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, (void *)k_l2_classify, THREADS,
                                                           L2_CLS_SMEM)) != cudaSuccess)
        return bail(e, "occupancy");
    P->blocks_l2cls = std::max(1, bps) * P->nsm;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
             &bps, pick_build(K, MODE_RAW), THREADS,
             P->smem_build)) != cudaSuccess)
        return bail(e, "occupancy");
    P->blocks_build = std::max(1, bps) * P->nsm;
    P->blocks_bgen = std::max(1, bps) * P->nsm;
    *out = P;
    int rc2 = tcg_agg_reset(P);
    if (rc2) {
        tcg_plan_destroy(P);
        *out = nullptr;
        return rc2;
    }
    if ((e = cudaStreamSynchronize(P->stream)) != cudaSuccess) {
        tcg_plan_destroy(P);
        *out = nullptr;
        return fail(TCG_E_CUDA, std::string("init: ") + cudaGetErrorString(e));
    }
    return TCG_OK;
}

int tcg_plan_destroy(tcg_plan *P) {
    if (!P) return TCG_OK;
    DeviceGuard guard(P->device);
    if (P->stream) cudaStreamSynchronize(P->stream);
    timing_resolve(P);
    void *ptrs[] = {P->d_adj, P->d_edges, P->d_tiles, P->d_lut, P->d_recs, P->d_dedup, P->d_tstats, P->d_l2pool, P->d_l2hash, P->d_l2u32, P->d_l2slots, P->d_l15pool, P->d_l15hash, P->d_l15slots, P->d_l15u32, P->d_oldlist, P->d_ovf, P->d_super, P->d_hash, P->d_slots, P->agg.keys, P->agg.cnt, P->agg.wit, P->agg.hist,
                    P->agg.bad, P->agg.overflow, P->d_ckey, P->d_ccnt, P->d_cwit, P->d_cn,
                    P->d_sig, P->d_key, P->d_ov, P->d_nr, P->d_st, P->d_splitA, P->d_splitB,
                    P->d_fbl, P->d_pext, P->d_splitstats, P->d_srep, P->d_sslots, P->d_repof};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    for (int i = 0; i < 2; ++i) {
        void *hp[] = {P->h_in[i], P->h_key[i], P->h_ov[i], P->h_nr[i], P->h_st[i]};
        for (void *q : hp)
            if (q) cudaFreeHost(q);
        void *dp[] = {P->sd_in[i], P->sd_key[i], P->sd_ov[i], P->sd_nr[i], P->sd_st[i]};
        for (void *q : dp)
            if (q) cudaFree(q);
        if (P->sst[i]) cudaStreamDestroy(P->sst[i]);
    }
    if (P->own) cudaStreamDestroy(P->own);
    delete P;
    return TCG_OK;
}

int tcg_plan_set_stream(tcg_plan *P, void *stream) {
    if (!P) return fail(TCG_E_ARG, "null plan");
    P->stream = stream ? (cudaStream_t)stream : P->own;
    return TCG_OK;
}

int tcg_plan_set_timing(tcg_plan *P, int enable) {
    if (!P) return fail(TCG_E_ARG, "null plan");
    DeviceGuard guard(P->device);
    timing_resolve(P);
    P->timing = enable ? 1 : 0;
    return TCG_OK;
}

int tcg_plan_set_dedup(tcg_plan *P, int enable) {
    if (!P) return fail(TCG_E_ARG, "null plan");
    P->dedup = enable < 0 ? -1 : (enable ? 1 : 0);
    return TCG_OK;
}

int tcg_tile_stats(tcg_plan *P, int64_t *out) {
    if (!P || !out) return fail(TCG_E_ARG, "null argument");
    DeviceGuard guard(P->device);
    unsigned long long c = 0;
    if (P->d_tstats) {
        CUDA_TRY(cudaStreamSynchronize(P->stream));
        CUDA_TRY(cudaMemcpy(&c, P->d_tstats, sizeof(c), cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemset(P->d_tstats, 0, sizeof(c)));
    }
    out[0] = P->tiles_built;
    out[1] = (int64_t)c + P->reps1_host;
    P->tiles_built = 0;
    P->reps1_host = 0;
    return TCG_OK;
}

int tcg_plan_set_level2(tcg_plan *P, int enable) {
    if (!P) return fail(TCG_E_ARG, "null plan");
    P->l2 = enable < 0 ? -1 : (enable ? 1 : 0);
    return TCG_OK;
}

int tcg_level2_stats(tcg_plan *P, int64_t *out) {
    if (!P || !out) return fail(TCG_E_ARG, "null argument");
    DeviceGuard guard(P->device);
    unsigned long long c[2] = {0, 0};
    if (P->d_tstats) {
        CUDA_TRY(cudaStreamSynchronize(P->stream));
        CUDA_TRY(cudaMemcpy(c, P->d_tstats + 1, sizeof(c), cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemset(P->d_tstats + 1, 0, sizeof(c)));
    }
    out[0] = P->l2_built;
    out[1] = (int64_t)c[0];
    out[2] = (int64_t)c[1];
    P->l2_built = 0;
    return TCG_OK;
}

int tcg_split_design(const tcg_desc *D, int64_t *out) {
    // host only (no device): the separator the sampler would use for D
    if (!D || !out) return fail(TCG_E_ARG, "null argument");
    HostPlan HP;
    int rc = build_host_plan(D, HP);
    if (rc) return rc;
    SplitDesign S;
    if (!split_design(D, HP.L, S)) {
        out[0] = 0;
        return TCG_OK;
    }
    out[0] = 1;
    out[1] = S.sp.nF;
    out[2] = S.pa.bits;
    out[3] = S.pb.bits;
    out[4] = (int64_t)S.Fm;
    out[5] = (int64_t)S.Am;
    out[6] = (int64_t)S.Bm;
    out[7] = (int64_t)(S.mean_nodes * 1000.0);
    out[8] = (int64_t)S.sp.stride * 4 * ((1ll << S.pa.bits) + (1ll << S.pb.bits));
    return TCG_OK;
}

int tcg_plan_set_split(tcg_plan *P, int enable) {
    if (!P) return fail(TCG_E_ARG, "null plan");
    P->split = enable < 0 ? -1 : (enable ? 1 : 0);
    return TCG_OK;
}

int tcg_split_stats(tcg_plan *P, int64_t *out) {
    if (!P || !out) return fail(TCG_E_ARG, "null argument");
    DeviceGuard guard(P->device);
    unsigned long long fb = 0;
    if (P->d_splitstats) {
        CUDA_TRY(cudaStreamSynchronize(P->stream));
        CUDA_TRY(cudaMemcpy(&fb, P->d_splitstats, 8, cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemset(P->d_splitstats, 0, 8));
    }
    out[0] = P->split_state;
    out[1] = P->split_draws;
    out[2] = (int64_t)fb;
    out[3] = P->split_state > 0 ? P->split_sp.nF : 0;
    out[4] = (int64_t)P->split_bytes;
    P->split_draws = 0;
    return TCG_OK;
}

int tcg_kernel_times(tcg_plan *P, double *ms, int64_t *counts) {
    if (!P || !ms || !counts) return fail(TCG_E_ARG, "null argument");
    DeviceGuard guard(P->device);
    timing_resolve(P);
    for (int i = 0; i < TCG_NKINDS; ++i) {
        ms[i] = P->t_ms[i];
        counts[i] = P->t_n[i];
        P->t_ms[i] = 0;
        P->t_n[i] = 0;
    }
    return TCG_OK;
}

int tcg_plan_info(const tcg_plan *P, int32_t *info, int ninfo) {
    if (!P || !info) return fail(TCG_E_ARG, "null argument");
    const int32_t v[10] = {P->d, P->K, P->nused, P->device, P->nsm, P->blocks_enum, P->threads,
                           P->maxreg, P->tile_bits[0], P->tile_bits[1]};
    for (int i = 0; i < ninfo && i < 10; ++i) info[i] = v[i];
    return TCG_OK;
}

static int launch_batch(tcg_plan *P, const uint64_t *d_sig, int64_t n, uint64_t *d_key,
                        uint8_t *d_ov, uint8_t *d_nr, int32_t *d_st,
                        cudaStream_t stream = nullptr) {
    if (!stream) stream = P->stream;
    if (n <= 0) return TCG_OK;
    void *fn = pick_batch(P->K, P->even);
    int64_t blocks = std::min<int64_t>(P->blocks_batch, (n + THREADS - 1) / THREADS);
    void *args[] = {&P->kp, &d_sig, &n, &d_key, &d_ov, &d_nr, &d_st};
    cudaEvent_t e3 = timing_begin(P, stream);
    CUDA_TRY(cudaLaunchKernel(fn, dim3((unsigned)blocks), dim3(THREADS), args, P->smem_batch,
                              stream));
    timing_end(P, TCG_KT_BATCH, e3, stream);
    P->launches++;
    return TCG_OK;
}

int tcg_classify_batch_device(tcg_plan *P, const uint64_t *d_sig, int64_t n, uint64_t *d_key,
                              uint8_t *d_ov, uint8_t *d_nr, int32_t *d_st) {
    if (!P) return fail(TCG_E_ARG, "null plan");
    DeviceGuard guard(P->device);
    return launch_batch(P, d_sig, n, d_key, d_ov, d_nr, d_st);
}

// Host-buffer batches run as a two-stream pipeline over pinned staging
// buffers: while chunk c is copied in / classified / copied out on one
// stream, the host moves chunk c-1's results out of the other slot.
static constexpr int64_t STAGE_CHUNK = 1 << 20;

static int ensure_staging(tcg_plan *P) {
    if (P->stage_ok) return TCG_OK;
    for (int i = 0; i < 2; ++i) {
        CUDA_TRY(cudaHostAlloc(&P->h_in[i], STAGE_CHUNK * 8, cudaHostAllocDefault));
        CUDA_TRY(cudaHostAlloc(&P->h_key[i], STAGE_CHUNK * 8, cudaHostAllocDefault));
        CUDA_TRY(cudaHostAlloc(&P->h_ov[i], STAGE_CHUNK, cudaHostAllocDefault));
        CUDA_TRY(cudaHostAlloc(&P->h_nr[i], STAGE_CHUNK, cudaHostAllocDefault));
        CUDA_TRY(cudaHostAlloc(&P->h_st[i], STAGE_CHUNK * 4, cudaHostAllocDefault));
        CUDA_TRY(cudaMalloc(&P->sd_in[i], STAGE_CHUNK * 8));
        CUDA_TRY(cudaMalloc(&P->sd_key[i], STAGE_CHUNK * 8));
        CUDA_TRY(cudaMalloc(&P->sd_ov[i], STAGE_CHUNK));
        CUDA_TRY(cudaMalloc(&P->sd_nr[i], STAGE_CHUNK));
        CUDA_TRY(cudaMalloc(&P->sd_st[i], STAGE_CHUNK * 4));
        CUDA_TRY(cudaStreamCreateWithFlags(&P->sst[i], cudaStreamNonBlocking));
    }
    P->stage_ok = true;
    return TCG_OK;
}

int tcg_classify_batch(tcg_plan *P, const uint64_t *sig, int64_t n, uint64_t *key, uint8_t *ov,
                       uint8_t *nr, int32_t *st) {
    if (!P || (n > 0 && (!sig || !key || !ov || !nr || !st))) return fail(TCG_E_ARG, "null argument");
    if (n <= 0) return TCG_OK;
    DeviceGuard guard(P->device);
    int rc = ensure_staging(P);
    if (rc) return rc;
    CUDA_TRY(cudaStreamSynchronize(P->stream));  // order after earlier work on the plan
    const int64_t nch = (n + STAGE_CHUNK - 1) / STAGE_CHUNK;
    for (int64_t c = 0; c < nch + 2; ++c) {
        const int sl = (int)(c & 1);
        if (c >= 2) {  // drain chunk c-2 from this slot
            const int64_t lo = (c - 2) * STAGE_CHUNK, len = std::min(STAGE_CHUNK, n - lo);
            CUDA_TRY(cudaStreamSynchronize(P->sst[sl]));
            std::memcpy(key + lo, P->h_key[sl], len * 8);
            std::memcpy(ov + lo, P->h_ov[sl], len);
            std::memcpy(nr + lo, P->h_nr[sl], len);
            std::memcpy(st + lo, P->h_st[sl], len * 4);
        }
        if (c < nch) {
            const int64_t lo = c * STAGE_CHUNK, len = std::min(STAGE_CHUNK, n - lo);
            cudaStream_t s = P->sst[sl];
            std::memcpy(P->h_in[sl], sig + lo, len * 8);
            CUDA_TRY(cudaMemcpyAsync(P->sd_in[sl], P->h_in[sl], len * 8, cudaMemcpyHostToDevice, s));
            rc = launch_batch(P, P->sd_in[sl], len, P->sd_key[sl], P->sd_ov[sl], P->sd_nr[sl],
                              P->sd_st[sl], s);
            if (rc) return rc;
            CUDA_TRY(cudaMemcpyAsync(P->h_key[sl], P->sd_key[sl], len * 8, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaMemcpyAsync(P->h_ov[sl], P->sd_ov[sl], len, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaMemcpyAsync(P->h_nr[sl], P->sd_nr[sl], len, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaMemcpyAsync(P->h_st[sl], P->sd_st[sl], len * 4, cudaMemcpyDeviceToHost, s));
        }
    }
    return TCG_OK;
}

int tcg_agg_reset(tcg_plan *P) {
    if (!P) return fail(TCG_E_ARG, "null plan");
    DeviceGuard guard(P->device);
    k_agg_clear<<<64, 256, 0, P->stream>>>(P->agg);
    CUDA_TRY(cudaGetLastError());
    P->launches++;
    P->pending_mode = -1;
    return TCG_OK;
}

// TCG_NO_L2=1 keeps sweeps on the level-1 tile classifier; results are identical.
static bool l2_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("TCG_NO_L2");
        return !(e && e[0] && e[0] != '0');
    }();
    return on;
}

static int l2_tail(tcg_plan *P, const TileTables &T, const TileTables *tt, uint32_t nrec,
                   uint32_t stride, uint64_t tile0);

// Two-stage level 2 for one batch of level-1 representatives.  Returns true
// when the batch is done; false (nothing consumed) when a record exceeded its
// super-node budget or the stage-2 records do not fit, and the caller runs the
// direct path.
static bool run_two_stage(tcg_plan *P, int mode, const TileTables *tt, const TileRec *recs,
                          const uint32_t *list1, const uint32_t *dup1, const uint32_t *mint1,
                          uint32_t i0, uint32_t nb, uint64_t tile0, uint64_t lo, uint64_t hi,
                          size_t cap, uint32_t stride, int &rc) {
    const TileTables &T = P->h_tiles[mode];
    // L15Bits stream: 3 nF + m + 1 bits per super-node, m <= L15_MAXM, nF <= 21;
    // one stride for every mode, so the pool's record capacity holds for all
    const uint32_t stride1 = (uint32_t)(1 + (L15_MAXM * (3 * 21 + L15_MAXM + 1) + 63) / 64);
    const uint32_t nrec1 = nb << T.la1;
    auto cuda_ok = [&](cudaError_t e, const char *what) {
        if (e != cudaSuccess) rc = fail(TCG_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
        return e == cudaSuccess;
    };
    if (nrec1 > P->l15_cap && nrec1 > P->l15_sized_for) {
        P->l15_sized_for = nrec1;
        size_t fr = 0, tot = 0;
        if (!cuda_ok(cudaStreamSynchronize(P->stream), "sync")) return false;
        if (!cuda_ok(cudaMemGetInfo(&fr, &tot), "meminfo")) return false;
        const size_t per = (size_t)stride1 * 8 + 8 + 4 * 6 + 16;
        fr += P->l15_cap * per;
        if ((size_t)nrec1 * per > fr / 2) return false;  // no room: direct path
        const size_t c1 = std::max<size_t>(nrec1, (P->chunk_cap / 2) << T.la1);
        const size_t c = c1 * per <= fr / 2 ? c1 : nrec1;
        cudaFree(P->d_l15pool);
        cudaFree(P->d_l15hash);
        cudaFree(P->d_l15slots);
        cudaFree(P->d_l15u32);
        P->d_l15pool = nullptr;
        P->d_l15hash = nullptr;
        P->d_l15slots = nullptr;
        P->d_l15u32 = nullptr;
        P->l15_cap = 0;
        if (!cuda_ok(cudaMalloc(&P->d_l15pool, sizeof(unsigned long long) * stride1 * c), "malloc l15") ||
            !cuda_ok(cudaMalloc(&P->d_l15hash, sizeof(unsigned long long) * c), "malloc l15") ||
            !cuda_ok(cudaMalloc(&P->d_l15slots, sizeof(unsigned long long) * 2 *
                                                    (size_t)next_pow2((uint32_t)c)), "malloc l15") ||
            !cuda_ok(cudaMalloc(&P->d_l15u32, sizeof(uint32_t) * (5 * c + 3)), "malloc l15"))
            return false;
        P->l15_cap = c;
    }
    if (nrec1 > P->l15_cap) return false;  // sized before and did not fit: direct path
    const size_t c = P->l15_cap;
    uint32_t *wts1 = P->d_l15u32, *poss1 = wts1 + c, *w15 = poss1 + c, *pos15 = w15 + c,
             *list15 = pos15 + c, *count15 = list15 + c, *failp = count15 + 1, *saved = failp + 1;
    unsigned long long *slots1 = P->d_l15slots, *pool1 = P->d_l15pool, *hash1 = P->d_l15hash;
    cudaStream_t st = P->stream;
    const uint32_t np2 = next_pow2(nrec1);
    if (!cuda_ok(cudaMemcpyAsync(saved, P->d_oldlist, 4, cudaMemcpyDeviceToDevice, st), "save") ||
        !cuda_ok(cudaMemsetAsync(failp, 0, 4, st), "memset") ||
        !cuda_ok(cudaMemsetAsync(count15, 0, 4, st), "memset") ||
        !cuda_ok(cudaMemsetAsync(slots1, 0xff, sizeof(unsigned long long) * 2 * (size_t)np2, st), "memset") ||
        !cuda_ok(cudaMemsetAsync(w15, 0, sizeof(uint32_t) * nrec1, st), "memset") ||
        !cuda_ok(cudaMemsetAsync(pos15, 0xff, sizeof(uint32_t) * nrec1, st), "memset"))
        return false;
    uint32_t *oldlist = P->d_oldlist + 1, *oldcount = P->d_oldlist;
    uint64_t t0 = tile0, a = lo, b = hi;
    uint32_t i0v = i0, nbv = nb, s1 = stride1;
    // grid sizes (CTAs per SM; measured, profiles/README.md): the stage-1 build
    // runs one pass (a whole grid: its per-record work varies, and the block
    // scheduler balances it better than a grid-stride loop), the stage-1 dedup 8,
    // stage 2 3 (= resident CTAs)
    auto env_grid = [](const char *name, uint64_t dflt) {
        const char *e = std::getenv(name);
        return e ? (uint64_t)std::max(1, std::atoi(e)) : dflt;
    };
    static const uint64_t gm1 = env_grid("TCG_L15_GRID", 1u << 20), gm1d = env_grid("TCG_L15D_GRID", 8),
                          gm2 = env_grid("TCG_L2F_GRID", 3);
    const unsigned g1 = (unsigned)std::min<uint64_t>((uint64_t)P->nsm * gm1, (nrec1 + THREADS - 1) / THREADS);
    const unsigned g1d = (unsigned)std::min<uint64_t>((uint64_t)P->nsm * gm1d, (nrec1 + THREADS - 1) / THREADS);
    const L15Lut *lutp = P->d_lut + mode;
    // row slot size (uint4 rows, 16..64; TCG_L15_STAGE=0 stages only <= 32-node tiles)
    // and where the lookup tables live (global by default, measured 0.5 % faster
    // than staging them; TCG_L15_LUTG=0 stages them in shared memory)
    static const int slotq_env = [] {
        const char *e = std::getenv("TCG_L15_SLOTQ");
        const char *f = std::getenv("TCG_L15_STAGE");
        if (f && std::atoi(f) == 0) return 16;
        return e ? std::max(16, std::min(64, std::atoi(e))) : 0;  // 0: fit 4 CTAs per SM
    }();
    static const int lutg_env = [] {
        const char *e = std::getenv("TCG_L15_LUTG");
        return e ? std::atoi(e) : 1;
    }();
    static const int l15_static = [] {
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, (const void *)k_l15_build);
        return (int)fa.sharedSizeBytes;
    }();
    int slotq = slotq_env, lut_smem = !lutg_env && T.l15sh < 0;  // tables unused with l15sh
    if (slotq == 0) {  // the widest slot that keeps 4 CTAs (= the register limit) per SM:
        // with the whole-grid launch 4 CTAs and 47-row slots beat 3 CTAs and 64 (profiles/README.md)
        const int tiles = (THREADS / 32) * (32 >> T.la1);
        int sm_smem = 0;  // per-SM shared memory (228 KB on B200), queried
        if (cudaDeviceGetAttribute(&sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor,
                                   P->device) != cudaSuccess || sm_smem <= 0) {
            cudaGetLastError();
            sm_smem = 228 * 1024;
        }
        const int budget = sm_smem / 4 - 1024 - l15_static - L2B_WORDS * 4 * THREADS -
                           (lut_smem ? (int)sizeof(L15Lut) : 0);
        slotq = std::max(16, std::min(64, budget / (tiles * 16)));
    }
    void *ab[] = {&tt, &recs, &list1, &dup1, &mint1, &i0v, &nbv, &t0, &a, &b, &pool1, &s1,
                  &hash1, &wts1, &poss1, &oldlist, &oldcount, &failp, &lutp, &slotq, &lut_smem};
    const size_t smem1 = (size_t)L2B_WORDS * 4 * THREADS + (size_t)(THREADS / 32) * (32 >> T.la1) * slotq * 16 +
                         (lut_smem ? sizeof(L15Lut) : 0);
    cudaEvent_t e0 = timing_begin(P);
    if (!cuda_ok(cudaLaunchKernel((void *)k_l15_build, dim3(g1), dim3(THREADS), ab, smem1, st), "l15 build"))
        return false;
    timing_end(P, TCG_KT_L15_BUILD, e0);
    e0 = timing_begin(P);
    uint32_t smask1 = 2 * np2 - 1;
    int wps2 = 0;  // stage-1 records carry their word count
    uint32_t nr1 = nrec1;
    void *ad[] = {&pool1, &s1, &nr1, &hash1, &wts1, &poss1, &slots1, &smask1, &w15, &pos15,
                  &list15, &count15, &wps2};
    if (!cuda_ok(cudaLaunchKernel((void *)k_l2_dedup, dim3(g1d), dim3(THREADS), ad, 0, st), "l15 dedup"))
        return false;
    uint32_t hostv[2] = {0, 0};  // count15, fail
    host_mark("l15 enqueued");
    if (!cuda_ok(cudaMemcpyAsync(hostv, count15, 8, cudaMemcpyDeviceToHost, st), "copy") ||
        !cuda_ok(cudaStreamSynchronize(st), "sync"))
        return false;
    host_mark("l15 synced");
    timing_end(P, TCG_KT_L15_DEDUP, e0);
    P->l15_built += nrec1;
    P->launches += 2;
    const uint32_t n15 = hostv[0];
    auto fallback = [&]() {
        P->l15_fallbacks++;
        cuda_ok(cudaMemcpyAsync(P->d_oldlist, saved, 4, cudaMemcpyDeviceToDevice, st), "restore");
        return false;
    };
    if (hostv[1] || ((size_t)n15 << T.la2) > cap) return fallback();
    // stage 2 into the ordinary level-2 buffers
    const uint32_t nrec = n15 << T.la2;
    uint32_t *wts = P->d_l2u32, *poss = wts + cap;
    unsigned long long *pool = P->d_l2pool, *hashes = P->d_l2hash;
    const unsigned g2 = (unsigned)std::min<uint64_t>((uint64_t)P->nsm * gm2, (nrec + THREADS - 1) / THREADS);
    uint32_t s2 = stride;
    void *a2[] = {&tt, &pool1, &s1, &list15, &count15, &w15, &pos15, &pool, &s2, &hashes, &wts,
                  &poss, &failp};
    const size_t smem2 = (size_t)(L2B_WORDS + L2B_CS) * 4 * THREADS;  // + B-relation words
    cudaEvent_t e1 = timing_begin(P);
    void *l2f = T.nA2 <= 4 ? (void *)k_l2_from_l15<4> : (void *)k_l2_from_l15<16>;
    if (!cuda_ok(cudaLaunchKernel(l2f, dim3(std::max(1u, g2)), dim3(THREADS), a2, smem2, st),
                 "l2 from l15"))
        return false;
    host_mark("l2f enqueued");
    if (!cuda_ok(cudaMemcpyAsync(hostv + 1, failp, 4, cudaMemcpyDeviceToHost, st), "copy") ||
        !cuda_ok(cudaStreamSynchronize(st), "sync"))
        return false;
    host_mark("l2f synced");
    timing_end(P, TCG_KT_L2_BUILD, e1);
    P->launches++;
    if (hostv[1]) return fallback();
    rc = l2_tail(P, T, tt, nrec, stride, tile0);
    return rc == 0;
}

// TCG_L2_TWOSTAGE=0 builds level-2 records directly (A/B); same results.
static bool l2_twostage_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("TCG_L2_TWOSTAGE");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Level-2 stage of one chunk (after the level-1 dedup): build the records of
// every (representative tile, A pattern), deduplicate them, classify the
// representatives.  Tiles the level-2 path does not take (range ends,
// fallback, > 32 nodes) are listed in d_oldlist for the level-1 classifier.
// The level-1 representative count comes back to the host (one small copy)
// to size the batches.
static int run_level2(tcg_plan *P, int mode, const TileTables *tt, const TileRec *recs,
                      const uint32_t *list1, const uint32_t *count1, const uint32_t *dup1,
                      const uint32_t *mint1, uint64_t tile0, uint64_t lo, uint64_t hi) {
    const TileTables &T = P->h_tiles[mode];
    uint32_t n1 = 0;
    host_mark("l1 enqueued");
    CUDA_TRY(cudaMemcpyAsync(&n1, count1, sizeof(n1), cudaMemcpyDeviceToHost, P->stream));
    CUDA_TRY(cudaStreamSynchronize(P->stream));
    host_mark("l1 synced");
    P->reps1_host += n1;
    CUDA_TRY(cudaMemsetAsync(P->d_oldlist, 0, sizeof(uint32_t), P->stream));
    if (n1 == 0) return TCG_OK;
    const int la = T.la;
    const int wps = T.l2even ? 2 : 1;  // record words per super-node
    const uint32_t stride = (uint32_t)(1 + wps * (32 - T.nB));
    // sized once for the whole chunk (every level-1 tile a representative), so
    // that later sweeps never reallocate inside a timed region
    const size_t want = std::max((size_t)n1, (size_t)P->chunk_cap / 2) << la;
    const size_t per_rec = stride * 8 + 8 + 4 * 6 + 16;
    // (re)size only when this want was not tried before: once the pool is as
    // large as memory allows, later sweeps must not query the driver again
    // (cudaMemGetInfo measured 2..90 ms on the box, inside the timed region)
    if ((want > P->l2_cap && want > P->l2_sized_for) || (int)stride != P->l2_stride) {
        size_t fr = 0, tot = 0;
        P->l2_sized_for = want;
        CUDA_TRY(cudaMemGetInfo(&fr, &tot));
        fr += P->l2_cap * per_rec;
        size_t cap = std::max<size_t>(want, P->l2_cap);
        while (cap > ((size_t)1 << 16) && cap * per_rec > fr / 2) cap >>= 1;
        if (cap > P->l2_cap || (int)stride != P->l2_stride) {
            cudaFree(P->d_l2pool);
            cudaFree(P->d_l2hash);
            cudaFree(P->d_l2u32);
            P->d_l2pool = nullptr;
            P->d_l2hash = nullptr;
            P->d_l2u32 = nullptr;
            P->l2_cap = 0;
            CUDA_TRY(cudaMalloc(&P->d_l2pool, sizeof(unsigned long long) * stride * cap));
            CUDA_TRY(cudaMalloc(&P->d_l2hash, sizeof(unsigned long long) * cap));
            CUDA_TRY(cudaMalloc(&P->d_l2u32, sizeof(uint32_t) * (5 * cap + 1)));
            cudaFree(P->d_l2slots);
            P->d_l2slots = nullptr;
            CUDA_TRY(cudaMalloc(&P->d_l2slots, sizeof(unsigned long long) * 2 *
                                                   (size_t)next_pow2((uint32_t)cap)));
            P->l2_cap = cap;
            P->l2_stride = (int)stride;
        }
    }
    const size_t cap = P->l2_cap;
    // Batches of level-1 representatives.  The direct build writes 2^la records
    // per tile into the level-2 pool, so its batches hold cap >> la tiles; the
    // two-stage path writes 2^la1 stage-1 records per tile into its own pool
    // and only the distinct ones' 2^la2 records into the level-2 pool, so it
    // takes every representative of the chunk in one batch -- one stage-1
    // deduplication window (C3: 2 -> 1 batch per step).  A batch the two-stage
    // path declines runs the direct path in cap >> la sub-batches.
    const uint32_t nbdir = (uint32_t)(cap >> la);
    const bool ts = T.ts && l2_twostage_enabled();
    const uint32_t nbmax = ts ? n1 : nbdir;
    for (uint32_t i0 = 0; i0 < n1; i0 += nbmax) {
        const uint32_t nbb = std::min(nbmax, n1 - i0);
        if (ts) {
            int rc2 = 0;
            const bool done = run_two_stage(P, mode, tt, recs, list1, dup1, mint1, i0, nbb, tile0,
                                            lo, hi, cap, stride, rc2);
            if (rc2) return rc2;
            if (done) continue;
        }
        for (uint32_t j0 = i0; j0 < i0 + nbb; j0 += nbdir) {
            uint32_t nb = std::min(nbdir, i0 + nbb - j0);
            uint32_t jv = j0;
            uint32_t nrec = nb << la;
            static const uint64_t gmb = [] {  // CTAs per SM of the direct level-2 build
                const char *e = std::getenv("TCG_L2B_GRID");
                return e ? (uint64_t)std::max(1, std::atoi(e)) : (uint64_t)8;
            }();
            const unsigned g12 = (unsigned)std::min<uint64_t>((uint64_t)P->nsm * gmb,
                                                              (nrec + THREADS - 1) / THREADS);
            unsigned long long *pool = P->d_l2pool, *hashes = P->d_l2hash;
            uint32_t *wts = P->d_l2u32, *poss = wts + cap;
            uint32_t *oldlist = P->d_oldlist + 1, *oldcount = P->d_oldlist;
            uint64_t t0 = tile0, a = lo, b = hi;
            void *a1[] = {&tt, &recs, &list1, &dup1, &mint1, &jv, &nb, &t0, &a, &b, &pool,
                          (void *)&stride, &hashes, &wts, &poss, &oldlist, &oldcount};
            cudaEvent_t e0 = timing_begin(P);
            const size_t l2b_smem = (size_t)L2B_WORDS * 4 * THREADS +
                                    (size_t)(THREADS / 32) * (32 >> std::min(la, 5)) * L2B_SLOT;
            void *kb = T.l2even ? (void *)k_l2_build<true> : (void *)k_l2_build<false>;
            CUDA_TRY(cudaLaunchKernel(kb, dim3(g12), dim3(THREADS), a1, l2b_smem, P->stream));
            timing_end(P, TCG_KT_L2_BUILD, e0);
            P->launches++;
            const int rc = l2_tail(P, T, tt, nrec, stride, tile0);
            if (rc) return rc;
        }
    }
    return TCG_OK;
}

// Deduplicate nrec level-2 records (pool / hashes / wts / poss as built) and
// classify the distinct ones.
static int l2_tail(tcg_plan *P, const TileTables &T, const TileTables *tt, uint32_t nrec,
                   uint32_t stride, uint64_t tile0) {
    if (nrec == 0) return TCG_OK;
    const size_t cap = P->l2_cap;
    uint32_t *wts = P->d_l2u32, *poss = wts + cap, *w2 = poss + cap, *pos2 = w2 + cap,
             *list2 = pos2 + cap, *count2 = list2 + cap;
    unsigned long long *slots = P->d_l2slots, *pool = P->d_l2pool, *hashes = P->d_l2hash;
    const int wps = T.l2even ? 2 : 1;
    const uint32_t np2 = next_pow2(nrec);
    CUDA_TRY(cudaMemsetAsync(slots, 0xff, sizeof(unsigned long long) * 2 * (size_t)np2,
                             P->stream));
    CUDA_TRY(cudaMemsetAsync(w2, 0, sizeof(uint32_t) * nrec, P->stream));
    CUDA_TRY(cudaMemsetAsync(pos2, 0xff, sizeof(uint32_t) * nrec, P->stream));
    CUDA_TRY(cudaMemsetAsync(count2, 0, sizeof(uint32_t), P->stream));
    const unsigned g12 = (unsigned)std::min<uint64_t>((uint64_t)P->nsm * 8,
                                                      (nrec + THREADS - 1) / THREADS);
    uint32_t smask = 2 * np2 - 1;
    int wpsv = wps;
    uint32_t nr = nrec, sv = stride;
    void *a2[] = {&pool, &sv, &nr, &hashes, &wts, &poss, &slots, &smask, &w2,
                  &pos2, &list2, &count2, &wpsv};
    cudaEvent_t e0d = timing_begin(P);
    CUDA_TRY(cudaLaunchKernel((void *)k_l2_dedup, dim3(g12), dim3(THREADS), a2, 0, P->stream));
    timing_end(P, TCG_KT_L2_DEDUP, e0d);
    P->l2_built += nrec;
    const unsigned g3 = (unsigned)std::min<uint64_t>(P->blocks_l2cls,
                                                     (nrec + CLS_WARPS - 1) / CLS_WARPS);
    unsigned long long *ts = P->d_tstats + 1;
    uint64_t t0 = tile0;
    void *a3[] = {&P->kp, &tt, &pool, &sv, &list2, &count2, &w2, &pos2, &t0,
                  &P->agg, &ts};
    cudaEvent_t e = timing_begin(P);
    if (T.l2even)
        CUDA_TRY(cudaLaunchKernel((void *)k_l2_classify_even, dim3(g3), dim3(THREADS), a3,
                                  L2E_CLS_SMEM, P->stream));
    else
        CUDA_TRY(cudaLaunchKernel((void *)k_l2_classify, dim3(g3), dim3(THREADS), a3,
                                  L2_CLS_SMEM, P->stream));
    timing_end(P, TCG_KT_L2_CLASSIFY, e);
    P->launches += 2;
    return TCG_OK;
}

// TCG_NO_SUPER_DEDUP=1 builds and compares the tiles of twin super-tiles too
// (A/B and debugging); results are identical.
static bool super_dedup_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("TCG_NO_SUPER_DEDUP");
        return !(e && e[0] && e[0] != '0');
    }();
    return on;
}

// TCG_NO_DEDUP=1 classifies every tile (A/B and debugging); results are identical.
static bool dedup_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("TCG_NO_DEDUP");
        return !(e && e[0] && e[0] != '0');
    }();
    return on;
}

constexpr uint64_t SPLIT_MIN_DRAWS = 1ull << 22;

// TCG_NO_SPLIT=1 samples with the flat kernel only (A/B and debugging); results are identical.
static bool split_enabled(const tcg_plan *P) {
    if (P->split >= 0) return P->split != 0;
    static const bool on = [] {
        const char *e = std::getenv("TCG_NO_SPLIT");
        return !(e && e[0] && e[0] != '0');
    }();
    return on;
}

// Design the separator and build the two component tables (once per plan,
// at the first sample; d >= 6).  Leaves split_state = -1 (flat sampling)
// when no separator fits the limits in split.cuh.
static int ensure_split(tcg_plan *P) {
    if (P->split_state) return TCG_OK;
    P->split_state = -1;
    if (P->d < 6) return TCG_OK;
    tcg_desc D{};
    D.degree = P->d;
    D.nv = P->h_nv;
    D.npts = P->h_npts;
    D.ne = (int32_t)P->h_eu.size();
    D.edge_u = P->h_eu.data();
    D.edge_v = P->h_ev.data();
    D.src = P->h_src.data();
    D.par = P->h_par.data();
    D.used = P->h_used.data();
    D.nap = (int32_t)P->h_apu.size();
    D.ap_u = P->h_apu.data();
    D.ap_v = P->h_apv.data();
    D.maxreg = P->maxreg;
    Layout L;
    L.d = P->d;
    L.K = P->K;
    L.H = 16 * P->K;
    L.npts = P->h_npts;
    L.pos = P->h_pos;
    SplitDesign S;
    if (!split_design(&D, L, S)) return TCG_OK;
    const size_t na = (size_t)1 << S.pa.bits, nb = (size_t)1 << S.pb.bits;
    const size_t ew = S.sp.stride;
    {  // the tables are an accelerator: without the memory, sample on the flat kernel
        size_t fr = 0, tot = 0;
        const size_t need = (na + nb) * ew * 4 + S.pext.size() * 8 + (SPL_LAUNCH + 1) * 4 + 8;
        if (cudaMemGetInfo(&fr, &tot) != cudaSuccess || need > fr / 2) {
            cudaGetLastError();
            return TCG_OK;
        }
    }
    CUDA_TRY(cudaMalloc(&P->d_splitA, na * ew * 4));
    CUDA_TRY(cudaMalloc(&P->d_splitB, nb * ew * 4));
    CUDA_TRY(cudaMalloc(&P->d_pext, S.pext.size() * 8));
    CUDA_TRY(cudaMalloc(&P->d_fbl, (SPL_LAUNCH + 1) * 4));
    CUDA_TRY(cudaMalloc(&P->d_splitstats, 8));
    CUDA_TRY(cudaMemsetAsync(P->d_splitstats, 0, 8, P->stream));
    CUDA_TRY(cudaMemcpyAsync(P->d_pext, S.pext.data(), S.pext.size() * 8, cudaMemcpyHostToDevice,
                             P->stream));
    P->split_bytes = (na + nb) * ew * 4;
    void *fb = pick_split_build(P->K);
    const size_t bsm = adj_bytes(P->K) + 32 * P->K;  // + F index per layout position
    CUDA_TRY(cudaFuncSetAttribute(fb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
    int bps = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fb, THREADS, bsm));
    for (int t = 0; t < 2; ++t) {
        SplitPart part = t ? S.pb : S.pa;
        uint32_t *tab = t ? P->d_splitB : P->d_splitA;
        uint32_t n = (uint32_t)(t ? nb : na);
        const unsigned grid = (unsigned)std::min<uint64_t>((uint64_t)std::max(1, bps) * P->nsm,
                                                           (n + THREADS - 1) / THREADS);
        void *args[] = {&P->kp, &part, &tab, &n};
        cudaEvent_t e0 = timing_begin(P);
        CUDA_TRY(cudaLaunchKernel(fb, dim3(grid), dim3(THREADS), args, bsm, P->stream));
        timing_end(P, TCG_KT_SPLIT_BUILD, e0);
        P->launches++;
    }
    S.sp.tabA = P->d_splitA;
    S.sp.tabB = P->d_splitB;
    S.sp.pext = P->d_pext;
    P->split_sp = S.sp;
    void *fs = pick_split(P->even);
    CUDA_TRY(cudaFuncSetAttribute(fs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SPLIT_SMEM));
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fs, THREADS, SPLIT_SMEM));
    P->blocks_split = std::max(1, bps) * P->nsm;
    void *fl = pick_list(P->K, P->even);
    CUDA_TRY(cudaFuncSetAttribute(fl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smem_enum));
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fl, THREADS, P->smem_enum));
    P->blocks_list = std::max(1, bps) * P->nsm;
    CUDA_TRY(cudaGetLastError());
    P->split_state = 1;
    return TCG_OK;
}

// Sampling through the split tables: launches of <= SPL_LAUNCH draws, each
// followed by the flat classification of the draws it left.
static int enqueue_split(tcg_plan *P, uint64_t k0, uint64_t k1, uint64_t seed, uint64_t mask) {
    void *fs = pick_split(P->even);
    void *fl = pick_list(P->K, P->even);
    for (uint64_t a = k0; a < k1;) {
        uint64_t count = std::min<uint64_t>(k1 - a, SPL_LAUNCH), base = a;
        CUDA_TRY(cudaMemsetAsync(P->d_fbl, 0, 4, P->stream));
        const uint64_t need = ((count + 31) / 32 * 32 + THREADS - 1) / THREADS;
        const unsigned blocks = (unsigned)std::min<uint64_t>(P->blocks_split, std::max<uint64_t>(1, need));
        uint32_t *fbl = P->d_fbl;
        void *as[] = {&P->kp, &P->split_sp, &base, &count, &seed, &mask, &P->agg, &fbl};
        cudaEvent_t e0 = timing_begin(P);
        CUDA_TRY(cudaLaunchKernel(fs, dim3(blocks), dim3(THREADS), as, SPLIT_SMEM, P->stream));
        timing_end(P, TCG_KT_SAMPLE_SPLIT, e0);
        const uint32_t *cfbl = fbl;
        unsigned long long *st = P->d_splitstats;
        void *al[] = {&P->kp, &base, &seed, &mask, &P->agg, &cfbl, &st};
        cudaEvent_t e1 = timing_begin(P);
        CUDA_TRY(cudaLaunchKernel(fl, dim3(P->blocks_list), dim3(THREADS), al, P->smem_enum, P->stream));
        timing_end(P, TCG_KT_SAMPLE_LIST, e1);
        P->launches += 2;
        P->split_draws += (int64_t)count;
        a += count;
    }
    return TCG_OK;
}

static int enqueue(tcg_plan *P, int mode, uint64_t start, uint64_t end, uint64_t seed,
                   uint64_t mask) {
    if (P->pending_mode >= 0 && P->pending_mode != mode)
        return fail(TCG_E_ARG, "aggregate already holds another domain; call tcg_agg_reset");
    if (mode == MODE_SAMPLE && P->pending_mode == MODE_SAMPLE &&
        (P->pending_seed != seed || P->pending_mask != mask))
        return fail(TCG_E_ARG, "aggregate already holds another sample stream");
    P->pending_mode = mode;
    P->pending_seed = seed;
    P->pending_mask = mask;
    if (mode != MODE_SAMPLE && P->tiles_ok[mode] && end > start) {
        // chunks of chunk_tiles() tiles: contract, deduplicate, classify
        void *fb = pick_build(P->K, mode);
        void *fc = pick_cls(P->K, P->even, mode);
        const TileTables *tt = P->d_tiles + mode;
        const int bits = P->tile_bits[mode];
        const uint64_t t_end = ((end - 1) >> bits) + 1;
        // a chunk covers <= chunk_index_limit() indices and <= 2^25 tiles (tile ids and
        // level-2 positions fit 32 bits)
        uint32_t chunk = (uint32_t)std::min<uint64_t>(chunk_tiles(), chunk_index_limit() >> bits);
        chunk = std::min<uint32_t>(chunk, next_pow2((uint32_t)std::min<uint64_t>(
                                              t_end - (start >> bits), 1u << 30)));
        if (chunk > P->chunk_cap && chunk > P->chunk_sized_for) {  // (re)allocate records + dedup table
            P->chunk_sized_for = chunk;
            CUDA_TRY(cudaStreamSynchronize(P->stream));
            size_t fr = 0, tot = 0;
            CUDA_TRY(cudaMemGetInfo(&fr, &tot));
            if (P->d_recs) fr += sizeof(TileRec) * (size_t)P->chunk_cap;
            const size_t per_tile = sizeof(TileRec) + 6 * sizeof(uint32_t) + 5 * 8;
            while (chunk > (1u << 14) && (size_t)chunk * per_tile > fr / 4) chunk >>= 1;
            if (chunk > P->chunk_cap) {
                cudaFree(P->d_recs);
                cudaFree(P->d_dedup);
                P->d_recs = nullptr;
                P->d_dedup = nullptr;
                P->chunk_cap = 0;
                cudaFree(P->d_oldlist);
                P->d_oldlist = nullptr;
                cudaFree(P->d_ovf);
                P->d_ovf = nullptr;
                CUDA_TRY(cudaMalloc(&P->d_ovf, sizeof(uint32_t) * ((size_t)chunk + 1)));
                CUDA_TRY(cudaMalloc(&P->d_recs, sizeof(TileRec) * (size_t)chunk));
                CUDA_TRY(cudaMalloc(&P->d_oldlist, sizeof(uint32_t) * ((size_t)chunk + 1)));
                CUDA_TRY(cudaMalloc(&P->d_dedup, sizeof(uint32_t) * (3 * (size_t)chunk + 1)));
                cudaFree(P->d_hash);
                cudaFree(P->d_slots);
                P->d_hash = nullptr;
                P->d_slots = nullptr;
                CUDA_TRY(cudaMalloc(&P->d_hash, sizeof(unsigned long long) * (size_t)chunk));
                cudaFree(P->d_repof);
                P->d_repof = nullptr;
                CUDA_TRY(cudaMalloc(&P->d_repof, sizeof(uint32_t) * (size_t)chunk));
                CUDA_TRY(cudaMalloc(&P->d_slots,
                                    sizeof(unsigned long long) * 2 * (size_t)next_pow2(chunk)));
                P->chunk_cap = chunk;
            }
        }
        chunk = std::min(chunk, P->chunk_cap);
        if (!P->d_tstats) {
            CUDA_TRY(cudaMalloc(&P->d_tstats, 3 * sizeof(unsigned long long)));
            CUDA_TRY(cudaMemsetAsync(P->d_tstats, 0, 3 * sizeof(unsigned long long), P->stream));
        }
        for (uint64_t t0 = start >> bits; t0 < t_end; t0 += chunk) {
            uint32_t nt = (uint32_t)std::min<uint64_t>(chunk, t_end - t0);
            uint64_t tile0 = t0;
            TileRec *recs = P->d_recs;
            unsigned long long *hashes = P->d_hash;
            const unsigned gb = (unsigned)((nt + THREADS - 1) / THREADS);
            const uint32_t *nolist = nullptr, *nocount = nullptr;
            cudaEvent_t e0 = timing_begin(P);
            const int sh = P->h_tiles[mode].sh;
            const uint32_t *srep = nullptr;  // super-tile twins (sh > 0 with deduplication)
            if (sh > 0) {
                // super-tiles: contract the shared part once per 2^sh tiles, then
                // each tile from its super record; fallback super-tiles go to the
                // generic kernel
                const uint64_t s0 = tile0 >> sh;
                const uint32_t nsup = (uint32_t)(((tile0 + nt - 1) >> sh) - s0 + 1);
                if (nsup > P->super_cap) {
                    CUDA_TRY(cudaStreamSynchronize(P->stream));
                    cudaFree(P->d_super);
                    P->d_super = nullptr;
                    P->super_cap = 0;
                    const size_t cap = std::max<size_t>(nsup, (P->chunk_cap >> sh) + 2);
                    CUDA_TRY(cudaMalloc(&P->d_super, sizeof(SuperRec) * cap));
                    cudaFree(P->d_srep);
                    cudaFree(P->d_sslots);
                    P->d_srep = nullptr;
                    P->d_sslots = nullptr;
                    CUDA_TRY(cudaMalloc(&P->d_srep, sizeof(uint32_t) * cap));
                    CUDA_TRY(cudaMalloc(&P->d_sslots, sizeof(unsigned long long) * 2 *
                                                          (size_t)next_pow2((uint32_t)cap)));
                    P->super_cap = cap;
                }
                SuperRec *sr = P->d_super;
                uint64_t s0v = s0;
                uint32_t nsv = nsup;
                void *as[] = {&P->kp, &tt, &s0v, &nsv, &sr};
                CUDA_TRY(cudaLaunchKernel(pick_super(P->K, mode),
                                          dim3((nsup + THREADS - 1) / THREADS), dim3(THREADS), as,
                                          P->smem_build, P->stream));
                const SuperRec *csr = sr;
                srep = nullptr;
                if ((P->dedup < 0 ? dedup_enabled() : P->dedup != 0) && super_dedup_enabled()) {
                    // twin super-tiles: their tiles are neither built nor compared
                    const uint32_t np2s = next_pow2(nsup);
                    CUDA_TRY(cudaMemsetAsync(P->d_sslots, 0xff, sizeof(unsigned long long) * 2 * np2s,
                                             P->stream));
                    uint32_t smask_s = 2 * np2s - 1;
                    uint64_t lo_s = start, hi_s = end;
                    uint32_t *srp = P->d_srep;
                    unsigned long long *ssl = P->d_sslots;
                    void *asd[] = {&tt, &csr, &nsv, &tile0, &nt, &lo_s, &hi_s, &ssl, &smask_s, &srp};
                    CUDA_TRY(cudaLaunchKernel((void *)k_super_dedup, dim3((nsup + THREADS - 1) / THREADS),
                                              dim3(THREADS), asd, 0, P->stream));
                    srep = P->d_srep;
                    P->launches++;
                }
                timing_end(P, TCG_KT_SUPER_BUILD, e0);
                e0 = timing_begin(P);
                uint32_t *ovf = P->d_ovf;
                CUDA_TRY(cudaMemsetAsync(ovf, 0, sizeof(uint32_t), P->stream));
                void *af[] = {&tt, &csr, &tile0, &nt, &recs, &hashes, &ovf, &srep};
                CUDA_TRY(cudaLaunchKernel((void *)k_tile_from_super,
                                          dim3((nt + THREADS - 1) / THREADS), dim3(THREADS), af,
                                          from_super_smem(P->h_tiles[mode].nf), P->stream));
                const uint32_t *ol = ovf + 1, *oc = ovf;
                void *ab[] = {&P->kp, &tt, &tile0, &nt, &recs, &hashes, &ol, &oc};
                CUDA_TRY(cudaLaunchKernel(fb, dim3(P->blocks_bgen), dim3(THREADS), ab,
                                          P->smem_build, P->stream));
                P->launches += 2;
            } else {
                void *ab[] = {&P->kp, &tt, &tile0, &nt, &recs, &hashes, &nolist, &nocount};
                CUDA_TRY(cudaLaunchKernel(fb, dim3(gb), dim3(THREADS), ab, P->smem_build,
                                          P->stream));
            }
            timing_end(P, TCG_KT_TILE_BUILD, e0);
            uint64_t lo = start, hi = end;
            const TileRec *crecs = recs;
            const uint32_t *list = nullptr, *cnt = nullptr, *dup = nullptr, *mint = nullptr;
            if (P->dedup < 0 ? dedup_enabled() : P->dedup != 0) {
                const size_t C = P->chunk_cap, Cn = next_pow2(nt);  // Cn <= next_pow2(C)
                unsigned long long *slots = P->d_slots;
                uint32_t *mnt = P->d_dedup, *dp = mnt + C, *ct = dp + C, *ls = ct + 1;
                const unsigned long long *chash = hashes;
                CUDA_TRY(cudaMemsetAsync(slots, 0xff, sizeof(unsigned long long) * 2 * Cn, P->stream));
                CUDA_TRY(cudaMemsetAsync(mnt, 0xff, sizeof(uint32_t) * nt, P->stream));
                CUDA_TRY(cudaMemsetAsync(dp, 0, sizeof(uint32_t) * nt, P->stream));
                CUDA_TRY(cudaMemsetAsync(ct, 0, sizeof(uint32_t), P->stream));
                uint32_t smask = (uint32_t)(2 * Cn - 1);
                int ibits = bits;
                TileRec *wrecs = recs;  // twins of never-merged tiles get a copy of the record
                int shv = sh;
                uint32_t *repof = srep ? P->d_repof : nullptr;
                void *ad[] = {&wrecs, &chash, &nt, &tile0, &ibits, &lo, &hi, &slots, &smask, &dp,
                              &mnt, &ls, &ct, &srep, &shv, &repof};
                const unsigned gd = (unsigned)((nt + THREADS - 1) / THREADS);
                cudaEvent_t ed = timing_begin(P);
                CUDA_TRY(cudaLaunchKernel((void *)k_tile_dedup, dim3(gd), dim3(THREADS), ad, 0,
                                          P->stream));
                if (srep) {  // tiles of twin super-tiles join their twins' groups
                    const uint32_t *crep = repof;
                    void *ap[] = {&crecs, &nt, &tile0, &shv, &srep, &crep, &dp, &mnt};
                    CUDA_TRY(cudaLaunchKernel((void *)k_super_prop, dim3(gd), dim3(THREADS), ap, 0,
                                              P->stream));
                    P->launches++;
                }
                timing_end(P, TCG_KT_TILE_DEDUP, ed);
                list = ls;
                cnt = ct;
                dup = dp;
                mint = mnt;
                P->launches++;
            }
            unsigned long long *tstats = P->d_tstats;
            if (list && P->l2_ok[mode] && (P->l2 < 0 ? l2_enabled() : P->l2 != 0)) {
                // level 2: the level-1 representatives' (tile, A) records, deduplicated
                int rc = run_level2(P, mode, tt, crecs, list, cnt, dup, mint, tile0, lo, hi);
                if (rc) return rc;
                list = P->d_oldlist + 1;  // tiles left to the level-1 classifier
                cnt = P->d_oldlist;
                tstats = P->d_tstats + 2;  // tiles the level-1 classifier takes
            }
            const unsigned gc = (unsigned)std::min<uint64_t>(P->blocks_cls,
                                                             (nt + CLS_WARPS - 1) / CLS_WARPS);
            P->tiles_built += nt;
            void *ac[] = {&P->kp, &tt, &crecs, &tile0, &nt, &lo, &hi, &P->agg,
                          &list, &cnt, &dup, &mint, &tstats};
            cudaEvent_t e1 = timing_begin(P);
            CUDA_TRY(cudaLaunchKernel(fc, dim3(gc), dim3(THREADS), ac, P->smem_cls, P->stream));
            timing_end(P, TCG_KT_TILE_CLASSIFY, e1);
            P->launches += 2;
        }
        return TCG_OK;
    }
    // the split tables (0.1-2.5 GB, built once per plan) pay off for large
    // samples; smaller ones use the flat kernel unless the tables exist or
    // the caller asked for the split path (tcg_plan_set_split(plan, 1))
    if (mode == MODE_SAMPLE && end > start && split_enabled(P) &&
        (P->split == 1 || P->split_state == 1 || end - start >= SPLIT_MIN_DRAWS)) {
        int rc = ensure_split(P);
        if (rc) return rc;
        if (P->split_state > 0) return enqueue_split(P, start, end, seed, mask);
    }
    void *fn = pick_enum(P->K, P->even, mode);
    for (uint64_t a = start; a < end;) {
        const uint64_t n = std::min<uint64_t>(end - a, LAUNCH_MAX);
        const uint64_t warps = (n + 31) / 32;
        const uint64_t need = (warps * 32 + THREADS - 1) / THREADS;
        const unsigned blocks = (unsigned)std::min<uint64_t>(P->blocks_enum, std::max<uint64_t>(1, need));
        uint64_t base = a, count = n;
        void *args[] = {&P->kp, &base, &count, &seed, &mask, &P->agg};
        cudaEvent_t e2 = timing_begin(P);
        CUDA_TRY(cudaLaunchKernel(fn, dim3(blocks), dim3(THREADS), args, P->smem_enum, P->stream));
        timing_end(P, TCG_KT_ENUMERATE, e2);
        P->launches++;
        a += n;
    }
    return TCG_OK;
}

int tcg_sweep_async(tcg_plan *P, int raw, uint64_t start, uint64_t end) {
    if (!P) return fail(TCG_E_ARG, "null plan");
    const int bits = raw ? P->kp.npts : P->kp.npts - 3;
    if (bits > 62) return fail(TCG_E_RANGE, "domain exceeds 62 index bits");
    const uint64_t domain = 1ull << bits;
    if (start > end || end > domain) return fail(TCG_E_RANGE, "sweep range outside the domain");
    DeviceGuard guard(P->device);
    return enqueue(P, raw ? MODE_RAW : MODE_REP, start, end, 0, 0);
}

int tcg_sample_async(tcg_plan *P, uint64_t seed, uint64_t k0, uint64_t k1, int nbits) {
    if (!P) return fail(TCG_E_ARG, "null plan");
    if (nbits < 0 || nbits > P->kp.npts - 3 || nbits > 62)
        return fail(TCG_E_RANGE, "nbits outside the representative domain");
    if (k0 > k1) return fail(TCG_E_RANGE, "bad draw range");
    DeviceGuard guard(P->device);
    const uint64_t mask = nbits >= 64 ? ~0ull : ((1ull << nbits) - 1ull);
    return enqueue(P, MODE_SAMPLE, k0, k1, seed, mask);
}

static uint64_t host_splitmix(uint64_t seed, uint64_t k) {
    uint64_t z = seed + (k + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static uint64_t host_rep_to_sigma(int d, uint64_t m) {
    const uint64_t low = m & ((1ull << (d - 1)) - 1ull);
    return (low << 2) | ((m >> (d - 1)) << (d + 2));
}

// What one plan's aggregate says about failures, before the table rule.
struct FetchOut {
    int cls_status = 0;        // smallest-index classification failure (0: none)
    int64_t cls_bad = -1;      // its index in the run's domain (m)
    uint64_t cls_order = 0;    // its position in enumeration order (sweep: m, sample: draw k)
    bool overflow = false;     // the device table dropped a key (> GCAP distinct)
    bool index_ordered = true; // witnesses are in enumeration order (sweeps; not samples)
};

// Reference _aggregate (kernels.py:389-391) refuses a NEW scheme once its table
// holds cap/2 = 32,768 (ameta[2]*2 >= cap with cap = 65,536) and the kernel
// stops at that index.  One sequential worker (workers=1) meets the schemes in
// index order, so the failing index is the 32,769th smallest witness.
constexpr int32_t REF_TABLE_LIMIT = 1 << 15;

static int64_t table_full_index(const tcg_agg *A) {
    std::vector<int64_t> w(A->witness, A->witness + A->n);
    std::nth_element(w.begin(), w.begin() + REF_TABLE_LIMIT, w.end());
    return w[REF_TABLE_LIMIT];
}

// Status and index a sweep_kernel / sample_kernel run would return.
static int settle(const tcg_agg *A, const FetchOut &F, int64_t *bad) {
    if (bad) *bad = -1;
    const bool full = F.overflow || A->n > REF_TABLE_LIMIT;
    const int64_t tbad = (full && A->n > REF_TABLE_LIMIT) ? table_full_index(A) : -1;
    if (F.cls_status) {
        // both fire: the earlier index wins (sweeps); samples report the
        // classification failure (first-draw positions of schemes are not kept)
        if (full && F.index_ordered && tbad >= 0 && tbad < F.cls_bad) {
            if (bad) *bad = tbad;
            return fail(TCG_TABLE_FULL, "scheme table full (32,768 distinct schemes)");
        }
        if (bad) *bad = F.cls_bad;
        return F.cls_status;
    }
    if (full) {
        if (bad) *bad = tbad;
        return fail(TCG_TABLE_FULL, "scheme table full (32,768 distinct schemes)");
    }
    return TCG_OK;
}

// Copy the device aggregate into A (sorted by key) and find the smallest
// failing index; library errors (< 0) only.
static int fetch_raw(tcg_plan *P, tcg_agg *A, FetchOut &F) {
    DeviceGuard guard(P->device);
    host_mark("fetch");
    CUDA_TRY(cudaMemsetAsync(P->d_cn, 0, 4, P->stream));
    k_agg_compact<<<64, 256, 0, P->stream>>>(P->agg, P->d_ckey, P->d_ccnt, P->d_cwit, P->d_cn);
    CUDA_TRY(cudaGetLastError());
    P->launches++;
    unsigned int n = 0, overflow = 0;
    unsigned long long hist[NHIST], badidx = 0;
    CUDA_TRY(cudaMemcpyAsync(&n, P->d_cn, 4, cudaMemcpyDeviceToHost, P->stream));
    CUDA_TRY(cudaMemcpyAsync(&overflow, P->agg.overflow, 4, cudaMemcpyDeviceToHost, P->stream));
    CUDA_TRY(cudaMemcpyAsync(hist, P->agg.hist, sizeof(hist), cudaMemcpyDeviceToHost, P->stream));
    CUDA_TRY(cudaMemcpyAsync(&badidx, P->agg.bad, 8, cudaMemcpyDeviceToHost, P->stream));
    CUDA_TRY(cudaStreamSynchronize(P->stream));
    host_mark("fetch synced");
    F = FetchOut{};
    F.overflow = overflow != 0;
    F.index_ordered = P->pending_mode != MODE_SAMPLE;
    if (badidx != ~0ull) {
        // recompute the failing patchwork's status (smallest failing index)
        uint64_t m = badidx, sigma;
        if (P->pending_mode == MODE_SAMPLE) {
            m = host_splitmix(P->pending_seed, badidx) & P->pending_mask;
            sigma = host_rep_to_sigma(P->d, m);
        } else if (P->pending_mode == MODE_REP) {
            sigma = host_rep_to_sigma(P->d, m);
        } else {
            sigma = m;
        }
        uint64_t key;
        uint8_t ov, nr;
        int32_t st = 0;
        int rc = tcg_classify_batch(P, &sigma, 1, &key, &ov, &nr, &st);
        if (rc) return rc;
        if (!st) return fail(TCG_E_CUDA, "device reported a failure the replay did not reproduce");
        F.cls_status = st;
        F.cls_bad = (int64_t)m;
        F.cls_order = badidx;
    }
    if ((int32_t)n > A->cap) return fail(TCG_E_RANGE, "caller's aggregate capacity too small");
    std::vector<unsigned long long> k(n), c(n), w(n);
    if (n) {
        CUDA_TRY(cudaMemcpy(k.data(), P->d_ckey, n * 8ull, cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemcpy(c.data(), P->d_ccnt, n * 8ull, cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemcpy(w.data(), P->d_cwit, n * 8ull, cudaMemcpyDeviceToHost));
    }
    std::vector<unsigned> ord(n);
    for (unsigned i = 0; i < n; ++i) ord[i] = i;
    std::sort(ord.begin(), ord.end(), [&](unsigned a, unsigned b) { return k[a] < k[b]; });
    int64_t total = 0;
    for (int i = 0; i < NHIST; ++i) {
        A->hist[i] = (int64_t)hist[i];
        total += (int64_t)hist[i];
    }
    A->total = total;
    A->n = (int32_t)n;
    for (unsigned i = 0; i < n; ++i) {
        A->key[i] = k[ord[i]];
        A->count[i] = (int64_t)c[ord[i]];
        A->witness[i] = (int64_t)w[ord[i]];
    }
    return TCG_OK;
}

int tcg_agg_fetch(tcg_plan *P, tcg_agg *A, int64_t *bad) {
    if (!P || !A) return fail(TCG_E_ARG, "null argument");
    FetchOut F;
    int rc = fetch_raw(P, A, F);
    if (rc) return rc;
    return settle(A, F, bad);
}

int tcg_sweep(tcg_plan *P, int raw, uint64_t start, uint64_t end, tcg_agg *A, int64_t *bad) {
    int rc = tcg_agg_reset(P);
    if (rc) return rc;
    rc = tcg_sweep_async(P, raw, start, end);
    if (rc) return rc;
    return tcg_agg_fetch(P, A, bad);
}

int tcg_sample(tcg_plan *P, uint64_t seed, uint64_t k0, uint64_t k1, int nbits, tcg_agg *A,
               int64_t *bad) {
    int rc = tcg_agg_reset(P);
    if (rc) return rc;
    rc = tcg_sample_async(P, seed, k0, k1, nbits);
    if (rc) return rc;
    return tcg_agg_fetch(P, A, bad);
}

// Merge per-device aggregates (count sum, witness min: sweep.py:168-180), then
// apply the failure rules once to the whole range, so the outcome does not
// depend on the number of devices: the classification failure earliest in
// enumeration order (sweep index or draw k) wins, the table rule applies to
// the merged scheme set.
static int merge_multi(std::vector<tcg_agg> &parts, std::vector<int> &rcs,
                       std::vector<FetchOut> &fo, tcg_agg *A, int64_t *bad) {
    for (size_t i = 0; i < parts.size(); ++i)
        if (rcs[i] < 0) return rcs[i];
    FetchOut F;
    for (auto &f : fo) {
        F.overflow |= f.overflow;
        F.index_ordered &= f.index_ordered;
        if (f.cls_status && (!F.cls_status || f.cls_order < F.cls_order)) {
            F.cls_status = f.cls_status;
            F.cls_bad = f.cls_bad;
            F.cls_order = f.cls_order;
        }
    }
    std::unordered_map<uint64_t, std::pair<int64_t, int64_t>> m;
    std::memset(A->hist, 0, sizeof(A->hist));
    A->total = 0;
    for (auto &p : parts) {
        for (int i = 0; i < NHIST; ++i) A->hist[i] += p.hist[i];
        A->total += p.total;
        for (int i = 0; i < p.n; ++i) {
            auto it = m.find(p.key[i]);
            if (it == m.end()) m.emplace(p.key[i], std::make_pair(p.count[i], p.witness[i]));
            else {
                it->second.first += p.count[i];
                it->second.second = std::min(it->second.second, p.witness[i]);
            }
        }
    }
    if ((int64_t)m.size() > A->cap) return fail(TCG_E_RANGE, "aggregate capacity too small");
    std::vector<uint64_t> keys;
    keys.reserve(m.size());
    for (auto &kv : m) keys.push_back(kv.first);
    std::sort(keys.begin(), keys.end());
    A->n = (int32_t)keys.size();
    for (size_t i = 0; i < keys.size(); ++i) {
        A->key[i] = keys[i];
        A->count[i] = m[keys[i]].first;
        A->witness[i] = m[keys[i]].second;
    }
    return settle(A, F, bad);
}

static int run_multi(tcg_plan **plans, int nplans, uint64_t a, uint64_t b, tcg_agg *A,
                     int64_t *bad, const std::function<int(tcg_plan *, uint64_t, uint64_t)> &fn) {
    if (!plans || nplans < 1 || !A) return fail(TCG_E_ARG, "bad arguments");
    for (int i = 0; i < nplans; ++i) {
        if (!plans[i]) return fail(TCG_E_ARG, "null plan");
        for (int j = 0; j < i; ++j)  // one host thread per plan: a plan may appear once
            if (plans[j] == plans[i]) return fail(TCG_E_ARG, "plan listed twice");
    }
    std::vector<tcg_agg> parts(nplans);
    std::vector<std::vector<uint64_t>> keys(nplans);
    std::vector<std::vector<int64_t>> cnts(nplans), wits(nplans);
    std::vector<int> rcs(nplans, 0);
    std::vector<FetchOut> fo(nplans);
    std::vector<std::thread> th;
    const uint64_t n = b - a;
    for (int i = 0; i < nplans; ++i) {
        keys[i].resize(GCAP);
        cnts[i].resize(GCAP);
        wits[i].resize(GCAP);
        parts[i] = tcg_agg{};
        parts[i].cap = GCAP;
        parts[i].key = keys[i].data();
        parts[i].count = cnts[i].data();
        parts[i].witness = wits[i].data();
        const uint64_t lo = a + (uint64_t)((unsigned __int128)n * i / nplans);
        const uint64_t hi = a + (uint64_t)((unsigned __int128)n * (i + 1) / nplans);
        th.emplace_back([&, i, lo, hi] {
            int rc = tcg_agg_reset(plans[i]);
            if (!rc) rc = fn(plans[i], lo, hi);
            if (!rc) rc = fetch_raw(plans[i], &parts[i], fo[i]);
            rcs[i] = rc;
        });
    }
    for (auto &t : th) t.join();
    return merge_multi(parts, rcs, fo, A, bad);
}

int tcg_sweep_multi(tcg_plan **plans, int nplans, int raw, uint64_t start, uint64_t end,
                    tcg_agg *A, int64_t *bad) {
    if (start > end) return fail(TCG_E_RANGE, "bad range");
    return run_multi(plans, nplans, start, end, A, bad,
                     [raw](tcg_plan *p, uint64_t lo, uint64_t hi) {
                         return tcg_sweep_async(p, raw, lo, hi);
                     });
}

int tcg_sample_multi(tcg_plan **plans, int nplans, uint64_t seed, uint64_t k0, uint64_t k1,
                     int nbits, tcg_agg *A, int64_t *bad) {
    if (k0 > k1) return fail(TCG_E_RANGE, "bad range");
    return run_multi(plans, nplans, k0, k1, A, bad,
                     [seed, nbits](tcg_plan *p, uint64_t lo, uint64_t hi) {
                         return tcg_sample_async(p, seed, lo, hi, nbits);
                     });
}


#include "api_multi.cuh"

#include "api_large.cuh"

}  // extern "C"
