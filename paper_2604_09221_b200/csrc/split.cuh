// split.cuh -- separator-split sampling (config C5: random sign draws).
// Included by tcg.cu inside its anonymous namespace (after the region pass,
// finish(), the scheme tables and the host layout helpers).
//
// A random draw shares no sign pattern with its neighbours in draw order, so
// the sweeps' tile contraction (amortised over 2^12 consecutive indices)
// does not apply.  Instead the lattice points are split once per
// triangulation by a small vertex separator F of T's edge graph into two
// parts A and B with no edge of T between them.  The same-sign components of
// A's diamond vertices then depend only on the signs of A's points (likewise
// for B), so they are tabulated once, in HBM:
//   table A: one entry per sign pattern of A's free points (2^bitsA entries),
//   table B: likewise (2^bitsB);
// an entry lists the part's components with their sign, their adjacency to
// the other components of the part and to the F vertices, and their
// antipodal links.  A draw is then classified on the contracted graph
//   nodes = F vertices (one node each) + A components + B components
// (<= 64 nodes, one u64 per node set) by the layer-free region pass of the
// tiles (node_pass), reading node rows straight from the draw's two entries.
// Antipodal links only join copies of one lattice point, so they never cross
// parts.  Draws whose graph does not fit, or whose contracted classification
// is not OK, go to a list that the flat kernel classifies exactly (status
// precedence, failing draw), so the aggregate is the reference's
// sample_kernel aggregate (kernels.py:447-462) bit for bit.

constexpr int SPL_MAXF = 32;     // separator vertices (graph nodes 0 .. nF-1)
constexpr int SPL_CAPC = 32;     // components per part entry
constexpr int SPL_MAXBITS = 24;  // free points per part (2^bits entries)
constexpr int SPL_MAXFB = 12;    // free separator points (two 6-bit sign tables)
constexpr int SPL_NBYTES = 8;    // sign-word bytes of the index extraction tables
constexpr uint64_t SPL_LAUNCH = 1ull << 26;  // draws per launch (= fallback list capacity)

// Kernel parameters of the sampler (staged into shared memory where indexed).
struct SplitParams {
    int nF, nFp, nbytes, maxnodes, prefetch;
    uint32_t stride;                    // u32 words per table entry
    const uint32_t *tabA, *tabB;
    // index extraction: byte j of sigma -> A index | B index << 24 | F bits << 48
    const unsigned long long *pext;     // [nbytes][256]
    uint32_t fadj[SPL_MAXF], flink[SPL_MAXF];  // F-F adjacency / antipodal links
    uint32_t fsign[2][64];              // F-vertex signs from the F bits (parity in [0])
};

// One table's build parameters.
struct SplitPart {
    int bits, npv, nF, nFp;
    uint32_t stride;
    uint32_t pm[MAXK];                    // the part's vertices (layout mask)
    uint8_t pt[SPL_MAXBITS];              // index bit i -> lattice point
    uint32_t fword[SPL_MAXF], fbit[SPL_MAXF];  // F vertices (layout word / bit)
};

// Entry layout (u32 words): [0] components (0xffff: more than SPL_CAPC),
// [1] component signs, [4 + f] components adjacent to F vertex f (f < nF),
// [4 + nFp + 4c] component c: {F vertices adjacent, components adjacent,
// components linked antipodally (self bit: a pair inside c), 0}.
__host__ __device__ constexpr uint32_t split_stride(int nFp) { return 4u + nFp + 4u * SPL_CAPC; }

template <int K>
__global__ void __launch_bounds__(THREADS) k_split_build(KParams p, SplitPart sp,
                                                         uint32_t *__restrict__ tab, uint32_t n) {
    extern __shared__ __align__(16) uint32_t smem[];
    int8_t *fidx = reinterpret_cast<int8_t *>(smem + 32 * K * K);  // layout position -> F vertex
    stage_adj<K>(p, smem);
    for (int i = threadIdx.x; i < 32 * K; i += blockDim.x) fidx[i] = -1;
    __syncthreads();
    for (int f = threadIdx.x; f < sp.nF; f += blockDim.x)
        fidx[32 * sp.fword[f] + __ffs(sp.fbit[f]) - 1] = (int8_t)f;
    __syncthreads();
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
        uint64_t sigma = 0;
        for (int i = 0; i < sp.bits; ++i) sigma |= (uint64_t)((x >> i) & 1u) << sp.pt[i];
        uint32_t SG[K], pm[K], zero[K];
        sign_words<K>(p, sigma, SG);
#pragma unroll
        for (int k = 0; k < K; ++k) {
            pm[k] = sp.pm[k];
            zero[k] = 0u;
        }
        Regions<K, SPL_CAPC> comps;
        region_pass<K, false, false, true, SPL_CAPC>(smem, SG, pm, zero, sp.npv, comps);
        uint32_t *e = tab + (size_t)x * sp.stride;
        const int nc = comps.nreg;
        if (nc > SPL_CAPC) {
            e[0] = 0xffffu;
            continue;
        }
        // component label of every part vertex, then each component's
        // neighbourhoods are read through the labels (O(|X|), not O(nc^2))
        uint8_t lab[32 * K];
        uint32_t sgn = 0;
        TCG_ASSERT(sp.nF <= SPL_MAXF && sp.bits <= SPL_MAXBITS);
        for (int c = 0; c < nc; ++c) {
            uint32_t s = 0;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const uint32_t r = comps.R[c][k];
                s |= r & SG[k];
                for (uint32_t w = r; w; w &= w - 1u) lab[32 * k + __ffs(w) - 1] = (uint8_t)c;
            }
            if (s) sgn |= 1u << c;
        }
        uint32_t fm[SPL_MAXF];
        for (int f = 0; f < SPL_MAXF; ++f) fm[f] = 0u;
        for (int c = 0; c < nc; ++c) {
            uint32_t adjP = 0, linkP = 0, adjF = 0;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const uint32_t xk = comps.X[c][k];
                const int ks = (k + K / 2) % K;  // antipodal partners: swap of halves
                const uint32_t pk = comps.R[c][ks] & p.bd[ks];
                for (uint32_t w = xk & pm[k]; w; w &= w - 1u) adjP |= 1u << lab[32 * k + __ffs(w) - 1];
                for (uint32_t w = pk & pm[k]; w; w &= w - 1u) linkP |= 1u << lab[32 * k + __ffs(w) - 1];
                for (uint32_t w = xk & ~pm[k]; w; w &= w - 1u) {
                    const int f = fidx[32 * k + __ffs(w) - 1];
                    if (f >= 0) {
                        adjF |= 1u << f;
                        fm[f] |= 1u << c;
                    }
                }
            }
            adjP &= ~(1u << c);
            reinterpret_cast<uint4 *>(e + 4 + sp.nFp)[c] = make_uint4(adjF, adjP, linkP, 0u);
        }
        e[0] = (uint32_t)nc;
        e[1] = sgn;
        for (int f = 0; f < sp.nF; ++f) e[4 + f] = fm[f];
    }
}

// The region graph of one draw, built while the regions close.
struct RegionGraph {
    uint32_t radj[MAXR];  // region adjacency (crossed edges), symmetric
    uint32_t selfm;       // regions with a crossed edge inside
    uint32_t oddmask;     // regions closing an orientation-reversing cycle (even degree)
    int nreg, nedges;
};

// Layer-free region pass over the contracted graph of one draw (node_pass
// with rows assembled from the two entries; one u64 per node set).  No
// per-region node sets are kept: every closed node carries its region id in
// five bit-planes (registers), and a closing region r finds the earlier
// regions it borders from the labels of its crossed neighbours that are
// already closed.  Each adjacent pair is met exactly once (at the later
// region's close), so the region graph, its edge count and the status inputs
// are complete when the pass ends.
template <bool EVEN, int V>
__device__ __forceinline__ void split_pass(const uint32_t *__restrict__ fadj_s,
                                           const uint32_t *__restrict__ flink_s,
                                           const uint32_t *__restrict__ ea,
                                           const uint32_t *__restrict__ eb, int nF, int nFp,
                                           int sB, int nn, unsigned long long sg,
                                           RegionGraph &out) {
    typedef unsigned long long u64;
    u64 un = nn >= 64 ? ~0ull : ((1ull << nn) - 1ull), f = 0, x = 0, q = 0, r = 0;
    u64 lab0 = 0, lab1 = 0, lab2 = 0, lab3 = 0, lab4 = 0, closed = 0;
    bool odd = false;
    int nreg = 0, nedges = 0;
    uint32_t oddmask = 0, selfm = 0;
    auto seed = [&]() {
        f = un & (0ull - un);
        r = un;
        un ^= f;
        x = 0ull;
        if (EVEN) q = 0ull;
        odd = false;
    };
    // V = 1: a closing region only records its crossed neighbours among the
    // closed nodes; the label lookups run after the pass (out of the divergent
    // close branch)
    constexpr int NSTEP = V >= 3 ? 4 : (V == 2 ? 3 : 2);  // frontier nodes per step
    u64 xs[V ? MAXR : 1];
    auto adjacency = [&](int rr, u64 w) {
        TCG_ASSERT(rr >= 0 && rr < MAXR);
        uint32_t A = 0;
        while (w) {
            const int n = __ffsll((long long)w) - 1;
            const int l = (int)((lab0 >> n) & 1ull) | (int)((lab1 >> n) & 1ull) << 1 |
                          (int)((lab2 >> n) & 1ull) << 2 | (int)((lab3 >> n) & 1ull) << 3 |
                          (int)((lab4 >> n) & 1ull) << 4;
            A |= 1u << l;
            const u64 m = (l & 1 ? lab0 : ~lab0) & (l & 2 ? lab1 : ~lab1) & (l & 4 ? lab2 : ~lab2) &
                          (l & 8 ? lab3 : ~lab3) & (l & 16 ? lab4 : ~lab4);
            w &= ~m;
        }
        out.radj[rr] = A;
        nedges += __popc(A);
        for (uint32_t a = A; a; a &= a - 1u) out.radj[__ffs(a) - 1] |= 1u << rr;
    };
    auto close = [&]() {
        if (nreg < MAXR) {
            const u64 rs = r ^ un;
            if (x & rs) selfm |= 1u << nreg;
            if (EVEN && odd) oddmask |= 1u << nreg;
            if (V) {
                xs[nreg] = x & closed;
            } else {
                adjacency(nreg, x & closed);
            }
            closed |= rs;
            if (nreg & 1) lab0 |= rs;
            if (nreg & 2) lab1 |= rs;
            if (nreg & 4) lab2 |= rs;
            if (nreg & 8) lab3 |= rs;
            if (nreg & 16) lab4 |= rs;
        }
        ++nreg;
    };
    const uint4 *ca = reinterpret_cast<const uint4 *>(ea + 4 + nFp);
    const uint4 *cb = reinterpret_cast<const uint4 *>(eb + 4 + nFp);
    const uint4 *fa = reinterpret_cast<const uint4 *>(ea + 4);
    const uint4 *fb = reinterpret_cast<const uint4 *>(eb + 4);
    // node row: F nodes take word v & 3 of two uint4s (the A and B entries'
    // masks), components one uint4 of their entry; the loads are issued
    // without branches so two nodes' loads are in flight together
    auto load = [&](int v, uint4 &t1, uint4 &t2) {
        TCG_ASSERT(v >= 0 && v < nn && nn <= 64);
        const bool isF = v < nF, inA = v < sB;
        TCG_ASSERT(isF || (inA ? v - nF : v - sB) < SPL_CAPC);
        const uint4 *pc = inA ? ca + (v - nF) : cb + (v - sB);
        t1 = __ldg(isF ? fa + (v >> 2) : pc);
        t2 = isF ? __ldg(fb + (v >> 2)) : make_uint4(0u, 0u, 0u, 0u);
    };
    auto expand = [&](int v, const uint4 &t1, const uint4 &t2) {
        u64 adj, link;
        if (v < nF) {
            const uint32_t wa = (v & 2) ? ((v & 1) ? t1.w : t1.z) : ((v & 1) ? t1.y : t1.x);
            const uint32_t wb = (v & 2) ? ((v & 1) ? t2.w : t2.z) : ((v & 1) ? t2.y : t2.x);
            adj = (u64)fadj_s[v] | ((u64)wa << nF) | ((u64)wb << sB);
            link = flink_s[v];
        } else {
            const int sh = v < sB ? nF : sB;
            adj = (u64)t1.x | ((u64)t1.y << sh);
            link = (u64)t1.z << sh;
        }
        const u64 sv = 0ull - ((sg >> v) & 1ull);
        const u64 o = sg ^ sv;  // nodes of the other sign
        x |= adj & o;
        if (EVEN) {
            // orientation parity per node: edges keep it, links flip it
            const u64 pv = 0ull - ((q >> v) & 1ull);
            const u64 te = adj & ~o, nt = te & un, np = link & un;
            const u64 eq = ~(q ^ pv);
            odd |= ((nt & np) | (te & ~un & ~eq) | (link & ~un & eq)) != 0ull;
            q |= (nt & pv) | (np & ~pv);
            const u64 n = nt | np;
            un ^= n;
            f |= n;
        } else {
            const u64 n = ((adj & ~o) | link) & un;
            un ^= n;
            f |= n;
        }
    };
    seed();
    while (true) {
        if (f == 0ull) {
            close();
            if (un == 0ull) break;
            seed();
        }
        // NSTEP frontier nodes per step: their row loads are issued together,
        // the expansions then run in order (the result is the sequential
        // pass's: a region's node set, crossed neighbourhood and parity verdict
        // do not depend on the visit order); missing nodes repeat v[0]
        int vs[NSTEP];
        uint4 t1[NSTEP], t2[NSTEP];
#pragma unroll
        for (int i = 0; i < NSTEP; ++i) {
            vs[i] = f ? __ffsll((long long)f) - 1 : vs[0];
            f &= f - 1ull;
        }
#pragma unroll
        for (int i = 0; i < NSTEP; ++i) load(vs[i], t1[i], t2[i]);
        expand(vs[0], t1[0], t2[0]);
#pragma unroll
        for (int i = 1; i < NSTEP; ++i)
            if (vs[i] != vs[0]) expand(vs[i], t1[i], t2[i]);
    }
    if (V)
        for (int rr = 0; rr < nreg && rr < MAXR; ++rr) adjacency(rr, xs[rr]);
    out.nreg = nreg;
    out.nedges = nedges;
    out.selfm = selfm;
    out.oddmask = oddmask;
}

// Status and key from the region graph, with finish()'s OK conditions
// (kernels.py:182-266): at most maxreg regions, a tree (nreg - 1 distinct
// region pairs, connected), and a root -- the one odd region with no crossed
// edge inside any region (even degree), or the one region with a crossed edge
// inside (odd degree).  Any other outcome is reported as NOT_A_TREE and the
// caller re-classifies the draw with the flat kernel (exact status).
template <bool EVEN>
__device__ __forceinline__ Result finish_graph(const RegionGraph &g, int maxreg) {
    Result res;
    res.nreg = g.nreg;
    res.key = 0ull;
    res.status = TCG_NOT_A_TREE;
    const int nreg = g.nreg;
    if (nreg > maxreg || nreg > MAXR || g.nedges != nreg - 1) return res;
    int root;
    if (EVEN) {
        if (__popc(g.oddmask) != 1 || g.selfm) return res;
        root = __ffs(g.oddmask) - 1;
    } else {
        if (__popc(g.selfm) != 1) return res;
        root = __ffs(g.selfm) - 1;
    }
    if (__popc(g.radj[root]) == nreg - 1) {  // the star at the root: root + nreg-1 leaves
        const int nb2 = 2 * (nreg - 1);
        res.status = TCG_OK;
        res.key = (1ull << nb2) | (0xAAAAAAAAAAAAAAAAull & ((1ull << nb2) - 1ull));
        return res;
    }
    if (nreg == 3) {  // two distinct pairs on three regions: the chain root - a - b
        res.status = TCG_OK;
        res.key = 28ull;
        return res;
    }
    uint64_t key;
    if (graph_key(g.radj, nreg, root, key)) {
        res.status = TCG_OK;
        res.key = key;
    }
    return res;
}

constexpr size_t SPLIT_SMEM_HEAD = (2 * SPL_MAXF + 128) * 4;
constexpr size_t SPLIT_SMEM = SPLIT_SMEM_HEAD + TABLE_SMEM;

// Sampler: draw k -> m = splitmix64(seed, k) & mask (kernels.py:447-462) ->
// sign word -> (A pattern, B pattern, F bits) by byte tables -> contracted
// classification.  fbl[0] counts the draws left to k_sample_list, fbl[1..]
// their offsets from `base`.
template <bool EVEN, int V>
__global__ void __launch_bounds__(THREADS, 3) k_sample_split(KParams p, SplitParams sp, uint64_t base,
                                                          uint64_t count, uint64_t seed,
                                                          uint64_t nbmask, DevAgg g,
                                                          uint32_t *__restrict__ fbl) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const unsigned long long *__restrict__ pext = sp.pext;  // 12-14 KB, L1-resident
    uint32_t *fadj_s = reinterpret_cast<uint32_t *>(smem_raw);
    uint32_t *flink_s = fadj_s + SPL_MAXF;
    uint32_t *fsign_s = flink_s + SPL_MAXF;
    CtaTable tab = carve_table(smem_raw + SPLIT_SMEM_HEAD);
    for (int i = threadIdx.x; i < SPL_MAXF; i += blockDim.x) {
        fadj_s[i] = sp.fadj[i];
        flink_s[i] = sp.flink[i];
    }
    for (int i = threadIdx.x; i < 128; i += blockDim.x) fsign_s[i] = sp.fsign[i >> 6][i & 63];
    tab.init();
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t wstride = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const int nF = sp.nF;
    for (uint64_t wb = warp * 32ull; wb < count; wb += wstride * 32ull) {
        const uint64_t idx = wb + lane;
        const bool valid = idx < count;
        const uint64_t gidx = base + idx;
        const uint64_t m = splitmix64(seed, gidx) & nbmask;
        const uint64_t sigma = rep_to_sigma(p.d, m);
        unsigned long long ix = 0;
#pragma unroll
        for (int j = 0; j < SPL_NBYTES; ++j)
            if (j < sp.nbytes) ix |= __ldg(pext + j * 256 + ((sigma >> (8 * j)) & 255u));
        TCG_ASSERT((ix & 0xffffffull) < (1ull << 24) && ((ix >> 24) & 0xffffffull) < (1ull << 24));
        const uint32_t *ea = sp.tabA + (size_t)(ix & 0xffffffull) * sp.stride;
        const uint32_t *eb = sp.tabB + (size_t)((ix >> 24) & 0xffffffull) * sp.stride;
        const uint32_t fb = (uint32_t)(ix >> 48);
        if (sp.prefetch && valid) {
            // both entries' lines into L2 at once; the region pass then reads
            // them at L2 latency instead of one HBM round trip per node row
            const char *a0 = reinterpret_cast<const char *>(ea), *b0 = reinterpret_cast<const char *>(eb);
#pragma unroll
            for (int l = 0; l < 6; ++l) {
                if (128 * l < sp.prefetch) {
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(a0 + 128 * l));
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(b0 + 128 * l));
                }
            }
        }
        const uint4 ha = __ldg(reinterpret_cast<const uint4 *>(ea));
        const uint4 hb = __ldg(reinterpret_cast<const uint4 *>(eb));
        const int sB = nF + (int)ha.x, nn = sB + (int)hb.x;
        const bool fits = valid && ha.x <= (uint32_t)SPL_CAPC && hb.x <= (uint32_t)SPL_CAPC &&
                          nn <= sp.maxnodes;
        Result r;
        r.status = TCG_ARENA_OVERFLOW;
        r.nreg = 1;
        r.key = 0ull;
        if (fits) {
            const unsigned long long sg = (unsigned long long)(fsign_s[fb & 63u] ^ fsign_s[64 + (fb >> 6)]) |
                                          ((unsigned long long)ha.y << nF) |
                                          ((unsigned long long)hb.y << sB);
            RegionGraph rg;
            split_pass<EVEN, V>(fadj_s, flink_s, ea, eb, nF, sp.nFp, sB, nn, sg, rg);
            r = finish_graph<EVEN>(rg, p.maxreg);
        }
        uint64_t k = 0;
        if (valid) {
            if (r.status == TCG_OK) {
                k = r.key;
            } else {
                const uint32_t pos = atomicAdd(fbl, 1u);
                TCG_ASSERT(pos < SPL_LAUNCH);
                fbl[1 + pos] = (uint32_t)idx;
            }
        }
        tab.add<false>(g, k, r.nreg, m);
    }
    __syncthreads();
    tab.flush(g);
}

// The draws k_sample_split left (list from fbl), classified by the flat
// kernel's classifier with exact status precedence (kernels.py:107-356).
template <int K, bool EVEN>
__global__ void __launch_bounds__(THREADS, K == 6 ? TCG_ENUM_MINB6 : 1)
    k_sample_list(KParams p, uint64_t base, uint64_t seed, uint64_t nbmask, DevAgg g,
                  const uint32_t *__restrict__ fbl, unsigned long long *__restrict__ stats) {
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t *adj_s = smem;
    CtaTable tab = carve_table(smem + 32 * K * K);
    stage_adj<K>(p, adj_s);
    tab.init();
    __syncthreads();
    const uint32_t count = *fbl;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(stats, (unsigned long long)count);
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t wstride = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t wb = warp * 32u; wb < count; wb += wstride * 32u) {
        const uint32_t i = wb + lane;
        const bool valid = i < count;
        const uint64_t gidx = base + (valid ? fbl[1 + i] : 0u);
        const uint64_t m = splitmix64(seed, gidx) & nbmask;
        const Result r = classify<K, EVEN>(p, adj_s, valid ? rep_to_sigma(p.d, m) : 0ull);
        uint64_t k = 0;
        if (valid) {
            if (r.status == TCG_OK) k = r.key;
            else atomicMin(g.bad, (unsigned long long)gidx);
        }
        tab.add<false>(g, k, r.nreg, m);
    }
    __syncthreads();
    tab.flush(g);
}


// TCG_SPLIT_V: 1 region adjacency after the pass (default; +6 % on bowtie8),
// 0 at each region close
inline void *pick_split(bool even) {
    static const int v = [] {
        const char *e = std::getenv("TCG_SPLIT_V");
        return e ? std::atoi(e) : 1;
    }();
    if (v == 1) return even ? (void *)k_sample_split<true, 1> : (void *)k_sample_split<false, 1>;
    if (v == 2) return even ? (void *)k_sample_split<true, 2> : (void *)k_sample_split<false, 2>;
    if (v == 3) return even ? (void *)k_sample_split<true, 3> : (void *)k_sample_split<false, 3>;
    return even ? (void *)k_sample_split<true, 0> : (void *)k_sample_split<false, 0>;
}

inline void *pick_list(int K, bool even) {
    if (K == 2) return even ? (void *)k_sample_list<2, true> : (void *)k_sample_list<2, false>;
    if (K == 4) return even ? (void *)k_sample_list<4, true> : (void *)k_sample_list<4, false>;
    return even ? (void *)k_sample_list<6, true> : (void *)k_sample_list<6, false>;
}

inline void *pick_split_build(int K) {
    if (K == 2) return (void *)k_split_build<2>;
    if (K == 4) return (void *)k_split_build<4>;
    return (void *)k_split_build<6>;
}
