// classify.cuh -- the per-patchwork classifier on the full diamond (region
// pass, status precedence, tree key), its batch / many-triangulation /
// enumeration kernels and the per-CTA scheme tables.  Included by tcg.cu
// inside its anonymous namespace.

// ------------------------------------------------------------------ helpers
template <int K>
__device__ __forceinline__ uint32_t sel(const uint32_t (&x)[K], int w) {
    uint32_t r = x[0];
#pragma unroll
    for (int k = 1; k < K; ++k) r = (w == k) ? x[k] : r;
    return r;
}

template <int K>
__device__ __forceinline__ bool any(const uint32_t (&x)[K]) {
    uint32_t r = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) r |= x[k];
    return r != 0;
}

// lowest set bit of a K-word mask: returns word index and bit; caller
// guarantees the mask is non-zero.
template <int K>
__device__ __forceinline__ void lowest(const uint32_t (&x)[K], int &w, int &b) {
    uint32_t word = x[K - 1];
    int wi = K - 1;
#pragma unroll
    for (int k = K - 2; k >= 0; --k) {
        const bool nz = x[k] != 0;
        word = nz ? x[k] : word;
        wi = nz ? k : wi;
    }
    w = wi;
    b = __ffs(word) - 1;
}

// Row v of a node table: K adjacency words (+ K partner words if ROWS, which
// are OR-ed into PL).  Vectorised shared-memory loads.
template <int K, bool ROWS>
__device__ __forceinline__ void load_row(const uint32_t *__restrict__ base, int v, uint32_t (&a)[K],
                                         uint32_t (&PL)[K]) {
    if constexpr (ROWS) {
        static_assert(K == 2, "contracted graphs use 64-node masks");
        const uint4 t = reinterpret_cast<const uint4 *>(base)[v];
        a[0] = t.x; a[1] = t.y;
        PL[0] |= t.z; PL[1] |= t.w;
    } else if constexpr (K == 2) {
        const uint2 t = reinterpret_cast<const uint2 *>(base)[v];
        a[0] = t.x; a[1] = t.y;
    } else if constexpr (K == 4) {
        const uint4 t = reinterpret_cast<const uint4 *>(base)[v];
        a[0] = t.x; a[1] = t.y; a[2] = t.z; a[3] = t.w;
    } else {
        const uint2 *r = reinterpret_cast<const uint2 *>(base) + 3 * v;
        const uint2 t0 = r[0], t1 = r[1], t2 = r[2];
        a[0] = t0.x; a[1] = t0.y; a[2] = t1.x; a[3] = t1.y; a[4] = t2.x; a[5] = t2.y;
    }
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t seed, uint64_t k) {
    // kernels.py:439-444
    uint64_t z = seed + (k + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t rep_to_sigma(int d, uint64_t m) {
    // free positions ascending take the bits of m (signs.py:188-206):
    // pinned set {0, 1, d+1} -> two shifted runs
    const uint64_t low = m & ((1ull << (d - 1)) - 1ull);
    return (low << 2) | ((m >> (d - 1)) << (d + 2));
}

// sign of every vertex, in the half-swap layout (see plan construction)
template <int K>
__device__ __forceinline__ void sign_words(const KParams &p, uint64_t sigma, uint32_t (&SG)[K]) {
    uint64_t q4 = 0;
#pragma unroll
    for (int r = 0; r < NQ4; ++r) {
        if (r < p.nq4)
            q4 |= ((sigma >> p.q4src[r]) & ((1ull << p.q4len[r]) - 1ull)) << p.q4dst[r];
    }
    const int sh = p.npts - 1;  // 2..54
    uint64_t lo = (sigma >> 1) | (q4 << sh);
    uint64_t hi = q4 >> (64 - sh);
    const uint64_t c = sigma & 1ull;
    if (p.center < 64) lo |= c << p.center;
    else hi |= c << (p.center - 64);
    const uint32_t w[3] = {(uint32_t)lo, (uint32_t)(lo >> 32), (uint32_t)hi};
#pragma unroll
    for (int k = 0; k < K / 2; ++k) {
        SG[k] = w[k] ^ p.jodd[k];
        SG[K / 2 + k] = SG[k] ^ p.parP[k];
    }
}

// Exact replay of kernels.py:199-230 (edge order) for the rare inputs where
// two order-dependent failures coexist.  Returns the status it produces.
template <int K, bool EVEN>
__device__ __noinline__ int ordered_scan(const KParams &p, const uint32_t (&SG)[K],
                                         const uint32_t (*regR)[K], int nreg, int root) {
    uint32_t sg[K];
#pragma unroll
    for (int k = 0; k < K; ++k) sg[k] = SG[k];
    uint32_t seen[MAXR];
    for (int r = 0; r < MAXR; ++r) seen[r] = 0;
    int nedges = 0;
    for (int e = 0; e < p.ne; ++e) {
        const uint32_t pk = p.edges[e];
        const int u = pk & 0xffff, v = pk >> 16;
        const int su = (sg[u >> 5] >> (u & 31)) & 1, sv = (sg[v >> 5] >> (v & 31)) & 1;
        if (su == sv) continue;
        int a = -1, b = -1;
        for (int r = 0; r < nreg && r < MAXR; ++r) {
            if ((regR[r][u >> 5] >> (u & 31)) & 1) a = r;
            if ((regR[r][v >> 5] >> (v & 31)) & 1) b = r;
        }
        if (a == b) {
            if (EVEN) return TCG_NONSEPARATING_OVAL;
            if (root < 0) root = a;
            else if (root != a) return TCG_ROOT_CONFLICT;
            continue;
        }
        if (a > b) { const int t = a; a = b; b = t; }
        if (!((seen[a] >> b) & 1u)) {
            seen[a] |= 1u << b;
            if (nedges >= nreg - 1) return TCG_NOT_A_TREE;
            ++nedges;
        }
    }
    return TCG_NOT_A_TREE;  // unreachable for the inputs routed here
}

// Rooted BFS over the region tree, then the AHU canonical key bottom-up:
// code(v) = 1 . sorted child codes . 0, children ordered by sentinel key
// (length first), leaves (key 0b110) emitted as one run; the root contributes
// only its child sequence.  Sets status (OK or DISCONNECTED).
__device__ __forceinline__ uint64_t tree_key(const uint32_t (&radj)[MAXR], int nreg, int root,
                                             int &status) {
    // rooted BFS over the region tree
    uint8_t order[MAXR], parent[MAXR];
    order[0] = (uint8_t)root;
    parent[root] = (uint8_t)root;
    uint32_t vis = 1u << root;
    int head = 0, tail = 1;
    while (head < tail) {
        const int r = order[head++];
        uint32_t nb = radj[r] & ~vis;
        vis |= nb;
        while (nb) {
            const int s2 = __ffs(nb) - 1;
            nb &= nb - 1;
            parent[s2] = (uint8_t)r;
            TCG_ASSERT(tail < MAXR && s2 < MAXR);
            order[tail++] = (uint8_t)s2;
        }
    }
    if (tail != nreg) { status = TCG_DISCONNECTED; return 0ull; }

    // AHU canonical key, bottom-up (children before parents)
    uint64_t skey[MAXR];
    uint64_t acc = 1;
    for (int k = nreg - 1; k >= 0; --k) {
        const int v = order[k];
        uint32_t ch = radj[v];
        if (k > 0) ch &= ~(1u << parent[v]);
        int nleaf = 0, h = 0;
        uint64_t buf[MAXR];
        while (ch) {
            const int c = __ffs(ch) - 1;
            ch &= ch - 1;
            const uint64_t ck = skey[c];
            if (ck == 6ull) {
                ++nleaf;
            } else {
                int j = h++;
                while (j > 0 && buf[j - 1] > ck) { buf[j] = buf[j - 1]; --j; }
                buf[j] = ck;
            }
        }
        acc = 1;
        if (nleaf) {
            const int nb2 = 2 * nleaf;
            acc = (1ull << nb2) | (0xAAAAAAAAAAAAAAAAull & ((1ull << nb2) - 1ull));
        }
        for (int i = 0; i < h; ++i) {
            const uint64_t c = buf[i];
            const int ln = 63 - __clzll(c);
            acc = (acc << ln) | (c ^ (1ull << ln));
        }
        if (k > 0) {
            const int il = 63 - __clzll(acc);
            skey[v] = (acc << 1) | (1ull << (il + 2));
        }
    }
    status = TCG_OK;
    return acc;
}

// ------------------------------------------------------------- classify one
// Regions of one patchwork as vertex (or node) masks.
template <int K, int CAP = MAXR>
struct Regions {
    uint32_t R[CAP][K];  // region vertex sets
    uint32_t X[CAP][K];  // crossed-edge neighbourhoods (COMPS mode: all neighbours)
    uint32_t oddmask;     // regions closing an orientation-reversing cycle
    int nreg;
};

// One breadth-first pass over the used vertices that labels regions.
//  * inside a layer all vertices share one sign (non-crossed edges join equal
//    signs), so `same` is a per-layer mask and a visited vertex costs
//    new = adj & unvS; unvS ^= new; F |= new; NB |= adj   (4 ops per word);
//  * a layer ends when its frontier empties; the next layer is seeded by the
//    antipodal partners of the layer (ROWS=false: swap of mask halves;
//    ROWS=true: per-node partner rows, for contracted graphs).  Partners have
//    the same sign in even degree and the opposite sign in odd degree;
//  * layers alternate orientation parity: a partner link between two nodes of
//    equal layer parity closes an odd cycle (the reference's parity
//    union-find, kernels.py:151-174).
// rows: per node K words of adjacency (+ K words of partner links if ROWS).
// COMPS: no antipodal jumps, so every "region" is one same-sign component and
// X collects all of its neighbours (used to contract a tile's fixed part).
#ifndef TCG_FLAT_BATCH
#define TCG_FLAT_BATCH 4  // measured: 1 / 2 / 3 / 4 / 6 / 8 / 12 -> C4 1.88 / 1.96 / 2.02 / 2.05 / 1.98 / 1.95 / 1.77e9 pairs/s
#endif
// BATCH > 1 (the full-diamond classifier): a lane whose layer has emptied waits
// for the next iteration that is a multiple of BATCH before running
// layer_end, so the lanes of a warp run their (divergent) layer ends together
// instead of in most iterations one by one; waiting lanes skip their pop.
template <int K, bool EVEN, bool ROWS, bool COMPS = false, int CAP = MAXR, int BATCH = 1>
__device__ __forceinline__ void region_pass(const uint32_t *__restrict__ rows,
                                            const uint32_t (&SG)[K], const uint32_t (&USED)[K],
                                            const uint32_t (&BD)[K], int nused,
                                            Regions<K, CAP> &out) {
    constexpr int HK = K / 2;
    uint32_t unvS[K], unvO[K], F[K], NB[K], XB[K], regS[K], LS[K], SAME[K], PL[K];
    uint32_t Ec[EVEN ? K : 1], Eo[EVEN ? K : 1];
    int nreg = 0;
    uint32_t oddmask = 0;
    bool odd = false;

    auto seed = [&](const uint32_t (&unv)[K]) {
        int w, b;
        lowest<K>(unv, w, b);
        const uint32_t nm = ((sel<K>(SG, w) >> b) & 1u) - 1u;  // seed sign s: s ? 0 : ~0
#pragma unroll
        for (int k = 0; k < K; ++k) {
            SAME[k] = SG[k] ^ nm;
            unvS[k] = unv[k] & SAME[k];
            unvO[k] = unv[k] & ~SAME[k];
            regS[k] = unv[k];
            LS[k] = unvS[k];
            F[k] = (k == w) ? (1u << b) : 0u;
            unvS[k] ^= F[k];
            XB[k] = 0u;
            NB[k] = 0u;
            PL[k] = 0u;
            if (EVEN) { Ec[k] = 0u; Eo[k] = 0u; }
        }
        odd = false;
    };

    auto layer_end = [&](bool more) {
        uint32_t L[K], unv[K], P[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            XB[k] |= COMPS ? NB[k] : (NB[k] & ~SAME[k]);
            NB[k] = 0u;
            L[k] = LS[k] ^ unvS[k];
            unv[k] = unvS[k] | unvO[k];
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            if (COMPS) {
                P[k] = 0u;
            } else if (ROWS) {
                P[k] = PL[k];
                PL[k] = 0u;
            } else {
                const int ks = (k + HK) % K;  // antipodal map = swap of halves
                P[k] = L[ks] & BD[ks];
            }
        }
        if (EVEN) {
            uint32_t hit = 0;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                Ec[k] |= L[k];
                hit |= P[k] & Ec[k];
            }
            odd |= hit != 0u;
        }
        uint32_t anyp = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            P[k] &= unv[k];
            anyp |= P[k];
        }
        if (anyp) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (!EVEN) {  // partners carry the opposite sign in odd degree
                    SAME[k] = ~SAME[k];
                    unvS[k] = unv[k] & SAME[k];
                    unvO[k] = unv[k] & ~SAME[k];
                }
                LS[k] = unvS[k];
                F[k] = P[k];
                unvS[k] ^= P[k];
                if (EVEN) {
                    const uint32_t t = Ec[k];
                    Ec[k] = Eo[k];
                    Eo[k] = t;
                }
            }
            return;
        }
        // region complete
        if (nreg < CAP) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                out.R[nreg][k] = regS[k] ^ unv[k];
                out.X[nreg][k] = XB[k];
            }
            if (EVEN && odd) oddmask |= 1u << nreg;
        }
        ++nreg;
        if (more) seed(unv);
    };

    seed(USED);
    for (int it = 0, pops = 0; pops < nused; ++it) {
        if (!any<K>(F)) {
            if (BATCH > 1 && it % BATCH != 0) continue;  // wait for the warp's batch
            layer_end(true);
        }
        ++pops;
        int w, b;
        lowest<K>(F, w, b);
        const int v = 32 * w + b;
        const uint32_t bit = 1u << b;
        uint32_t a[K];
        load_row<K, ROWS>(rows, v, a, PL);
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint32_t nw = a[k] & unvS[k];
            unvS[k] ^= nw;
            F[k] = (F[k] ^ ((k == w) ? bit : 0u)) | nw;
            NB[k] |= a[k];
        }
    }
    layer_end(false);
    out.nreg = nreg;
    out.oddmask = oddmask;
}

// AHU key of the region tree rooted at `root` (the same code as tree_key:
// children sorted by sentinel key, leaves first as one run) without per-region
// arrays: the levels of the rooted tree are bit masks, and only the internal
// non-root regions -- a handful in practice -- keep a code, in register slots.
// Returns false (caller falls back to the flat kernel) when the tree is
// disconnected, deeper than SPL_MAXD or has more than SPL_SLOTS internal
// non-root regions.
constexpr int SPL_MAXD = 8;
constexpr int SPL_SLOTS = 8;
__device__ __forceinline__ bool graph_key(const uint32_t (&radj)[MAXR], int nreg, int root,
                                          uint64_t &key) {
    uint32_t lev[SPL_MAXD + 1];
    uint32_t vis = 1u << root, internal = 0u;
    lev[0] = vis;
    int depth = 0;
#pragma unroll
    for (int k = 0; k < SPL_MAXD; ++k) {
        lev[k + 1] = 0u;
        if (k == depth) {
            uint32_t nxt = 0u;
            for (uint32_t l = lev[k]; l; l &= l - 1u) {
                const int v = __ffs(l) - 1;
                const uint32_t ch = radj[v] & ~vis;
                if (ch) internal |= 1u << v;
                nxt |= ch;
            }
            vis |= nxt;
            lev[k + 1] = nxt;
            if (nxt) depth = k + 1;
        }
    }
    if (__popc(vis) != nreg) return false;  // disconnected or deeper than SPL_MAXD
    if (__popc(internal & ~(1u << root)) > SPL_SLOTS) return false;
    int snode[SPL_SLOTS];
    uint64_t scode[SPL_SLOTS];
#pragma unroll
    for (int i = 0; i < SPL_SLOTS; ++i) {
        snode[i] = -1;
        scode[i] = 0ull;
    }
    int nslot = 0;
    uint64_t acc = 1ull;
#pragma unroll
    for (int k = SPL_MAXD - 1; k >= 0; --k) {
        if (k >= depth) continue;
        for (uint32_t l = lev[k] & internal; l; l &= l - 1u) {
            const int v = __ffs(l) - 1;
            const uint32_t ch = radj[v] & lev[k + 1];
            const int nleaf = __popc(ch & ~internal);
            // codes of the internal children, ascending (register insertion)
            uint64_t buf[SPL_SLOTS];
            int h = 0;
#pragma unroll
            for (int i = 0; i < SPL_SLOTS; ++i) buf[i] = ~0ull;
            for (uint32_t c = ch & internal; c; c &= c - 1u) {
                const int cv = __ffs(c) - 1;
                uint64_t ck = 0ull;
#pragma unroll
                for (int i = 0; i < SPL_SLOTS; ++i) ck = snode[i] == cv ? scode[i] : ck;
#pragma unroll
                for (int i = SPL_SLOTS - 1; i >= 0; --i)  // shift the larger ones, place ck
                    buf[i] = (i > 0 && buf[i > 0 ? i - 1 : 0] > ck) ? buf[i > 0 ? i - 1 : 0]
                                                                    : (buf[i] > ck ? ck : buf[i]);
                ++h;
            }
            acc = 1ull;
            if (nleaf) {
                const int nb2 = 2 * nleaf;
                acc = (1ull << nb2) | (0xAAAAAAAAAAAAAAAAull & ((1ull << nb2) - 1ull));
            }
#pragma unroll
            for (int i = 0; i < SPL_SLOTS; ++i) {
                if (i < h) {
                    const uint64_t c = buf[i];
                    const int ln = 63 - __clzll(c);
                    acc = (acc << ln) | (c ^ (1ull << ln));
                }
            }
            if (k > 0) {
                const int il = 63 - __clzll(acc);
                const uint64_t code = (acc << 1) | (1ull << (il + 2));
#pragma unroll
                for (int i = 0; i < SPL_SLOTS; ++i)
                    if (i == nslot) {
                        snode[i] = v;
                        scode[i] = code;
                    }
                ++nslot;
            }
        }
    }
    key = acc;
    return true;
}

// Region graph -> status (reference precedence) -> rooted tree -> AHU key.
// EXACT: replay the two order-dependent status collisions in edge order
// (only meaningful for the flat diamond layout); otherwise report a failure
// and let the host recompute the exact status through the flat kernel.
template <int K, bool EVEN, bool EXACT>
__device__ __forceinline__ Result finish(const KParams &p, const uint32_t (&SG)[K],
                                         const Regions<K> &rg, int maxreg) {
    Result res;
    const int nreg = rg.nreg;
    res.nreg = nreg;
    res.key = 0;
    if (nreg > maxreg || nreg > MAXR) {  // kernels.py:182: ids 0..maxreg-1 allowed
        res.status = TCG_TOO_MANY_REGIONS;
        return res;
    }
    int root = -1;
    if (EVEN) {
        const int c = __popc(rg.oddmask);
        if (c == 0) { res.status = TCG_NO_ODD_REGION; return res; }
        if (c > 1) { res.status = TCG_MANY_ODD_REGIONS; return res; }
        root = __ffs(rg.oddmask) - 1;
    } else {
        // the pseudoline region: the first region with a crossed edge inside
        for (int r = 0; r < nreg; ++r) {
            uint32_t t = 0;
#pragma unroll
            for (int k = 0; k < K; ++k) t |= rg.X[r][k] & rg.R[r][k];
            if (t) { root = r; break; }
        }
    }
    // Fast path, flat trees (92 % of degree-7 patchworks): every other
    // region touches only the root across crossed edges.  Then the region
    // graph is the star at the root -- nreg-1 edges, connected, no crossed
    // edge inside a non-root region -- so no status can fire and the key is
    // the root with nreg-1 leaf children.  Anything else takes the general
    // path below (which also settles every status exactly).
    if (root >= 0) {
        bool flat = true;
        uint32_t rroot[K];
#pragma unroll
        for (int k = 0; k < K; ++k) rroot[k] = rg.R[root][k];
        if (EVEN) {
            uint32_t t = 0;
#pragma unroll
            for (int k = 0; k < K; ++k) t |= rg.X[root][k] & rroot[k];
            flat = t == 0u;
        }
        for (int r = 0; r < nreg && flat; ++r) {
            if (r == root) continue;
            uint32_t out = 0, in = 0;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                out |= rg.X[r][k] & ~rroot[k];
                in |= rg.X[r][k];
            }
            flat = out == 0u && in != 0u;
        }
        if (flat) {
            const int nb2 = 2 * (nreg - 1);
            res.status = TCG_OK;
            res.key = (1ull << nb2) | (0xAAAAAAAAAAAAAAAAull & ((1ull << nb2) - 1ull));
            return res;
        }
    }
    // region graph from crossed-edge neighbourhoods
    uint32_t radj[MAXR];
    uint32_t selfm = 0;
    int nedges = 0;
    for (int r = 0; r < nreg; ++r) radj[r] = 0u;
    for (int r = 0; r < nreg; ++r) {
        uint32_t x[K];
        uint32_t t = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            x[k] = rg.X[r][k];
            t |= x[k] & rg.R[r][k];
        }
        if (t) selfm |= 1u << r;
        for (int r2 = r + 1; r2 < nreg; ++r2) {
            uint32_t u = 0;
#pragma unroll
            for (int k = 0; k < K; ++k) u |= x[k] & rg.R[r2][k];
            if (u) {
                radj[r] |= 1u << r2;
                radj[r2] |= 1u << r;
                ++nedges;
            }
        }
    }
    const bool toomany = nedges > nreg - 1;  // mid-loop NOT_A_TREE will fire
    if (EVEN) {
        if (toomany && selfm) {
            if constexpr (EXACT) res.status = ordered_scan<K, EVEN>(p, SG, rg.R, nreg, root);
            else res.status = TCG_NOT_A_TREE;
            return res;
        }
        if (toomany) { res.status = TCG_NOT_A_TREE; return res; }
        if (selfm) { res.status = TCG_NONSEPARATING_OVAL; return res; }
    } else {
        const bool conflict = __popc(selfm) >= 2;
        if (toomany && conflict) {
            if constexpr (EXACT) res.status = ordered_scan<K, EVEN>(p, SG, rg.R, nreg, -1);
            else res.status = TCG_NOT_A_TREE;
            return res;
        }
        if (toomany) { res.status = TCG_NOT_A_TREE; return res; }
        if (conflict) { res.status = TCG_ROOT_CONFLICT; return res; }
        if (!selfm) { res.status = TCG_NO_PSEUDOLINE; return res; }
        root = __ffs(selfm) - 1;
    }
    if (nedges != nreg - 1) { res.status = TCG_NOT_A_TREE; return res; }
    // a tree on nreg <= 3 nodes is connected; its key is closed-form:
    // 1 = <no oval>, 0b110 = one oval, 0b11010 = two leaves under the root,
    // 0b11100 = a chain (one oval inside another)
    if (nreg <= 3) {
        res.status = TCG_OK;
        res.key = nreg == 1 ? 1ull : (nreg == 2 ? 6ull : (__popc(radj[root]) == 2 ? 26ull : 28ull));
        return res;
    }
    // register-slot AHU key (graph_key); the array version for trees it declines
    if (graph_key(radj, nreg, root, res.key)) res.status = TCG_OK;
    else res.key = tree_key(radj, nreg, root, res.status);
    return res;
}

template <int K, bool EVEN>
__device__ __forceinline__ Result classify(const KParams &p, const uint32_t *__restrict__ adj,
                                           uint64_t sigma) {
    uint32_t SG[K];
    sign_words<K>(p, sigma, SG);
    uint32_t used[K], bd[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        used[k] = p.used[k];
        bd[k] = p.bd[k];
    }
    Regions<K> rg;
    region_pass<K, EVEN, false, false, MAXR, TCG_FLAT_BATCH>(adj, SG, used, bd, p.nused, rg);
    return finish<K, EVEN, true>(p, SG, rg, p.maxreg);
}

// ------------------------------------------------------------------ kernels
template <int K>
__device__ __forceinline__ void stage_adj(const KParams &p, uint32_t *adj_s) {
    const int n = 32 * K * K;  // 2H rows of K words, H = 16K
    for (int i = threadIdx.x; i < n; i += blockDim.x) adj_s[i] = p.adj[i];
}

template <int K, bool EVEN>
__global__ void __launch_bounds__(THREADS) k_batch(KParams p, const uint64_t *__restrict__ sig,
                                                   int64_t n, uint64_t *__restrict__ key,
                                                   uint8_t *__restrict__ ovals,
                                                   uint8_t *__restrict__ nreg,
                                                   int32_t *__restrict__ status) {
    extern __shared__ __align__(16) uint32_t smem[];
    stage_adj<K>(p, smem);
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += stride) {
        const Result r = classify<K, EVEN>(p, smem, sig[t]);
        key[t] = r.status == TCG_OK ? r.key : 0ull;
        ovals[t] = r.status == TCG_OK ? (uint8_t)(r.nreg - 1) : 0xff;
        nreg[t] = (uint8_t)min(r.nreg, 255);
        status[t] = r.status;
    }
}

// Many triangulations of one degree (config C4): a work item is
// (triangulation, first pair, pair count) over pairs sorted by triangulation;
// each CTA stages its item's descriptor and adjacency rows in shared memory,
// so consecutive CTAs classify on different topologies.
template <int K, bool EVEN>
__global__ void __launch_bounds__(THREADS) k_multi(const KParams *__restrict__ kps,
                                                   const int4 *__restrict__ items,
                                                   const uint64_t *__restrict__ sig,
                                                   uint64_t *__restrict__ key,
                                                   uint8_t *__restrict__ ovals,
                                                   uint8_t *__restrict__ nreg,
                                                   int32_t *__restrict__ status) {
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ KParams kp_s;
    const int4 it = items[blockIdx.x];  // x = triangulation, y = first, z = count
    if (threadIdx.x == 0) kp_s = kps[it.x];
    __syncthreads();
    stage_adj<K>(kp_s, smem);
    __syncthreads();
    for (int t = threadIdx.x; t < it.z; t += blockDim.x) {
        const int64_t i = (int64_t)it.y + t;
        const Result r = classify<K, EVEN>(kp_s, smem, sig[i]);
        key[i] = r.status == TCG_OK ? r.key : 0ull;
        ovals[i] = r.status == TCG_OK ? (uint8_t)(r.nreg - 1) : 0xff;
        nreg[i] = (uint8_t)min(r.nreg, 255);
        status[i] = r.status;
    }
}

__device__ __forceinline__ uint32_t hash_slot(uint64_t key, int bits) {
    return (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> (64 - bits));
}

__device__ void global_insert(const DevAgg &g, uint64_t key, uint64_t cnt, uint64_t wit) {
    uint32_t h = hash_slot(key, GCAP_BITS);
    for (int probe = 0; probe < GCAP; ++probe) {
        const unsigned long long prev = atomicCAS(&g.keys[h], 0ull, (unsigned long long)key);
        if (prev == 0ull || prev == key) {
            atomicAdd(&g.cnt[h], (unsigned long long)cnt);
            atomicMin(&g.wit[h], (unsigned long long)wit);
            return;
        }
        h = (h + 1) & (GCAP - 1);
    }
    atomicOr(g.overflow, 1u);
}

// Per-CTA scheme table in shared memory (flushed to the global table).
struct CtaTable {  // 64-bit counts: a tiled launch covers up to 2^32 weighted patchworks
    unsigned long long *key, *wit;
    unsigned long long *cnt, *hist;

    __device__ void init() {
        for (int i = threadIdx.x; i < TBL; i += blockDim.x) {
            key[i] = 0ull;
            wit[i] = ~0ull;
            cnt[i] = 0ull;
        }
        for (int i = threadIdx.x; i < NHIST; i += blockDim.x) hist[i] = 0ull;
    }

    // Warp-aggregated insert of one result per lane (all 32 lanes call).
    // WITNESS_BY_LEADER: lanes are in increasing index order, so the group
    // leader holds the group's minimal index (sweeps); otherwise every lane
    // offers its own index (random draws).
    template <bool WITNESS_BY_LEADER>
    __device__ __forceinline__ void add(const DevAgg &g, uint64_t k, int nreg, uint64_t m,
                                        uint32_t weight = 1u) {
        const int lane = threadIdx.x & 31;
        const unsigned grp = __match_any_sync(0xffffffffu, k);
        if (k == 0ull) return;
        const int leader = __ffs(grp) - 1;
        int slot = -1;
        if (lane == leader) {
            uint32_t h = hash_slot(k, TBL_BITS);
            for (int probe = 0; probe < TBL_PROBES; ++probe) {
                const unsigned long long cur = key[h];
                if (cur == k) { slot = (int)h; break; }
                if (cur == 0ull) {
                    const unsigned long long prev = atomicCAS(&key[h], 0ull, k);
                    if (prev == 0ull || prev == k) { slot = (int)h; break; }
                }
                h = (h + 1) & (TBL - 1);
            }
            const unsigned long long c = (unsigned long long)__popc(grp) * weight;
            TCG_ASSERT(nreg >= 1 && nreg <= NHIST);
            atomicAdd(&hist[nreg - 1], c);
            if (slot >= 0) {
                atomicAdd(&cnt[slot], c);
                if (WITNESS_BY_LEADER) atomicMin(&wit[slot], (unsigned long long)m);
            } else {  // table saturated: straight to the global table
                global_insert(g, k, c, WITNESS_BY_LEADER ? m : ~0ull);
            }
        }
        if (!WITNESS_BY_LEADER) {
            slot = __shfl_sync(grp, slot, leader);
            if (slot >= 0) atomicMin(&wit[slot], (unsigned long long)m);
            else global_insert(g, k, 0ull, m);
        }
    }

    __device__ void flush(const DevAgg &g) {
        for (int i = threadIdx.x; i < TBL; i += blockDim.x) {
            const unsigned long long kk = key[i];
            if (kk != 0ull) global_insert(g, kk, cnt[i], wit[i]);
        }
        for (int i = threadIdx.x; i < NHIST; i += blockDim.x)
            if (hist[i]) atomicAdd(&g.hist[i], hist[i]);
    }
};

constexpr size_t TABLE_SMEM = TBL * 3 * sizeof(unsigned long long) +
                              NHIST * sizeof(unsigned long long);

__device__ __forceinline__ CtaTable carve_table(void *at) {
    CtaTable t;
    t.key = reinterpret_cast<unsigned long long *>(at);
    t.wit = t.key + TBL;
    t.cnt = t.wit + TBL;
    t.hist = t.cnt + TBL;
    return t;
}

// Enumeration kernel: raw / representative sweep or counter-based sample.
// Persistent grid; each warp walks 32 consecutive indices per step.
template <int K, bool EVEN, int MODE>
#ifndef TCG_ENUM_MINB6
#define TCG_ENUM_MINB6 3  // d = 8, 9: cap registers for 3 resident CTAs (measured +14 % on bowtie8)
#endif
__global__ void __launch_bounds__(THREADS, K == 6 ? TCG_ENUM_MINB6 : 1) k_enumerate(KParams p, uint64_t base, uint64_t count,
                                                       uint64_t seed, uint64_t nbmask, DevAgg g) {
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t *adj_s = smem;
    CtaTable tab = carve_table(smem + 32 * K * K);
    stage_adj<K>(p, adj_s);
    tab.init();
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t wstride = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t wb = warp * 32ull; wb < count; wb += wstride * 32ull) {
        const uint64_t idx = wb + lane;
        const bool valid = idx < count;
        const uint64_t gidx = base + idx;  // m (sweeps) or draw number k (sample)
        uint64_t m, sigma;
        if (MODE == MODE_SAMPLE) {
            m = splitmix64(seed, gidx) & nbmask;
            sigma = rep_to_sigma(p.d, m);
        } else if (MODE == MODE_REP) {
            m = gidx;
            sigma = rep_to_sigma(p.d, m);
        } else {
            m = gidx;
            sigma = m;
        }
        const Result r = classify<K, EVEN>(p, adj_s, valid ? sigma : 0ull);
        uint64_t k = 0;
        if (valid) {
            if (r.status == TCG_OK) k = r.key;
            else atomicMin(g.bad, (unsigned long long)gidx);
        }
        tab.add<MODE != MODE_SAMPLE>(g, k, r.nreg, m);
    }
    __syncthreads();
    tab.flush(g);
}
