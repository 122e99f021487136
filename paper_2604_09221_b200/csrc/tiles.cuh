// tiles.cuh -- sweep tiles: contraction of a tile's fixed part (super-tiles,
// tile records), exact record deduplication and the level-1 tile classifier.
// Included by tcg.cu inside its anonymous namespace.

// ---------------------------------------------------------- tile contraction
// A sweep tile is 2^TILE_BITS consecutive indices aligned to its size: every
// index in it shares all sign bits except those of a few "free" lattice
// points (raw: points 0..9, i.e. the j-axis and two more; representative:
// the first 10 free positions).  Their diamond copies are the free vertices.
// Once per tile, warp 0 labels the same-sign components of the remaining
// (fixed) vertices and contracts each to one node; every lane then
// classifies its patchwork on the contracted graph -- at most 64 nodes
// (components + free vertices), one 64-bit mask per set -- with the same
// region pass (ROWS mode: per-node adjacency and antipodal-link rows).
// Any tile whose contraction does not fit falls back to the flat kernel.
constexpr int TILE_BITS_MAX = 12;
constexpr int MAXC = 48;  // fixed components per tile
constexpr int MAXF = 32;  // free vertices
constexpr int MAXM = 24;  // mid vertices of a super-tile
// level-1 list entries for a single A slice: tile | (a + 1) << slice_shift(la)
// (a + 1 <= 2^la takes la + 1 bits; tile ids < 2^(31 - la), which the chunk
// size guarantees: <= 2^35 indices = 2^(30 - la) tiles)
__host__ __device__ constexpr int slice_shift(int la) { return 31 - la; }
constexpr int SUPER_BITS_MAX = 6;

struct alignas(16) TileTables {  // per plan and domain (raw / representative), device memory
    int nf, nfixed, bits, maxnodes;  // maxnodes: contraction size limit (64; lower only in tests)
    uint32_t fixed[MAXK];                  // used and not free (layout mask)
    uint32_t fword[MAXF], fbit[MAXF];      // layout word / bit of free node f
    unsigned long long fadj[MAXF];         // free-free adjacency (bit g = free node g)
    unsigned long long fpl[MAXF];          // free-free antipodal links
    unsigned long long fcopy[TILE_BITS_MAX];  // free nodes whose sign is index bit i
    unsigned long long fpar;               // sign-extension parity of the free nodes
    // free-node sign words for the tile-local index: fsign[0][low & 63] ^
    // fsign[1][(low >> 6) & 63] (parity folded into fsign[0])
    unsigned long long fsign[2][64];
    // level-2 contraction (odd degree): index bits 0..4 are the B points (one
    // per lane), bits 5..bits-1 the A points fixed per level-2 record
    int l2, nB, NA, la;                     // enabled, B nodes, A patterns = 2^la
    int l2shift, l2even;                    // B nodes = free nodes l2shift .. +nB-1 (or -1)
    // two-stage level 2 (odd degree, 4 A bits): stage 1 fixes A1 = tile bits 5,6,
    // stage 2 the A2 = bits 7,8.  F space (stage-1 free nodes) = B nodes 0..nB-1,
    // then A2 nodes nB..nB+nA2-1.
    int ts, nA2;
    uint32_t fa1, fa2;                      // free-node masks of A1 / A2 nodes
    int32_t l15sh;                          // B | A1 | A2 contiguous: F index = f or f - l15sh (else -1: lookup tables)
    int8_t l15F[MAXF];                      // free node -> F index (or -1)
    uint32_t a2sign[16];                    // A2-node signs (A2 index space) per A2 pattern
    int la1, la2;                           // A1 = tile bits 5 .. 4+la1, A2 = the la2 = la - la1 above
    int l15max;                             // stage-1 super-node budget (TCG_L15_MAXM tests the fallback)
    uint32_t a2adjA2[16], a2linkA2[16];     // A2-A2 adjacency / links (A2 space)
    uint32_t a2adjB[16], a2linkB[16];       // A2-B adjacency / links (B space)
    uint32_t fa, fbm;                       // free-node masks of A and B nodes
    int8_t l2j[MAXF];                       // free node -> B index (or -1)
    uint32_t l2adjB[16], l2linkB[16];       // B-B adjacency / links (B index space)
    uint32_t l2bsign[32];                   // B-node signs for tile-local bits 0..4
    uint32_t freem[MAXK];                   // free vertices (layout mask)
    int8_t vfree[32 * MAXK];                // layout position -> free node (or -1)
    // super-tiles (k_super_build / k_tile_from_super): 2^sh consecutive tiles share
    // every sign except those of the "mid" points (tile-index bits 0..sh-1)
    int sh, nm, nsfixed, pad2;              // sh = 0: off
    uint32_t sfixed[MAXK];                  // fixed vertices that are not mid vertices
    uint16_t mpos[MAXM];                    // layout positions of the mid vertices, ascending
    uint32_t msign[1 << SUPER_BITS_MAX];    // mid-vertex signs (bit j) for mid pattern x
};

// Contracted tile, written by k_tile_build and staged into shared memory by
// k_tile_classify.
struct TileRec {
    uint4 rows[64];  // per node: adjacency (x, y), antipodal links (z, w)
    unsigned long long sgn_fixed;
    int n, nnodes, fallback, pad;
};

// Graphs of <= 32 nodes (all of d = 6, 99 % of d = 7) store only the low
// adjacency and link words, packed as uint2 at the start of rows[]: a quarter
// of the bytes to write, deduplicate and stage.
__device__ __forceinline__ const uint2 *rows2(const TileRec *r) {
    return reinterpret_cast<const uint2 *>(r->rows);
}

__device__ __forceinline__ void store_row(TileRec *rec, int node, int nn, unsigned long long adj,
                                          unsigned long long pl) {
    if (nn <= 32)
        reinterpret_cast<uint2 *>(rec->rows)[node] = make_uint2((uint32_t)adj, (uint32_t)pl);
    else
        rec->rows[node] = make_uint4((uint32_t)adj, (uint32_t)(adj >> 32), (uint32_t)pl,
                                     (uint32_t)(pl >> 32));
}

// Record hash, accumulated by the builders as they write the rows (the
// deduplication only uses it to find candidates; equality is decided by
// comparing the records word by word).
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

struct RecHash {
    uint32_t h1 = 0x243F6A88u, h2 = 0x85A308D3u;
    __device__ __forceinline__ void row(unsigned long long adj, unsigned long long pl) {
        const uint32_t ah = (uint32_t)(adj >> 32), ph = (uint32_t)(pl >> 32);
        h1 = (h1 ^ (uint32_t)adj ^ __funnelshift_l(ah, ah, 16)) * 0x9E3779B1u;
        h1 ^= h1 >> 15;
        h2 = (h2 ^ (uint32_t)pl ^ __funnelshift_l(ph, ph, 16)) * 0x85EBCA77u;
        h2 ^= h2 >> 13;
    }
    __device__ __forceinline__ unsigned long long fin(unsigned long long sgn, int n, int nn) const {
        return mix64(((unsigned long long)h1 << 32 | h2) ^
                     mix64(sgn ^ ((unsigned long long)nn << 56) ^ ((unsigned long long)n << 48)));
    }
};

// Region pass over a contracted graph (<= 64 nodes, one u64 per set) without
// layers: antipodal links are followed in the same step as edges, so a lane
// only branches when a region ends.  Each popped node v uses its own sign:
//   new = unvisited & ((adj & same_v) | links_v);   XB |= adj & ~same_v.
// Even degree: orientation parity is tracked per node (edges keep it, links
// flip it); any edge or link whose ends violate the 2-colouring closes an odd
// cycle (the reference's parity union-find, kernels.py:151-174).
template <bool EVEN>
__device__ __forceinline__ void node_pass(const uint4 *__restrict__ rows, uint32_t sg0,
                                          uint32_t sg1, uint32_t u0, uint32_t u1, int nn,
                                          Regions<2> &out) {
    // two 32-bit halves per node set: lo = nodes 0..31, hi = nodes 32..63
    uint32_t un0 = u0, un1 = u1, f0 = 0, f1 = 0, x0 = 0, x1 = 0, q0 = 0, q1 = 0, r0 = 0, r1 = 0;
    bool odd = false;
    int nreg = 0;
    uint32_t oddmask = 0;
    auto seed = [&]() {
        const bool lo = un0 != 0u;
        const uint32_t w = lo ? un0 : un1;
        const uint32_t low = w & (0u - w);
        r0 = un0;
        r1 = un1;
        f0 = lo ? low : 0u;
        f1 = lo ? 0u : low;
        un0 ^= f0;
        un1 ^= f1;
        x0 = x1 = 0u;
        if (EVEN) q0 = q1 = 0u;
        odd = false;
    };
    auto close = [&]() {
        if (nreg < MAXR) {
            out.R[nreg][0] = r0 ^ un0;
            out.R[nreg][1] = r1 ^ un1;
            out.X[nreg][0] = x0;
            out.X[nreg][1] = x1;
            if (EVEN && odd) oddmask |= 1u << nreg;
        }
        ++nreg;
    };
    seed();
    for (int it = 0; it < nn; ++it) {
        if ((f0 | f1) == 0u) {
            close();
            seed();
        }
        const bool lo = f0 != 0u;
        const uint32_t w = lo ? f0 : f1;
        const int b = __ffs(w) - 1;
        const uint32_t rest = w & (w - 1u);
        f0 = lo ? rest : f0;
        f1 = lo ? f1 : rest;
        const int v = lo ? b : b + 32;
        const uint4 row = rows[v];
        // opp = nodes whose sign differs from v's: SG ^ (s_v ? ~0 : 0)
        const uint32_t sv = (uint32_t)((int32_t)((lo ? sg0 : sg1) << (31 - b)) >> 31);
        const uint32_t o0 = sg0 ^ sv, o1 = sg1 ^ sv;
        x0 |= row.x & o0;
        x1 |= row.y & o1;
        if (EVEN) {
            // parity of v (equal-parity mask pv): edges keep it, links flip it
            const uint32_t pv = (uint32_t)((int32_t)((lo ? q0 : q1) << (31 - b)) >> 31);
            const uint32_t te0 = row.x & ~o0, te1 = row.y & ~o1;
            const uint32_t nt0 = te0 & un0, nt1 = te1 & un1;
            const uint32_t np0 = row.z & un0, np1 = row.w & un1;
            const uint32_t eq0 = ~(q0 ^ pv), eq1 = ~(q1 ^ pv);
            const uint32_t bad = (nt0 & np0) | (nt1 & np1) | (te0 & ~un0 & ~eq0) |
                                 (te1 & ~un1 & ~eq1) | (row.z & ~un0 & eq0) | (row.w & ~un1 & eq1);
            odd |= bad != 0u;
            q0 |= (nt0 & pv) | (np0 & ~pv);
            q1 |= (nt1 & pv) | (np1 & ~pv);
            const uint32_t n0 = nt0 | np0, n1 = nt1 | np1;
            un0 ^= n0;
            un1 ^= n1;
            f0 |= n0;
            f1 |= n1;
        } else {
            const uint32_t n0 = ((row.x & ~o0) | row.z) & un0;
            const uint32_t n1 = ((row.y & ~o1) | row.w) & un1;
            un0 ^= n0;
            un1 ^= n1;
            f0 |= n0;
            f1 |= n1;
        }
    }
    close();
    out.nreg = nreg;
    out.oddmask = oddmask;
}

// node_pass for contracted graphs of at most 32 nodes: one 32-bit word per set.
template <bool EVEN>
__device__ __forceinline__ void node_pass1(const uint4 *__restrict__ rows, uint32_t sg,
                                           uint32_t used, int nn, Regions<1> &out) {
    uint32_t un = used, f = 0, x = 0, q = 0, r = 0;
    bool odd = false;
    int nreg = 0;
    uint32_t oddmask = 0;
    auto seed = [&]() {
        f = un & (0u - un);
        r = un;
        un ^= f;
        x = 0u;
        if (EVEN) q = 0u;
        odd = false;
    };
    auto close = [&]() {
        if (nreg < MAXR) {
            out.R[nreg][0] = r ^ un;
            out.X[nreg][0] = x;
            if (EVEN && odd) oddmask |= 1u << nreg;
        }
        ++nreg;
    };
    seed();
    for (int it = 0; it < nn; ++it) {
        if (f == 0u) {
            close();
            seed();
        }
        const int v = __ffs(f) - 1;
        f &= f - 1u;
        const uint4 row = rows[v];
        const uint32_t sv = (uint32_t)((int32_t)(sg << (31 - v)) >> 31);
        const uint32_t o = sg ^ sv;  // nodes of the other sign
        x |= row.x & o;
        if (EVEN) {
            const uint32_t pv = (uint32_t)((int32_t)(q << (31 - v)) >> 31);
            const uint32_t te = row.x & ~o, nt = te & un, np = row.z & un;
            const uint32_t eq = ~(q ^ pv);
            odd |= ((nt & np) | (te & ~un & ~eq) | (row.z & ~un & eq)) != 0u;
            q |= (nt & pv) | (np & ~pv);
            const uint32_t n = nt | np;
            un ^= n;
            f |= n;
        } else {
            const uint32_t n = ((row.x & ~o) | row.z) & un;
            un ^= n;
            f |= n;
        }
    }
    close();
    out.nreg = nreg;
    out.oddmask = oddmask;
}

// Two independent patchworks of one tile per thread, stepped in lock-step:
// the region opens/closes stay branches, but both shared-memory row loads
// and both expansions sit in one basic block, so their latencies overlap.
template <bool EVEN>
struct NP1 {
    uint32_t un, f, x, q, r, oddmask;
    bool odd;
    int nreg;
    __device__ __forceinline__ void start(uint32_t used) {
        un = used;
        nreg = 0;
        oddmask = 0u;
        seed();
    }
    __device__ __forceinline__ void seed() {
        f = un & (0u - un);
        r = un;
        un ^= f;
        x = 0u;
        if (EVEN) q = 0u;
        odd = false;
    }
    __device__ __forceinline__ void close(Regions<1> &out) {
        if (nreg < MAXR) {
            out.R[nreg][0] = r ^ un;
            out.X[nreg][0] = x;
            if (EVEN && odd) oddmask |= 1u << nreg;
        }
        ++nreg;
    }
    __device__ __forceinline__ void expand(const uint32_t rx, const uint32_t rz, int v,
                                           uint32_t sg) {
        const uint32_t sv = (uint32_t)((int32_t)(sg << (31 - v)) >> 31);
        const uint32_t o = sg ^ sv;
        x |= rx & o;
        if (EVEN) {
            const uint32_t pv = (uint32_t)((int32_t)(q << (31 - v)) >> 31);
            const uint32_t te = rx & ~o, nt = te & un, np = rz & un;
            const uint32_t eq = ~(q ^ pv);
            odd |= ((nt & np) | (te & ~un & ~eq) | (rz & ~un & eq)) != 0u;
            q |= (nt & pv) | (np & ~pv);
            const uint32_t n = nt | np;
            un ^= n;
            f |= n;
        } else {
            const uint32_t n = ((rx & ~o) | rz) & un;
            un ^= n;
            f |= n;
        }
    }
    __device__ __forceinline__ void finish(Regions<1> &out) {
        close(out);
        out.nreg = nreg;
        out.oddmask = oddmask;
    }
};

template <bool EVEN>
__device__ __forceinline__ void node_pass1x2(const uint32_t *__restrict__ ax,
                                             const uint32_t *__restrict__ az, uint32_t sga,
                                             uint32_t sgb, uint32_t used, int nn,
                                             Regions<1> &oa, Regions<1> &ob) {
    NP1<EVEN> a, b;
    a.start(used);
    b.start(used);
    for (int it = 0; it < nn; ++it) {
        if (a.f == 0u) {
            a.close(oa);
            a.seed();
        }
        if (b.f == 0u) {
            b.close(ob);
            b.seed();
        }
        const int va = __ffs(a.f) - 1, vb = __ffs(b.f) - 1;
        a.f &= a.f - 1u;
        b.f &= b.f - 1u;
        const uint32_t xa = ax[va], xb = ax[vb], za = az[va], zb = az[vb];
        a.expand(xa, za, va, sga);
        b.expand(xb, zb, vb, sgb);
    }
    a.finish(oa);
    b.finish(ob);
}

template <bool EVEN>
__device__ __forceinline__ Result classify_tile(const KParams &p, const TileTables &tt,
                                                const uint4 *rows,
                                                unsigned long long sgn_fixed, int n, int nn,
                                                uint32_t low) {
    // signs of the free nodes: two table lookups on the tile-local index
    const unsigned long long fs = tt.fsign[0][low & 63u] ^ tt.fsign[1][(low >> 6) & 63u];
    const unsigned long long sg = sgn_fixed | (fs << n);
    const unsigned long long used = nn >= 64 ? ~0ull : ((1ull << nn) - 1ull);
    if (nn <= 32) {  // tile-uniform: a warp owns the tile
        Regions<1> r1;
        node_pass1<EVEN>(rows, (uint32_t)sg, (uint32_t)used, nn, r1);
        const uint32_t SG1[1] = {(uint32_t)sg};
        return finish<1, EVEN, false>(p, SG1, r1, p.maxreg);
    }
    Regions<2> rg;
    node_pass<EVEN>(rows, (uint32_t)sg, (uint32_t)(sg >> 32), (uint32_t)used,
                    (uint32_t)(used >> 32), nn, rg);
    const uint32_t SG[2] = {(uint32_t)sg, (uint32_t)(sg >> 32)};
    return finish<2, EVEN, false>(p, SG, rg, p.maxreg);
}

template <int K, int MODE>
__device__ __forceinline__ void build_lane(const KParams &p, const uint32_t *__restrict__ adj_s,
                                           const TileTables &tt_r, uint64_t tile0, uint32_t t,
                                           TileRec *__restrict__ recs,
                                           unsigned long long *__restrict__ hashes) {
    RecHash hs;
    const TileTables *tt = &tt_r;
    const uint64_t base = (tile0 + t) << tt->bits;
    const uint64_t sigma = MODE == MODE_REP ? rep_to_sigma(p.d, base) : base;
    uint32_t SG[K], fixed[K], zero[K];
    sign_words<K>(p, sigma, SG);
#pragma unroll
    for (int k = 0; k < K; ++k) {
        fixed[k] = tt->fixed[k];
        zero[k] = 0u;
    }
    Regions<K, MAXC> comps;
    region_pass<K, false, false, true, MAXC>(adj_s, SG, fixed, zero, tt->nfixed, comps);
    const int n = comps.nreg, nf = tt->nf, nn = n + nf;
    TileRec *rec = recs + t;
    const bool fits = n <= MAXC && nn <= tt->maxnodes;
    unsigned long long sbits = 0;
    if (fits) {
        unsigned long long fadj_c[MAXF];  // free node f -> comps adjacent to it
        for (int f = 0; f < nf; ++f) fadj_c[f] = 0ull;
        for (int c = 0; c < n; ++c) {
            uint32_t X[K], R[K], P[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                X[k] = comps.X[c][k];
                R[k] = comps.R[c][k];
            }
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int ks = (k + K / 2) % K;
                P[k] = R[ks] & p.bd[ks];
            }
            unsigned long long adj = 0, pl = 0;
            for (int c2 = 0; c2 < n; ++c2) {
                uint32_t a = 0, q = 0;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    a |= X[k] & comps.R[c2][k];
                    q |= P[k] & comps.R[c2][k];
                }
                if (a && c2 != c) adj |= 1ull << c2;
                if (q) pl |= 1ull << c2;
            }
            for (int f = 0; f < nf; ++f)
                if (sel<K>(X, tt->fword[f]) & tt->fbit[f]) {
                    adj |= 1ull << (n + f);
                    fadj_c[f] |= 1ull << c;
                }
            uint32_t sg = 0;
#pragma unroll
            for (int k = 0; k < K; ++k) sg |= R[k] & SG[k];
            if (sg) sbits |= 1ull << c;
            store_row(rec, c, nn, adj, pl);
            hs.row(adj, pl);
        }
        for (int f = 0; f < nf; ++f) {
            const unsigned long long adj = (tt->fadj[f] << n) | fadj_c[f];
            const unsigned long long pl = tt->fpl[f] << n;
            store_row(rec, n + f, nn, adj, pl);
            hs.row(adj, pl);
        }
    }
    hashes[t] = hs.fin(sbits, n, nn);
    rec->sgn_fixed = sbits;
    rec->n = n;
    rec->nnodes = nn;
    rec->fallback = fits ? 0 : 1;
}
// list != nullptr: only the tiles list[0 .. *count) (the ones k_tile_from_super
// left: super-tiles whose contraction does not fit), grid-stride.
template <int K, int MODE>
__global__ void __launch_bounds__(THREADS) k_tile_build_lanes(KParams p,
                                                              const TileTables *__restrict__ tt_g,
                                                              uint64_t tile0, uint32_t ntiles,
                                                              TileRec *__restrict__ recs,
                                                              unsigned long long *__restrict__ hashes,
                                                              const uint32_t *__restrict__ list,
                                                              const uint32_t *__restrict__ count) {
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t *adj_s = smem;
    TileTables *tt = reinterpret_cast<TileTables *>(smem + 32 * K * K);
    stage_adj<K>(p, adj_s);
    for (int i = threadIdx.x; i < (int)(sizeof(TileTables) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t *>(tt)[i] = reinterpret_cast<const uint32_t *>(tt_g)[i];
    __syncthreads();
    const uint32_t nwork = list ? *count : ntiles;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nwork;
         i += gridDim.x * blockDim.x)
        build_lane<K, MODE>(p, adj_s, *tt, tile0, list ? list[i] : i, recs, hashes);
}


// ------------------------------------------------------------ super-tiles
// A super-tile is 2^sh consecutive tiles: they share the signs of every
// fixed vertex except the "mid" vertices (copies of the points of tile-index
// bits 0..sh-1).  k_super_build contracts the remaining ("super-fixed")
// vertices once per super-tile, exactly as k_tile_build_lanes contracts a
// tile, and keeps the mid vertices as single nodes: SN nodes = super
// components + mid vertices, ordered by their lowest layout position.
// k_tile_from_super then gives each tile (one per lane) its mid signs and
// merges same-sign SN neighbours -- a breadth-first pass over <= 64 nodes
// instead of ~100 vertices -- and emits the tile record.  Components come out
// ordered by their lowest vertex, as in k_tile_build_lanes, so the records
// are byte-identical to the direct contraction (tested: dedup counts and
// reports agree with TCG_BUILD_GENERIC=1).
#ifndef FS_BATCH
#define FS_BATCH 2  // k_tile_from_super pass 2: close batching (1 / 2 / 4 / 8: 21.25 / 21.08 / 21.11 / 21.15 ms per C3 step)
#endif
struct SuperRec {
    unsigned long long adj[64];   // SN-node adjacency (no self bit)
    unsigned long long link[64];  // SN-node antipodal links (self bit: pair inside the node)
    unsigned long long fsn[MAXF]; // free node -> adjacent SN nodes
    uint32_t fadj[64];            // SN node -> adjacent free nodes
    unsigned long long sgn;       // signs of the component nodes (mid nodes: 0)
    uint8_t msn[MAXM];            // SN index of mid vertex j
    int nsn, fallback;
};

template <int K, int MODE>
__global__ void __launch_bounds__(THREADS) k_super_build(KParams p,
                                                         const TileTables *__restrict__ tt_g,
                                                         uint64_t s0, uint32_t nsup,
                                                         SuperRec *__restrict__ srecs) {
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t *adj_s = smem;
    TileTables *tt = reinterpret_cast<TileTables *>(smem + 32 * K * K);
    stage_adj<K>(p, adj_s);
    for (int i = threadIdx.x; i < (int)(sizeof(TileTables) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t *>(tt)[i] = reinterpret_cast<const uint32_t *>(tt_g)[i];
    __syncthreads();
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nsup;
         i += gridDim.x * blockDim.x) {
        const uint64_t base = ((s0 + i) << tt->sh) << tt->bits;
        const uint64_t sigma = MODE == MODE_REP ? rep_to_sigma(p.d, base) : base;
        uint32_t SG[K], sf[K], zero[K];
        sign_words<K>(p, sigma, SG);
#pragma unroll
        for (int k = 0; k < K; ++k) {
            sf[k] = tt->sfixed[k];
            zero[k] = 0u;
        }
        Regions<K, MAXC> comps;
        region_pass<K, false, false, true, MAXC>(adj_s, SG, sf, zero, tt->nsfixed, comps);
        SuperRec *S = srecs + i;
        const int n = comps.nreg, nm = tt->nm, nsn = n + nm;
        if (n > MAXC || nsn > 64) {
            S->nsn = nsn;
            S->fallback = 1;
            continue;
        }
        // SN order: merge the components (ascending lowest vertex) with the mid vertices
        uint8_t ord[64];  // c, or 64 + j for mid vertex j
        {
            int ci = 0, mj = 0;
            for (int q = 0; q < nsn; ++q) {
                bool takec = ci < n;
                if (takec && mj < nm) {
                    int w, b;
                    uint32_t R[K];
#pragma unroll
                    for (int k = 0; k < K; ++k) R[k] = comps.R[ci][k];
                    lowest<K>(R, w, b);
                    takec = 32 * w + b < (int)tt->mpos[mj];
                }
                ord[q] = takec ? (uint8_t)ci++ : (uint8_t)(64 + mj++);
            }
        }
        auto node = [&](int q, uint32_t (&R)[K], uint32_t (&NB)[K]) {
            const int o = ord[q];
            if (o < 64) {
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    R[k] = comps.R[o][k];
                    NB[k] = comps.X[o][k];
                }
            } else {
                const int pos = tt->mpos[o - 64];
                uint32_t dummy[K];
                load_row<K, false>(adj_s, pos, NB, dummy);
#pragma unroll
                for (int k = 0; k < K; ++k) R[k] = (k == (pos >> 5)) ? (1u << (pos & 31)) : 0u;
            }
        };
        unsigned long long sgn = 0;
        unsigned long long fsn[MAXF];
        for (int f = 0; f < tt->nf; ++f) fsn[f] = 0ull;
        for (int q = 0; q < nsn; ++q) {
            uint32_t R[K], NB[K], P[K];
            node(q, R, NB);
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const int ks = (k + K / 2) % K;
                P[k] = R[ks] & p.bd[ks];
            }
            unsigned long long adj = 0, pl = 0;
            for (int q2 = 0; q2 < nsn; ++q2) {
                uint32_t R2[K], NB2[K];
                const int o2 = ord[q2];
                if (o2 < 64) {
#pragma unroll
                    for (int k = 0; k < K; ++k) R2[k] = comps.R[o2][k];
                } else {
                    const int pos = tt->mpos[o2 - 64];
#pragma unroll
                    for (int k = 0; k < K; ++k)
                        R2[k] = (k == (pos >> 5)) ? (1u << (pos & 31)) : 0u;
                }
                (void)NB2;
                uint32_t a = 0, l = 0;
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    a |= NB[k] & R2[k];
                    l |= P[k] & R2[k];
                }
                if (a && q2 != q) adj |= 1ull << q2;
                if (l) pl |= 1ull << q2;
            }
            uint32_t fb = 0;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                uint32_t x = NB[k] & tt->freem[k];
                while (x) {
                    const int f = tt->vfree[32 * k + __ffs(x) - 1];
                    x &= x - 1u;
                    fb |= 1u << f;
                    fsn[f] |= 1ull << q;
                }
            }
            S->adj[q] = adj;
            S->link[q] = pl;
            S->fadj[q] = fb;
            const int o = ord[q];
            if (o < 64) {
                uint32_t sg = 0;
#pragma unroll
                for (int k = 0; k < K; ++k) sg |= R[k] & SG[k];
                if (sg) sgn |= 1ull << q;
            } else {
                S->msn[o - 64] = (uint8_t)q;
            }
        }
        for (int f = 0; f < tt->nf; ++f) S->fsn[f] = fsn[f];
        S->sgn = sgn;
        S->nsn = nsn;
        S->fallback = 0;
    }
}

// One tile per lane: mid signs, merge same-sign SN neighbours (labels are
// lane-private bytes in shared memory, bank = lane), then one more pass per
// component to collect its neighbours, links and free neighbours and write
// the row.  Tiles of fallback super-tiles are listed in ovf for
// k_tile_build_lanes.
constexpr size_t FROM_SUPER_SMEM = sizeof(TileTables) + (16 + MAXF) * 4 * THREADS;  // max
inline size_t from_super_smem(int nf) { return sizeof(TileTables) + (size_t)(16 + nf) * 4 * THREADS; }

// Super-tile deduplication.  Every tile record of a super-tile is a function
// of the super record (its used part) and the tile's mid pattern alone, so
// two super-tiles with equal super records have equal tile records at equal
// mid offsets: the tiles of a duplicate super-tile are not built or compared
// -- each joins the tile-dedup group of its twin in the representative
// super-tile (k_super_prop).  Only super-tiles whose tiles are all full
// (inside the chunk and the index range) and whose contraction fit take part.
// C3: 131,072 super-tiles per step, ~74,000 distinct.
__device__ __forceinline__ unsigned long long super_hash(const SuperRec *__restrict__ r, int nf, int nm) {
    unsigned long long h = 0x9E3779B97F4A7C15ull ^ (unsigned long long)r->nsn;
    for (int k = 0; k < r->nsn; ++k) {
        h = mix64(h ^ r->adj[k]);
        h = mix64(h ^ r->link[k] ^ ((unsigned long long)r->fadj[k] << 7));
    }
    for (int f = 0; f < nf; ++f) h = mix64(h ^ r->fsn[f]);
    for (int j = 0; j < nm; ++j) h = mix64(h ^ ((unsigned long long)r->msn[j] << (8 * (j & 7))));
    return mix64(h ^ r->sgn);
}

__device__ __forceinline__ bool super_equal(const SuperRec *__restrict__ a, const SuperRec *__restrict__ b,
                                            int nf, int nm) {
    if (a->nsn != b->nsn || a->sgn != b->sgn) return false;
    unsigned long long d = 0;
    for (int k = 0; k < a->nsn; ++k)
        d |= (a->adj[k] ^ b->adj[k]) | (a->link[k] ^ b->link[k]) | (unsigned long long)(a->fadj[k] ^ b->fadj[k]);
    for (int f = 0; f < nf; ++f) d |= a->fsn[f] ^ b->fsn[f];
    for (int j = 0; j < nm; ++j) d |= (unsigned long long)(a->msn[j] ^ b->msn[j]);
    return d == 0ull;
}

// srep[s] = s (a representative, or not eligible) or the representative's index.
__global__ void __launch_bounds__(THREADS) k_super_dedup(const TileTables *__restrict__ tt_g,
                                                         const SuperRec *__restrict__ srecs, uint32_t nsup,
                                                         uint64_t tile0, uint32_t ntiles,
                                                         uint64_t start, uint64_t end,
                                                         unsigned long long *__restrict__ slots,
                                                         uint32_t smask, uint32_t *__restrict__ srep) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nsup) return;
    const int sh = tt_g->sh, bits = tt_g->bits, nf = tt_g->nf, nm = tt_g->nm;
    const uint64_t g0 = (((tile0 >> sh) + s) << sh), g1 = g0 + (1ull << sh);  // global tiles
    const SuperRec *r = srecs + s;
    uint32_t out = s;
    if (!r->fallback && g0 >= tile0 && g1 <= tile0 + ntiles && (g0 << bits) >= start &&
        (g1 << bits) <= end) {
        const unsigned long long h = super_hash(r, nf, nm);
        const unsigned long long tag = (h >> 32) << 32;
        uint32_t at = (uint32_t)h & smask;
        while (true) {
            unsigned long long cur = slots[at];
            if (cur == ~0ull) {
                const unsigned long long prev = atomicCAS(&slots[at], ~0ull, tag | s);
                if (prev == ~0ull) break;  // representative
                cur = prev;
            }
            TCG_ASSERT((cur & 0xffffffffull) < nsup);
            if ((cur & 0xffffffff00000000ull) == tag && super_equal(r, srecs + (uint32_t)cur, nf, nm)) {
                out = (uint32_t)cur;
                break;
            }
            at = (at + 1) & smask;
        }
    }
    srep[s] = out;
}

// The tiles of duplicate super-tiles join their twins' groups (after
// k_tile_dedup has settled the groups in repof).  A twin whose contraction
// did not fit is never merged; k_tile_dedup copied its record and listed the
// tile on its own.
__global__ void __launch_bounds__(THREADS) k_super_prop(const TileRec *__restrict__ recs,
                                                        uint32_t ntiles, uint64_t tile0, int sh,
                                                        const uint32_t *__restrict__ srep,
                                                        const uint32_t *__restrict__ repof,
                                                        uint32_t *__restrict__ dup,
                                                        uint32_t *__restrict__ mint) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntiles) return;
    const uint64_t gt = tile0 + t;
    const uint32_t si = (uint32_t)((gt >> sh) - (tile0 >> sh));
    const uint32_t rs = srep[si];
    if (rs == si) return;
    const uint32_t tw = (uint32_t)(((((tile0 >> sh) + rs) << sh) | (gt & ((1ull << sh) - 1ull))) - tile0);
    TCG_ASSERT(tw < ntiles);  // the representative may sit before or after the twin
    if (recs[tw].fallback) return;
    const uint32_t R = repof[tw];
    TCG_ASSERT(R < ntiles);
    atomicAdd(&dup[R], 1u);
    atomicMin(&mint[R], t);
}

__global__ void __launch_bounds__(THREADS) k_tile_from_super(const TileTables *__restrict__ tt_g,
                                                             const SuperRec *__restrict__ srecs,
                                                             uint64_t tile0, uint32_t ntiles,
                                                             TileRec *__restrict__ recs,
                                                             unsigned long long *__restrict__ hashes,
                                                             uint32_t *__restrict__ ovf,
                                                             const uint32_t *__restrict__ srep) {
    extern __shared__ __align__(16) uint32_t smem[];
    TileTables *tt = reinterpret_cast<TileTables *>(smem);
    uint8_t *lb = reinterpret_cast<uint8_t *>(smem + sizeof(TileTables) / 4 + threadIdx.x);
    for (int i = threadIdx.x; i < (int)(sizeof(TileTables) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t *>(tt)[i] = reinterpret_cast<const uint32_t *>(tt_g)[i];
    __syncthreads();
    const int h = tt->sh, nf = tt->nf, nm = tt->nm;
    const uint64_t sbase = tile0 >> h;
    auto label = [&](int v) -> uint32_t { return lb[(v >> 2) * (4 * THREADS) + (v & 3)]; };
    // labels of the SN nodes in x, as a node mask (one lookup per set bit;
    // 32-bit halves: __ffs is cheaper than __ffsll)
    auto labels_of = [&](unsigned long long x) -> unsigned long long {
        unsigned long long r = 0;
        for (uint32_t w = (uint32_t)x; w; w &= w - 1u) r |= 1ull << label(__ffs(w) - 1);
        for (uint32_t w = (uint32_t)(x >> 32); w; w &= w - 1u) r |= 1ull << label(31 + __ffs(w));
        return r;
    };
    uint32_t *FCs = smem + sizeof(TileTables) / 4 + 16 * THREADS + threadIdx.x;  // [nf] lane-private
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < ntiles;
         t += gridDim.x * blockDim.x) {
        const uint64_t gt = tile0 + t;
        const SuperRec *S = srecs + ((gt >> h) - sbase);
        TileRec *rec = recs + t;
        if (srep && srep[(gt >> h) - sbase] != (uint32_t)((gt >> h) - sbase)) continue;  // twin built
        if (S->fallback) {
            ovf[1 + atomicAdd(ovf, 1u)] = t;
            continue;
        }
        const int nsn = S->nsn;
        const uint32_t ms = tt->msign[gt & ((1u << h) - 1u)];
        unsigned long long sg = S->sgn;
        for (int j = 0; j < nm; ++j) sg |= (unsigned long long)((ms >> j) & 1u) << S->msn[j];
        const unsigned long long all = nsn >= 64 ? ~0ull : ((1ull << nsn) - 1ull);
        // pass 1: label the merged components.  One flat loop of nsn pops (every
        // lane of a warp shares the super record, so the trip count is uniform);
        // a component closes when its frontier empties.
        unsigned long long unv = all, seeds = 0, sbits = 0, F = 0, same = 0;
        int n = -1;
        for (int it = 0; it < nsn; ++it) {
            if (F == 0ull) {
                const unsigned long long seed = unv & (0ull - unv);
                const bool s1 = (sg & seed) != 0ull;
                same = s1 ? sg : ~sg;
                F = seed;
                unv ^= seed;
                seeds |= seed;
                ++n;
                if (s1) sbits |= 1ull << n;
            }
            const int v = __ffsll((long long)F) - 1;
            F &= F - 1ull;
            TCG_ASSERT(v >= 0 && v < 64 && n < 64);
            lb[(v >> 2) * (4 * THREADS) + (v & 3)] = (uint8_t)n;
            const unsigned long long nw = S->adj[v] & unv & same;
            unv ^= nw;
            F |= nw;
        }
        ++n;
        const int nn = n + nf;
        const bool fits = n <= MAXC && nn <= tt->maxnodes;
        RecHash hs;
        if (fits) {
            // pass 2: the same traversal again, collecting each component's
            // neighbours / links / free neighbours; rows are written as the
            // components close
            unsigned long long sd = seeds, M = 0, CG = 0, LK = 0;
            uint32_t FB = 0;
            unv = all;
            F = 0;
            int c = -1;
            const bool fcs = n <= 32;  // free rows by scattering the components' free bits
            if (fcs)
                for (int f = 0; f < nf; ++f) FCs[f * THREADS] = 0u;
            auto close = [&]() {
                const unsigned long long adj = ((unsigned long long)FB << n) | labels_of(CG & ~M);
                const unsigned long long pl = labels_of(LK);
                if (fcs)
                    for (uint32_t y = FB; y; y &= y - 1u) {
                        TCG_ASSERT(__ffs(y) - 1 < nf && c < 32);
                        FCs[(__ffs(y) - 1) * THREADS] |= 1u << c;
                    }
                store_row(rec, c, nn, adj, pl);
                hs.row(adj, pl);
            };
            // a lane whose component has ended waits for the warp's next
            // multiple of FS_BATCH iterations, so the closes run together
            for (int it = 0, pops = 0; pops < nsn; ++it) {
                if (F == 0ull) {
                    if (FS_BATCH > 1 && c >= 0 && it % FS_BATCH != 0) continue;
                    if (c >= 0) close();
                    const unsigned long long seed = sd & (0ull - sd);
                    sd ^= seed;
                    same = (sg & seed) ? sg : ~sg;
                    F = seed;
                    unv ^= seed;
                    M = CG = LK = 0ull;
                    FB = 0u;
                    ++c;
                }
                ++pops;
                const int v = __ffsll((long long)F) - 1;
                F &= F - 1ull;
                M |= 1ull << v;
                const unsigned long long a = S->adj[v];
                CG |= a;
                LK |= S->link[v];
                FB |= S->fadj[v];
                const unsigned long long nw = a & unv & same;
                unv ^= nw;
                F |= nw;
            }
            close();
            for (int f = 0; f < nf; ++f) {
                const unsigned long long fc = fcs ? (unsigned long long)FCs[f * THREADS]
                                                  : labels_of(S->fsn[f]);
                const unsigned long long adj = (tt->fadj[f] << n) | fc, pl = tt->fpl[f] << n;
                store_row(rec, n + f, nn, adj, pl);
                hs.row(adj, pl);
            }
        }
        const unsigned long long sgf = fits ? sbits : 0ull;
        hashes[t] = hs.fin(sgf, n, nn);
        rec->sgn_fixed = sgf;
        rec->n = n;
        rec->nnodes = nn;
        rec->fallback = fits ? 0 : 1;
    }
}

// Tile deduplication.  A tile's classification depends only on its contracted
// record (rows, fixed signs, sizes) and the tile-local index, so tiles with
// byte-identical records produce identical results index by index.  One
// thread per tile probes an open-addressing table keyed by the record hash
// the builder computed (slot = hash tag << 32 | tile); a slot whose tag
// matches is compared word by word (never by hash alone) and an equal record
// absorbs the tile: dup[rep] += 1, mint[rep] = min tile id (the witness of
// every scheme in the group is the smallest index, which lies in the group's
// smallest tile).  Representatives are appended to list[] (warp-aggregated);
// partial tiles (range ends) and fallback tiles are never merged.
constexpr unsigned long long SLOT_EMPTY = ~0ull;

__device__ __forceinline__ bool rec_equal(const TileRec *__restrict__ a,
                                          const TileRec *__restrict__ b) {
    if (a->n != b->n || a->nnodes != b->nnodes || a->sgn_fixed != b->sgn_fixed) return false;
    const int nn = a->nnodes;
    TCG_ASSERT(nn >= 0 && nn <= 64);
    uint32_t diff = 0;
    if (nn <= 32) {  // uint2 rows: compare two per uint4, the last one by halves
        const uint4 *x = a->rows, *y = b->rows;
        const int full = nn >> 1;
#pragma unroll 4
        for (int i = 0; i < full; ++i) {
            const uint4 p = x[i], q = y[i];
            diff |= (p.x ^ q.x) | (p.y ^ q.y) | (p.z ^ q.z) | (p.w ^ q.w);
        }
        if (nn & 1) {
            const uint2 p = rows2(a)[nn - 1], q = rows2(b)[nn - 1];
            diff |= (p.x ^ q.x) | (p.y ^ q.y);
        }
    } else {
#pragma unroll 4
        for (int i = 0; i < nn; ++i) {
            const uint4 p = a->rows[i], q = b->rows[i];
            diff |= (p.x ^ q.x) | (p.y ^ q.y) | (p.z ^ q.z) | (p.w ^ q.w);
        }
    }
    return diff == 0u;
}

__global__ void __launch_bounds__(THREADS) k_tile_dedup(TileRec *__restrict__ recs,
                                                        const unsigned long long *__restrict__ hashes,
                                                        uint32_t ntiles, uint64_t tile0, int bits,
                                                        uint64_t start, uint64_t end,
                                                        unsigned long long *__restrict__ slots,
                                                        uint32_t smask, uint32_t *__restrict__ dup,
                                                        uint32_t *__restrict__ mint,
                                                        uint32_t *__restrict__ list,
                                                        uint32_t *__restrict__ count,
                                                        const uint32_t *__restrict__ srep, int sh,
                                                        uint32_t *__restrict__ repof) {
    const int lane = threadIdx.x & 31;
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    bool rep = false;
    bool twin = false;  // a tile of a duplicate super-tile (record not built)
    if (t < ntiles && srep) {
        const uint64_t gt = tile0 + t;
        const uint32_t si = (uint32_t)((gt >> sh) - (tile0 >> sh)), rs = srep[si];
        if (rs != si) {
            twin = true;
            const uint32_t tw = (uint32_t)(((((tile0 >> sh) + rs) << sh) | (gt & ((1ull << sh) - 1ull))) - tile0);
            if (recs[tw].fallback) {  // never merged: the tile is its own representative
                const uint4 *src = reinterpret_cast<const uint4 *>(recs + tw);
                uint4 *dst = reinterpret_cast<uint4 *>(recs + t);
                for (int i = 0; i < (int)(sizeof(TileRec) / 16); ++i) dst[i] = src[i];
                rep = true;
                repof[t] = t;
            }
        }
    }
    if (t < ntiles && !twin) {
        const TileRec *r = recs + t;
        const uint64_t b0 = (tile0 + t) << bits, b1 = (tile0 + t + 1) << bits;
        if (r->fallback || b0 < start || b1 > end) {
            rep = true;
            if (repof) repof[t] = t;
        } else {
            const unsigned long long h = hashes[t];
            const unsigned long long tag = (h >> 32) << 32;
            uint32_t at = (uint32_t)h & smask;
            while (true) {
                unsigned long long cur = slots[at];
                if (cur == SLOT_EMPTY) {
                    const unsigned long long prev = atomicCAS(&slots[at], SLOT_EMPTY, tag | t);
                    if (prev == SLOT_EMPTY) {
                        rep = true;
                        if (repof) repof[t] = t;
                        break;
                    }
                    cur = prev;
                }
                if ((cur & 0xffffffff00000000ull) == tag) {
                    const uint32_t o = (uint32_t)cur;
                    TCG_ASSERT(o < ntiles);
                    if (rec_equal(r, recs + o)) {
                        atomicAdd(&dup[o], 1u);
                        atomicMin(&mint[o], t);
                        if (repof) repof[t] = o;
                        break;
                    }
                }
                at = (at + 1) & smask;
            }
        }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, rep);
    if (bal) {
        uint32_t base = 0;
        if (lane == __ffs(bal) - 1) base = atomicAdd(count, (uint32_t)__popc(bal));
        base = __shfl_sync(0xffffffffu, base, __ffs(bal) - 1);
        TCG_ASSERT(!rep || base + __popc(bal & ((1u << lane) - 1u)) < ntiles);
        if (rep) list[base + __popc(bal & ((1u << lane) - 1u))] = t;
    }
}

// Classify every index of [start, end) that falls in tiles tile0 .. tile0+ntiles-1.
// One warp owns a whole tile at a time (its contracted graph staged in a
// per-warp shared-memory slot), so warps never wait on each other.
constexpr int CLS_WARPS = THREADS / 32;


template <int K, bool EVEN, int MODE>
__global__ void __launch_bounds__(THREADS) k_tile_classify(KParams p,
                                                           const TileTables *__restrict__ tt_g,
                                                           const TileRec *__restrict__ recs,
                                                           uint64_t tile0, uint32_t ntiles,
                                                           uint64_t start, uint64_t end,
                                                           DevAgg g, const uint32_t *__restrict__ list,
                                                           const uint32_t *__restrict__ count,
                                                           const uint32_t *__restrict__ dup,
                                                           const uint32_t *__restrict__ mint,
                                                           unsigned long long *__restrict__ tstats) {
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t *adj_s = smem;
    CtaTable tab = carve_table(smem + 32 * K * K);
    TileTables *tt = reinterpret_cast<TileTables *>(
        reinterpret_cast<char *>(smem) + 32 * K * K * 4 + TABLE_SMEM);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    TileRec *rec = reinterpret_cast<TileRec *>(tt + 1) + w;
    stage_adj<K>(p, adj_s);
    for (int i = threadIdx.x; i < (int)(sizeof(TileTables) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t *>(tt)[i] = reinterpret_cast<const uint32_t *>(tt_g)[i];
    tab.init();
    __syncthreads();
    const int bits = tt->bits;
    const uint32_t tsize = 1u << bits;
    // list != nullptr: classify only the representatives, each with the weight
    // of its duplicate group and the group's smallest tile as the witness base
    const uint32_t nwork = list ? *count : ntiles;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(tstats, (unsigned long long)nwork);
    for (uint32_t i = blockIdx.x * CLS_WARPS + w; i < nwork; i += gridDim.x * CLS_WARPS) {
        // list entries: tile, or tile | (a + 1) << 24 for the 32-index slice of
        // A pattern a only (a slice the level-2 path could not take)
        const uint32_t e = list ? list[i] : i;
        const int ssh = slice_shift(tt->la);
        const uint32_t t = e & ((1u << ssh) - 1u), sub = e >> ssh;
        const uint32_t lo0 = sub ? (sub - 1u) << 5 : 0u, lo1 = sub ? lo0 + 32u : tsize;
        const uint32_t weight = list ? 1u + dup[t] : 1u;
        const uint32_t tw = list ? min(t, mint[t]) : t;
        const TileRec *src = recs + t;
        const int nn = src->nnodes;
        const bool fb = src->fallback != 0;
        // nn <= 32: the node pass reads only the low adjacency and link words;
        // stage them as two 32-word arrays (one bank per node: no conflicts)
        uint32_t *ax = reinterpret_cast<uint32_t *>(rec->rows), *az = ax + 32;
        if (!fb && nn <= 32) {
            if (lane < nn) {
                const uint2 row = rows2(src)[lane];
                ax[lane] = row.x;
                az[lane] = row.y;
            }
        } else {
            if (lane < nn) rec->rows[lane] = src->rows[lane];
            if (lane + 32 < nn) rec->rows[lane + 32] = src->rows[lane + 32];
        }
        const int n = src->n;
        const unsigned long long sgf = src->sgn_fixed;
        __syncwarp();
        const uint64_t base = (tile0 + tw) << bits;
        if (!fb && nn <= 32 && !sub) {  // two patchworks per thread (tile sizes are >= 64)
            const uint32_t used = nn >= 32 ? ~0u : ((1u << nn) - 1u);
            for (uint32_t low = lane; low < tsize; low += 64) {
                const unsigned long long fa =
                    tt->fsign[0][low & 63u] ^ tt->fsign[1][(low >> 6) & 63u];
                const unsigned long long fb2 =
                    tt->fsign[0][(low + 32) & 63u] ^ tt->fsign[1][((low + 32) >> 6) & 63u];
                const uint32_t sga = (uint32_t)(sgf | (fa << n));
                const uint32_t sgb = (uint32_t)(sgf | (fb2 << n));
                Regions<1> ra, rb;
                node_pass1x2<EVEN>(ax, az, sga, sgb, used, nn, ra, rb);
#pragma unroll 1
                for (int h = 0; h < 2; ++h) {
                    const uint64_t m = base + low + 32u * h;
                    const bool valid = m >= start && m < end;
                    const uint32_t SG1[1] = {h ? sgb : sga};
                    const Result r = finish<1, EVEN, false>(p, SG1, h ? rb : ra, p.maxreg);
                    uint64_t k = 0;
                    if (valid) {
                        if (r.status == TCG_OK) k = r.key;
                        else atomicMin(g.bad, (unsigned long long)m);
                    }
                    tab.add<true>(g, k, r.nreg, m, weight);
                }
            }
            __syncwarp();
            continue;
        }
        for (uint32_t low = lo0 + lane; low < lo1; low += 32) {
            const uint64_t m = base + low;
            const bool valid = m >= start && m < end;
            Result r;
            if (fb) {
                const uint64_t sigma = MODE == MODE_REP ? rep_to_sigma(p.d, m) : m;
                r = classify<K, EVEN>(p, adj_s, valid ? sigma : 0ull);
            } else {
                r = classify_tile<EVEN>(p, *tt, rec->rows, sgf, n, nn, low);
            }
            uint64_t k = 0;
            if (valid) {
                if (r.status == TCG_OK) k = r.key;
                else atomicMin(g.bad, (unsigned long long)m);
            }
            tab.add<true>(g, k, r.nreg, m, weight);
        }
        __syncwarp();
    }
    __syncthreads();
    tab.flush(g);
}
