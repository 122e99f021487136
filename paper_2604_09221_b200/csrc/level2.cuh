// level2.cuh -- level-2 records (A points fixed per record; direct and
// two-stage builds), their deduplication and the level-2 classifiers.
// Included by tcg.cu inside its anonymous namespace.

// ------------------------------------------------------------ level 2
// Level-2 contraction of a representative tile (odd degree, <= 64 nodes).
// Fix the signs of the A points (tile-local index bits 5..bits-1) as well:
// the fixed components and the A nodes then merge, through same-sign edges
// and antipodal links, into "super-nodes" -- subsets of regions whatever
// the B signs (bits 0..4) are.  A super-node mixes signs, so its edges to a
// B node are recorded by the sign of the member they leave from (plusB /
// minusB); edges between two super-nodes are always crossed (a same-sign
// edge would have merged them).  One record (header + one u64 per
// super-node) describes 32 patchworks, one per lane.  Records built from
// different tiles coincide far more often than level-1 records do, and are
// deduplicated the same way (exact comparison, weights add, witness = the
// smallest (tile, A) position of the group).
//   word[s] = crossS | (plusB | minusB << nB | linkB << 2nB | self << 3nB) << 32

__device__ __forceinline__ uint32_t l2_compress(const TileTables &tt, uint32_t freemask) {
    if (tt.l2shift >= 0) return (freemask >> tt.l2shift) & ((1u << tt.nB) - 1u);
    uint32_t r = 0;
    while (freemask) {
        const int f = __ffs(freemask) - 1;
        freemask &= freemask - 1u;
        r |= 1u << tt.l2j[f];
    }
    return r;
}

// <= 32-node records (98 % at d=7): the same super-node BFS without
// per-super-node arrays in local memory.  Node labels (bytes) and the
// cross-adjacency words cs[q] are lane-private shared memory (bank = lane);
// when super-node q closes, its crossed neighbours that are already labelled
// (earlier super-nodes) set cs[q] and cs[q2] -- every pair is met once, from
// its later end -- and the record's high half (B-node words, self flag) is
// written immediately; the low halves (cs) follow at the end.
constexpr int L2B_CS = 24;          // super-nodes per level-2 record (also <= 32 - nB)
constexpr int L2B_WORDS = 16 + L2B_CS;  // labels (64 nodes, 4 per word) | cs[L2B_CS]
constexpr int L2B_SLOT = 256;       // staged rows per tile: 32 x uint2 (wider tiles read global)
// level 2 needs tile bits >= 6 (la >= 1): at most 16 tiles per warp
constexpr size_t L2B_SMEM = (size_t)L2B_WORDS * 4 * THREADS + (THREADS / 32) * 16 * L2B_SLOT;

template <typename MT>
__device__ __forceinline__ int l2_build_lbl(const TileTables &tt,
                                            const TileRec *__restrict__ rec,
                                            const uint4 *__restrict__ R4, uint32_t a, int mmax,
                                            unsigned long long *out, unsigned long long &hout,
                                            uint32_t *mine) {
    constexpr bool WIDE = sizeof(MT) == 8;
    const int n = rec->n, nB = tt.nB;
    uint8_t *lb = reinterpret_cast<uint8_t *>(mine);
    uint32_t *cs = mine + 16 * THREADS;
    const uint32_t lowA = a << 5;
    const unsigned long long fsA = tt.fsign[0][lowA & 63u] ^ tt.fsign[1][(lowA >> 6) & 63u];
    const MT one = 1;
    const MT sg1 = (MT)rec->sgn_fixed | ((MT)((uint32_t)fsA & tt.fa) << n);
    const MT G = (n >= 8 * (int)sizeof(MT) ? ~(MT)0 : ((one << n) - one)) | ((MT)tt.fa << n);
    const MT FBn = (MT)tt.fbm << n;
    uint32_t *out32 = reinterpret_cast<uint32_t *>(out);
    MT unv = G, done = 0;
    uint32_t hh = 0x9E3779B9u;
    int m = 0;
    auto label = [&](int v) -> uint32_t { return lb[(v >> 2) * (4 * THREADS) + (v & 3)]; };
    while (unv) {
        if (m == mmax) return -1;
        MT f = unv & ((MT)0 - unv);
        unv ^= f;
        MT M = f, cg = 0, pb = 0, mb = 0, lk = 0;
        while (f) {
            const int u = WIDE ? __ffsll((long long)f) - 1 : __ffs((uint32_t)f) - 1;
            f &= f - one;
            TCG_ASSERT(u >= 0 && u < 64 && m < 64);
            lb[(u >> 2) * (4 * THREADS) + (u & 3)] = (uint8_t)m;
            MT rx, ry;
            if constexpr (WIDE) {
                const uint4 r = R4[u];
                rx = (MT)r.x | ((MT)r.y << 32);
                ry = (MT)r.z | ((MT)r.w << 32);
            } else {
                const uint2 r = reinterpret_cast<const uint2 *>(R4)[u];
                rx = r.x;
                ry = r.y;
            }
            const MT s = (sg1 >> u) & one;
            const MT diff = sg1 ^ ((MT)0 - s);  // nodes of the other sign
            const MT nw = ((rx & ~diff) | ry) & unv;
            unv ^= nw;
            f |= nw;
            M |= nw;
            cg |= rx & G & diff;
            const MT bp = rx & FBn;
            pb |= s ? bp : (MT)0;
            mb |= s ? (MT)0 : bp;
            lk |= ry & FBn;
        }
        // crossed neighbours in earlier super-nodes (labelled): both ends' cs words
        uint32_t c = 0;
        const MT x = cg & done;
        for (uint32_t w = (uint32_t)x; w; w &= w - 1u) c |= 1u << label(__ffs(w) - 1);
        if constexpr (WIDE)
            for (uint32_t w = (uint32_t)(x >> 32); w; w &= w - 1u) c |= 1u << label(31 + __ffs(w));
        TCG_ASSERT(m < L2B_CS);
        cs[m * THREADS] = c;
        for (uint32_t y = c; y; y &= y - 1u) cs[(__ffs(y) - 1) * THREADS] |= 1u << m;
        const uint32_t self = (cg & M) != (MT)0;
        const uint32_t hi = l2_compress(tt, (uint32_t)(pb >> n)) |
                            l2_compress(tt, (uint32_t)(mb >> n)) << nB |
                            l2_compress(tt, (uint32_t)(lk >> n)) << (2 * nB) | self << (3 * nB);
        out32[2 * (1 + m) + 1] = hi;
        hh = (hh ^ hi) * 0x85EBCA77u;
        hh ^= hh >> 13;
        done |= M;
        ++m;
    }
    out[0] = (unsigned long long)m;
    uint32_t hl = 0xC2B2AE3Du;
    for (int q = 0; q < m; ++q) {
        const uint32_t c = cs[q * THREADS];
        out32[2 * (1 + q)] = c;
        hl = (hl ^ c) * 0x9E3779B1u;
        hl ^= hl >> 15;
    }
    hout = mix64(((unsigned long long)hh << 32 | hl) + 0x51ED2701ull * (unsigned long long)(m + 1));
    return m;
}

// Level 2 in even degree.  Antipodal partners carry the same sign, and a
// region's orientation matters (the root is its unique region with an
// orientation-reversing cycle), so a super-node keeps each member's parity
// relative to its seed (same-sign edges keep it, links flip it) and an odd
// flag (a member reached with both parities).  Its record is two words:
//   word0 = cs | self << 30 | odd << 31
//   word1 = P10 | P11 << nB | P00 << 2nB | P01 << 3nB | LK0 << 4nB | LK1 << 5nB
// where Psp = B nodes adjacent to members of sign s and parity p, LKp = B
// nodes linked to members of parity p.
template <typename MT>
__device__ __forceinline__ int l2_build_even(const TileTables &tt,
                                             const TileRec *__restrict__ rec,
                                             const uint4 *__restrict__ R4, uint32_t a, int mmax,
                                             unsigned long long *out, unsigned long long &hout,
                                             uint32_t *mine) {
    constexpr bool WIDE = sizeof(MT) == 8;
    const int n = rec->n, nB = tt.nB;
    uint8_t *lb = reinterpret_cast<uint8_t *>(mine);
    uint32_t *cs = mine + 16 * THREADS;
    const uint32_t lowA = a << 5;
    const unsigned long long fsA = tt.fsign[0][lowA & 63u] ^ tt.fsign[1][(lowA >> 6) & 63u];
    const MT one = 1;
    const MT sg1 = (MT)rec->sgn_fixed | ((MT)((uint32_t)fsA & tt.fa) << n);
    const MT G = (n >= 8 * (int)sizeof(MT) ? ~(MT)0 : ((one << n) - one)) | ((MT)tt.fa << n);
    const MT FBn = (MT)tt.fbm << n;
    MT unv = G, done = 0, q = 0;  // q: parity-1 nodes (relative to their super-node's seed)
    unsigned long long hh = 0x9E3779B97F4A7C15ull;
    int m = 0;
    auto label = [&](int v) -> uint32_t { return lb[(v >> 2) * (4 * THREADS) + (v & 3)]; };
    auto cmp = [&](MT x) -> unsigned long long { return l2_compress(tt, (uint32_t)(x >> n)); };
    while (unv) {
        if (m == mmax) return -1;
        MT f = unv & ((MT)0 - unv);
        unv ^= f;
        MT M = f, cg = 0, p10 = 0, p11 = 0, p00 = 0, p01 = 0, lk0 = 0, lk1 = 0;
        bool odd = false;
        while (f) {
            const int u = WIDE ? __ffsll((long long)f) - 1 : __ffs((uint32_t)f) - 1;
            f &= f - one;
            TCG_ASSERT(u >= 0 && u < 64 && m < 64);
            lb[(u >> 2) * (4 * THREADS) + (u & 3)] = (uint8_t)m;
            MT rx, ry;
            if constexpr (WIDE) {
                const uint4 r = R4[u];
                rx = (MT)r.x | ((MT)r.y << 32);
                ry = (MT)r.z | ((MT)r.w << 32);
            } else {
                const uint2 r = reinterpret_cast<const uint2 *>(R4)[u];
                rx = r.x;
                ry = r.y;
            }
            const MT s = (sg1 >> u) & one, pu = (q >> u) & one;
            const MT diff = sg1 ^ ((MT)0 - s);        // nodes of the other sign
            const MT eqm = pu ? q : ~q;                 // nodes with u's parity
            const MT te = rx & ~diff & G, tl = ry & G;  // same-sign edges keep, links flip
            const MT nt = te & unv, np = tl & unv;
            odd |= ((nt & np) | (te & ~unv & ~eqm) | (tl & ~unv & eqm)) != (MT)0;
            q |= pu ? nt : np;
            const MT nw = nt | np;
            unv ^= nw;
            f |= nw;
            M |= nw;
            cg |= rx & G & diff;
            const MT bp = rx & FBn, bl = ry & FBn;
            if (s) {
                if (pu) p11 |= bp; else p10 |= bp;
            } else {
                if (pu) p01 |= bp; else p00 |= bp;
            }
            if (pu) lk1 |= bl; else lk0 |= bl;
        }
        uint32_t c = 0;
        const MT x = cg & done;
        for (uint32_t w = (uint32_t)x; w; w &= w - 1u) c |= 1u << label(__ffs(w) - 1);
        if constexpr (WIDE)
            for (uint32_t w = (uint32_t)(x >> 32); w; w &= w - 1u) c |= 1u << label(31 + __ffs(w));
        const uint32_t self = (cg & M) != (MT)0;
        TCG_ASSERT(m < L2B_CS);
        cs[m * THREADS] = c | self << 30 | (uint32_t)odd << 31;
        for (uint32_t y = c; y; y &= y - 1u) cs[(__ffs(y) - 1) * THREADS] |= 1u << m;
        const unsigned long long w1 = cmp(p10) | cmp(p11) << nB | cmp(p00) << (2 * nB) |
                                      cmp(p01) << (3 * nB) | cmp(lk0) << (4 * nB) |
                                      cmp(lk1) << (5 * nB);
        out[2 + 2 * m] = w1;
        hh = mix64(hh ^ w1);
        done |= M;
        ++m;
    }
    out[0] = (unsigned long long)m;
    uint32_t hl = 0xC2B2AE3Du;
    for (int k = 0; k < m; ++k) {
        const uint32_t c = cs[k * THREADS];
        out[1 + 2 * k] = c;
        hl = (hl ^ c) * 0x9E3779B1u;
        hl ^= hl >> 15;
    }
    hout = mix64((hh ^ hl) + 0x51ED2701ull * (unsigned long long)(m + 1));
    return m;
}

// One thread per (representative tile, A pattern) of list1[i0 .. i0+nb).
// Tiles the level-2 path cannot take go to oldlist for the level-1
// classifier: whole tiles (entry = tile: range ends, fallback) or single A
// slices whose super-node graph is too large (entry = tile | (a + 1) << 24).
template <bool EVEN>
__global__ void __launch_bounds__(THREADS) k_l2_build(const TileTables *__restrict__ tt_g,
                                                      const TileRec *__restrict__ recs,
                                                      const uint32_t *__restrict__ list1,
                                                      const uint32_t *__restrict__ dup1,
                                                      const uint32_t *__restrict__ mint1,
                                                      uint32_t i0, uint32_t nb, uint64_t tile0,
                                                      uint64_t start, uint64_t end,
                                                      unsigned long long *__restrict__ pool,
                                                      uint32_t stride,
                                                      unsigned long long *__restrict__ hashes,
                                                      uint32_t *__restrict__ wts,
                                                      uint32_t *__restrict__ poss,
                                                      uint32_t *__restrict__ oldlist,
                                                      uint32_t *__restrict__ oldcount) {
    __shared__ TileTables tts;
    extern __shared__ __align__(16) uint32_t l2smem[];
    uint32_t *mine = l2smem + threadIdx.x;
    for (int i = threadIdx.x; i < (int)(sizeof(TileTables) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t *>(&tts)[i] = reinterpret_cast<const uint32_t *>(tt_g)[i];
    __syncthreads();
    const TileTables &tt = tts;
    const int la = tt.la, bits = tt.bits;
    const int mmax = min(32 - tt.nB, L2B_CS);
    const uint32_t nrec = nb << la;
    // the 2^la lanes of one tile stage its (<= 32-node) rows in shared memory
    // first: the breadth-first pass then reads rows at shared-memory latency
    const int lane = threadIdx.x & 31, lpt = la < 5 ? la : 5;
    uint4 *slot = reinterpret_cast<uint4 *>(l2smem + L2B_WORDS * THREADS) +
                  (L2B_SLOT / 16) * ((threadIdx.x >> 5) * (32 >> lpt) + (lane >> lpt));
    for (uint32_t jb = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); jb < nrec;
         jb += gridDim.x * blockDim.x) {  // warp-uniform
        const uint32_t j = jb + lane;
        const bool valid = j < nrec;
        const uint32_t i = i0 + (j >> la), a = j & ((1u << la) - 1u);
        const uint32_t t = valid ? list1[i] : 0u;
        const TileRec *rec = recs + t;
        if (valid && rec->nnodes <= 32) {  // 256 bytes of uint2 rows
            const uint4 *src = rec->rows;
            for (int q = lane & ((1 << lpt) - 1); q < 16; q += 1 << lpt) slot[q] = src[q];
        }
        __syncwarp();
        if (valid) {
            const int nn = rec->nnodes;
            const uint64_t b0 = (tile0 + t) << bits, b1 = (tile0 + t + 1) << bits;
            if (rec->fallback || b0 < start || b1 > end) {
                if (a == 0) oldlist[atomicAdd(oldcount, 1u)] = t;
                wts[j] = 0u;
            } else {
                unsigned long long *out = pool + (size_t)j * stride;
                unsigned long long h = 0;
                int m;
                if constexpr (EVEN)
                    m = nn <= 32 ? l2_build_even<uint32_t>(tt, rec, slot, a, mmax, out, h, mine)
                                 : l2_build_even<unsigned long long>(tt, rec, rec->rows, a, mmax, out,
                                                                     h, mine);
                else
                    m = nn <= 32 ? l2_build_lbl<uint32_t>(tt, rec, slot, a, mmax, out, h, mine)
                                 : l2_build_lbl<unsigned long long>(tt, rec, rec->rows, a, mmax, out,
                                                                    h, mine);
                if (m < 0) {
                    oldlist[atomicAdd(oldcount, 1u)] = t | ((a + 1u) << slice_shift(la));
                    wts[j] = 0u;
                } else {
                    hashes[j] = h;
                    wts[j] = 1u + dup1[t];
                    poss[j] = (min(t, mint1[t]) << la) | a;
                }
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------- two-stage level 2
// Stage 1 (k_l15_build, one lane per (representative tile, A1 pattern)):
// fix the A1 nodes (tile bits 5, 6) and merge components + A1 nodes into
// super-nodes, keeping their relations to the F nodes (B and A2) by member
// sign; a record is a bit stream (L15Bits) of, per super-node,
//   F relations = plusF | minusF << nF | linkF << 2nF   (3 nF bits), then
//   cs row (m bits) + self flag (1 bit),
// 3 nF + m + 1 bits per super-node (~23 words at C3 against 41 for two
// words per super-node), and records are deduplicated like level-2 records.  Stage 2 (k_l2_from_l15, one
// lane per (distinct stage-1 record, A2 pattern)) fixes the A2 nodes and
// merges again, emitting ordinary level-2 records (same format and hash as
// k_l2_build, so the rest of the pipeline is unchanged).  Either stage sets
// *fail when a record would exceed its super-node budget; the host then
// redoes the batch on the direct path.
// dynamic shared memory of k_l15_build: labels | cs, then one 1 KB row slot
// per tile of each warp (at least 2 A1 bits: <= 8 tiles per warp)
constexpr size_t L15_SMEM_MAX = (size_t)L2B_WORDS * 4 * THREADS + (THREADS / 32) * 8 * 1024 + 4096;
constexpr int L15_MAXM = L2B_CS;  // stage-1 super-nodes (cs bit 31 is the self flag)

// F-space compression by byte lookup tables (k_l15_build stages them in shared memory)
struct L15Lut {
    uint32_t b[4][256];  // byte k of a free-node mask -> its F bits
};

__device__ __forceinline__ unsigned long long l15_compress(const L15Lut &L, uint32_t fm) {
    return (unsigned long long)(L.b[0][fm & 0xffu] | L.b[1][(fm >> 8) & 0xffu] |
                                L.b[2][(fm >> 16) & 0xffu] | L.b[3][fm >> 24]);
}

// Stage-1 record bit stream (words 1..): the m super-nodes' F relations
// (3 nF bits each), then their cs rows (m bits) + self flag (1 bit) each;
// word 0 = m | stream words << 16.  Unused high bits of the last word are 0,
// so equal records are equal word for word.
struct L15Bits {
    unsigned long long acc = 0;
    int nacc = 0, wi = 1;
    __device__ __forceinline__ void put(unsigned long long *out, unsigned long long v, int nb) {
        // v < 2^nb, 1 <= nb <= 63
        acc |= v << nacc;
        nacc += nb;
        if (nacc >= 64) {
            out[wi++] = acc;
            nacc -= 64;
            acc = nacc ? v >> (nb - nacc) : 0ull;
        }
    }
    __device__ __forceinline__ int finish(unsigned long long *out) {
        if (nacc) out[wi++] = acc;
        return wi - 1;
    }
};

__device__ __forceinline__ unsigned long long l15_bits(const unsigned long long *r1, int pos, int nb) {
    const int w = pos >> 6, o = pos & 63;
    unsigned long long v = __ldg(r1 + 1 + w) >> o;
    if (o + nb > 64) v |= __ldg(r1 + 2 + w) << (64 - o);
    return v & ((1ull << nb) - 1ull);
}

template <typename MT>
__device__ __forceinline__ int l15_build(const TileTables &tt, const L15Lut &lut,
                                         const TileRec *__restrict__ rec,
                                         const uint4 *__restrict__ R4, uint32_t a1,
                                         unsigned long long *out, unsigned long long &hout,
                                         uint32_t *mine) {
    constexpr bool WIDE = sizeof(MT) == 8;
    const int n = rec->n, nF = tt.nB + tt.nA2;
    uint8_t *lb = reinterpret_cast<uint8_t *>(mine);
    uint32_t *cs = mine + 16 * THREADS;
    const uint32_t lowA = a1 << 5;
    const unsigned long long fsA = tt.fsign[0][lowA & 63u] ^ tt.fsign[1][(lowA >> 6) & 63u];
    const MT one = 1;
    const MT sg1 = (MT)rec->sgn_fixed | ((MT)((uint32_t)fsA & tt.fa1) << n);
    const MT G = (n >= 8 * (int)sizeof(MT) ? ~(MT)0 : ((one << n) - one)) | ((MT)tt.fa1 << n);
    const MT nsg1 = ~sg1;
    const uint32_t fbm32 = tt.fbm | tt.fa2;
    MT unv = G, done = 0;
    unsigned long long hh = 0x9E3779B97F4A7C15ull;
    int m = 0;
    L15Bits bw;
    auto label = [&](int v) -> uint32_t { return lb[(v >> 2) * (4 * THREADS) + (v & 3)]; };
    while (unv) {
        if (m == tt.l15max) return -1;
        MT f = unv & ((MT)0 - unv);
        unv ^= f;
        MT M = f, cg = 0;
        uint32_t pb = 0, mb = 0, lk = 0;  // F relations in free-node space
        while (f) {
            const int u = WIDE ? __ffsll((long long)f) - 1 : __ffs((uint32_t)f) - 1;
            f &= f - one;
            TCG_ASSERT(u >= 0 && u < 64 && m < 64);
            lb[(u >> 2) * (4 * THREADS) + (u & 3)] = (uint8_t)m;
            MT rx, ry;
            if constexpr (WIDE) {
                const uint4 r = R4[u];
                rx = (MT)r.x | ((MT)r.y << 32);
                ry = (MT)r.z | ((MT)r.w << 32);
            } else {
                const uint2 r = reinterpret_cast<const uint2 *>(R4)[u];
                rx = r.x;
                ry = r.y;
            }
            const MT s = (sg1 >> u) & one;
            const MT diff = s ? nsg1 : sg1;
            const MT nw = ((rx & ~diff) | ry) & unv;
            unv ^= nw;
            f |= nw;
            M |= nw;
            cg |= rx & diff;  // only read as cg & done / cg & M, both inside G
            const uint32_t bp = (uint32_t)(rx >> n) & fbm32;
            pb |= s ? bp : 0u;
            mb |= s ? 0u : bp;
            lk |= (uint32_t)(ry >> n) & fbm32;
        }
        uint32_t c = 0;
        const MT x = cg & done;
        for (uint32_t w = (uint32_t)x; w; w &= w - 1u) c |= 1u << label(__ffs(w) - 1);
        if constexpr (WIDE)
            for (uint32_t w = (uint32_t)(x >> 32); w; w &= w - 1u) c |= 1u << label(31 + __ffs(w));
        const uint32_t self = (cg & M) != (MT)0;
        TCG_ASSERT(m < L2B_CS);
        cs[m * THREADS] = c | self << 31;
        for (uint32_t y = c; y; y &= y - 1u) cs[(__ffs(y) - 1) * THREADS] |= 1u << m;
        unsigned long long w1;
        if (tt.l15sh >= 0) {  // contiguous B | A1 | A2 free nodes (A1 bits are 0 here)
            const uint32_t bmk = (1u << tt.nB) - 1u, sh = (uint32_t)tt.l15sh;
            const uint32_t xp = pb, xm = mb, xl = lk;
            w1 = (unsigned long long)((xp & bmk) | ((xp >> sh) & ~bmk)) |
                 (unsigned long long)((xm & bmk) | ((xm >> sh) & ~bmk)) << nF |
                 (unsigned long long)((xl & bmk) | ((xl >> sh) & ~bmk)) << (2 * nF);
        } else {
            w1 = l15_compress(lut, pb) | l15_compress(lut, mb) << nF | l15_compress(lut, lk) << (2 * nF);
        }
        bw.put(out, w1, 3 * nF);
        hh = mix64(hh ^ w1);
        done |= M;
        ++m;
    }
    uint32_t hl = 0xC2B2AE3Du;
    for (int k = 0; k < m; ++k) {
        const uint32_t c = cs[k * THREADS];
        bw.put(out, (unsigned long long)(c & 0xffffffu) | (unsigned long long)(c >> 31) << m, m + 1);
        hl = (hl ^ c) * 0x9E3779B1u;
        hl ^= hl >> 15;
    }
    const int nw = bw.finish(out);
    out[0] = (unsigned long long)m | (unsigned long long)nw << 16;
    hout = mix64((hh ^ hl) + 0x51ED2701ull * (unsigned long long)(m + 1));
    return m;
}

// One lane per (representative tile, A1 pattern) of list1[i0 .. i0+nb): 4 per tile.
__global__ void __launch_bounds__(THREADS) k_l15_build(const TileTables *__restrict__ tt_g,
                                                       const TileRec *__restrict__ recs,
                                                       const uint32_t *__restrict__ list1,
                                                       const uint32_t *__restrict__ dup1,
                                                       const uint32_t *__restrict__ mint1,
                                                       uint32_t i0, uint32_t nb, uint64_t tile0,
                                                       uint64_t start, uint64_t end,
                                                       unsigned long long *__restrict__ pool,
                                                       uint32_t stride,
                                                       unsigned long long *__restrict__ hashes,
                                                       uint32_t *__restrict__ wts,
                                                       uint32_t *__restrict__ poss,
                                                       uint32_t *__restrict__ oldlist,
                                                       uint32_t *__restrict__ oldcount,
                                                       uint32_t *__restrict__ fail,
                                                       const L15Lut *__restrict__ lut_g,
                                                       int slotq, int lut_smem) {
    __shared__ TileTables tts;
    extern __shared__ __align__(16) uint32_t l2smem[];
    uint32_t *mine = l2smem + threadIdx.x;
    // dynamic shared memory: labels | cs (lane-private), one row slot of
    // slotq uint4 rows per tile of each warp, then (lut_smem) the lookup tables
    const int nslot = (THREADS / 32) * (32 >> tt_g->la1);
    uint32_t *lutsm = l2smem + L2B_WORDS * THREADS + nslot * slotq * 4;
    const L15Lut &luts = lut_smem ? *reinterpret_cast<const L15Lut *>(lutsm) : *lut_g;
    for (int i = threadIdx.x; i < (int)(sizeof(TileTables) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t *>(&tts)[i] = reinterpret_cast<const uint32_t *>(tt_g)[i];
    for (int i = threadIdx.x; i < (int)(sizeof(L15Lut) / 4); i += blockDim.x)
        if (lut_smem) lutsm[i] = reinterpret_cast<const uint32_t *>(lut_g)[i];
    __syncthreads();
    const TileTables &tt = tts;
    const int bits = tt.bits;
    const int la1 = tt.la1;
    const uint32_t nrec = nb << la1;
    const int lane = threadIdx.x & 31;
    // one row slot per tile of the warp: 16 uint4 hold <= 32-node rows (uint2);
    // tiles of 33..slotq nodes (all of d = 7 at 2^12-index tiles have > 32)
    // are staged too, wider ones read their rows from global memory
    uint4 *slot = reinterpret_cast<uint4 *>(l2smem + L2B_WORDS * THREADS) +
                  slotq * ((threadIdx.x >> 5) * (32 >> tt.la1) + (lane >> tt.la1));
    for (uint32_t jb = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); jb < nrec;
         jb += gridDim.x * blockDim.x) {  // warp-uniform
        const uint32_t j = jb + lane;
        const bool valid = j < nrec;
        const uint32_t i = i0 + (j >> la1), a1 = j & ((1u << la1) - 1u);
        const uint32_t t = valid ? list1[i] : 0u;
        const TileRec *rec = recs + t;
        if (valid && (rec->nnodes <= 32 || rec->nnodes <= slotq)) {  // uint2 rows, or nnodes uint4 rows
            const uint4 *src = rec->rows;
            const int nq = rec->nnodes <= 32 ? 16 : rec->nnodes;
            for (int q = lane & ((1 << la1) - 1); q < nq; q += 1 << la1) slot[q] = src[q];
        }
        __syncwarp();
        if (valid) {
            const int nn = rec->nnodes;
            const uint64_t b0 = (tile0 + t) << bits, b1 = (tile0 + t + 1) << bits;
            if (rec->fallback || b0 < start || b1 > end) {
                if (a1 == 0) oldlist[atomicAdd(oldcount, 1u)] = t;
                wts[j] = 0u;
            } else {
                unsigned long long *out = pool + (size_t)j * stride;
                unsigned long long h = 0;
                const int m = nn <= 32 ? l15_build<uint32_t>(tt, luts, rec, slot, a1, out, h, mine)
                                       : l15_build<unsigned long long>(tt, luts, rec, nn <= slotq ? slot : rec->rows,
                                                                       a1, out, h, mine);
                if (m < 0) {
                    atomicOr(fail, 1u);
                    wts[j] = 0u;
                } else {
                    hashes[j] = h;
                    wts[j] = 1u + dup1[t];
                    poss[j] = (min(t, mint1[t]) << la1) | a1;
                }
            }
        }
        __syncwarp();
    }
}

// One lane per (distinct stage-1 record list15[i], A2 pattern): 4 per record.
// NA: A2 nodes the per-record sameA / crossA rows are sized for.  NA <= 4
// (d = 7 raw, 2^12-index tiles: nA2 = 3) keeps them in registers (static
// indices); the general instance (16) keeps the dynamically indexed arrays,
// which live in local memory.
template <int NA>
__global__ void __launch_bounds__(THREADS) k_l2_from_l15(const TileTables *__restrict__ tt_g,
                                                         const unsigned long long *__restrict__ pool1,
                                                         uint32_t stride1,
                                                         const uint32_t *__restrict__ list15,
                                                         const uint32_t *__restrict__ count15,
                                                         const uint32_t *__restrict__ w15,
                                                         const uint32_t *__restrict__ pos15,
                                                         unsigned long long *__restrict__ pool,
                                                         uint32_t stride,
                                                         unsigned long long *__restrict__ hashes,
                                                         uint32_t *__restrict__ wts,
                                                         uint32_t *__restrict__ poss,
                                                         uint32_t *__restrict__ fail) {
    __shared__ TileTables tts;
    extern __shared__ __align__(16) uint32_t l2smem[];
    uint32_t *mine = l2smem + threadIdx.x;
    uint8_t *lb = reinterpret_cast<uint8_t *>(mine);
    uint32_t *cs = mine + 16 * THREADS, *hw = cs + L2B_CS * THREADS;
    for (int i = threadIdx.x; i < (int)(sizeof(TileTables) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t *>(&tts)[i] = reinterpret_cast<const uint32_t *>(tt_g)[i];
    __syncthreads();
    const TileTables &tt = tts;
    const int nB = tt.nB, nA2 = tt.nA2, nF = nB + nA2;
    const uint32_t bm = (1u << nB) - 1u, a2m = (1u << nA2) - 1u;
    const unsigned long long fm = (1ull << nF) - 1ull;
    const int mmax = min(32 - nB, L2B_CS);
    const int la2 = tt.la2;
    const uint32_t nrec = *count15 << la2;
    // stage-1 super-node s of an m1-node record (L15Bits): w1 = F relations,
    // w0 = cs | self << 31
    auto rw1 = [&](const unsigned long long *r1, int s2) -> unsigned long long {
        return l15_bits(r1, 3 * nF * s2, 3 * nF);
    };
    auto rw0 = [&](const unsigned long long *r1, int s2, int m1) -> uint32_t {
        const uint32_t x = (uint32_t)l15_bits(r1, m1 * 3 * nF + s2 * (m1 + 1), m1 + 1);
        return (x & ((1u << m1) - 1u)) | (x >> m1) << 31;
    };
    auto label = [&](int v) -> uint32_t { return lb[(v >> 2) * (4 * THREADS) + (v & 3)]; };
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < nrec; j += gridDim.x * blockDim.x) {
        const uint32_t j1 = list15[j >> la2], a2 = j & ((1u << la2) - 1u);
        const unsigned long long *r1 = pool1 + (size_t)j1 * stride1;
        const int m1 = (int)(r1[0] & 0xffffu);
        const uint32_t SA2 = tt.a2sign[a2];
        // A2 rows toward the stage-1 super-nodes (same-sign or linked / crossed)
        uint32_t sameA[NA], crossA[NA];
#pragma unroll
        for (int k = 0; k < NA; ++k) sameA[k] = crossA[k] = 0u;
        for (int s = 0; s < m1; ++s) {
            const unsigned long long w1 = rw1(r1, s);
            const uint32_t pA = (uint32_t)(w1 >> nB) & a2m, mA = (uint32_t)(w1 >> (nF + nB)) & a2m,
                           lA = (uint32_t)(w1 >> (2 * nF + nB)) & a2m;
            const uint32_t same = (pA & SA2) | (mA & ~SA2) | lA, cross = (pA & ~SA2) | (mA & SA2);
            if constexpr (NA <= 4) {  // bits >= nA2 are zero (a2m)
#pragma unroll
                for (int k = 0; k < NA; ++k) {
                    sameA[k] |= ((same >> k) & 1u) << s;
                    crossA[k] |= ((cross >> k) & 1u) << s;
                }
            } else {
                for (uint32_t y = same; y; y &= y - 1u) sameA[__ffs(y) - 1] |= 1u << s;
                for (uint32_t y = cross; y; y &= y - 1u) crossA[__ffs(y) - 1] |= 1u << s;
            }
        }
        const int nn = m1 + nA2;
        if (nn > 32) {  // 32-bit node masks: the host redoes the batch directly
            atomicOr(fail, 1u);
            wts[j] = 0u;
            continue;
        }
        const uint32_t G = nn >= 32 ? ~0u : ((1u << nn) - 1u);
        uint32_t unv = G, done = 0, hh = 0x9E3779B9u;
        unsigned long long *out = pool + (size_t)j * stride;
        int m = 0;
        bool bad = false;
        while (unv) {
            if (m == mmax) { bad = true; break; }
            uint32_t f = unv & (0u - unv);
            unv ^= f;
            uint32_t M = f, cg = 0, pb = 0, mb = 0, lk = 0, selfany = 0;
            while (f) {
                const int v = __ffs(f) - 1;
                f &= f - 1u;
                TCG_ASSERT(v >= 0 && v < 64 && m < 64);
                lb[(v >> 2) * (4 * THREADS) + (v & 3)] = (uint8_t)m;
                uint32_t same, cross;
                if (v < m1) {
                    const unsigned long long w0 = rw0(r1, v, m1), w1 = rw1(r1, v);
                    const uint32_t pA = (uint32_t)(w1 >> nB) & a2m,
                                   mA = (uint32_t)(w1 >> (nF + nB)) & a2m,
                                   lA = (uint32_t)(w1 >> (2 * nF + nB)) & a2m;
                    same = ((pA & SA2) | (mA & ~SA2) | lA) << m1;
                    cross = ((uint32_t)w0 & 0x7fffffffu) | (((pA & ~SA2) | (mA & SA2)) << m1);
                    selfany |= (uint32_t)w0 >> 31;
                    pb |= (uint32_t)(w1 & fm) & bm;
                    mb |= (uint32_t)((w1 >> nF) & fm) & bm;
                    lk |= (uint32_t)((w1 >> (2 * nF)) & fm) & bm;
                } else {
                    const int k = v - m1;
                    const uint32_t sk = (SA2 >> k) & 1u, own = sk ? SA2 : ~SA2;
                    uint32_t sAk, cAk;
                    if constexpr (NA <= 4) {
                        sAk = sameA[0];
                        cAk = crossA[0];
#pragma unroll
                        for (int q = 1; q < NA; ++q) {
                            sAk = k == q ? sameA[q] : sAk;
                            cAk = k == q ? crossA[q] : cAk;
                        }
                    } else {
                        sAk = sameA[k];
                        cAk = crossA[k];
                    }
                    same = sAk | (((tt.a2adjA2[k] & own) | tt.a2linkA2[k]) << m1);
                    cross = cAk | ((tt.a2adjA2[k] & ~own & a2m) << m1);
                    if (sk) pb |= tt.a2adjB[k];
                    else mb |= tt.a2adjB[k];
                    lk |= tt.a2linkB[k];
                }
                const uint32_t nw = same & unv;
                unv ^= nw;
                f |= nw;
                M |= nw;
                cg |= cross;
            }
            uint32_t c = 0;
            for (uint32_t w = cg & done; w; w &= w - 1u) c |= 1u << label(__ffs(w) - 1);
            TCG_ASSERT(m < L2B_CS);
            cs[m * THREADS] = c;
            for (uint32_t y = c; y; y &= y - 1u) cs[(__ffs(y) - 1) * THREADS] |= 1u << m;
            const uint32_t self = ((cg & M) != 0u) | selfany;
            hw[m * THREADS] = pb | mb << nB | lk << (2 * nB) | self << (3 * nB);
            done |= M;
            ++m;
        }
        if (bad) {
            atomicOr(fail, 1u);
            wts[j] = 0u;
            continue;
        }
        // canonical order: super-nodes sorted by their B-relation word (stable),
        // so that equal graphs reached through different node numberings give
        // equal records (the classification is invariant under relabelling)
        // rank of super-node q in label slot q, the inverse in slot 32 + rank
        // (lane-private bytes: slot v at (v >> 2) * 4 * THREADS + (v & 3))
        auto slot8 = [&](int v) -> uint8_t & { return lb[(v >> 2) * (4 * THREADS) + (v & 3)]; };
        for (int q = 0; q < m; ++q) {
            const uint32_t hq = hw[q * THREADS];
            int r = 0;
            for (int q2 = 0; q2 < m; ++q2) {
                const uint32_t h2 = hw[q2 * THREADS];
                r += (h2 < hq) || (h2 == hq && q2 < q);
            }
            slot8(q) = (uint8_t)r;
            slot8(32 + r) = (uint8_t)q;
        }
        out[0] = (unsigned long long)m;
        uint32_t hl = 0xC2B2AE3Du;
        for (int r = 0; r < m; ++r) {
            const int q = slot8(32 + r);
            uint32_t c = 0;
            for (uint32_t y = cs[q * THREADS]; y; y &= y - 1u) c |= 1u << slot8(__ffs(y) - 1);
            const uint32_t hi = hw[q * THREADS];
            out[1 + r] = (unsigned long long)c | (unsigned long long)hi << 32;
            hh = (hh ^ hi) * 0x85EBCA77u;
            hh ^= hh >> 13;
            hl = (hl ^ c) * 0x9E3779B1u;
            hl ^= hl >> 15;
        }
        hashes[j] = mix64(((unsigned long long)hh << 32 | hl) + 0x51ED2701ull * (unsigned long long)(m + 1));
        wts[j] = w15[j1];
        const uint32_t p1 = pos15[j1];
        const int la1 = tt.la1;
        poss[j] = ((p1 >> la1) << (la1 + la2)) | (a2 << la1) | (p1 & ((1u << la1) - 1u));
    }
}

// One thread per level-2 record: exact deduplication (hash, then word-by-word).
#ifndef L2D_PRE
#define L2D_PRE 8  // record words k_l2_dedup fetches before probing
#endif
__global__ void __launch_bounds__(THREADS) k_l2_dedup(const unsigned long long *__restrict__ pool,
                                                      uint32_t stride, uint32_t nrec,
                                                      const unsigned long long *__restrict__ hashes,
                                                      const uint32_t *__restrict__ wts,
                                                      const uint32_t *__restrict__ poss,
                                                      unsigned long long *__restrict__ slots,
                                                      uint32_t smask,
                                                      uint32_t *__restrict__ w2,
                                                      uint32_t *__restrict__ pos2,
                                                      uint32_t *__restrict__ list2,
                                                      uint32_t *__restrict__ count2, int wps) {
    // slot = hash tag << 32 | record; a tag match is confirmed word by word
    // (wps = record words per super-node: 1 odd degree, 2 even)
    const int lane = threadIdx.x & 31;
    const uint32_t tot = gridDim.x * blockDim.x;
    const uint32_t jmax = (nrec + 31u) & ~31u;  // whole warps iterate together
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < jmax; j += tot) {
        bool isnew = false;
        const uint32_t wj = j < nrec ? wts[j] : 0u;
        if (wj) {
            const unsigned long long h = hashes[j];
            const unsigned long long tag = (h >> 32) << 32;
            const unsigned long long *mine = pool + (size_t)j * stride;
            // the record's first words, fetched with its length and alongside the
            // first probe (a tag match -- every duplicate -- compares them); words
            // past the record's end lie inside its slot (stride >= 5) and are unused
            const int npre = min(L2D_PRE, (int)stride - 1);
            const unsigned long long m = mine[0];
            unsigned long long pw[L2D_PRE];
#pragma unroll
            for (int q = 0; q < L2D_PRE; ++q) pw[q] = q < npre ? mine[1 + q] : 0ull;
            const int nw = wps ? wps * (int)m : (int)(m >> 16);  // wps 0: stage-1 (L15Bits)
            uint32_t at = (uint32_t)h & smask;
            while (true) {
                unsigned long long cur = slots[at];
                if (cur == SLOT_EMPTY) {
                    const unsigned long long prev = atomicCAS(&slots[at], SLOT_EMPTY, tag | j);
                    if (prev == SLOT_EMPTY) {
                        isnew = true;
                        atomicAdd(&w2[j], wj);
                        atomicMin(&pos2[j], poss[j]);
                        break;
                    }
                    cur = prev;
                }
                if ((cur & 0xffffffff00000000ull) == tag) {
                    const uint32_t o = (uint32_t)cur;
                    TCG_ASSERT(o < nrec && at <= smask);
                    const unsigned long long *ow = pool + (size_t)o * stride;
                    unsigned long long diff = ow[0] ^ m;
#pragma unroll
                    for (int q = 0; q < L2D_PRE; ++q)
                        if (q < npre && q < nw) diff |= ow[1 + q] ^ pw[q];
#pragma unroll 4
                    for (int q = npre + 1; q <= nw; ++q) diff |= ow[q] ^ mine[q];
                    if (diff == 0ull) {
                        atomicAdd(&w2[o], wj);
                        atomicMin(&pos2[o], poss[j]);
                        break;
                    }
                }
                at = (at + 1) & smask;
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, isnew);
        if (bal) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(count2, (uint32_t)__popc(bal));
            base = __shfl_sync(0xffffffffu, base, 0);
            TCG_ASSERT(!isnew || base + __popc(bal & ((1u << lane) - 1u)) < nrec);
            if (isnew) list2[base + __popc(bal & ((1u << lane) - 1u))] = j;
        }
    }
}

// Level-2 node pass.  Node rows (shared memory, SoA by node):
//   same  = (A & ~T) | (B & T) | (s_v ? Cp : Cm) | L
//   cross = (A &  T) | (B & ~T) | (s_v ? Cm : Cp) | X,   T = S ^ (s_v ? ~0 : 0)
// super-node: A = minusB, B = plusB, Cp = Cm = 0, L = linkB, X = crossS | self
// B node:     A = adjB, B = 0, Cp = plusS, Cm = minusS, L = linkBB | linkS, X = 0
// (S = the lane's B-node signs; super-nodes carry sign 0).
struct L2Rows {
    uint32_t A[32], B[32], Cp[32], Cm[32], L[32], X[32];
    unsigned long long W[32];
};

__device__ __forceinline__ void l2_node_pass(const L2Rows &rw, uint32_t S, int nn,
                                             Regions<1> &out) {
    uint32_t un = nn >= 32 ? ~0u : ((1u << nn) - 1u), f = 0, x = 0, r = 0;
    int nreg = 0;
    auto seed = [&]() {
        f = un & (0u - un);
        r = un;
        un ^= f;
        x = 0u;
    };
    seed();
    for (int it = 0; it < nn; ++it) {
        if (f == 0u) {
            if (nreg < MAXR) {
                out.R[nreg][0] = r ^ un;
                out.X[nreg][0] = x;
            }
            ++nreg;
            seed();
        }
        const int v = __ffs(f) - 1;
        f &= f - 1u;
        const uint32_t sv = (S >> v) & 1u;
        const uint32_t T = S ^ (0u - sv);
        const uint32_t a = rw.A[v], b = rw.B[v], cp = rw.Cp[v], cm = rw.Cm[v];
        const uint32_t same = (a & ~T) | (b & T) | (sv ? cp : cm) | rw.L[v];
        x |= (a & T) | (b & ~T) | (sv ? cm : cp) | rw.X[v];
        const uint32_t nw = same & un;
        un ^= nw;
        f |= nw;
    }
    if (nreg < MAXR) {
        out.R[nreg][0] = r ^ un;
        out.X[nreg][0] = x;
    }
    out.nreg = nreg + 1;
    out.oddmask = 0u;
}

constexpr size_t L2_CLS_SMEM = TABLE_SMEM + sizeof(TileTables) + CLS_WARPS * sizeof(L2Rows);

// One warp per representative level-2 record; lane b classifies B pattern b.
__global__ void __launch_bounds__(THREADS) k_l2_classify(KParams p,
                                                         const TileTables *__restrict__ tt_g,
                                                         const unsigned long long *__restrict__ pool,
                                                         uint32_t stride,
                                                         const uint32_t *__restrict__ list2,
                                                         const uint32_t *__restrict__ count2,
                                                         const uint32_t *__restrict__ w2,
                                                         const uint32_t *__restrict__ pos2,
                                                         uint64_t tile0, DevAgg g,
                                                         unsigned long long *__restrict__ tstats) {
    extern __shared__ __align__(16) uint32_t smem[];
    CtaTable tab = carve_table(smem);
    TileTables *tt = reinterpret_cast<TileTables *>(reinterpret_cast<char *>(smem) + TABLE_SMEM);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    L2Rows *rw = reinterpret_cast<L2Rows *>(tt + 1) + w;
    for (int i = threadIdx.x; i < (int)(sizeof(TileTables) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t *>(tt)[i] = reinterpret_cast<const uint32_t *>(tt_g)[i];
    tab.init();
    __syncthreads();
    const int nB = tt->nB, bits = tt->bits;
    const uint32_t bm = (1u << nB) - 1u;
    const uint32_t n2 = *count2;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(tstats, (unsigned long long)n2);
    const uint32_t Sb = tt->l2bsign[lane];
    for (uint32_t i = blockIdx.x * CLS_WARPS + w; i < n2; i += gridDim.x * CLS_WARPS) {
        const uint32_t j = list2[i];
        const unsigned long long *rec = pool + (size_t)j * stride;
        const int m = (int)rec[0];
        if (lane < m) rw->W[lane] = rec[1 + lane];
        __syncwarp();
        if (lane < m) {
            const unsigned long long wd = rw->W[lane];
            const uint32_t hi = (uint32_t)(wd >> 32);
            rw->A[lane] = ((hi >> nB) & bm) << m;
            rw->B[lane] = (hi & bm) << m;
            rw->Cp[lane] = 0u;
            rw->Cm[lane] = 0u;
            rw->L[lane] = ((hi >> (2 * nB)) & bm) << m;
            rw->X[lane] = (uint32_t)wd | (((hi >> (3 * nB)) & 1u) << lane);
        }
        if (lane < nB) {
            uint32_t ps = 0, ms = 0, ls = 0;
            for (int q = 0; q < m; ++q) {
                const uint32_t hi = (uint32_t)(rw->W[q] >> 32);
                ps |= ((hi >> lane) & 1u) << q;
                ms |= ((hi >> (nB + lane)) & 1u) << q;
                ls |= ((hi >> (2 * nB + lane)) & 1u) << q;
            }
            const int v = m + lane;
            rw->A[v] = tt->l2adjB[lane] << m;
            rw->B[v] = 0u;
            rw->Cp[v] = ps;
            rw->Cm[v] = ms;
            rw->L[v] = (tt->l2linkB[lane] << m) | ls;
            rw->X[v] = 0u;
        }
        __syncwarp();
        Regions<1> rg;
        l2_node_pass(*rw, Sb << m, m + nB, rg);
        const uint32_t SG1[1] = {0u};
        const Result r = finish<1, false, false>(p, SG1, rg, p.maxreg);
        const uint64_t mw = (tile0 << bits) + ((uint64_t)pos2[j] << 5) + lane;
        uint64_t k = 0;
        if (r.status == TCG_OK) k = r.key;
        else atomicMin(g.bad, (unsigned long long)mw);
        tab.add<true>(g, k, r.nreg, mw, w2[j]);
        __syncwarp();
    }
    __syncthreads();
    tab.flush(g);
}

// Even-degree level-2 classification.  Rows per node v (super-nodes 0..m-1,
// B nodes m..m+nB-1), with T = the lane's B-sign mask S for a super-node
// and all-ones / all-zeros by the B node's own sign:
//   E0 = T&F0 | ~T&F2 | F5 | AB&~(S^T)    neighbours at the same parity
//   E1 = T&F1 | ~T&F3 | F4 | LB           neighbours at the other parity
//   X  = T&(F2|F3) | ~T&(F0|F1) | CS | AB&(S^T)   crossed neighbours
// F0..F5 = P10, P11, P00, P01, LK0, LK1 (super-nodes: B masks; B nodes: the
// transposed super-node masks), AB / LB = static B-B adjacency / links, CS =
// super-node crossed adjacency (+ self bit), ODD = odd super-nodes.
struct L2RowsE {
    uint32_t F[6][32], AB[32], LB[32], CS[32];
    unsigned long long W0[32], W1[32];
};

__device__ __forceinline__ void l2_node_pass_even(const L2RowsE &rw, uint32_t S, uint32_t oddn,
                                                  int m, int nn, Regions<1> &out) {
    uint32_t un = nn >= 32 ? ~0u : ((1u << nn) - 1u), f = 0, x = 0, r = 0, q = 0, oddmask = 0;
    bool odd = false;
    int nreg = 0;
    auto seed = [&]() {
        f = un & (0u - un);
        r = un;
        un ^= f;
        x = 0u;
        odd = false;
    };
    auto close = [&]() {
        if (nreg < MAXR) {
            out.R[nreg][0] = r ^ un;
            out.X[nreg][0] = x;
            if (odd) oddmask |= 1u << nreg;
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
        const uint32_t T = v < m ? S : (0u - ((S >> v) & 1u));
        const uint32_t f0 = rw.F[0][v], f1 = rw.F[1][v], f2 = rw.F[2][v], f3 = rw.F[3][v];
        const uint32_t ab = rw.AB[v];
        const uint32_t e0 = (T & f0) | (~T & f2) | rw.F[5][v] | (ab & ~(S ^ T));
        const uint32_t e1 = (T & f1) | (~T & f3) | rw.F[4][v] | rw.LB[v];
        x |= (T & (f2 | f3)) | (~T & (f0 | f1)) | rw.CS[v] | (ab & (S ^ T));
        const uint32_t pv = (q >> v) & 1u;
        const uint32_t eqm = pv ? q : ~q;
        const uint32_t nt = e0 & un, np = e1 & un;
        odd |= ((nt & np) | (e0 & ~un & ~eqm) | (e1 & ~un & eqm) | (oddn & (1u << v))) != 0u;
        q |= pv ? nt : np;
        un ^= nt | np;
        f |= nt | np;
    }
    close();
    out.nreg = nreg;
    out.oddmask = oddmask;
}

constexpr size_t L2E_CLS_SMEM = TABLE_SMEM + sizeof(TileTables) + CLS_WARPS * sizeof(L2RowsE);

__global__ void __launch_bounds__(THREADS) k_l2_classify_even(KParams p,
                                                              const TileTables *__restrict__ tt_g,
                                                              const unsigned long long *__restrict__ pool,
                                                              uint32_t stride,
                                                              const uint32_t *__restrict__ list2,
                                                              const uint32_t *__restrict__ count2,
                                                              const uint32_t *__restrict__ w2,
                                                              const uint32_t *__restrict__ pos2,
                                                              uint64_t tile0, DevAgg g,
                                                              unsigned long long *__restrict__ tstats) {
    extern __shared__ __align__(16) uint32_t smem[];
    CtaTable tab = carve_table(smem);
    TileTables *tt = reinterpret_cast<TileTables *>(reinterpret_cast<char *>(smem) + TABLE_SMEM);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    L2RowsE *rw = reinterpret_cast<L2RowsE *>(tt + 1) + w;
    for (int i = threadIdx.x; i < (int)(sizeof(TileTables) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t *>(tt)[i] = reinterpret_cast<const uint32_t *>(tt_g)[i];
    tab.init();
    __syncthreads();
    const int nB = tt->nB, bits = tt->bits;
    const uint32_t bm = (1u << nB) - 1u;
    const uint32_t n2 = *count2;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(tstats, (unsigned long long)n2);
    const uint32_t Sb = tt->l2bsign[lane];
    for (uint32_t i = blockIdx.x * CLS_WARPS + w; i < n2; i += gridDim.x * CLS_WARPS) {
        const uint32_t j = list2[i];
        const unsigned long long *rec = pool + (size_t)j * stride;
        const int m = (int)rec[0];
        if (lane < m) {
            rw->W0[lane] = rec[1 + 2 * lane];
            rw->W1[lane] = rec[2 + 2 * lane];
        }
        __syncwarp();
        uint32_t oddn = 0;
        {
            const bool od = lane < m && ((uint32_t)rw->W0[lane] >> 31);
            oddn = __ballot_sync(0xffffffffu, od);
        }
        if (lane < m) {
            const uint32_t c = (uint32_t)rw->W0[lane];
            const unsigned long long w1 = rw->W1[lane];
#pragma unroll
            for (int k = 0; k < 6; ++k) rw->F[k][lane] = (uint32_t)((w1 >> (k * nB)) & bm) << m;
            rw->AB[lane] = 0u;
            rw->LB[lane] = 0u;
            rw->CS[lane] = (c & 0x3fffffffu) | (((c >> 30) & 1u) << lane);
        }
        if (lane < nB) {
            uint32_t t[6] = {0u, 0u, 0u, 0u, 0u, 0u};
            for (int s = 0; s < m; ++s) {
                const unsigned long long w1 = rw->W1[s];
#pragma unroll
                for (int k = 0; k < 6; ++k) t[k] |= (uint32_t)((w1 >> (k * nB + lane)) & 1u) << s;
            }
            const int v = m + lane;
#pragma unroll
            for (int k = 0; k < 6; ++k) rw->F[k][v] = t[k];
            rw->AB[v] = tt->l2adjB[lane] << m;
            rw->LB[v] = tt->l2linkB[lane] << m;
            rw->CS[v] = 0u;
        }
        __syncwarp();
        Regions<1> rg;
        l2_node_pass_even(*rw, Sb << m, oddn, m, m + nB, rg);
        const uint32_t SG1[1] = {0u};
        const Result r = finish<1, true, false>(p, SG1, rg, p.maxreg);
        const uint64_t mw = (tile0 << bits) + ((uint64_t)pos2[j] << 5) + lane;
        uint64_t k = 0;
        if (r.status == TCG_OK) k = r.key;
        else atomicMin(g.bad, (unsigned long long)mw);
        tab.add<true>(g, k, r.nreg, mw, w2[j]);
        __syncwarp();
    }
    __syncthreads();
    tab.flush(g);
}
