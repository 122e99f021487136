// host_plan.cuh -- host side of a plan: device guard, per-kernel timing,
// kernel pickers, chunk sizes, the vertex layout, the tile tables and the
// validated host plan.  Included by tcg.cu inside its anonymous namespace.


struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// TCG_HOST_TRACE=1: host timestamps (us since the previous mark) around the
// pipeline's synchronisation points, to stderr (diagnostics only).
static void host_mark(const char *what) {
    static const bool on = [] {
        const char *e = std::getenv("TCG_HOST_TRACE");
        return e && e[0] && e[0] != '0';
    }();
    if (!on) return;
    static auto prev = std::chrono::steady_clock::now();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[tcg] %-22s +%9.1f us\n", what,
                 std::chrono::duration<double, std::micro>(now - prev).count());
    prev = now;
}

// Per-kernel timing: events bracket each launch on the plan's stream and are
// resolved after the next synchronisation (tcg_agg_fetch / tcg_kernel_times).
cudaEvent_t timing_begin(tcg_plan *P, cudaStream_t st = nullptr) {
    if (!P->timing) return nullptr;
    cudaEvent_t a;
    cudaEventCreate(&a);
    cudaEventRecord(a, st ? st : P->stream);
    return a;
}

void timing_end(tcg_plan *P, int kind, cudaEvent_t a, cudaStream_t st = nullptr) {
    if (!P->timing || !a) return;
    cudaEvent_t b;
    cudaEventCreate(&b);
    cudaEventRecord(b, st ? st : P->stream);
    P->tev.push_back({kind, {a, b}});
}

void timing_resolve(tcg_plan *P) {
    for (auto &t : P->tev) {
        float ms = 0.f;
        cudaEventSynchronize(t.second.second);
        cudaEventElapsedTime(&ms, t.second.first, t.second.second);
        P->t_ms[t.first] += ms;
        P->t_n[t.first] += 1;
        cudaEventDestroy(t.second.first);
        cudaEventDestroy(t.second.second);
    }
    P->tev.clear();
}

template <int K, bool EVEN>
void *enum_fn(int mode) {
    switch (mode) {
        case MODE_RAW: return (void *)k_enumerate<K, EVEN, MODE_RAW>;
        case MODE_REP: return (void *)k_enumerate<K, EVEN, MODE_REP>;
        default: return (void *)k_enumerate<K, EVEN, MODE_SAMPLE>;
    }
}

void *pick_enum(int K, bool even, int mode) {
    if (K == 2) return even ? enum_fn<2, true>(mode) : enum_fn<2, false>(mode);
    if (K == 4) return even ? enum_fn<4, true>(mode) : enum_fn<4, false>(mode);
    return even ? enum_fn<6, true>(mode) : enum_fn<6, false>(mode);
}

template <int K>
void *build_fn(int mode) {
    return mode == MODE_RAW ? (void *)k_tile_build_lanes<K, MODE_RAW>
                            : (void *)k_tile_build_lanes<K, MODE_REP>;
}


template <int K>
void *super_fn(int mode) {
    return mode == MODE_RAW ? (void *)k_super_build<K, MODE_RAW> : (void *)k_super_build<K, MODE_REP>;
}

void *pick_super(int K, int mode) {
    if (K == 2) return super_fn<2>(mode);
    if (K == 4) return super_fn<4>(mode);
    return super_fn<6>(mode);
}

void *pick_build(int K, int mode) {
    if (K == 2) return build_fn<2>(mode);
    if (K == 4) return build_fn<4>(mode);
    return build_fn<6>(mode);
}

template <int K, bool EVEN>
void *cls_fn(int mode) {
    return mode == MODE_RAW ? (void *)k_tile_classify<K, EVEN, MODE_RAW>
                            : (void *)k_tile_classify<K, EVEN, MODE_REP>;
}

void *pick_cls(int K, bool even, int mode) {
    if (K == 2) return even ? cls_fn<2, true>(mode) : cls_fn<2, false>(mode);
    if (K == 4) return even ? cls_fn<4, true>(mode) : cls_fn<4, false>(mode);
    return even ? cls_fn<6, true>(mode) : cls_fn<6, false>(mode);
}

size_t build_smem(int K) { return (size_t)32 * K * K * 4 + sizeof(TileTables); }

size_t cls_smem(int K) {
    return (size_t)32 * K * K * 4 + TABLE_SMEM + sizeof(TileTables) + CLS_WARPS * sizeof(TileRec);
}

// Tiles per contraction chunk (records: 1 KiB each).  Deduplication works
// within a chunk, and larger chunks find many more duplicates (C3: 1.6x at
// 2^20 tiles, 2.4x at 2^23), so the default is 2^24 tiles (18 GB of records,
// allocated on demand and only as large as the sweep needs, halved while it
// would take more than a quarter of the free HBM).  TCG_CHUNK_LOG2 (14..24)
// overrides.
// indices per chunk (TCG_CHUNK_INDEX_LOG2, 32..35; default 2^35): larger chunks
// deduplicate over a larger window (C3 at 2^9-index tiles: 158x at 2^32,
// 244x at 2^33, 379x at 2^34); 2^35 is the whole C3 domain in one window.
// At most chunk_tiles() = 2^25 tiles; 2^35 indices = 2^(30 - la) tiles keeps
// level-1 slice entries (tile < 2^(31 - la)) and level-2 positions
// (tile << la < 2^30) in 32 bits.
static uint64_t chunk_index_limit() {
    static const uint64_t c = [] {
        int lg = 35;
        if (const char *e = std::getenv("TCG_CHUNK_INDEX_LOG2")) lg = std::max(32, std::min(35, std::atoi(e)));
        return 1ull << lg;
    }();
    return c;
}

static uint32_t chunk_tiles() {
    static const uint32_t c = [] {
        int lg = 25;
        if (const char *e = std::getenv("TCG_CHUNK_LOG2")) lg = std::max(14, std::min(25, std::atoi(e)));
        return 1u << lg;
    }();
    return c;
}

static uint32_t next_pow2(uint32_t x) {
    uint32_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

void *pick_batch(int K, bool even) {
    if (K == 2) return even ? (void *)k_batch<2, true> : (void *)k_batch<2, false>;
    if (K == 4) return even ? (void *)k_batch<4, true> : (void *)k_batch<4, false>;
    return even ? (void *)k_batch<6, true> : (void *)k_batch<6, false>;
}

size_t adj_bytes(int K) { return (size_t)32 * K * K * sizeof(uint32_t); }

size_t enum_smem(int K) { return adj_bytes(K) + TABLE_SMEM; }

// Vertex layout.  H = 16K bits per half.  P-half (points p > -p
// lexicographically, i.e. i > 0 or (i == 0 and j > 0)):
//   bits [0, npts-1)      : first-quadrant points except the origin, in
//                           A(d) index order (bit = index - 1), so their
//                           signs are sigma >> 1;
//   bits [npts-1, d^2+d)  : mirrored quadrant (i > 0, j < 0), in A(d) order
//                           of (i, |j|); signs = compressed sigma ^ (j odd);
//   bit d^2+d             : the origin.
// N-half: bit H + b holds the antipode of P-half bit b, whose sign is the
// P-half sign ^ ((|i|+|j|) & 1).  The antipodal map is therefore a swap of
// the two halves.
struct Layout {
    int d, K, H, npts;
    std::vector<int> pos;  // lex vertex -> bit position
};

int point_index(int d, int i, int j) { return i * (d + 1) - i * (i - 1) / 2 + j; }

int build_layout(const tcg_desc *D, Layout &L) {
    const int d = D->degree;
    L.d = d;
    L.npts = (d + 1) * (d + 2) / 2;
    const int half = d * d + d + 1;  // P-half incl. the origin
    L.K = half <= 32 ? 2 : (half <= 64 ? 4 : 6);
    L.H = 16 * L.K;
    // q4 rank of (i, j), i > 0, j > 0
    std::vector<int> q4rank(L.npts, -1);
    int r = 0;
    for (int i = 1; i <= d; ++i)
        for (int j = 1; j <= d - i; ++j) q4rank[point_index(d, i, j)] = r++;
    // lexicographic diamond points
    std::vector<std::pair<int, int>> pts;
    for (int i = -d; i <= d; ++i) {
        const int a = d - std::abs(i);
        for (int j = -a; j <= a; ++j) pts.emplace_back(i, j);
    }
    if ((int)pts.size() != D->nv) return fail(TCG_E_ARG, "nv does not match the degree");
    auto ppos = [&](int i, int j) -> int {  // P-half position of a P-half point
        if (j >= 0) return point_index(d, i, j) - 1;
        return (L.npts - 1) + q4rank[point_index(d, i, -j)];
    };
    L.pos.assign(D->nv, -1);
    for (int v = 0; v < D->nv; ++v) {
        const int i = pts[v].first, j = pts[v].second;
        if (i == 0 && j == 0) L.pos[v] = d * d + d;
        else if (i > 0 || (i == 0 && j > 0)) L.pos[v] = ppos(i, j);
        else L.pos[v] = L.H + ppos(-i, -j);
    }
    return TCG_OK;
}


// Free vertices of a tile (index bits 0..bits-1) and the fixed mask.
bool build_tiles_bits(const tcg_desc *D, const Layout &L, int mode, int bits, TileTables &T) {
    const int d = D->degree;
    const int npts = D->npts;
    const int dom_bits = mode == MODE_RAW ? npts : npts - 3;
    if (d < 5 || bits > TILE_BITS_MAX || dom_bits < bits + 2) return false;
    std::memset(&T, 0, sizeof(T));
    std::memset(T.vfree, 0xff, sizeof(T.vfree));
    T.bits = bits;
    T.maxnodes = 64;
    if (const char *e = std::getenv("TCG_TILE_MAXNODES")) T.maxnodes = std::max(0, std::min(64, std::atoi(e)));
    int sbit[TILE_BITS_MAX];
    for (int i = 0; i < bits; ++i)
        sbit[i] = mode == MODE_RAW ? i : (i < d - 1 ? i + 2 : i - (d - 1) + d + 2);
    std::vector<int> fnode(D->nv, -1), vbit(D->nv, -1);
    for (int v = 0; v < D->nv; ++v) {
        if (!D->used[v]) continue;
        for (int i = 0; i < bits; ++i)
            if (sbit[i] == D->src[v]) vbit[v] = i;
        if (vbit[v] < 0) {
            const int pos = L.pos[v];
            T.fixed[pos >> 5] |= 1u << (pos & 31);
            ++T.nfixed;
        }
    }
    // free nodes numbered by tile bit (then vertex): the B, A1 and A2 nodes of
    // the two-stage level 2 are contiguous free-node ranges, so the stage-1
    // F-space compression is a shift (TileTables::l15sh)
    int nf = 0;
    std::vector<int> vorder;
    for (int i = 0; i < bits; ++i)
        for (int v = 0; v < D->nv; ++v)
            if (D->used[v] && vbit[v] == i) vorder.push_back(v);
    for (const int v : vorder) {
        const int bit = vbit[v];
        const int pos = L.pos[v];
        if (nf >= MAXF) return false;
        fnode[v] = nf;
        T.fword[nf] = (uint32_t)(pos >> 5);
        T.fbit[nf] = 1u << (pos & 31);
        T.freem[pos >> 5] |= 1u << (pos & 31);
        T.vfree[pos] = (int8_t)nf;
        T.fpar |= (unsigned long long)(D->par[v] & 1) << nf;
        T.fcopy[bit] |= 1ull << nf;
        ++nf;
    }
    T.nf = nf;
    for (int h = 0; h < 2; ++h)
        for (int x = 0; x < 64; ++x) {
            unsigned long long w = h == 0 ? T.fpar : 0ull;
            for (int i = 0; i < 6; ++i)
                if (((x >> i) & 1) && 6 * h + i < bits) w ^= T.fcopy[6 * h + i];
            T.fsign[h][x] = w;
        }
    for (int e = 0; e < D->ne; ++e) {
        const int fu = fnode[D->edge_u[e]], fv = fnode[D->edge_v[e]];
        if (fu >= 0 && fv >= 0) {
            T.fadj[fu] |= 1ull << fv;
            T.fadj[fv] |= 1ull << fu;
        }
    }
    // level-2 tables (filled after fadj / fpl below)
    auto l2_tables = [&]() {
        T.l2 = 0;
        if (bits < 6 || bits > 12 || nf > 32) return;
        T.l2even = d % 2 == 0;
        uint32_t fb = 0, fa = 0;
        for (int i = 0; i < bits; ++i) (i < 5 ? fb : fa) |= (uint32_t)T.fcopy[i];
        const int nB = __builtin_popcount(fb);
        if (nB > 10 || nB == 0) return;
        T.fbm = fb;
        T.fa = fa;
        T.nB = nB;
        T.la = bits - 5;
        T.NA = 1 << T.la;
        int j = 0;
        int fj[32];
        for (int f = 0; f < MAXF; ++f) T.l2j[f] = -1;
        for (int f = 0; f < nf; ++f)
            if ((fb >> f) & 1u) {
                T.l2j[f] = (int8_t)j;
                fj[j++] = f;
            }
        auto comp = [&](unsigned long long x) {
            uint32_t r = 0;
            for (int f = 0; f < nf; ++f)
                if (((x >> f) & 1ull) && T.l2j[f] >= 0) r |= 1u << T.l2j[f];
            return r;
        };
        for (int q = 0; q < nB; ++q) {
            T.l2adjB[q] = comp(T.fadj[fj[q]] & fb);
            T.l2linkB[q] = comp(T.fpl[fj[q]] & fb);
        }
        for (int b = 0; b < 32; ++b) T.l2bsign[b] = comp(T.fsign[0][b] & fb);
        T.l2shift = -1;
        if (fb >> __builtin_ctz(fb) == (1u << nB) - 1u) T.l2shift = __builtin_ctz(fb);
        T.l2 = 1;
        // two-stage tables
        T.ts = 0;
        // A1 = the fewest low A bits (>= 2) that leave an F space of <= 21 nodes
        int la1 = 2;
        uint32_t fa1 = 0, fa2 = 0;
        int nA2 = 0;
        for (; la1 <= T.la - 1; ++la1) {
            fa1 = fa2 = 0;
            for (int i = 5; i < bits; ++i) (i < 5 + la1 ? fa1 : fa2) |= (uint32_t)T.fcopy[i];
            nA2 = __builtin_popcount(fa2);
            if (nA2 <= 16 && nB + nA2 <= 21) break;
        }
        if (!T.l2even && T.la >= 4 && la1 <= 4 && la1 < T.la && nA2 > 0 && nA2 <= 16 &&
            nB + nA2 <= 21) {
            T.la1 = la1;
            T.la2 = T.la - la1;
            T.l15max = L15_MAXM;
            if (const char *e = std::getenv("TCG_L15_MAXM"))
                T.l15max = std::max(1, std::min(L15_MAXM, std::atoi(e)));
            T.fa1 = fa1;
            T.fa2 = fa2;
            {
                const int n1 = __builtin_popcount(fa1);
                const bool contig = fb == (1u << nB) - 1u && fa1 == ((1u << n1) - 1u) << nB &&
                                    fa2 == ((1u << nA2) - 1u) << (nB + n1);
                T.l15sh = contig && !std::getenv("TCG_L15_LUT") ? n1 : -1;
            }
            T.nA2 = nA2;
            int a2j[MAXF], a2f[16], k = 0;
            for (int f = 0; f < MAXF; ++f) { T.l15F[f] = -1; a2j[f] = -1; }
            for (int f = 0; f < nf; ++f) {
                if (T.l2j[f] >= 0) T.l15F[f] = T.l2j[f];
                if ((fa2 >> f) & 1u) {
                    a2j[f] = k;
                    a2f[k] = f;
                    T.l15F[f] = (int8_t)(nB + k);
                    ++k;
                }
            }
            auto compA2 = [&](unsigned long long x) {
                uint32_t r = 0;
                for (int f = 0; f < nf; ++f)
                    if (((x >> f) & 1ull) && a2j[f] >= 0) r |= 1u << a2j[f];
                return r;
            };
            for (int q = 0; q < nA2; ++q) {
                const int f = a2f[q];
                T.a2adjA2[q] = compA2(T.fadj[f] & fa2);
                T.a2linkA2[q] = compA2(T.fpl[f] & fa2);
                T.a2adjB[q] = comp(T.fadj[f] & fb);
                T.a2linkB[q] = comp(T.fpl[f] & fb);
            }
            for (int x = 0; x < (1 << T.la2); ++x) {  // tile-local index of the A2 bits
                const uint32_t low = (uint32_t)x << (5 + la1);
                T.a2sign[x] = compA2((T.fsign[0][low & 63u] ^ T.fsign[1][(low >> 6) & 63u]) & fa2);
            }
            T.ts = 1;
        }
    };
    for (int a = 0; a < D->nap; ++a) {
        const int fu = fnode[D->ap_u[a]], fv = fnode[D->ap_v[a]];
        if ((fu >= 0) != (fv >= 0)) return false;  // cannot happen: p and -p share src
        if (fu >= 0) {
            T.fpl[fu] |= 1ull << fv;
            T.fpl[fv] |= 1ull << fu;
        }
    }
    l2_tables();
    // super-tiles: mid points = index bits bits .. bits+sh-1; the largest sh <= 6
    // (TCG_SUPER_BITS) whose mid vertices fit MAXM
    T.sh = 0;
    int hmax = SUPER_BITS_MAX;
    if (const char *e = std::getenv("TCG_SUPER_BITS")) hmax = std::atoi(e);
    if (const char *e = std::getenv("TCG_BUILD_GENERIC"))
        if (e[0] && e[0] != '0') hmax = 0;
    for (int h = std::max(0, std::min(hmax, SUPER_BITS_MAX)); h > 0 && T.sh == 0; --h) {
        if (dom_bits >= bits + h + 1) {
            auto point_of = [&](int ib) {  // index bit -> lattice point
                return mode == MODE_RAW ? ib : (ib < d - 1 ? ib + 2 : ib - (d - 1) + d + 2);
            };
            std::vector<std::pair<int, int>> mids;  // (layout position, vertex)
            std::vector<int> mbit(D->nv, -1);
            for (int v = 0; v < D->nv; ++v) {
                if (!D->used[v] || fnode[v] >= 0) continue;
                for (int i = 0; i < h; ++i)
                    if (point_of(bits + i) == D->src[v]) mbit[v] = i;
                if (mbit[v] >= 0) mids.push_back({L.pos[v], v});
            }
            std::sort(mids.begin(), mids.end());
            if ((int)mids.size() <= MAXM && !mids.empty()) {
                T.sh = h;
                T.nm = (int)mids.size();
                for (int k = 0; k < MAXK; ++k) T.sfixed[k] = T.fixed[k];
                for (int j = 0; j < T.nm; ++j) {
                    const int pos = mids[j].first, v = mids[j].second;
                    T.mpos[j] = (uint16_t)pos;
                    T.sfixed[pos >> 5] &= ~(1u << (pos & 31));
                    for (int x = 0; x < (1 << h); ++x)
                        T.msign[x] |= (uint32_t)(((x >> mbit[v]) & 1) ^ (D->par[v] & 1)) << j;
                }
                T.nsfixed = T.nfixed - T.nm;
            }
        }
    }
    return T.nfixed > 0 && nf > 0;
}

// Tile size: 2^bits indices.  Larger tiles amortise the contraction but add
// free vertices (lane work); since contraction runs one tile per lane it is
// cheap, so the default picks the largest tile whose contracted graph
// (free vertices + the fixed part's components) usually fits one 32-bit
// word: at most 16 free vertices (d=7 raw: 2^8 indices, the j-axis).
// Degree 8-9 graphs exceed 32 nodes anyway, so they take 2^10.
// TCG_TILE_BITS overrides.
// Odd degrees up to 7 run the two-stage level 2 (which also takes 33..64-node
// tiles), so they allow 29 free vertices: d=7 raw tiles are 2^12 indices
// (measured on C3: 7.48e11 patchworks/s vs 7.11e11 at 2^11, 5.07e11 at 2^10,
// 3.49e11 at 2^9; with the direct level 2, 2^9 had been best).
bool build_tiles(const tcg_desc *D, const Layout &L, int mode, TileTables &T) {
    int want = D->degree >= 8 ? 10 : 12;
    int fmax = D->degree >= 8 ? 28 : (D->degree % 2 ? 29 : 16);
    if (const char *e = std::getenv("TCG_TILE_BITS")) {
        want = std::atoi(e);
        fmax = MAXF;
    }
    for (int bits = std::min(want, TILE_BITS_MAX); bits >= 6; --bits)
        if (build_tiles_bits(D, L, mode, bits, T) && T.nf <= fmax) return true;
    return false;
}

// Host-side plan: layout, masks, adjacency rows and edge list of one
// triangulation, validated against the reference's sign-extension tables.
struct HostPlan {
    int d = 0, K = 0, even = 0, nused = 0;
    KParams kp{};
    Layout L;
    std::vector<uint32_t> adj, edges;
};

int build_host_plan(const tcg_desc *D, HostPlan &HP) {
    if (!D) return fail(TCG_E_ARG, "null descriptor");
    const int d = D->degree;
    if (d < 1) return fail(TCG_E_ARG, "degree must be >= 1");
    if (d > 9)
        return fail(TCG_E_UNSUPPORTED,
                    "degree > 9 exceeds the 64-bit sign word / 96-bit half-mask layout");
    if (D->nv != 2 * d * d + 2 * d + 1) return fail(TCG_E_ARG, "nv != 2d^2+2d+1");
    if (D->npts != (d + 1) * (d + 2) / 2) return fail(TCG_E_ARG, "npts mismatch");
    if (D->maxreg < 1 || D->maxreg > MAXR) return fail(TCG_E_UNSUPPORTED, "maxreg out of range");
    if (D->ne < 1) return fail(TCG_E_ARG, "empty edge list");
    Layout &L = HP.L;
    int rc = build_layout(D, L);
    if (rc) return rc;
    const int K = L.K, H = L.H;
    HP.d = d;
    HP.K = K;
    HP.even = (d % 2 == 0);
    KParams &kp = HP.kp;
    kp = KParams{};
    kp.d = d;
    kp.npts = D->npts;
    kp.maxreg = D->maxreg;
    kp.center = d * d + d;
    kp.ne = D->ne;
    std::vector<std::pair<int, int>> pts;
    for (int i = -d; i <= d; ++i) {
        const int a = d - std::abs(i);
        for (int j = -a; j <= a; ++j) pts.emplace_back(i, j);
    }
    auto setbit = [&](uint32_t *m, int pos) { m[pos >> 5] |= 1u << (pos & 31); };
    int nused = 0;
    for (int v = 0; v < D->nv; ++v)
        if (D->used[v]) {
            setbit(kp.used, L.pos[v]);
            ++nused;
        }
    kp.nused = nused;
    HP.nused = nused;
    for (int a = 0; a < D->nap; ++a) {
        const int u = D->ap_u[a], v = D->ap_v[a];
        if (u < 0 || u >= D->nv || v < 0 || v >= D->nv)
            return fail(TCG_E_ARG, "antipodal pair out of range");
        const int pu = L.pos[u], pv = L.pos[v];
        if (std::abs(pu - pv) != H) return fail(TCG_E_ARG, "antipodal pair is not (p, -p)");
        if (std::abs(pts[u].first) + std::abs(pts[u].second) != d)
            return fail(TCG_E_ARG, "antipodal pair off the diamond boundary");
        setbit(kp.bd, pu);
        setbit(kp.bd, pv);
    }
    // sign-extension tables -> P-half masks; verify they are the reference's
    for (int v = 0; v < D->nv; ++v) {
        const int i = pts[v].first, j = pts[v].second;
        const int want_src = point_index(d, std::abs(i), std::abs(j));
        const int want_par = ((i < 0 ? -i : 0) + (j < 0 ? -j : 0)) & 1;
        if (D->src[v] != want_src || D->par[v] != want_par)
            return fail(TCG_E_ARG, "src/par tables differ from the reflected sign extension");
        const int pos = L.pos[v];
        if (pos < H && !(i == 0 && j == 0)) {
            if (((std::abs(i) + std::abs(j)) & 1) != 0) kp.parP[pos >> 5] |= 1u << (pos & 31);
            if (j < 0 && ((-j) & 1)) kp.jodd[pos >> 5] |= 1u << (pos & 31);
        }
    }
    // mirrored-quadrant compress runs: row i contributes (i,1..d-i)
    {
        int nq = 0, dst = 0;
        for (int i = 1; i <= d - 1; ++i) {
            kp.q4src[nq] = (uint8_t)point_index(d, i, 1);
            kp.q4len[nq] = (uint8_t)(d - i);
            kp.q4dst[nq] = (uint8_t)dst;
            dst += d - i;
            ++nq;
        }
        kp.nq4 = nq;
    }
    // adjacency rows and edge list in layout positions
    HP.adj.assign((size_t)2 * H * K, 0u);
    HP.edges.assign(D->ne, 0u);
    for (int e = 0; e < D->ne; ++e) {
        const int u = D->edge_u[e], v = D->edge_v[e];
        if (u < 0 || u >= D->nv || v < 0 || v >= D->nv || u == v)
            return fail(TCG_E_ARG, "edge endpoint out of range");
        const int pu = L.pos[u], pv = L.pos[v];
        HP.adj[(size_t)pu * K + (pv >> 5)] |= 1u << (pv & 31);
        HP.adj[(size_t)pv * K + (pu >> 5)] |= 1u << (pu & 31);
        HP.edges[e] = (uint32_t)pu | ((uint32_t)pv << 16);
    }
    return TCG_OK;
}
