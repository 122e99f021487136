// split_design.cuh -- host side of the separator-split sampler (split.cuh):
// the separator search and the per-plan tables.  Included by tcg.cu inside
// its anonymous namespace, after the vertex layout helpers.

// The separator, the two parts and every per-plan table of the sampler.
struct SplitDesign {
    SplitParams sp{};  // device pointers are filled by the caller
    SplitPart pa{}, pb{};
    std::vector<unsigned long long> pext;  // [nbytes * 256]
    int nfpts = 0;                         // separator points
    unsigned long long Fm = 0, Am = 0, Bm = 0;  // point masks of F and the two sides
    double mean_nodes = 0;                 // estimated contracted-graph size
};

// Separator search over the point graph of T (npts <= 55: one u64 per set).
// Candidates: for a few hundred pseudo-random linear orders of the points
// and every balanced cut of each order, the minimum vertex cover of the
// edges crossing the cut (Koenig, from a maximum bipartite matching) is a
// separator; the components of the rest are distributed over the two tables
// to balance their index bits.  The best candidates by separator size are
// scored by simulating random sign patterns (mean contracted-graph size plus
// a penalty for graphs over 64 nodes); the lowest score wins.
static bool split_design(const tcg_desc *D, const Layout &L, SplitDesign &S) {
    typedef unsigned long long u64;
    const int d = D->degree, npts = D->npts, nv = D->nv;
    if (npts > 62) return false;
    std::vector<u64> nb(npts, 0ull);
    for (int e = 0; e < D->ne; ++e) {
        const int a = D->src[D->edge_u[e]], b = D->src[D->edge_v[e]];
        if (a != b) {
            nb[a] |= 1ull << b;
            nb[b] |= 1ull << a;
        }
    }
    std::vector<int> copies(npts, 0);
    for (int v = 0; v < nv; ++v)
        if (D->used[v]) ++copies[D->src[v]];
    const u64 pinned = (1ull << 0) | (1ull << 1) | (1ull << (d + 1));
    const u64 all = (npts == 64) ? ~0ull : ((1ull << npts) - 1ull);
    std::vector<std::pair<int, int>> ij(npts);
    for (int i = 0, k = 0; i <= d; ++i)
        for (int j = 0; j <= d - i; ++j) ij[k++] = {i, j};
    const size_t budget = (size_t)[] {
        const char *e = std::getenv("TCG_SPLIT_MAXMB");
        return e ? std::atol(e) : 4096l;
    }() << 20;

    struct Cand {
        u64 F, A, B;
        int cost, maxbits;
    };
    std::vector<Cand> cands;
    auto popc = [](u64 x) { return __builtin_popcountll(x); };
    auto consider = [&](u64 F) {
        for (const Cand &c : cands)
            if (c.F == F) return;
        int nFv = 0;
        for (int p = 0; p < npts; ++p)
            if ((F >> p) & 1ull) nFv += copies[p];
        if (nFv > SPL_MAXF || popc(F & ~pinned) > SPL_MAXFB) return;
        // components of the rest, largest first onto the lighter table
        std::vector<std::pair<int, u64>> comps;
        u64 left = all & ~F;
        while (left) {
            u64 c = left & (0ull - left), fr = c;
            while (fr) {
                const int p = __builtin_ctzll(fr);
                fr &= fr - 1ull;
                const u64 nw = nb[p] & left & ~c & ~F;
                c |= nw;
                fr |= nw;
            }
            left &= ~c;
            comps.push_back({popc(c & ~pinned), c});
        }
        std::sort(comps.begin(), comps.end(), [](const std::pair<int, u64> &a, const std::pair<int, u64> &b) {
            return a.first != b.first ? a.first > b.first : a.second < b.second;
        });
        u64 A = 0, B = 0;
        int ba = 0, bb = 0;
        for (auto &c : comps) {
            if (ba <= bb) { A |= c.second; ba += c.first; }
            else { B |= c.second; bb += c.first; }
        }
        if (!A || !B || std::max(ba, bb) > SPL_MAXBITS) return;
        const size_t stride = split_stride((nFv + 3) & ~3);
        if (((1ull << ba) + (1ull << bb)) * stride * 4 > budget) return;
        cands.push_back({F, A, B, nFv, std::max(ba, bb)});
    };
    uint64_t rs = 0x9E3779B97F4A7C15ull;
    auto rnd = [&]() {  // splitmix64, uniform in [0, 1)
        rs += 0x9E3779B97F4A7C15ull;
        u64 z = rs;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return (double)((z ^ (z >> 31)) >> 11) * (1.0 / 9007199254740992.0);
    };
    std::vector<int> order(npts);
    std::vector<double> key(npts);
    for (int trial = 0; trial < 240; ++trial) {
        const double a = 2 * rnd() - 1, b = 2 * rnd() - 1, noise = 0.4 * rnd();
        for (int p = 0; p < npts; ++p) {
            order[p] = p;
            key[p] = a * ij[p].first + b * ij[p].second + noise * rnd();
        }
        std::sort(order.begin(), order.end(), [&](int x, int y) { return key[x] < key[y]; });
        u64 Lm = 0;
        for (int cut = 0; cut < npts - 1; ++cut) {
            Lm |= 1ull << order[cut];
            if (cut < npts / 5 || cut > 4 * npts / 5) continue;
            // maximum matching on the crossing edges (Kuhn), then Koenig's cover
            std::vector<int> mr(npts, -1), ml(npts, -1);
            std::function<bool(int, u64 &)> aug = [&](int l, u64 &seen) -> bool {
                u64 rr = nb[l] & ~Lm & ~seen;
                while (rr) {
                    const int r = __builtin_ctzll(rr);
                    rr &= rr - 1ull;
                    seen |= 1ull << r;
                    if (mr[r] < 0 || aug(mr[r], seen)) {
                        mr[r] = l;
                        ml[l] = r;
                        return true;
                    }
                }
                return false;
            };
            for (u64 ls = Lm; ls;) {
                const int l = __builtin_ctzll(ls);
                ls &= ls - 1ull;
                u64 seen = 0;
                aug(l, seen);
            }
            u64 Z = 0, fr = 0;
            for (u64 ls = Lm; ls;) {
                const int l = __builtin_ctzll(ls);
                ls &= ls - 1ull;
                if (ml[l] < 0) fr |= 1ull << l;
            }
            Z = fr;
            while (fr) {
                const int u = __builtin_ctzll(fr);
                fr &= fr - 1ull;
                if ((Lm >> u) & 1ull) {
                    u64 rr = nb[u] & ~Lm & ~Z;  // non-matching edges L -> R
                    Z |= rr;
                    fr |= rr;
                } else if (mr[u] >= 0 && !((Z >> mr[u]) & 1ull)) {
                    Z |= 1ull << mr[u];  // matching edge R -> L
                    fr |= 1ull << mr[u];
                }
            }
            consider((Lm & ~Z) | (~Lm & all & Z));
        }
    }
    if (cands.empty()) return false;
    std::sort(cands.begin(), cands.end(), [](const Cand &x, const Cand &y) {
        return x.cost != y.cost ? x.cost < y.cost : x.maxbits < y.maxbits;
    });
    if (cands.size() > 96) cands.resize(96);
    // score by simulation: same-sign components of each part (union-find)
    std::vector<int> uf(nv);
    std::function<int(int)> find = [&](int x) {
        while (uf[x] != x) x = uf[x] = uf[uf[x]];
        return x;
    };
    double best = 1e30;
    int bi = -1;
    const int NS = 128;
    for (int ci = 0; ci < (int)cands.size(); ++ci) {
        const Cand &c = cands[ci];
        double tot = 0, over = 0;
        rs = 0xD1B54A32D192ED03ull;
        for (int s = 0; s < NS; ++s) {
            const u64 sig = ((u64)(rnd() * 9007199254740992.0) | ((u64)(rnd() * 1024.0) << 53)) & all & ~pinned;
            for (int v = 0; v < nv; ++v) uf[v] = v;
            auto part = [&](int v) { return (c.A >> D->src[v]) & 1ull ? 0 : ((c.B >> D->src[v]) & 1ull ? 1 : -1); };
            auto sgn = [&](int v) { return (int)(((sig >> D->src[v]) & 1ull) ^ (D->par[v] & 1)); };
            for (int e = 0; e < D->ne; ++e) {
                const int u = D->edge_u[e], v = D->edge_v[e];
                const int pu = part(u);
                if (pu >= 0 && pu == part(v) && sgn(u) == sgn(v)) uf[find(u)] = find(v);
            }
            int n = c.cost;
            for (int v = 0; v < nv; ++v)
                if (D->used[v] && part(v) >= 0 && find(v) == v) ++n;
            tot += n;
            over += n > 64;
        }
        const double sc = tot / NS + 300.0 * over / NS;
        if (sc < best) {
            best = sc;
            bi = ci;
            S.mean_nodes = tot / NS;
        }
    }
    const Cand &c = cands[bi];
    if (const char *e = std::getenv("TCG_SPLIT_DEBUG"))
        if (e[0] && e[0] != '0')
            std::fprintf(stderr, "[tcg split] %zu candidates; F = %d points / %d vertices, "
                         "mean contracted graph %.1f nodes, score %.1f\n",
                         cands.size(), popc(c.F), c.cost, S.mean_nodes, best);
    // F vertices in layout order; part vertex masks; index ranks
    std::vector<std::pair<int, int>> fv;
    SplitPart *parts[2] = {&S.pa, &S.pb};
    const u64 pm[2] = {c.A, c.B};
    *parts[0] = SplitPart{};
    *parts[1] = SplitPart{};
    for (int v = 0; v < nv; ++v) {
        if (!D->used[v]) continue;
        const int p = D->src[v], pos = L.pos[v];
        if ((c.F >> p) & 1ull) fv.push_back({pos, v});
        for (int t = 0; t < 2; ++t)
            if ((pm[t] >> p) & 1ull) {
                parts[t]->pm[pos >> 5] |= 1u << (pos & 31);
                ++parts[t]->npv;
            }
    }
    std::sort(fv.begin(), fv.end());
    const int nF = (int)fv.size();
    std::vector<int> fnode(nv, -1);
    for (int f = 0; f < nF; ++f) fnode[fv[f].second] = f;
    SplitParams &sp = S.sp;
    sp = SplitParams{};
    sp.nF = nF;
    sp.nFp = (nF + 3) & ~3;
    sp.stride = split_stride(sp.nFp);
    sp.nbytes = (npts + 7) / 8;
    sp.maxnodes = 64;
    if (const char *e = std::getenv("TCG_SPLIT_MAXNODES")) sp.maxnodes = std::max(1, std::min(64, std::atoi(e)));
    // bytes of each entry prefetched into L2 per draw (TCG_SPLIT_PREFETCH; off by
    // default: 256 / 768 B measured 7 % / 19 % slower on bowtie8)
    sp.prefetch = 0;
    if (const char *e = std::getenv("TCG_SPLIT_PREFETCH")) sp.prefetch = std::max(0, std::atoi(e));
    for (int e = 0; e < D->ne; ++e) {
        const int fu = fnode[D->edge_u[e]], fw = fnode[D->edge_v[e]];
        if (fu >= 0 && fw >= 0) {
            sp.fadj[fu] |= 1u << fw;
            sp.fadj[fw] |= 1u << fu;
        }
    }
    for (int a = 0; a < D->nap; ++a) {
        const int fu = fnode[D->ap_u[a]], fw = fnode[D->ap_v[a]];
        if (fu >= 0 && fw >= 0) {
            sp.flink[fu] |= 1u << fw;
            sp.flink[fw] |= 1u << fu;
        }
    }
    int rank[64];
    int nrank[3] = {0, 0, 0};  // A, B, F free points
    for (int p = 0; p < npts; ++p) {
        rank[p] = -1;
        if ((pinned >> p) & 1ull) continue;
        const int t = ((c.A >> p) & 1ull) ? 0 : (((c.B >> p) & 1ull) ? 1 : 2);
        rank[p] = nrank[t]++;
        if (t < 2) parts[t]->pt[rank[p]] = (uint8_t)p;
    }
    S.nfpts = popc(c.F);
    S.Fm = c.F;
    S.Am = c.A;
    S.Bm = c.B;
    uint32_t parm = 0, cm[SPL_MAXFB] = {};
    for (int f = 0; f < nF; ++f) {
        const int v = fv[f].second, p = D->src[v];
        parm |= (uint32_t)(D->par[v] & 1) << f;
        if (rank[p] >= 0) cm[rank[p]] |= 1u << f;
    }
    for (int x = 0; x < 64; ++x) {
        uint32_t w0 = parm, w1 = 0;
        for (int i = 0; i < 6; ++i)
            if ((x >> i) & 1) {
                w0 ^= cm[i];
                w1 ^= cm[6 + i];
            }
        sp.fsign[0][x] = w0;
        sp.fsign[1][x] = w1;
    }
    S.pext.assign((size_t)sp.nbytes * 256, 0ull);
    for (int j = 0; j < sp.nbytes; ++j)
        for (int v = 0; v < 256; ++v) {
            u64 w = 0;
            for (int b = 0; b < 8; ++b) {
                const int p = 8 * j + b;
                if (p >= npts || !((v >> b) & 1) || rank[p] < 0) continue;
                const int t = ((c.A >> p) & 1ull) ? 0 : (((c.B >> p) & 1ull) ? 1 : 2);
                w |= 1ull << (rank[p] + (t == 0 ? 0 : (t == 1 ? 24 : 48)));
            }
            S.pext[(size_t)j * 256 + v] = w;
        }
    for (int t = 0; t < 2; ++t) {
        SplitPart &P = *parts[t];
        P.bits = nrank[t];
        P.nF = nF;
        P.nFp = sp.nFp;
        P.stride = sp.stride;
        for (int f = 0; f < nF; ++f) {
            const int pos = fv[f].first;
            P.fword[f] = (uint32_t)(pos >> 5);
            P.fbit[f] = 1u << (pos & 31);
        }
    }
    return true;
}
