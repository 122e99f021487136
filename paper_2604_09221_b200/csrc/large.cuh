// large.cuh -- the any-degree kernel (one CTA per patchwork, reference vertex
// numbering).  Included by tcg.cu inside its anonymous namespace.

// ------------------------------------------------------------ any degree
// Generic path for degrees the bit-mask layout does not cover (d > 9; any d
// works): one CTA per patchwork, state in shared memory, vertex numbering
// and edge order exactly the reference's.  Components by a lock-free
// union-find over the non-crossed edges (CAS hooking of the larger root onto
// the smaller, path halving); the parity union-find over the 2d antipodal
// pairs, region ids, odd flags and any status collision are replayed by one
// thread in the reference's order (kernels.py:151-230); the crossed-edge
// region pairs are deduplicated in a shared hash set; the rooted tree comes
// back as a parent array for the host to render.
struct LargeParams {
    int d, nv, ne, nap, npts, maxreg, words;  // words = u64 per sign row
    const int32_t *eu, *ev, *src, *apu, *apv;
    const uint8_t *par, *used;
};

constexpr int LHASH = 8192;  // region-pair hash set (pairs <= maxreg - 1 on valid input)

__device__ __forceinline__ int lfind(int *p, int x) {
    while (true) {
        const int px = p[x];
        if (px == x) return x;
        const int ppx = p[px];
        if (ppx != px) p[x] = ppx;  // path halving (benign race: only shortens paths)
        x = px;
    }
}

__device__ int lfind2(int *p2, uint8_t *par2, int x, int &parity) {
    int root = x, pp = 0;
    while (p2[root] != root) {
        pp ^= par2[root];
        root = p2[root];
    }
    int v = x, acc = pp;
    while (p2[v] != v) {
        const int nxt = p2[v];
        const int step = par2[v];
        p2[v] = root;
        par2[v] = (uint8_t)acc;
        acc ^= step;
        v = nxt;
    }
    parity = pp;
    return root;
}

// insert (a, b) into the pair set; returns true if it was new
__device__ __forceinline__ bool pair_insert(uint32_t *hs, uint32_t key) {
    uint32_t h = (key * 2654435761u) & (LHASH - 1);
    for (int probe = 0; probe < LHASH; ++probe) {
        const uint32_t prev = atomicCAS(&hs[h], 0xffffffffu, key);
        if (prev == 0xffffffffu) return true;
        if (prev == key) return false;
        h = (h + 1) & (LHASH - 1);
    }
    return false;
}

__global__ void __launch_bounds__(THREADS) k_large(LargeParams P, const uint64_t *__restrict__ sig,
                                                   int64_t n, int32_t *__restrict__ status,
                                                   int32_t *__restrict__ nreg_out,
                                                   int32_t *__restrict__ parent_out) {
    extern __shared__ __align__(16) uint32_t smem[];
    const int nv = P.nv;
    int *p1 = reinterpret_cast<int *>(smem);       // [nv] component union-find
    int *rid = p1 + nv;                            // [nv] region id per vertex
    int *p2 = rid + nv;                            // [nv] parity union-find (by vertex id)
    uint32_t *hs = reinterpret_cast<uint32_t *>(p2 + nv);  // [LHASH]
    int *deg = reinterpret_cast<int *>(hs + LHASH);        // [maxreg + 1] CSR offsets
    int *adjl = deg + P.maxreg + 1;                        // [2 * maxreg]
    int *bfs = adjl + 2 * P.maxreg;                        // [maxreg]
    int *rpar = bfs + P.maxreg;                            // [maxreg]
    uint8_t *sg = reinterpret_cast<uint8_t *>(rpar + P.maxreg);  // [nv]
    uint8_t *par2 = sg + nv;                                     // [nv]
    uint8_t *odd2 = par2 + nv;                                   // [nv]
    __shared__ int s_nreg, s_status, s_root, s_nedges, s_selfm, s_self1, s_self2;
    for (int64_t t = blockIdx.x; t < n; t += gridDim.x) {
        const uint64_t *row = sig + t * P.words;
        for (int v = threadIdx.x; v < nv; v += blockDim.x) {
            const int k = P.src[v];
            sg[v] = (uint8_t)(((row[k >> 6] >> (k & 63)) & 1ull) ^ P.par[v]);
            p1[v] = v;
            p2[v] = v;
            par2[v] = 0;
            odd2[v] = 0;
        }
        for (int i = threadIdx.x; i < LHASH; i += blockDim.x) hs[i] = 0xffffffffu;
        __syncthreads();
        for (int e = threadIdx.x; e < P.ne; e += blockDim.x) {
            int u = P.eu[e], v = P.ev[e];
            if (sg[u] != sg[v]) continue;
            while (true) {
                u = lfind(p1, u);
                v = lfind(p1, v);
                if (u == v) break;
                if (u < v) { const int tmp = u; u = v; v = tmp; }
                if (atomicCAS(&p1[u], u, v) == u) break;
            }
        }
        __syncthreads();
        // flatten in two phases: roots found read-only (into rid, free until the
        // region ids below), then stored.  A halving find here could land a stale
        // non-root ancestor in p1[v] after v's own thread stored the root.
        for (int v = threadIdx.x; v < nv; v += blockDim.x) {
            int x = v;
            while (p1[x] != x) x = p1[x];
            rid[v] = x;
        }
        __syncthreads();
        for (int v = threadIdx.x; v < nv; v += blockDim.x) p1[v] = rid[v];
        __syncthreads();
        if (threadIdx.x == 0) {
            // parity union-find over the antipodal pairs (components named by root vertex)
            for (int a = 0; a < P.nap; ++a) {
                const int cu = p1[P.apu[a]], cv = p1[P.apv[a]];
                int pu, pv;
                int ru = lfind2(p2, par2, cu, pu), rv = lfind2(p2, par2, cv, pv);
                if (ru == rv) {
                    if (pu == pv) odd2[ru] = 1;
                } else {
                    // deterministic: hook the larger root onto the smaller
                    if (ru > rv) { const int tmp = ru; ru = rv; rv = tmp; const int tp = pu; pu = pv; pv = tp; }
                    p2[rv] = ru;
                    par2[rv] = (uint8_t)(pu ^ pv ^ 1);
                    if (odd2[rv]) odd2[ru] = 1;
                }
            }
            // dense region ids in vertex order (the reference's first-occurrence order)
            int nreg = 0, nodd = 0, oddr = -1, st = TCG_OK;
            for (int v = 0; v < nv; ++v) {
                if (!P.used[v] || p1[v] != v) continue;
                int pp;
                const int r = lfind2(p2, par2, v, pp);
                if (r == v) {
                    if (nreg >= P.maxreg) { st = TCG_TOO_MANY_REGIONS; break; }
                    rid[v] = nreg;
                    if (odd2[v]) { ++nodd; oddr = nreg; }
                    ++nreg;
                }
            }
            if (st == TCG_OK) {
                for (int v = 0; v < nv; ++v) {
                    if (!P.used[v] || p1[v] != v) continue;
                    int pp;
                    const int r = lfind2(p2, par2, v, pp);
                    rid[v] = rid[r];
                }
            }
            if (st == TCG_OK && P.d % 2 == 0) {
                if (nodd == 0) st = TCG_NO_ODD_REGION;
                else if (nodd > 1) st = TCG_MANY_ODD_REGIONS;
            }
            s_nreg = nreg;
            s_status = st;
            s_root = P.d % 2 == 0 ? oddr : -1;
            s_nedges = 0;
            s_selfm = 0;
            s_self1 = -1;
            s_self2 = -1;
        }
        __syncthreads();
        for (int v = threadIdx.x; v < nv; v += blockDim.x)
            if (P.used[v]) rid[v] = rid[p1[v]];
        __syncthreads();
        if (s_status == TCG_OK) {
            for (int e = threadIdx.x; e < P.ne; e += blockDim.x) {
                const int u = P.eu[e], v = P.ev[e];
                if (sg[u] == sg[v]) continue;
                int a = rid[u], b = rid[v];
                if (a == b) {
                    atomicAdd(&s_selfm, 1);
                    if (atomicCAS(&s_self1, -1, a) != -1 && s_self1 != a) atomicExch(&s_self2, a);
                    continue;
                }
                if (a > b) { const int tmp = a; a = b; b = tmp; }
                if (pair_insert(hs, ((uint32_t)a << 16) | (uint32_t)b)) atomicAdd(&s_nedges, 1);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && s_status == TCG_OK) {
            const int nreg = s_nreg;
            const bool even = P.d % 2 == 0;
            const bool toomany = s_nedges > nreg - 1;
            const bool anomaly = toomany || (even && s_selfm) || (!even && s_self2 >= 0);
            int st = TCG_OK, root = s_root;
            if (anomaly) {
                // exact replay in the reference's edge order (kernels.py:199-230)
                for (int i = 0; i < LHASH; ++i) hs[i] = 0xffffffffu;
                int ne2 = 0;
                root = even ? s_root : -1;
                for (int e = 0; e < P.ne && st == TCG_OK; ++e) {
                    const int u = P.eu[e], v = P.ev[e];
                    if (sg[u] == sg[v]) continue;
                    int a = rid[u], b = rid[v];
                    if (a == b) {
                        if (even) st = TCG_NONSEPARATING_OVAL;
                        else if (root < 0) root = a;
                        else if (root != a) st = TCG_ROOT_CONFLICT;
                        continue;
                    }
                    if (a > b) { const int tmp = a; a = b; b = tmp; }
                    if (pair_insert(hs, ((uint32_t)a << 16) | (uint32_t)b)) {
                        if (ne2 >= nreg - 1) st = TCG_NOT_A_TREE;
                        ++ne2;
                    }
                }
                if (st == TCG_OK) st = TCG_NOT_A_TREE;  // unreachable for anomalous inputs
            } else if (!even) {
                if (s_self1 < 0) st = TCG_NO_PSEUDOLINE;
                root = s_self1;
            }
            if (st == TCG_OK && s_nedges != nreg - 1) st = TCG_NOT_A_TREE;
            if (st == TCG_OK) {
                // CSR over the deduplicated pairs, BFS from the root
                for (int r = 0; r <= nreg; ++r) deg[r] = 0;
                for (int i = 0; i < LHASH; ++i) {
                    const uint32_t k = hs[i];
                    if (k == 0xffffffffu) continue;
                    deg[(k >> 16) + 1]++;
                    deg[(k & 0xffff) + 1]++;
                }
                for (int r = 0; r < nreg; ++r) deg[r + 1] += deg[r];
                for (int r = 0; r < nreg; ++r) rpar[r] = deg[r];
                for (int i = 0; i < LHASH; ++i) {
                    const uint32_t k = hs[i];
                    if (k == 0xffffffffu) continue;
                    const int a = (int)(k >> 16), b = (int)(k & 0xffff);
                    adjl[rpar[a]++] = b;
                    adjl[rpar[b]++] = a;
                }
                for (int r = 0; r < nreg; ++r) rpar[r] = -1;
                int head = 0, tail = 1;
                bfs[0] = root;
                rpar[root] = root;
                while (head < tail) {
                    const int r = bfs[head++];
                    for (int k = deg[r]; k < deg[r + 1]; ++k) {
                        const int s2 = adjl[k];
                        if (rpar[s2] < 0) {
                            rpar[s2] = r;
                            bfs[tail++] = s2;
                        }
                    }
                }
                if (tail != nreg) st = TCG_DISCONNECTED;
            }
            s_status = st;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            status[t] = s_status;
            nreg_out[t] = s_nreg;
        }
        if (s_status == TCG_OK)
            for (int r = threadIdx.x; r < s_nreg; r += blockDim.x)
                parent_out[t * P.maxreg + r] = rpar[r];
        __syncthreads();
    }
}
