/*
 * tcg.h -- C ABI of the sm_100a patchwork classifier (libtcg.so).
 *
 * Drop-in boundary for the reference's compiled hot path.  The reference
 * (arXiv 2604.09221 companion package `tcurves`) crosses from Python into
 * native code at three numba dispatchers; each entry point below replaces
 * one of them:
 *
 *   tcg_plan_create       <- classify.py:24-55   Classifier.__init__ / plan():
 *                            the plan tuple (d, nv, npts, edge_u, edge_v, src,
 *                            par, used, ap_u, ap_v, maxreg) is passed verbatim
 *                            as tcg_desc (same arrays, same vertex numbering)
 *   tcg_classify_batch    <- kernels.py:366-368  classify_bits_kernel(plan, scr, bits)
 *                            (called at classify.py:94), batched: n sign words
 *   tcg_sweep             <- kernels.py:423-436  sweep_kernel(plan, scr, agg, bits,
 *                            start, end) (called per chunk at sweep.py:153, merged
 *                            at sweep.py:168-180); one call covers the whole range
 *   tcg_sample            <- kernels.py:447-462  sample_kernel(plan, scr, agg, bits,
 *                            seed, k0, k1, nbits) (sweep.py:245-246)
 *   tcg_*_multi           <- sweep.py:143-180    _run_chunks' thread pool, one host
 *                            thread per device instead of per CPU worker
 *
 * Differences the caller must know (everything else is the reference's):
 *  - Schemes come back as 64-bit canonical tree keys (AHU balanced
 *    parentheses with a sentinel bit), not strings; the host renders the
 *    reference string once per distinct key (paper_2604_09221_b200/scheme.py).
 *    ovals = (bit_length(key) - 1) / 2.
 *  - Sign vectors travel as one uint64 word per patchwork: bit k = sign of
 *    lattice point k (d <= 9).
 *  - The aggregate is keyed by tree key; counts add and witnesses take the
 *    minimum index exactly as in _aggregate (kernels.py:379-420).  Hash
 *    collisions are impossible (the key is the exact tree code).
 *
 * Status codes are the reference's (kernels.py:20-31); negative values are
 * library errors.  All buffers passed to tcg_classify_batch / tcg_sweep /
 * tcg_sample / tcg_agg_fetch are HOST buffers owned by the caller; the
 * library owns every device buffer.  Calls on one plan are serialised on
 * that plan's stream; different plans (devices) may be driven from
 * different host threads concurrently.
 */
#ifndef TCG_H
#define TCG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    TCG_OK = 0,
    TCG_TOO_MANY_REGIONS = 1,
    TCG_NO_ODD_REGION = 2,
    TCG_MANY_ODD_REGIONS = 3,
    TCG_NO_PSEUDOLINE = 4,
    TCG_ROOT_CONFLICT = 5,
    TCG_NONSEPARATING_OVAL = 6,
    TCG_NOT_A_TREE = 7,
    TCG_DISCONNECTED = 8,
    TCG_ARENA_OVERFLOW = 9,
    TCG_TABLE_FULL = 10,
    TCG_HASH_COLLISION = 11,
    /* library errors */
    TCG_E_ARG = -1,
    TCG_E_CUDA = -2,
    TCG_E_UNSUPPORTED = -3,
    TCG_E_RANGE = -4
};

/* The reference plan tuple (classify.py:47-49), flat.  Vertex numbering is
 * the lexicographic diamond order (diamond.py:25-31); edges are in the
 * reference's sorted order (diamond.py:102). */
typedef struct tcg_desc {
    int32_t degree;
    int32_t nv;
    int32_t npts;
    int32_t ne;
    const int32_t *edge_u; /* [ne] */
    const int32_t *edge_v; /* [ne] */
    const int32_t *src;    /* [nv] index into A(d) */
    const uint8_t *par;    /* [nv] sign-extension parity */
    const uint8_t *used;   /* [nv] */
    int32_t nap;
    const int32_t *ap_u; /* [nap] antipodal pairs */
    const int32_t *ap_v; /* [nap] */
    int32_t maxreg;      /* harnack_bound(d) + 2 */
} tcg_desc;

typedef struct tcg_plan tcg_plan;

/* Aggregate of a sweep / sample (the reference's agg 9-tuple, sweep.py:118-130,
 * reduced to its observable content).  key/count/witness are caller-owned
 * arrays of `cap` entries; `n` is set to the number of distinct schemes. */
typedef struct tcg_agg {
    int64_t hist[64]; /* oval histogram, bins 0..maxreg */
    int64_t total;
    int32_t n;
    int32_t cap;
    uint64_t *key;
    int64_t *count;
    int64_t *witness; /* minimal index in the run's own domain */
} tcg_agg;

/* Plan lifetime.  device < 0 selects the current device. */
int tcg_plan_create(const tcg_desc *desc, int device, tcg_plan **out);
int tcg_plan_destroy(tcg_plan *plan);
/* Use an external cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream);
 * NULL restores the plan's own stream. */
int tcg_plan_set_stream(tcg_plan *plan, void *cuda_stream);
/* info[0]=degree info[1]=mask words K info[2]=used vertices info[3]=device
 * info[4]=SM count info[5]=CTAs per launch info[6]=threads per CTA
 * info[7]=maxreg info[8]/info[9]=tile bits for raw/representative sweeps
 * (0 = sweeps of that domain use the flat kernel) */
int tcg_plan_info(const tcg_plan *plan, int32_t *info, int ninfo);
/* Per-kernel device time (CUDA events on the plan's stream around every
 * launch) while enabled.  tcg_kernel_times returns and clears the totals:
 * ms[TCG_NKINDS] / counts[TCG_NKINDS], indexed by the TCG_KT_* kinds. */
#define TCG_KT_TILE_BUILD 0    /* k_tile_from_super (+ k_tile_build_lanes): tile contraction */
#define TCG_KT_TILE_CLASSIFY 1 /* k_tile_classify: level-1 tile classification */
#define TCG_KT_ENUMERATE 2     /* k_enumerate: flat per-patchwork sweeps / sampling */
#define TCG_KT_BATCH 3         /* k_batch: explicit sign words */
#define TCG_KT_TILE_DEDUP 4    /* k_tile_dedup: level-1 record deduplication */
#define TCG_KT_L2_BUILD 5      /* k_l2_build / k_l2_from_l15: level-2 records */
#define TCG_KT_L2_DEDUP 6      /* k_l2_dedup: level-2 record deduplication */
#define TCG_KT_L2_CLASSIFY 7   /* k_l2_classify: level-2 classification */
#define TCG_KT_SUPER_BUILD 8   /* k_super_build: super-tile contraction */
#define TCG_KT_L15_BUILD 9     /* k_l15_build: two-stage level 2, stage 1 */
#define TCG_KT_L15_DEDUP 10    /* k_l2_dedup on the stage-1 records */
#define TCG_KT_SPLIT_BUILD 11  /* k_split_build: the sampler's component tables (once per plan) */
#define TCG_KT_SAMPLE_SPLIT 12 /* k_sample_split: sampling on the separator-contracted graph */
#define TCG_KT_SAMPLE_LIST 13  /* k_sample_list: draws the split sampler left to the flat classifier */
#define TCG_NKINDS 14
int tcg_plan_set_timing(tcg_plan *plan, int enable);
int tcg_kernel_times(tcg_plan *plan, double *ms, int64_t *counts);
/* Tile deduplication (exhaustive sweeps): tiles whose contracted records are
 * identical are classified once and counted with their multiplicity (the
 * witness is taken from the group's smallest tile, so reports are unchanged).
 * enable: 1 on, 0 off, -1 default (on unless TCG_NO_DEDUP=1). */
int tcg_plan_set_dedup(tcg_plan *plan, int enable);
/* out[0] = tiles contracted, out[1] = distinct tiles (level-1 representatives;
 * = out[0] without deduplication) since the last call
 * (synchronises the plan's stream); resets both. */
int tcg_tile_stats(tcg_plan *plan, int64_t *out);
/* Level-2 contraction (odd degree sweeps, on by default with deduplication;
 * TCG_NO_L2=1 or enable=0 turns it off): each representative tile is split
 * into 2^(b-5) records of 32 patchworks with the other tile bits fixed, and
 * equal records are classified once (exact, like tile deduplication).
 * tcg_level2_stats: out[0] = records built, out[1] = records classified,
 * out[2] = tiles the level-1 classifier took while level 2 ran (range ends,
 * graphs over 32 nodes, fallback tiles); all since the last call. */
int tcg_plan_set_level2(tcg_plan *plan, int enable);
int tcg_level2_stats(tcg_plan *plan, int64_t *out);
/* Separator-split sampling (d >= 6; on by default for samples of >= 2^22
 * draws, and for any sample once the tables exist; enable=1 forces it,
 * TCG_NO_SPLIT=1 or enable=0 samples with the flat kernel only -- results are
 * identical).  At the first such sample the plan picks a small vertex separator F of T's edge
 * graph and tabulates, for every sign pattern of each side, the same-sign
 * components of that side's diamond vertices (device memory, once); each draw
 * is then classified on the graph of F's vertices plus the two sides'
 * components.  Draws whose graph exceeds 64 nodes, or whose status is not OK,
 * are re-classified by the flat kernel.  If the tables would take more than
 * half of the free device memory the plan samples with the flat kernel.
 * tcg_split_stats: out[0] = state
 * (1 ready, -1 unavailable: flat sampling, 0 not built yet), out[1] = draws
 * sampled through the split kernel, out[2] = of those, draws the flat kernel
 * took, out[3] = separator vertices, out[4] = table bytes; counts since the
 * last call (synchronises the plan's stream). */
int tcg_plan_set_split(tcg_plan *plan, int enable);
int tcg_split_stats(tcg_plan *plan, int64_t *out);
/* The separator design for a descriptor, on the host (no device needed):
 * out[0] = 1 if the split sampler applies, out[1] = separator vertices,
 * out[2] / out[3] = index bits of the two tables, out[4..6] = lattice-point
 * masks of the separator F and the two sides A, B, out[7] = estimated mean
 * contracted-graph size x 1000, out[8] = table bytes. */
int tcg_split_design(const tcg_desc *desc, int64_t *out);

/* classify_bits_kernel, batched.  sigma[t] bit k = sign of point k.
 * Outputs per patchwork: tree key, oval count, region count, status. */
int tcg_classify_batch(tcg_plan *plan, const uint64_t *sigma, int64_t n, uint64_t *key,
                       uint8_t *ovals, uint8_t *nreg, int32_t *status);
/* Same with DEVICE pointers, asynchronous on the plan's stream. */
int tcg_classify_batch_device(tcg_plan *plan, const uint64_t *d_sigma, int64_t n,
                              uint64_t *d_key, uint8_t *d_ovals, uint8_t *d_nreg,
                              int32_t *d_status);

/* sweep_kernel over [start, end) of the representative (raw=0) or raw
 * (raw=1) domain; sample_kernel over draws [k0, k1) with nbits-bit indices.
 * Return TCG_OK or the status of the failing patchwork with the smallest
 * index (*bad = that index: m for sweeps, the drawn m of the earliest failing
 * draw for samples), or a negative library error.
 * TCG_TABLE_FULL follows the reference's threshold (kernels.py:389-391: a
 * new scheme is refused once 32,768 are stored): it is returned when the run
 * meets more than 32,768 distinct schemes, with *bad = the 32,769th smallest
 * witness -- the index where one sequential worker (workers=1) stops.  If a
 * classification failure comes first in index order, that status wins.  For
 * samples, whose witnesses are not in draw order, a classification failure
 * always wins and *bad is the 32,769th smallest witness m.  Exact while the
 * device table (65,536 schemes) has not overflowed.  HASH_COLLISION cannot
 * occur (keys are exact tree codes). */
int tcg_sweep(tcg_plan *plan, int raw, uint64_t start, uint64_t end, tcg_agg *agg, int64_t *bad);
int tcg_sample(tcg_plan *plan, uint64_t seed, uint64_t k0, uint64_t k1, int nbits, tcg_agg *agg,
               int64_t *bad);

/* Split-phase form (accumulate on the device across calls, fetch once).
 * tcg_agg_reset zeroes the device aggregate; the *_async calls only
 * enqueue work on the plan's stream; tcg_agg_fetch synchronises, copies
 * the aggregate back and resolves errors like tcg_sweep. */
int tcg_agg_reset(tcg_plan *plan);
int tcg_sweep_async(tcg_plan *plan, int raw, uint64_t start, uint64_t end);
int tcg_sample_async(tcg_plan *plan, uint64_t seed, uint64_t k0, uint64_t k1, int nbits);
int tcg_agg_fetch(tcg_plan *plan, tcg_agg *agg, int64_t *bad);

/* Multi-device: contiguous shards of the range, one host thread per plan
 * (plans on distinct devices, or several distinct plans on one device),
 * merged on the host (count sum, witness min).  A plan may appear only once
 * (TCG_E_ARG otherwise: its stream and aggregate are single-owner).  The
 * failure rules above are applied to the merged run -- the earliest failure
 * in enumeration order (index for sweeps, draw k for samples) -- so output and
 * status are identical for any number of plans. */
int tcg_sweep_multi(tcg_plan **plans, int nplans, int raw, uint64_t start, uint64_t end,
                    tcg_agg *agg, int64_t *bad);
int tcg_sample_multi(tcg_plan **plans, int nplans, uint64_t seed, uint64_t k0, uint64_t k1,
                     int nbits, tcg_agg *agg, int64_t *bad);

/* Many triangulations of one degree on one device (config C4, SURVEY
 * section 8f row 2): pairs (tri[t], sigma[t]) are grouped by triangulation
 * and every CTA classifies one group on its own topology.  Host buffers;
 * outputs in the input order; the call pipelines chunks of 2^22 pairs
 * through pinned staging (host threads copy in and out while the GPU copies
 * and classifies the neighbouring chunks).  tcg_multi_last_ms = device time
 * of the last call's classification kernels (CUDA events, summed). */
typedef struct tcg_multi tcg_multi;
int tcg_multi_create(const tcg_desc *descs, int32_t ntri, int device, tcg_multi **out);
int tcg_multi_destroy(tcg_multi *m);
int tcg_multi_classify(tcg_multi *m, const int32_t *tri, const uint64_t *sigma, int64_t n,
                       uint64_t *key, uint8_t *ovals, uint8_t *nreg, int32_t *status);
double tcg_multi_last_ms(const tcg_multi *m);

/* Any degree (d > 9 included) for single patchworks and batches; sweeps and
 * samples stay d <= 9 as in the reference (62-bit index cap, sweep.py:32).
 * One CTA per patchwork.  sigma_rows: n rows of ceil(npts/64) uint64 words
 * (bit k of a row = sign of point k).  Outputs: status[n], nreg[n] and, for
 * status 0, the rooted region tree as parent[n][maxreg] (parent[t][r] of
 * region r; the root is its own parent); the scheme is rendered on the host
 * (ovals = nreg - 1). */
typedef struct tcg_large tcg_large;
int tcg_large_create(const tcg_desc *desc, int device, tcg_large **out);
int tcg_large_destroy(tcg_large *g);
int tcg_large_classify(tcg_large *g, const uint64_t *sigma_rows, int64_t n, int32_t *status,
                       int32_t *nreg, int32_t *parent);

/* Diagnostics. */
const char *tcg_last_error(void);
int tcg_device_count(void);
int64_t tcg_launch_count(const tcg_plan *plan); /* kernels this plan launched */
const char *tcg_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TCG_H */
