/*
 * tsb.h -- C ABI of the B200 (sm_100a) tilesampler library, libtsb.so.
 *
 * Drop-in boundary for the reference `tilesampler` hot path (colour-class
 * Glauber sweeps + CFTP).  Plain pointers and sizes only; host buffers use the
 * reference's own layouts and dtypes, so a binding is a few ctypes lines
 * (see INTEGRATION.md).  Reference paths are relative to
 * /root/reference/pkg/src/tilesampler/.
 *
 * Conventions
 *  - Every entry point returns a status (0 = OK).  Non-zero codes map to the
 *    reference exception taxonomy (errors.py:4-69); tsb_last_error() gives the
 *    message of the calling thread's last failure.
 *  - Handles own device memory; callers own host buffers.  A handle is used by
 *    one host thread at a time; distinct handles are independent.
 *  - Work is enqueued on the handle's stream (tsb_*_set_stream to share a
 *    torch stream).  *_download and *_sync synchronise that stream.
 *  - Chain k's result depends only on its own seed, never on batching or on
 *    which device ran it (reference contract sweeps.py:286-292, cftp.py:11-14).
 *  - There is no CPU fallback: without an sm_100 device every call fails
 *    with TSB_E_NODEVICE.
 */
#ifndef TSB_H
#define TSB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    TSB_OK = 0,
    TSB_E_VALUE = 1,        /* ValueError                                     */
    TSB_E_INCONSISTENT = 2, /* InconsistencyError   (errors.py:24-25)         */
    TSB_E_CAPACITY = 3,     /* CapacityError        (errors.py:32-33)         */
    TSB_E_CUDA = 4,         /* RuntimeError: CUDA failure                     */
    TSB_E_NODEVICE = 5,     /* RuntimeError: no sm_100 device                 */
    TSB_E_CONVERGENCE = 6,  /* ConvergenceCapExceeded (errors.py:64-65)       */
    TSB_E_DOMAIN = 7,       /* DomainError          (errors.py:8-9)           */
    TSB_E_UNTILEABLE = 8,   /* UntileableDomain     (errors.py:56-57)         */
    TSB_E_INFEASIBLE = 9    /* InfeasibleBoundary   (errors.py:52-53)         */
};

/* ---------------------------------------------------------------- library */
const char *tsb_last_error(void);
int tsb_abi_version(void);
/* SM count, compute capability and L2 size of `device`. */
/* Number of 4-connected components of the nonzero cells of a (rows x cols)
 * uint8 grid (GPU union-find): the Domain checks of lattice.py:99-132
 * (faces connected <=> 1 component; no hole <=> the complement padded by one
 * ring of cells is 1 component) without the reference's Python DFS. */
int tsb_grid_components(int device, const uint8_t *grid, int rows, int cols, int64_t *ncomp);
/* TriDomain checks (lozenge.py:185-210) on the device: number of
 * edge-connected components of the up/down triangles ((sx, sy) uint8 grids;
 * up(x,y) touches down(x,y), down(x-1,y), down(x,y-1)) and the Euler
 * characteristic V - E + F (simply connected <=> 1). */
int tsb_tri_check(int device, const uint8_t *up, const uint8_t *down, int sx, int sy, int64_t *ncomp,
                  int64_t *euler);
int tsb_device_info(int device, int *sm_count, int *cc_major, int *cc_minor, int64_t *l2_bytes);

/* ------------------------------------------------------------------- RNG */
/* StreamFamily(seed, (rows, cols)).uniform_grid(step, tag) -> out[rows*cols]
 * float64, computed on the device.  Replaces rng.py:105-123 (and the batched
 * key_grid_batch/uniform_from_keys, rng.py:138-162).  Host output buffer. */
int tsb_uniform_grid(int device, uint64_t seed, int rows, int cols, uint64_t step, int tag,
                     double *out);

/* --------------------------------------------------------------- dominoes */
typedef struct tsb_domino tsb_domino;

/* A batch of `nchains` domino chains on the (side x side) vertex grid,
 * side = Domain.n + 1 (lattice.py:267-280).  `faces` is the Domain.faces
 * grid ((side-1) x (side-1), uint8/bool, row-major) or NULL for the full box;
 * it bounds the work region and the crossable edges. */
int tsb_domino_create(int device, int side, int nchains, const uint8_t *faces, tsb_domino **out);
int tsb_domino_destroy(tsb_domino *h);
/* One chain of the `side` x `side` grid holding only the global rows
 * [row_lo, row_hi) (plus a zero margin): state planes, domain planes and
 * tiles cover the window, so N strip ranks hold 1/N of a lattice each.
 * Rows keep their global indices (coins and colours are unchanged).  Whole-grid
 * operations (upload / download / heights / extremal / cftp / observables)
 * fail with TSB_E_VALUE; use tsb_domino_upload_rows / download_rows.  `faces`
 * is the full (side-1)^2 grid (NULL: all faces). */
int tsb_domino_create_window(int device, int side, int row_lo, int row_hi, const uint8_t *faces, tsb_domino **out);
/* Rows [r0, r0+nrows) of chain 0 from / to a host (nrows, side) uint8
 * tilestate grid (the reference layout); any handle, rows within its window.
 * The "up" bit of a window's first row refers to a row the window does not
 * hold: it is not checked on upload and reads back as 0. */
int tsb_domino_upload_rows(tsb_domino *h, int r0, int nrows, const uint8_t *rows);
int tsb_domino_download_rows(tsb_domino *h, int r0, int nrows, uint8_t *rows);
/* Use an external cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream). */
int tsb_domino_set_stream(tsb_domino *h, void *stream);
/* SweepPlan.p_up, (side x side) float64 (sweeps.py:170-179).  Converted
 * exactly to integer thresholds: u < p  <=>  (x >> 11) < ceil(p * 2^53). */
int tsb_domino_set_p_up(tsb_domino *h, const double *p_up);
/* The same for p_up that depends only on the vertex parity (Uniform:
 * 0.5 / 0.5; VolumeWeights without overrides: q^(+-4)/(1+q^(+-4)),
 * sweeps.py:134-150): no (side x side) grid is built or stored. */
int tsb_domino_set_p_up_parity(tsb_domino *h, double p_even, double p_odd);

/* Tiling.states batch (n, side, side) uint8 <-> device state.  Upload
 * rejects grids that are not edge-consistent or that cross a non-crossable
 * edge with TSB_E_INCONSISTENT. */
int tsb_domino_upload(tsb_domino *h, int chain0, int n, const uint8_t *states);
int tsb_domino_download(tsb_domino *h, int chain0, int n, uint8_t *states);

/* n_steps sweeps of chains [chain0, chain0+n) with per-chain seeds, step
 * counter starting at step0 (the reference always uses step0 = 0; a walk of
 * a+b steps equals a walk of a steps followed by one of b steps at step0=a).
 * Replaces the fused hook _fused_walk(out, site_keys, global_keys, p_up,
 * n_steps) (sweeps.py:272-275, 306-309; _kernels.py:35-69), with seeds in
 * place of the materialised key grids (keys are derived on the device). */
int tsb_domino_walk(tsb_domino *h, int chain0, int n, const uint64_t *seeds, uint64_t step0,
                    uint64_t n_steps);
/* One sweep with an explicit colour (0 = BLACK, 1 = WHITE) at `step`
 * (sweeps.py:322-342). */
int tsb_domino_sweep(tsb_domino *h, int chain0, int n, const uint64_t *seeds, uint64_t step,
                     int color);
int tsb_domino_sync(tsb_domino *h);

/* Strip sharding (multi-GPU): restrict sweeps to the tile bands
 * covering rows [row_lo, row_hi) (row_hi < 0: all rows).  Rows outside the
 * window are left untouched; a K-sweep walk keeps rows at distance >= K from
 * the window edge exact (the dependency radius is one row per sweep). */
int tsb_domino_set_window(tsb_domino *h, int row_lo, int row_hi);
/* Packed device rows for halo exchange: rows [r0, r0+nrows) of `chain`
 * (r0 >= -1, -1 = guard row) copied to / from device memory, row_bytes each. */
int tsb_domino_row_bytes(tsb_domino *h, int64_t *bytes);
int tsb_domino_get_rows(tsb_domino *h, int chain, int r0, int nrows, void *dev_dst);
int tsb_domino_set_rows(tsb_domino *h, int chain, int r0, int nrows, const void *dev_src);

/* Device-driven strip exchange (replaces the host-driven
 * halo swap of strips.py): rank owns rows [lo, hi) of chain 0 and sweeps them
 * plus `halo` rows per side; tsb_domino_strip_init allocates the exchange
 * region (halo staging + flags) and writes its CUDA IPC handle (64 bytes,
 * cudaIpcMemHandle_t) to ipc_handle_out (nullable); connect opens the up /
 * down neighbours' handles (NULL at the lattice edge) -- or, for handles in
 * one process, connect_local links them directly.  strip_walk enqueues
 * n_steps sweeps with a peer-memory halo push + flag wait every `halo`
 * sweeps entirely in the handle's stream (no host synchronisation);
 * the strip rows are bit-identical to a single-GPU walk. */
int tsb_domino_strip_init(tsb_domino *h, int lo, int hi, int halo, void *ipc_handle_out);
int tsb_domino_strip_connect(tsb_domino *h, const void *up_handle, const void *dn_handle);
int tsb_domino_strip_connect_local(tsb_domino *h, tsb_domino *up, tsb_domino *dn);
int tsb_domino_strip_walk(tsb_domino *h, uint64_t seed, uint64_t step0, uint64_t n_steps);
/* The same walk one round at a time: strip_seed once, then per round phase 0
 * (k <= halo sweeps from step0, then push; epoch += 1) and phase 1 (flag wait
 * + pull).  Running phase 0 on all ranks before phase 1 lets several handles
 * share one GPU (tests) without depending on concurrent streams. */
int tsb_domino_strip_seed(tsb_domino *h, uint64_t seed);
int tsb_domino_strip_step(tsb_domino *h, uint64_t step0, uint64_t k, int phase);
/* Synchronise and report: TSB_E_CUDA if a flag wait gave up (~20 s without
 * the neighbour's push; the epoch is returned in timed_out_epoch). */
int tsb_domino_strip_status(tsb_domino *h, uint64_t *epoch, uint64_t *timed_out_epoch);
int tsb_domino_strip_close(tsb_domino *h);

/* Height function of chain `chain` (lattice.py:537-580): int32 (side x side),
 * 0 outside Domain.vertex_mask, h(ref) = 0 at the reference vertex
 * (lattice.py:197-203).  TSB_E_INCONSISTENT when the state does not
 * integrate. */
int tsb_domino_heights(tsb_domino *h, int chain, int ref_r, int ref_c, int32_t *out);
/* Thurston's maximal / minimal tilings of the handle's domain written into
 * chains chain_max / chain_min (lattice.py:734-754).  TSB_E_UNTILEABLE when
 * the domain has no tiling (the reference returns None). */
int tsb_domino_extremal(tsb_domino *h, int chain_max, int chain_min, int ref_r, int ref_c);

/* On-device observables (stats.py:187-245).  Adds the
 * indicator "domino-orientation" (1 where a face is covered by a horizontal
 * domino, stats.py:187-200) of chains [chain0, chain0+n) to the caller's
 * device accumulator acc_dev ((side-1)^2 uint32 counts, face-major); faces
 * outside the domain stay 0.  density_map = acc / (#states added). */
int tsb_domino_orientation_add(tsb_domino *h, int chain0, int n, uint32_t *acc_dev);

/* Heights of chains [chain0, chain0+n) (height_function, lattice.py:537-551,
 * reference vertex (ref_r, ref_c)) added to the caller's device int64
 * accumulator acc_dev (side^2, row-major; 0 outside vertex_mask): the mean
 * height function = acc / (#states added).  TSB_E_INCONSISTENT as
 * tsb_domino_heights. */
int tsb_domino_height_sum_add(tsb_domino *h, int chain0, int n, int ref_r, int ref_c, long long *acc_dev);

/* Sample-archive record of chain `chain` (stats.py:146-153
 * _serialize_state): the tilestates joined by single spaces in decimal, as one
 * line without the newline, formatted on the device.  With out == NULL or
 * cap < the record length only *len is set (size query). */
int tsb_domino_serialize(tsb_domino *h, int chain, char *out, size_t cap, size_t *len);

/* ------------------------------------------------------------------ CFTP */
/* Progress callback: (round, steps = sum_{i<=round} 2^i, samples collapsed so
 * far, batch size, user) -- the reference's progress hook (cftp.py:130-136). */
typedef void (*tsb_progress_fn)(int round_no, uint64_t steps, int collapsed, int total, void *user);

/* K7: flags[j] = 1 iff chains chain0+2j and chain0+2j+1 hold identical states
 * (collapse_check / (top == bot).all(), cftp.py:71-75, 120). */
int tsb_domino_coalesced(tsb_domino *h, int chain0, int npairs, uint8_t *flags);
/* Copy chain `src` into chains dst0, dst0+step, ... (n copies). */
int tsb_domino_replicate(tsb_domino *h, int src, int dst0, int step, int n);
/* Monotone CFTP for `count` samples with chain master seeds `masters`
 * (cftp_sample_many / run_cftp_batch, cftp.py:86-139, 161-213): doubling
 * rounds, pair seeds derive_seed(m, r, 0x51ED2701), newest pair first, each
 * round restarted from top0 (T_max) / bot0 (T_min) host grids.  Writes the
 * coalesced bottom state of sample k to out_states[k] ((count, side, side)
 * uint8) and the round it collapsed in to collapsed_round[k] (nullable).
 * Needs nchains >= 2*count + 2.  TSB_E_CONVERGENCE after max_doublings. */
int tsb_domino_cftp(tsb_domino *h, const uint8_t *top0, const uint8_t *bot0, const uint64_t *masters,
                    int count, int max_doublings, uint8_t *out_states, int32_t *collapsed_round,
                    tsb_progress_fn progress, void *user);

/* ------------------------------------------------------------- six-vertex */
typedef struct tsb_sv tsb_sv;

/* `nchains` six-vertex chains on the n x n vertex grid; state = face heights
 * (n+1) x (n+1) int32 (FaceHeights, sixvertex.py:199-210), stored on the
 * device as one bit per face (h mod 4). */
int tsb_sv_create(int device, int n, int nchains, tsb_sv **out);
int tsb_sv_destroy(tsb_sv *h);
int tsb_sv_set_stream(tsb_sv *h, void *stream);
/* Heat-bath p_high for the 32 local patterns: index (max ? 16 : 0) | NW<<3 |
 * NE<<2 | SW<<1 | SE, where a diagonal bit is set when that diagonal face
 * differs from the centre by 2 (sixvertex.py:354-442). */
int tsb_sv_set_p_high(tsb_sv *h, const double *p_high);
/* Height batches (n, n+1, n+1) int32; upload rejects grids whose adjacent
 * faces do not differ by exactly 1 (TSB_E_INCONSISTENT). */
int tsb_sv_upload(tsb_sv *h, int chain0, int n, const int32_t *heights);
int tsb_sv_download(tsb_sv *h, int chain0, int n, int32_t *heights);
/* sv_random_walk_batch (sixvertex.py:445-467): class from the global coin. */
int tsb_sv_walk(tsb_sv *h, int chain0, int n, const uint64_t *seeds, uint64_t step0, uint64_t n_steps);
/* sv_sweep (sixvertex.py:470-486): one sweep of an explicit face class 0..3. */
int tsb_sv_sweep(tsb_sv *h, int chain0, int n, const uint64_t *seeds, uint64_t step, int face_class);
int tsb_sv_sync(tsb_sv *h);
/* sv_extremal (sixvertex.py:534-562) from the ring heights of
 * _ring_heights (ring: (n+1)^2 int32, interior ignored) into chains
 * chain_max / chain_min; heights to hmax / hmin (nullable).
 * TSB_E_INFEASIBLE when the ring heights are incompatible. */
int tsb_sv_extremal(tsb_sv *h, const int32_t *ring, int chain_max, int chain_min, int32_t *hmax, int32_t *hmin);
/* Indicator observables of stats.py:213-228 added to a device uint32
 * accumulator: observable 0 "h-edge" (n, n+1), 1 "v-edge" (n+1, n),
 * 2 "c-vertex" (n, n). */
int tsb_sv_observe_add(tsb_sv *h, int chain0, int n, int observable, uint32_t *acc_dev);
/* Face heights summed into a device int64 accumulator ((n+1)^2): the mean
 * height function = acc / (#states added). */
int tsb_sv_height_sum_add(tsb_sv *h, int chain0, int n, long long *acc_dev);
/* Class-run collapsing for the six-vertex walk (default on; env
 * TSB_SV_COLLAPSE=0): the c-flip is a heat-bath move, so a sweep followed by
 * a sweep of the same class is skipped; bit-identical results. */
int tsb_sv_set_collapse(tsb_sv *h, int on);
/* Archive record: h_edges then v_edges ravelled as '0'/'1' (stats.py:146-153);
 * size query as tsb_domino_serialize. */
int tsb_sv_serialize(tsb_sv *h, int chain, char *out, size_t cap, size_t *len);
int tsb_sv_coalesced(tsb_sv *h, int chain0, int npairs, uint8_t *flags);
int tsb_sv_replicate(tsb_sv *h, int src, int dst0, int step, int n);
/* sv_cftp (sixvertex.py:565-622): as tsb_domino_cftp with height grids. */
int tsb_sv_cftp(tsb_sv *h, const int32_t *top0, const int32_t *bot0, const uint64_t *masters, int count,
                int max_doublings, int32_t *out_heights, int32_t *collapsed_round, tsb_progress_fn progress,
                void *user);

/* ---------------------------------------------------------------- lozenges */
typedef struct tsb_loz tsb_loz;

/* `nchains` lozenge chains of a TriDomain with triangle grids up/down
 * ((sx, sy) uint8/bool, lozenge.py:144-282); state = LozengeTiling.edges
 * (3, sx+1, sy+1) bool (lozenge.py:285-301) as three device bit planes. */
int tsb_loz_create(int device, int sx, int sy, int nchains, const uint8_t *up, const uint8_t *down, tsb_loz **out);
int tsb_loz_destroy(tsb_loz *h);
int tsb_loz_set_stream(tsb_loz *h, void *stream);
/* loz_p_up_grid (lozenge.py:545-566), (sx+1, sy+1) float64. */
int tsb_loz_set_p_up(tsb_loz *h, const double *p_up);
/* Edge batches (n, 3, sx+1, sy+1) uint8 0/1; upload rejects crossed edges
 * whose two triangles are not both in the domain (TSB_E_INCONSISTENT). */
int tsb_loz_upload(tsb_loz *h, int chain0, int n, const uint8_t *edges);
int tsb_loz_download(tsb_loz *h, int chain0, int n, uint8_t *edges);
/* loz_random_walk_batch (lozenge.py:600-622). */
int tsb_loz_walk(tsb_loz *h, int chain0, int n, const uint64_t *seeds, uint64_t step0, uint64_t n_steps);
/* loz_sweep (lozenge.py:625-646): one sweep of colour class 0..2. */
int tsb_loz_sweep(tsb_loz *h, int chain0, int n, const uint64_t *seeds, uint64_t step, int color);
int tsb_loz_sync(tsb_loz *h);
/* loz_heights (lozenge.py:414-447): int32 (sx+1, sy+1), 0 outside the mask. */
int tsb_loz_heights(tsb_loz *h, int chain, int ref_x, int ref_y, int32_t *out);
/* loz_heights of chains [chain0, chain0+n) added to a device int64
 * accumulator ((sx+1) x (sy+1)): mean height function = acc / #states. */
int tsb_loz_height_sum_add(tsb_loz *h, int chain0, int n, int ref_x, int ref_y, long long *acc_dev);
/* loz_extremal (lozenge.py:762-775) into chains chain_max / chain_min;
 * TSB_E_UNTILEABLE when the domain has no tiling. */
int tsb_loz_extremal(tsb_loz *h, int chain_max, int chain_min, int ref_x, int ref_y);
/* Class-run collapsing for the lozenge walk (default on; env
 * TSB_LZ_COLLAPSE=0), as tsb_sv_set_collapse. */
int tsb_loz_set_collapse(tsb_loz *h, int on);
/* Archive record: edges (3, X, Y) ravelled as '0'/'1' (stats.py:146-153). */
int tsb_loz_serialize(tsb_loz *h, int chain, char *out, size_t cap, size_t *len);
int tsb_loz_coalesced(tsb_loz *h, int chain0, int npairs, uint8_t *flags);
int tsb_loz_replicate(tsb_loz *h, int src, int dst0, int step, int n);
/* loz_cftp (lozenge.py:778-827): as tsb_domino_cftp with edge grids. */
int tsb_loz_cftp(tsb_loz *h, const uint8_t *top0, const uint8_t *bot0, const uint64_t *masters, int count,
                 int max_doublings, uint8_t *out_edges, int32_t *collapsed_round, tsb_progress_fn progress,
                 void *user);

/* Run collapsing (default on; env TSB_DOM_COLLAPSE=0 turns it off at
 * creation): a sweep whose successor in the same walk has the same colour is
 * skipped.  The move is a heat-bath update (_kernels.py:46-55: a rotateable
 * vertex becomes 12 iff u < p_up, else 3, whatever its state) and a colour's
 * rotateable set cannot change while only that colour moves, so the last
 * sweep of a run of equal colours alone decides the state: results are
 * bit-identical, about half of the sweeps are executed. */
int tsb_domino_set_collapse(tsb_domino *h, int on);

/* One-shot form of the fused hook: evolves a host (nchains, side, side)
 * uint8 batch in place (upload + walk + download). */
int tsb_domino_walk_host(int device, uint8_t *states, int nchains, int side, const uint64_t *seeds,
                         const double *p_up, const uint8_t *faces, uint64_t n_steps);

#ifdef __cplusplus
}
#endif
#endif /* TSB_H */
