// Domino tilings: bit-plane state, colour-class Glauber sweep, codecs.
//
// Reference path (relative to /root/reference/pkg/src/tilesampler/):
//   _kernels.py:35-69  domino_walk   (the fused CPU kernel this replaces)
//   sweeps.py:209-316  sweep_batch / random_walk_batch
//   lattice.py:51-61, 267-280  tilestate bits and the Tiling grid
//
// Device state (per chain): two bit planes over the (side x side) vertex grid,
// interleaved as one uint2 {V, H} per (row, 32-column word):
//   V[r] bit c  = vertical edge (r,c)-(r+1,c) crossed  (= "down" bit 2 of (r,c)
//                 = "up" bit 1 of (r+1,c))
//   H[r] bit c  = horizontal edge (r,c)-(r,c+1) crossed (= "right" bit 8 of
//                 (r,c) = "left" bit 4 of (r,c+1))
// Each edge is stored once: 2 bits per vertex instead of the reference's
// 8-bit tilestate.  Rows -1 and `side` are zero guard rows.  The tilestate of
// (r,c) is  V[r-1]c | V[r]c << 1 | H[r]c-1 << 2 | H[r]c << 3.
//
// A sweep of colour `col` rotates every active vertex ((r+c)%2 == col) whose
// state is 3 (V[r-1],V[r] set, H[r]c-1,H[r]c clear) or 12 (the reverse) with
// its own (site, step) coin; a rotation toggles its four incident edges.  The
// reference's "update the other colour" pass is implicit: the other colour's
// tilestates are read off the same edges.  Same-colour vertices share no
// edge, so a sweep is a pure function of the previous state and is computed
// out of place (double buffer).
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "domino.cuh"
#include "tsb_fire.cuh"

namespace tsb {

constexpr int kTileRows = 15;   // output rows per block tile (+1 halo fire row)
constexpr int kTileWords = 62;  // output words per tile: 64 loaded (2 per lane), 1 halo word each side
constexpr int kPad = 2;         // zero words left of every state row (lane 0's halo of the first tile)
#ifndef TSB_MROWS
#define TSB_MROWS 16
#endif
constexpr int kMRows = TSB_MROWS;  // rows per temporally blocked tile (warps per block)
constexpr int kMBlocks = 48 / kMRows;  // resident blocks per SM (48 warps)
constexpr int kMK = 2;          // sweeps per temporally blocked launch
constexpr int kMOut = kMRows - 2 * kMK;  // exact output rows per temporally blocked tile
constexpr size_t kPipeMinBytes = 96ull << 20;  // launches whose two state buffers exceed this use the pipelined kernel
constexpr int kOrderThreads = 1024;     // adaptive dispatch order (replay_tail_kernel): one block
constexpr int kOrderClasses = 4;
constexpr int kOrderPer = 8;            // tiles per thread: launches of more tiles use the pipelined kernel
constexpr size_t kMSmem = 2 * sizeof(uint2) * kMRows * 32 + sizeof(uint32_t) * kMRows * 64 + 2 * kMRows * 1024;

struct SweepCtx {
    const uint2 *src;          // chain 0, row 0, word 0 (after the kPad left pad)
    uint2 *dst;
    const uint64_t *seedinfo;  // [n][2] = {family base, global key}
    const uint64_t *tgrid;     // per-site thresholds (mode 2), (side x side)
    const uint64_t *step_dev;  // graph replays: step = *step_dev + step
    int ntiles;
    const uint8_t *colors;     // graph replays: [n][kGraphSweeps] colours (null: direct launch)
    const int2 *tiles;         // non-empty tiles {word chunk, row band}
    uint64_t t0, t1;           // thresholds for even / odd parity (modes 0, 1)
    size_t chain_stride;       // uint2 per chain (incl. guard rows)
    int side, pitch;
    uint64_t step;
    int color_override;  // -1: colour from the global coin (direct launches)
    const int *order;    // multi-sweep adaptive order: canonical index of the tile of block b (tiles permuted)
    unsigned *cost;      // multi-sweep: per-tile block duration in cycles (null: not measured)
    // compacted walks (walk_compact): executed sweeps of chain z are
    // xlist[z * xpitch + j], j < xcnt[z] = (step - step_dev[0]) | colour << 31;
    // launch sweep s takes entry *xbase + step + s (null: colour table)
    const uint32_t *xlist;
    const int *xcnt;
    const uint64_t *xbase;
    int xpitch;
};

// Sweep selection of the multi-sweep kernels (template MODE, so each variant
// carries only its own code): 0 every sweep, colours from the replay's
// table; 1 the table's skip flags too (run collapsing inside the launches,
// strip walks); 2 compacted executed-sweep lists (run-collapsed walks).
enum { kSelPlain = 0, kSelSkip = 1, kSelList = 2 };

// Both sweeps of a kMK = 2 launch resolved up front, so their loads (list
// cursor, entries / colour bytes) are in flight together instead of one
// dependent round trip per sweep.
struct Sweeps2 {
    uint64_t step0, step1;
    int color0, color1;
    bool on0, on1;
};

template <int MODE>
__device__ __forceinline__ Sweeps2 sweeps_of(const SweepCtx &c, int z, uint64_t step0) {
    Sweeps2 w;
    if constexpr (MODE == kSelList) {
        const uint64_t j = *c.xbase + c.step;
        const int n = c.xcnt[z];
        const uint32_t *l = c.xlist + (size_t)z * c.xpitch;
        const uint64_t base = c.step_dev[0];
        w.on0 = j < (uint64_t)n;
        w.on1 = j + 1 < (uint64_t)n;
        const uint32_t e0 = w.on0 ? l[j] : 0u, e1 = w.on1 ? l[j + 1] : 0u;
        w.step0 = base + (e0 & 0x7FFFFFFFu);
        w.step1 = base + (e1 & 0x7FFFFFFFu);
        w.color0 = (int)(e0 >> 31);
        w.color1 = (int)(e1 >> 31);
    } else {
        const uint8_t *cl = c.colors + z * kGraphSweeps + (int)c.step;
        const int c0 = cl[0], c1 = cl[1];
        w.step0 = step0;
        w.step1 = step0 + 1ull;
        w.color0 = c0 & 1;
        w.color1 = c1 & 1;
        w.on0 = MODE == kSelPlain || !(c0 & 2);
        w.on1 = MODE == kSelPlain || !(c1 & 2);
    }
    return w;
}

// Step and colour of sweep s of a multi-sweep launch for chain z; false when
// the sweep is not executed (a collapsed run, or past the chain's list).
template <int MODE>
__device__ __forceinline__ bool sweep_of(const SweepCtx &c, int z, int s, uint64_t step0, uint64_t *step,
                                         int *color) {
    if constexpr (MODE == kSelList) {
        const uint64_t j = *c.xbase + c.step + (uint64_t)s;
        if (j >= (uint64_t)c.xcnt[z]) return false;
        const uint32_t e = c.xlist[(size_t)z * c.xpitch + j];
        *step = c.step_dev[0] + (e & 0x7FFFFFFFu);
        *color = (int)(e >> 31);
        return true;
    } else {
        const int ci = c.colors[z * kGraphSweeps + (int)c.step + s];
        *step = step0 + (uint64_t)s;
        *color = ci & 1;
        return MODE == kSelPlain || !(ci & 2);
    }
}

// One sweep, one block per non-empty tile of kTileRows x 62 words (512
// threads).  Warp k owns row r = r0+k; each lane owns two adjacent words
// (16-byte loads; lanes 0 and 31 hold one halo word each, so horizontal
// neighbours are shuffles).  Rows carry kPad zero words on the left and zero
// padding on the right, and every word outside the domain is zero, so loads
// need no predication.
//   phase 0: V of every row -> shared (the row above for the fire test)
//   phase 1: fire row F(r) of every row (warp 15 = halo row r0+15) -> shared
//   phase 2: warps 0..14 toggle the four incident edges of every firing vertex:
//            V[r] ^= F(r) ^ F(r+1),   H[r] ^= F(r) ^ F(r) >> 1 (carry from the next word).
template <int TM>
__global__ void __launch_bounds__(32 * (kTileRows + 1), 3)
    domino_sweep_kernel(SweepCtx c) {
    __shared__ uint2 vs[kTileRows + 1][32];
    __shared__ uint2 fs[kTileRows + 1][32];
    __shared__ uint16_t queue[kTileRows + 1][1024];
    __shared__ uint32_t fres[kTileRows + 1][64];
    const int lane = threadIdx.x & 31;
    const int k = threadIdx.x >> 5;
    const int2 tile = c.tiles[blockIdx.x];
    const int r = tile.y * kTileRows + k;
    const int wa = tile.x * kTileWords - 2 + 2 * lane;  // words wa, wa+1; outputs wa+1 .. wa+62 of lane 0..31
    const int z = blockIdx.z;
    const bool live = r < c.side;  // rows >= side are the zero guard row or beyond: never loaded / stored
    const uint2 *row = c.src + (size_t)z * c.chain_stride + (ptrdiff_t)r * c.pitch;
    // Programmatic dependent launch: let the next sweep's grid start its
    // prologue now, and wait for the previous sweep's stores before loading.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    uint4 cur = make_uint4(0u, 0u, 0u, 0u);
    if (live) cur = __ldg(reinterpret_cast<const uint4 *>(row + wa));
    uint32_t vua = 0, vub = 0;
    if (k == 0) {  // the tile's first row reads the row above from global (guard row at r = -1)
        const uint4 q = __ldg(reinterpret_cast<const uint4 *>(row - c.pitch + wa));
        vua = q.x;
        vub = q.z;
    }
    // colour: per-replay table (graph mode) or the global coin; BLACK iff
    // u < 1/2 <=> bit 63 of the draw is 0 (_kernels.py:44-45, sweeps.py:266-269)
    int color;
    uint64_t step;
    if (c.colors) {
        step = *c.step_dev + c.step;
        color = c.colors[z * kGraphSweeps + (int)c.step] & 1;  // single sweeps are never skipped
    } else {
        step = c.step;
        color = c.color_override >= 0 ? c.color_override
                                      : (int)(mix64(c.seedinfo[2 * z + 1] + (step + 1ull) * kGold) >> 63);
    }
    vs[k][lane] = make_uint2(cur.x, cur.z);
    __syncthreads();
    if (k > 0) {
        const uint2 u = vs[k - 1][lane];
        vua = u.x;
        vub = u.y;
    }
    // lane 0's first word is a pure halo (its fire row feeds no output); lane
    // 31's second word only feeds bit 0 into the H carry of its first word.
    const uint32_t act = ((r + color) & 1) ? 0xAAAAAAAAu : 0x55555555u;
    const uint32_t hl = __shfl_up_sync(0xffffffffu, cur.w, 1);
    const uint32_t la = (cur.y << 1) | (hl >> 31);
    const uint32_t lb = (cur.w << 1) | (cur.y >> 31);
    // rotateable (state 3 or 12): up, down, not-left, not-right agree; state 3 = rotateable with up set
    const uint32_t ra = ~((vua ^ cur.x) | (vua ^ ~la) | (vua ^ ~cur.y)) & (lane == 0 ? 0u : act);
    const uint32_t rb = ~((vub ^ cur.z) | (vub ^ ~lb) | (vub ^ ~cur.w)) & (lane == 31 ? act & 1u : act);
    const uint32_t ia = vua, ib = vub;
    uint2 f = make_uint2(0u, 0u);
    if (__any_sync(0xffffffffu, (ra | rb) != 0u)) {
        const uint64_t t = (TM == 1 && color) ? c.t1 : c.t0;
        f = warp_fire<TM>(ra, rb, ia, ib, queue[k], fres[k], c.seedinfo, c.tgrid, t, c.side, z, r, wa, step);
    }
    const uint32_t fa = f.x, fb = f.y;
    fs[k][lane] = f;
    __syncthreads();
    if (k == kTileRows || !live) return;  // warp-uniform
    const uint2 fn = fs[k + 1][lane];     // F(r+1)
    const uint32_t frb = __shfl_down_sync(0xffffffffu, fa, 1);
    const uint32_t nva = cur.x ^ fa ^ fn.x;
    const uint32_t nvb = cur.z ^ fb ^ fn.y;
    const uint32_t nha = cur.y ^ fa ^ (fa >> 1) ^ (fb << 31);
    const uint32_t nhb = cur.w ^ fb ^ (fb >> 1) ^ (frb << 31);
    uint2 *out = c.dst + (size_t)z * c.chain_stride + (ptrdiff_t)r * c.pitch;
    if (lane > 0 && lane < 31) *reinterpret_cast<uint4 *>(out + wa) = make_uint4(nva, nha, nvb, nhb);
    else if (lane == 0) out[wa + 1] = make_uint2(nvb, nhb);
    else out[wa] = make_uint2(nva, nha);
}

// Temporal blocking: kMK sweeps per launch.  A block holds kMRows rows
// (warp k owns row r0 - kMK + k, two words per lane as above) entirely in
// registers/shared memory and sweeps them kMK times; rows and halo words next
// to the unloaded outside go stale by one row / bit per sweep, so after kMK
// sweeps the central kMOut rows and the 62 interior words are exact and are
// the only ones stored.  Per sweep it costs two block barriers and the fire
// test; loads, stores, addressing and the launch are paid once per kMK sweeps.
// Used inside the graph replays (colours from the per-replay table).
#ifdef TSB_TIMING
// Debug builds only (nvcc -DTSB_TIMING): %globaltimer stamps of block 0..N of
// each multi-sweep launch in a replay -> g_tt[launch][block][phase].
__device__ unsigned long long g_tt[16][2048][6];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define TT(ph) \
    if (threadIdx.x == 0 && blockIdx.x < 2048 && c.step / kMK < 16) g_tt[c.step / kMK][blockIdx.x][ph] = gtimer()
#else
#define TT(ph)
#endif

// Coins whose outcome cannot reach a stored bit are not drawn.  Row k's fire
// row touches rows k-1 and k, and the fire test of a row reads the row above,
// so sweep s of a kMK = 2 tile needs fire rows s+1 .. kMRows-1-s; across
// columns a fire moves one column per sweep, so the left halo word (lane 0,
// word a) matters only at bit 31 in sweep 0, the right halo word (lane 31,
// word b) at bits 0-1 in sweep 0 and bit 0 in sweep 1.  Skipped sites keep
// their state; they lie in the stale halo, which is never stored.
static_assert(kMK == 2, "need masks are derived for two sweeps per launch");
#ifndef TSB_NEED_MASKS
#define TSB_NEED_MASKS 1
#endif
__device__ __forceinline__ uint32_t need_a(int s, int k, int lane) {
    if (!TSB_NEED_MASKS) return 0xFFFFFFFFu;
    if (k < s + 1 || k > kMRows - 1 - s) return 0u;
    return lane == 0 ? (s == 0 ? 0x80000000u : 0u) : 0xFFFFFFFFu;
}
__device__ __forceinline__ uint32_t need_b(int s, int k, int lane) {
    if (!TSB_NEED_MASKS) return 0xFFFFFFFFu;
    if (k < s + 1 || k > kMRows - 1 - s) return 0u;
    return lane == 31 ? (s == 0 ? 3u : 1u) : 0xFFFFFFFFu;
}

// kMK sweeps of one tile held in registers (cur) and shared memory, then the
// exact central rows are stored.
template <int TM, int MODE>
__device__ __forceinline__ void multi_tile(const SweepCtx &c, uint2 (*vs)[32], uint2 (*fs)[32], uint32_t (*fres)[64],
                                           uint16_t (*queue)[1024], int k, int lane, int z, int r, int wa,
                                           bool in_grid, uint4 cur, const Sweeps2 &sw) {
    const uint32_t act0 = (r & 1) ? 0xAAAAAAAAu : 0x55555555u;  // active sites of colour 0 (BLACK: r+c even)
    static_assert(kMK == 2, "two sweeps per launch");
#pragma unroll 1
    for (int s = 0; s < kMK; ++s) {
        if (!(s ? sw.on1 : sw.on0)) continue;  // block-uniform
        const uint64_t step = s ? sw.step1 : sw.step0;
        const int color = s ? sw.color1 : sw.color0;
        vs[k][lane] = make_uint2(cur.x, cur.z);
        __syncthreads();
        uint32_t vua = 0u, vub = 0u;
        if (k > 0) {
            const uint2 u = vs[k - 1][lane];
            vua = u.x;
            vub = u.y;
        }
        const uint32_t act = color ? ~act0 : act0;
        // lane 0's word a and lane 31's word b are halo words: their
        // neighbour bits from the shuffles wrap around but only feed bits
        // that are never stored (stale-halo argument above)
        const uint32_t hl = __shfl_up_sync(0xffffffffu, cur.w, 1);
        const uint32_t la = (cur.y << 1) | (hl >> 31);
        const uint32_t lb = (cur.w << 1) | (cur.y >> 31);
        // rotateable: state 3 (up and down edges crossed, left and right not)
        // or 12 (the reverse), i.e. up, down, not-left and not-right agree;
        // the state-3 sites are the rotateable ones with the up edge crossed
        uint32_t ra = ~((vua ^ cur.x) | (vua ^ ~la) | (vua ^ ~cur.y)) & act;
        uint32_t rb = ~((vub ^ cur.z) | (vub ^ ~lb) | (vub ^ ~cur.w)) & act;
        uint2 f = make_uint2(0u, 0u);
        if (__any_sync(0xffffffffu, (ra | rb) != 0u)) {
            // the masks only where coins are drawn: the frozen bulk never pays them
            ra &= need_a(s, k, lane);
            rb &= need_b(s, k, lane);
            const uint64_t t = (TM == 1 && color) ? c.t1 : c.t0;
            f = warp_fire<TM>(ra, rb, vua, vub, queue[k], fres[k], c.seedinfo, c.tgrid, t, c.side, z, r, wa, step);
        }
        fs[k][lane] = f;
        __syncthreads();
        const uint2 fn = k + 1 < kMRows ? fs[k + 1][lane] : make_uint2(0u, 0u);  // F(r+1)
        const uint32_t frb = __shfl_down_sync(0xffffffffu, f.x, 1);
        const uint32_t nva = cur.x ^ f.x ^ fn.x;
        const uint32_t nvb = cur.z ^ f.y ^ fn.y;
        const uint32_t nha = cur.y ^ f.x ^ (f.x >> 1) ^ (f.y << 31);
        const uint32_t nhb = cur.w ^ f.y ^ (f.y >> 1) ^ (frb << 31);
        // rows outside the grid stay zero without masking: a vertex on the
        // first or last grid row is never rotateable (its outer edges cannot
        // be crossed), so no fire reaches them
        cur = make_uint4(nva, nha, nvb, nhb);
        TT(3 + s);
    }
    if (k >= kMK && k < kMRows - kMK && in_grid) {  // warp-uniform
        uint2 *out = c.dst + (size_t)z * c.chain_stride + (ptrdiff_t)r * c.pitch;
        if (lane > 0 && lane < 31) *reinterpret_cast<uint4 *>(out + wa) = cur;
        else if (lane == 0) out[wa + 1] = make_uint2(cur.z, cur.w);
        else out[wa] = make_uint2(cur.x, cur.y);
    }
}

#define MULTI_SMEM                                                                                          \
    extern __shared__ __align__(16) unsigned char dsm[];                                                    \
    uint2(*vs)[32] = reinterpret_cast<uint2(*)[32]>(dsm);                                                   \
    uint2(*fs)[32] = reinterpret_cast<uint2(*)[32]>(dsm + sizeof(uint2) * kMRows * 32);                     \
    uint32_t(*fres)[64] = reinterpret_cast<uint32_t(*)[64]>(dsm + 2 * sizeof(uint2) * kMRows * 32);         \
    uint16_t(*queue)[1024] =                                                                                \
        reinterpret_cast<uint16_t(*)[1024]>(dsm + 2 * sizeof(uint2) * kMRows * 32 + sizeof(uint32_t) * kMRows * 64)

template <int TM, int MODE>
__global__ void __launch_bounds__(32 * kMRows, kMBlocks) domino_multi_kernel(SweepCtx c) {
    TT(0);
    MULTI_SMEM;
    __shared__ long long t_start;
    const int lane = threadIdx.x & 31;
    const int k = threadIdx.x >> 5;
    const int2 tile = c.tiles[blockIdx.x];  // adaptive order: c.tiles is the permuted list
    const int r = tile.y * kMOut - kMK + k;
    const int wa = tile.x + 2 * lane;  // band-aligned tile: tile.x = first loaded word (even)
    const int z = blockIdx.z;
    const bool in_grid = r >= 0 && r < c.side;
    const uint2 *row = c.src + (size_t)z * c.chain_stride + (ptrdiff_t)r * c.pitch;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    TT(1);
    asm volatile("griddepcontrol.wait;" ::: "memory");
    TT(2);
    if (c.cost && threadIdx.x == 0) t_start = clock64();
    uint4 cur = make_uint4(0u, 0u, 0u, 0u);
    if (in_grid) cur = __ldg(reinterpret_cast<const uint4 *>(row + wa));
    multi_tile<TM, MODE>(c, vs, fs, fres, queue, k, lane, z, r, wa, in_grid, cur,
                         sweeps_of<MODE>(c, z, *c.step_dev + c.step));
    if (c.cost && threadIdx.x == 0) c.cost[c.order[blockIdx.x]] = (unsigned)(clock64() - t_start);  // after the last barrier
    TT(5);
}

// Streaming launches, pipelined: persistent blocks (3 per SM) walk the tile
// list with a grid stride; each thread's 16-byte slice of the tiles
// kPipeStages-1 ahead is fetched with cp.async into the thread's own
// shared-memory slots while the current tile is swept, so the HBM latency
// of a tile overlaps the sweeps of the previous one (two tiles in flight
// measured slower at C4, 63.0 vs 58.7 us per sweep).
// A thread only ever reads the slot it filled itself, so
// cp.async.wait_group needs no block barrier.
constexpr int kPipeStages = 2;
constexpr size_t kPipeSmem = kMSmem + kPipeStages * sizeof(uint4) * 32 * kMRows;

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}

template <int TM, int MODE>
__global__ void __launch_bounds__(32 * kMRows, kMBlocks) domino_multi_pipe_kernel(SweepCtx c) {
    MULTI_SMEM;
    uint4 *slot = reinterpret_cast<uint4 *>(dsm + kMSmem) + threadIdx.x;  // [kPipeStages][blockDim]
    const int lane = threadIdx.x & 31;
    const int k = threadIdx.x >> 5;
    const int z = blockIdx.z;
    const uint2 *base = c.src + (size_t)z * c.chain_stride;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // the launch's two sweeps (steps, colours, skip flags) are the same for
    // every tile: resolved once per block
    const Sweeps2 sw = sweeps_of<MODE>(c, z, *c.step_dev + c.step);
    auto fetch = [&](int2 t, int b) {
        const int r = t.y * kMOut - kMK + k;
        uint4 *dst = slot + b * 32 * kMRows;
        if (r >= 0 && r < c.side) cp_async16(dst, base + (ptrdiff_t)r * c.pitch + t.x + 2 * lane);
        else *dst = make_uint4(0u, 0u, 0u, 0u);
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // tile coordinates are read two tiles ahead, so the list load's latency
    // hides behind a tile's sweeps instead of stalling the next fetch
    const int G = gridDim.x;
    int2 t_cur = (int)blockIdx.x < c.ntiles ? c.tiles[blockIdx.x] : make_int2(0, 0);
    int2 t_nxt = (int)blockIdx.x + G < c.ntiles ? c.tiles[blockIdx.x + G] : make_int2(0, 0);
    int b = 0;
    if ((int)blockIdx.x < c.ntiles) fetch(t_cur, 0);
    for (int i = blockIdx.x; i < c.ntiles; i += G, b ^= 1) {
        const int nx = i + G;
        const int2 t_nn = nx + G < c.ntiles ? c.tiles[nx + G] : make_int2(0, 0);
        if (nx < c.ntiles) {
            fetch(t_nxt, b ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");  // this tile's group has landed
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        const uint4 cur = slot[b * 32 * kMRows];
        const int r = t_cur.y * kMOut - kMK + k;
        multi_tile<TM, MODE>(c, vs, fs, fres, queue, k, lane, z, r, t_cur.x + 2 * lane, r >= 0 && r < c.side, cur, sw);
        t_cur = t_nxt;
        t_nxt = t_nn;
    }
}

// The same temporal blocking with ONE {V,H} word per lane (tiles of 30 output
// words): chosen for narrow lattices (e.g. CFTP at Aztec 512, W = 33 words),
// where the 62-word tiles would leave half of every warp outside the domain.
// Lanes 0 and 31 hold the halo words.
template <int TM, int MODE>
__global__ void __launch_bounds__(32 * kMRows, kMBlocks) domino_multi1_kernel(SweepCtx c) {
    extern __shared__ __align__(16) unsigned char dsm[];
    uint32_t(*vs)[32] = reinterpret_cast<uint32_t(*)[32]>(dsm);
    uint32_t(*fs)[32] = reinterpret_cast<uint32_t(*)[32]>(dsm + sizeof(uint2) * kMRows * 32);
    uint32_t(*fres)[64] = reinterpret_cast<uint32_t(*)[64]>(dsm + 2 * sizeof(uint2) * kMRows * 32);
    uint16_t(*queue)[1024] =
        reinterpret_cast<uint16_t(*)[1024]>(dsm + 2 * sizeof(uint2) * kMRows * 32 + sizeof(uint32_t) * kMRows * 64);
    const int lane = threadIdx.x & 31;
    const int k = threadIdx.x >> 5;
    const int2 tile = c.tiles[blockIdx.x];
    const int r = tile.y * kMOut - kMK + k;
    const int wa = tile.x + lane;  // tile.x = first loaded word
    const int z = blockIdx.z;
    const bool in_grid = r >= 0 && r < c.side;
    const uint2 *row = c.src + (size_t)z * c.chain_stride + (ptrdiff_t)r * c.pitch;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    uint2 cur = make_uint2(0u, 0u);
    if (in_grid) cur = __ldg(row + wa);
    const uint64_t step0 = *c.step_dev + c.step;
    const uint32_t act0 = (r & 1) ? 0xAAAAAAAAu : 0x55555555u;
#pragma unroll 1
    for (int s = 0; s < kMK; ++s) {
        uint64_t step;
        int color;
        if (!sweep_of<MODE>(c, z, s, step0, &step, &color)) continue;  // block-uniform
        vs[k][lane] = cur.x;
        __syncthreads();
        const uint32_t vu = k > 0 ? vs[k - 1][lane] : 0u;
        const uint32_t act = color ? ~act0 : act0;
        const uint32_t hl = __shfl_up_sync(0xffffffffu, cur.y, 1);  // lane 0: halo, wraps harmlessly
        const uint32_t la = (cur.y << 1) | (hl >> 31);
        const uint32_t ra = ~((vu ^ cur.x) | (vu ^ ~la) | (vu ^ ~cur.y)) & act;  // as multi_tile
        const uint32_t ia = vu;
        uint32_t f = 0u;
        if (__any_sync(0xffffffffu, ra != 0u)) {
            const uint64_t t = (TM == 1 && color) ? c.t1 : c.t0;
            const uint32_t rn = ra & (lane == 31 ? need_b(s, k, 31) : need_a(s, k, lane));
            f = warp_fire<TM, 1>(rn, 0u, ia, 0u, queue[k], fres[k], c.seedinfo, c.tgrid, t, c.side, z, r, wa, step).x;
        }
        fs[k][lane] = f;
        __syncthreads();
        const uint32_t fn = k + 1 < kMRows ? fs[k + 1][lane] : 0u;  // F(r+1)
        const uint32_t fr = __shfl_down_sync(0xffffffffu, f, 1);
        cur = make_uint2(cur.x ^ f ^ fn, cur.y ^ f ^ (f >> 1) ^ (fr << 31));
    }
    if (k >= kMK && k < kMRows - kMK && in_grid && lane > 0 && lane < 31) {
        uint2 *out = c.dst + (size_t)z * c.chain_stride + (ptrdiff_t)r * c.pitch;
        out[wa] = cur;
    }
}

// Small lattices: one block per chain keeps the whole chain in shared memory
// for all n_steps sweeps of a walk (one launch, no global traffic between
// sweeps).  Thread t owns the (row, word) items t, t + blockDim, ...; per
// sweep: fire words F (each warp deals the coins of its rotateable active
// sites to its lanes), barrier, edge toggles in place, barrier.  The same
// rotate/update semantics as the tiled kernels (_kernels.py:35-69); chosen
// for tiny lattices and for batches of small lattices (CFTP) -- see
// resident_smem for the rule.
constexpr int kResThreads = 1024;
constexpr int kResMaxItems = 512;
constexpr int kResMinChains = 16;
constexpr size_t kResScratch = (8 + 4 + 2 * 16) * 32 * 32;  // per-warp site bases, fire words, coin queues

struct ResCtx {
    uint2 *state;              // chain 0, row 0, word 0; updated in place
    const uint64_t *seedinfo;  // [n][2]
    const uint64_t *tgrid;
    uint64_t t0, t1;
    size_t chain_stride;
    int side, pitch, W;
    uint64_t step0, n_steps;
    int collapse;
};

// Coins of a warp's rotateable active sites, dealt round-robin to its lanes
// (two splitmix64 chains per lane per round, as warp_fire): lane l's word
// starts at site sb and has rotateable bits ra (ia: the site is in state 3).
template <int TM>
__device__ __forceinline__ uint32_t res_coins(uint32_t ra, uint32_t ia, uint64_t sb, uint16_t *queue, uint32_t *fres,
                                              uint64_t *sbase, uint64_t base, uint64_t salt, uint64_t t,
                                              const uint64_t *__restrict__ tgrid) {
    const int lane = threadIdx.x & 31;
    const int cnt = __popc(ra);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    int pos = incl - cnt;
    for (uint32_t m = ra; m; m &= m - 1) {  // job = is3 << 10 | lane << 5 | bit
        const int b = __ffs(m) - 1;
        queue[pos++] = (uint16_t)((((ia >> b) & 1u) << 10) | (lane << 5) | b);
    }
    fres[lane] = 0u;
    sbase[lane] = sb;
    __syncwarp();
    for (int j = lane; j < total; j += 64) {
        const bool two = j + 32 < total;
        const uint32_t q0 = queue[j], q1 = two ? queue[j + 32] : q0;
        const uint64_t s0 = sbase[(q0 >> 5) & 31u] + (q0 & 31u), s1 = sbase[(q1 >> 5) & 31u] + (q1 & 31u);
        const uint64_t x0 = mix64(mix64(base + (s0 + 1ull) * kGold) + salt);
        const uint64_t x1 = mix64(mix64(base + (s1 + 1ull) * kGold) + salt);
        const uint64_t t0 = TM == 2 ? __ldg(tgrid + s0) : t;
        const uint64_t t1 = TM == 2 ? __ldg(tgrid + s1) : t;
        if (((x0 >> 11) < t0) == (bool)((q0 >> 10) & 1u)) atomicOr(&fres[(q0 >> 5) & 31u], 1u << (q0 & 31u));
        if (two && ((x1 >> 11) < t1) == (bool)((q1 >> 10) & 1u)) atomicOr(&fres[(q1 >> 5) & 31u], 1u << (q1 & 31u));
    }
    __syncwarp();
    const uint32_t f = fres[lane];
    __syncwarp();  // fres / sbase / queue are reused by the warp's next item
    return f;
}

template <int TM>
__global__ void __launch_bounds__(kResThreads, 1) domino_resident_kernel(ResCtx c) {
    extern __shared__ __align__(16) unsigned char dsm[];
    const int side = c.side, W = c.W, items = side * W;
    const int warp = threadIdx.x >> 5;
    uint64_t *sbase = reinterpret_cast<uint64_t *>(dsm) + 32 * warp;                         // [32 warps][32]
    uint32_t *fres = reinterpret_cast<uint32_t *>(dsm + 8 * 32 * 32) + 32 * warp;              // [32][32]
    uint16_t *queue = reinterpret_cast<uint16_t *>(dsm + 12 * 32 * 32) + 512 * warp;           // [32][512]
    unsigned char *st = dsm + kResScratch;
    uint2 *S = reinterpret_cast<uint2 *>(st);                                     // (side + 2) x W, guard rows
    uint32_t *F = reinterpret_cast<uint32_t *>(st + sizeof(uint2) * (size_t)(side + 2) * W);  // (side + 1) x (W + 1)
    const int z = blockIdx.x;
    uint2 *g = c.state + (size_t)z * c.chain_stride;
    for (int i = threadIdx.x; i < (side + 2) * W; i += blockDim.x) {
        const int r = i / W - 1, w = i - (r + 1) * W;
        S[i] = (r >= 0 && r < side) ? g[(ptrdiff_t)r * c.pitch + w] : make_uint2(0u, 0u);
    }
    for (int i = threadIdx.x; i < (side + 1) * (W + 1); i += blockDim.x) F[i] = 0u;
    const uint64_t base = c.seedinfo[2 * z], gkey = c.seedinfo[2 * z + 1];
    __syncthreads();
#pragma unroll 1
    for (uint64_t s = 0; s < c.n_steps; ++s) {
        const uint64_t step = c.step0 + s;
        const uint64_t salt = (step + 1ull) * kGold;
        const int color = (int)(mix64(gkey + salt) >> 63);  // BLACK iff u < 1/2 (sweeps.py:266-269)
        // collapsed run (color_entry): the next sweep has the same colour
        if (c.collapse && s + 1 < c.n_steps && (int)(mix64(gkey + salt + kGold) >> 63) == color) continue;
        const uint64_t t = (TM == 1 && color) ? c.t1 : c.t0;
        for (int i0 = 0; i0 < items; i0 += blockDim.x) {  // warp-uniform trip count
            const int i = i0 + threadIdx.x;
            const int r = i / W, w = i - r * W;
            uint32_t ra = 0u, ia = 0u;
            if (i < items) {
                const uint2 cur = S[i + W];
                const uint32_t vu = S[i].x;
                const uint32_t hp = w > 0 ? S[i + W - 1].y : 0u;
                const uint32_t act0 = (r & 1) ? 0xAAAAAAAAu : 0x55555555u;
                const uint32_t la = (cur.y << 1) | (hp >> 31);
                ia = vu & cur.x & ~(la | cur.y);
                ra = (ia | (~(vu | cur.x) & la & cur.y)) & (color ? ~act0 : act0);
            }
            uint32_t f = 0u;
            if (__any_sync(0xffffffffu, ra != 0u))
                f = res_coins<TM>(ra, ia, (uint64_t)r * (uint64_t)side + 32ull * (uint64_t)w, queue, fres, sbase,
                                  base, salt, t, c.tgrid);
            if (i < items) F[r * (W + 1) + w] = f;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < items; i += blockDim.x) {
            const int r = i / W, w = i - r * W;
            const uint32_t *fr = F + r * (W + 1) + w;
            const uint32_t f = fr[0], fn = fr[W + 1], fx = fr[1];
            const uint2 cur = S[i + W];
            S[i + W] = make_uint2(cur.x ^ f ^ fn, cur.y ^ f ^ (f >> 1) ^ (fx << 31));
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < items; i += blockDim.x) {
        const int r = i / W, w = i - r * W;
        g[(ptrdiff_t)r * c.pitch + w] = S[i + W];
    }
}

// CFTP's coupled pairs (cftp.py:115-119): chains 2z and 2z+1 run from T_max /
// T_min with the SAME seeds, so every coin is shared.  One block sweeps the
// tile in both chains and draws each coin once, for the union of the two
// chains' rotateable sites: with c = (u < p_up), a site fires in a chain iff
// it is rotateable there and c equals its "state 3" bit -- exactly what two
// independent sweeps compute.  Narrow (1 word per lane) tiles.
template <int TM, int MODE>
__global__ void __launch_bounds__(32 * kMRows, kMBlocks) domino_multi1c_kernel(SweepCtx c) {
    extern __shared__ __align__(16) unsigned char dsm[];
    uint32_t(*vs)[kMRows][32] = reinterpret_cast<uint32_t(*)[kMRows][32]>(dsm);
    uint32_t(*fs)[kMRows][32] = reinterpret_cast<uint32_t(*)[kMRows][32]>(dsm + 2 * sizeof(uint32_t) * kMRows * 32);
    uint32_t(*fres)[64] = reinterpret_cast<uint32_t(*)[64]>(dsm + 2 * sizeof(uint2) * kMRows * 32);
    uint16_t(*queue)[1024] =
        reinterpret_cast<uint16_t(*)[1024]>(dsm + 2 * sizeof(uint2) * kMRows * 32 + sizeof(uint32_t) * kMRows * 64);
    const int lane = threadIdx.x & 31;
    const int k = threadIdx.x >> 5;
    const int2 tile = c.tiles[blockIdx.x];
    const int r = tile.y * kMOut - kMK + k;
    const int wa = tile.x + lane;
    const int zt = 2 * blockIdx.z;  // top chain; bottom = zt + 1
    const bool in_grid = r >= 0 && r < c.side;
    const uint2 *rowt = c.src + (size_t)zt * c.chain_stride + (ptrdiff_t)r * c.pitch;
    const uint2 *rowb = rowt + c.chain_stride;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    uint2 ct = make_uint2(0u, 0u), cb = make_uint2(0u, 0u);
    if (in_grid) {
        ct = __ldg(rowt + wa);
        cb = __ldg(rowb + wa);
    }
    const uint64_t step0 = *c.step_dev + c.step;
    const uint32_t act0 = (r & 1) ? 0xAAAAAAAAu : 0x55555555u;
#pragma unroll 1
    for (int s = 0; s < kMK; ++s) {
        uint64_t step;
        int color;
        if (!sweep_of<MODE>(c, zt, s, step0, &step, &color)) continue;  // block-uniform
        vs[0][k][lane] = ct.x;
        vs[1][k][lane] = cb.x;
        __syncthreads();
        const uint32_t vut = k > 0 ? vs[0][k - 1][lane] : 0u, vub = k > 0 ? vs[1][k - 1][lane] : 0u;
        const uint32_t act = color ? ~act0 : act0;
        const uint32_t hlt = __shfl_up_sync(0xffffffffu, ct.y, 1), hlb = __shfl_up_sync(0xffffffffu, cb.y, 1);
        const uint32_t lat = (ct.y << 1) | (hlt >> 31), lab = (cb.y << 1) | (hlb >> 31);
        // as multi_tile: rotateable = the four edge bits agree (left, right
        // inverted); state 3 = rotateable with the up edge crossed
        const uint32_t rat = ~((vut ^ ct.x) | (vut ^ ~lat) | (vut ^ ~ct.y)) & act;
        const uint32_t rab = ~((vub ^ cb.x) | (vub ^ ~lab) | (vub ^ ~cb.y)) & act;
        const uint32_t iat = vut, iab = vub;
        const uint32_t un = rat | rab;
        uint32_t ft = 0u, fb = 0u;
        if (__any_sync(0xffffffffu, un != 0u)) {
            const uint64_t t = (TM == 1 && color) ? c.t1 : c.t0;
            // coin bits: 1 where u < p_up, on the union of both chains' sites
            const uint32_t cu =
                warp_fire_body<TM, 1>(un, 0u, 0xFFFFFFFFu, 0u, queue[k], fres[k], c.seedinfo, c.tgrid, t, c.side, zt, r,
                                 wa, step).x;
            ft = rat & ~(cu ^ iat);
            fb = rab & ~(cu ^ iab);
        }
        fs[0][k][lane] = ft;
        fs[1][k][lane] = fb;
        __syncthreads();
        const uint32_t fnt = k + 1 < kMRows ? fs[0][k + 1][lane] : 0u, fnb = k + 1 < kMRows ? fs[1][k + 1][lane] : 0u;
        const uint32_t frt = __shfl_down_sync(0xffffffffu, ft, 1), frb = __shfl_down_sync(0xffffffffu, fb, 1);
        ct = make_uint2(ct.x ^ ft ^ fnt, ct.y ^ ft ^ (ft >> 1) ^ (frt << 31));
        cb = make_uint2(cb.x ^ fb ^ fnb, cb.y ^ fb ^ (fb >> 1) ^ (frb << 31));
    }
    if (k >= kMK && k < kMRows - kMK && in_grid && lane > 0 && lane < 31) {
        uint2 *out = c.dst + (size_t)zt * c.chain_stride + (ptrdiff_t)r * c.pitch;
        out[wa] = ct;
        out[wa + c.chain_stride] = cb;
    }
}

// Colour tables (graph mode): the colour of every sweep of a replay (bit 0)
// and, with run collapsing, a skip flag (bit 1): a sweep whose successor in
// the same walk has the same colour is skipped.  The domino move is a heat-bath update -- a rotateable
// vertex becomes 12 iff u < p_up and 3 otherwise, whatever its state
// (_kernels.py:46-55) -- and while one colour is swept the other colour does
// not move, so the rotateable set of that colour cannot change within a run
// of equal colours and only the last sweep of the run decides the state.
// Skipping the others gives the identical state (tests: every golden walk,
// oracle walks, CFTP samples and traces, with TSB_DOM_COLLAPSE=0 and 1).
// color_entry: the table entry of `step` for a chain with global key g, the
// colour bit and the skip bit (the next sweep of the walk, which ends at `end`, has
// the same colour).  Tables of kGraphSweeps entries per chain are written by
// set_walk_kernel (a walk's first replay) and replay_tail_kernel (the next).
__device__ __forceinline__ uint8_t color_entry(uint64_t g, uint64_t step, uint64_t end, int collapse) {
    const int col = (int)(mix64(g + (step + 1ull) * kGold) >> 63);
    int skip = 0;
    if (collapse && step + 1ull < end) skip = (int)(mix64(g + (step + 2ull) * kGold) >> 63) == col;
    return (uint8_t)(col | (skip << 1));
}

// --------------------------------------------------------------- codecs
// Row ranges and crossable-edge planes from Domain.faces
// (vertex_mask lattice.py:190-195; crossable = both faces of the edge in
// the domain, lattice.py:67-78, 639-689).
__device__ __forceinline__ bool face_in(const uint8_t *faces, int nf, int r, int c) {
    return r >= 0 && c >= 0 && r < nf && c < nf && faces[(size_t)r * nf + c] != 0;
}

__global__ void domain_planes_kernel(const uint8_t *faces, int side, int W, int pitch,
                                     uint4 *dom, uint32_t *fbits, int2 *range, int r0, int win_lo, int win_hi) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = r0 + (int)blockIdx.y;  // global row (row windows: only the allocated rows)
    if (w >= W) return;
    const int nf = side - 1;
    uint32_t cv = 0, ch = 0, ev = 0, eh = 0, fb = 0;
    bool any = false;
    for (int b = 0; b < 32; ++b) {
        const int cc = w * 32 + b;
        if (cc >= side) break;
        const bool ful = face_in(faces, nf, r - 1, cc - 1), fur = face_in(faces, nf, r - 1, cc);
        const bool fdl = face_in(faces, nf, r, cc - 1), fdr = face_in(faces, nf, r, cc);
        if (ful || fur || fdl || fdr) any = true;
        if (fdl && fdr) cv |= 1u << b;  // edge down: faces (r,c-1),(r,c)
        if (fur && fdr) ch |= 1u << b;  // edge right: faces (r-1,c),(r,c)
        if ((fdl || fdr) && r + 1 < side) ev |= 1u << b;
        if ((fur || fdr) && cc + 1 < side) eh |= 1u << b;
        if (fdr) fb |= 1u << b;  // face (r, c)
    }
    dom[(size_t)r * pitch + w] = make_uint4(cv, ch, ev, eh);
    fbits[(size_t)r * pitch + w] = fb;
    if (any && r >= win_lo && r < win_hi) {  // swept rows: the window's (tiles never start outside it)
        atomicMin(&range[r].x, w);
        atomicMax(&range[r].y, w + 1);
    }
}

__global__ void fix_ranges_kernel(int2 *range, int side) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < side && range[r].x >= range[r].y) range[r] = make_int2(0, 0);
}

// Tiling.states (n, side, side) uint8 -> {V, H} planes, with validation:
// values < 16, every edge bit mirrored by the neighbour (lattice.py:432-450),
// no crossed edge leaving the grid or the domain.
__global__ void pack_kernel(const uint8_t *bytes, int side, int W, int pitch, size_t chain_stride,
                            const uint4 *dom, uint2 *state, int *bad) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y;
    const int z = blockIdx.z;
    if (w >= W) return;
    const uint8_t *g = bytes + (size_t)z * side * side;
    const uint4 cr = dom[(size_t)r * pitch + w];
    uint32_t v = 0, h = 0;
    int err = 0;
    for (int b = 0; b < 32; ++b) {
        const int cc = w * 32 + b;
        if (cc >= side) break;
        const uint8_t s = g[(size_t)r * side + cc];
        if (s >= 16) err |= 1;
        const bool up = s & 1, dn = s & 2, lf = s & 4, rt = s & 8;
        const bool up_n = r > 0 ? (g[(size_t)(r - 1) * side + cc] & 2) != 0 : false;
        const bool lf_n = cc > 0 ? (g[(size_t)r * side + cc - 1] & 8) != 0 : false;
        if (up != up_n || lf != lf_n) err |= 2;
        if (dn && !((cr.x >> b) & 1u)) err |= 4;
        if (rt && !((cr.y >> b) & 1u)) err |= 4;
        if (dn) v |= 1u << b;
        if (rt) h |= 1u << b;
    }
    state[(size_t)z * chain_stride + (size_t)(r + 1) * pitch + w] = make_uint2(v, h);
    if (err) atomicOr(bad, err);
}

__global__ void unpack_kernel(const uint2 *state, int side, int pitch, size_t chain_stride,
                              uint8_t *bytes) {
    const int cc = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y;
    const int z = blockIdx.z;
    if (cc >= side) return;
    const uint2 *s = state + (size_t)z * chain_stride + (size_t)(r + 1) * pitch;
    const int w = cc >> 5, b = cc & 31;
    const uint32_t up = (s[w - pitch].x >> b) & 1u;
    const uint32_t dn = (s[w].x >> b) & 1u;
    const uint32_t rt = (s[w].y >> b) & 1u;
    const uint32_t lf = cc > 0 ? (s[(cc - 1) >> 5].y >> ((cc - 1) & 31)) & 1u : 0u;
    bytes[(size_t)z * side * side + (size_t)r * side + cc] = (uint8_t)(up | dn << 1 | lf << 2 | rt << 3);
}

// Rows [r0, r0 + gridDim.y) of chain 0 from / to a (rows, side) uint8 grid
// (row windows, host-driven strip exchange): the same codec as pack_kernel /
// unpack_kernel; the first row's "up" bits are not checked (the row above is
// not in the grid).
__global__ void pack_rows_kernel(const uint8_t *bytes, int r0, int side, int W, int pitch, const uint4 *dom,
                                 uint2 *state, int *bad) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y, r = r0 + i;
    if (w >= W) return;
    const uint8_t *g = bytes + (size_t)i * side;
    const uint4 cr = dom[(size_t)r * pitch + w];
    uint32_t v = 0, hz = 0;
    int err = 0;
    for (int b = 0; b < 32; ++b) {
        const int cc = w * 32 + b;
        if (cc >= side) break;
        const uint8_t st = g[cc];
        if (st >= 16) err |= 1;
        const bool up = st & 1, dn = st & 2, lf = st & 4, rt = st & 8;
        const bool lf_n = cc > 0 ? (g[cc - 1] & 8) != 0 : false;
        if (lf != lf_n) err |= 2;
        if (i > 0 && up != ((g[cc - side] & 2) != 0)) err |= 2;
        if (dn && !((cr.x >> b) & 1u)) err |= 4;
        if (rt && !((cr.y >> b) & 1u)) err |= 4;
        if (dn) v |= 1u << b;
        if (rt) hz |= 1u << b;
    }
    state[(size_t)(r + 1) * pitch + w] = make_uint2(v, hz);
    if (err) atomicOr(bad, err);
}

__global__ void unpack_rows_kernel(const uint2 *state, int r0, int side, int pitch, uint8_t *bytes) {
    const int cc = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y, r = r0 + i;
    if (cc >= side) return;
    const uint2 *s = state + (size_t)(r + 1) * pitch;
    const int w = cc >> 5, b = cc & 31;
    const uint32_t up = (s[w - pitch].x >> b) & 1u;
    const uint32_t dn = (s[w].x >> b) & 1u;
    const uint32_t rt = (s[w].y >> b) & 1u;
    const uint32_t lf = cc > 0 ? (s[(cc - 1) >> 5].y >> ((cc - 1) & 31)) & 1u : 0u;
    bytes[(size_t)i * side + cc] = (uint8_t)(up | dn << 1 | lf << 2 | rt << 3);
}

}  // namespace tsb

using namespace tsb;

namespace tsb {

int ensure_bytes(tsb_domino *h, size_t need) {
    if (h->bytes_cap >= need) return TSB_OK;
    TSB_CUDA(cudaStreamSynchronize(h->stream));
    if (h->bytes) TSB_CUDA(cudaFree(h->bytes));
    h->bytes = nullptr;
    TSB_CUDA(cudaMalloc(&h->bytes, need));
    h->bytes_cap = need;
    return TSB_OK;
}

int check_range(tsb_domino *h, int chain0, int n) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    if (chain0 < 0 || n < 0 || chain0 + n > h->nchains)
        return fail(TSB_E_VALUE, "chains [%d, %d) outside the handle's %d chains", chain0, chain0 + n,
                    h->nchains);
    return TSB_OK;
}

int push_seeds(tsb_domino *h, int n, const uint64_t *seeds) {
    TSB_CUDA(cudaEventSynchronize(h->seed_ev));  // staging free again
    if ((int)h->gkeys.size() < n) h->gkeys.resize(n);
    for (int i = 0; i < n; ++i) {
        const uint64_t b = family_base(seeds[i]);
        h->seed_pinned[2 * i] = b;
        h->seed_pinned[2 * i + 1] = global_key(b);
        h->gkeys[i] = global_key(b);
    }
    TSB_CUDA(cudaMemcpyAsync(h->seedinfo, h->seed_pinned, sizeof(uint64_t) * 2 * n,
                             cudaMemcpyHostToDevice, h->stream));
    TSB_CUDA(cudaEventRecord(h->seed_ev, h->stream));
    return TSB_OK;
}

int launch_sweep(tsb_domino *h, int chain0, int n, uint64_t step, int color_override, cudaStream_t stream,
                 const uint64_t *step_dev) {
    SweepCtx c;
    const size_t off = (size_t)chain0 * h->chain_stride + h->pitch + kPad;  // row 0, word 0
    c.src = h->buf[h->cur] + off;
    c.dst = h->buf[h->cur ^ 1] + off;
    c.seedinfo = h->seedinfo;
    c.tgrid = h->tgrid;
    c.step_dev = step_dev;
    c.colors = step_dev ? h->colors : nullptr;
    c.tiles = h->tiles + h->win_t0;
    c.ntiles = h->win_tn;
    c.t0 = h->t0;
    c.t1 = h->t1;
    c.chain_stride = h->chain_stride;
    c.side = h->side;
    c.pitch = h->pitch;
    c.step = step;
    c.color_override = color_override;
    c.order = nullptr;
    c.cost = nullptr;
    c.xlist = nullptr;
    c.xcnt = nullptr;
    c.xbase = nullptr;
    c.xpitch = 0;
    h->cur ^= 1;
    if (h->ntiles == 0) return TSB_OK;
    cudaLaunchConfig_t cfg = {};
    if (h->win_tn == 0) return TSB_OK;
    cfg.gridDim = dim3(h->win_tn, 1, n);
    cfg.blockDim = dim3(32 * (kTileRows + 1));
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    switch (h->tmode) {
        case 0: TSB_CUDA(cudaLaunchKernelEx(&cfg, domino_sweep_kernel<0>, c)); break;
        case 1: TSB_CUDA(cudaLaunchKernelEx(&cfg, domino_sweep_kernel<1>, c)); break;
        default: TSB_CUDA(cudaLaunchKernelEx(&cfg, domino_sweep_kernel<2>, c)); break;
    }
    return TSB_OK;
}

// The pipelined kernel pays off once a launch streams from HBM: the two state
// buffers of the launched rows exceed what L2 keeps (Aztec 8192 and up, C4
// windows down to 1/4); L2-resident launches use one short-lived block per tile
// with the adaptive order (a 1/8 window of Aztec 16384: 9.6 -> 8.0 us/sweep).
static bool pipe_launch(const tsb_domino *h, int n) {
    if (h->m_pipe >= 0) return h->m_pipe == 1;
    const size_t bytes = 2 * sizeof(uint2) * (size_t)h->win_rows * h->pitch * (size_t)n;
    return bytes > kPipeMinBytes || (size_t)h->win_mn * (size_t)n > (size_t)kOrderThreads * kOrderPer;
}

// Whole-domain launches of the one-block-per-tile kernel use the adaptive
// dispatch order (reorder_tiles); TSB_DOM_ADAPT=0 keeps band-major order.
static bool adaptive_order(const tsb_domino *h, int n) {
    // row windows (strips) only with several waves of tiles: on the ~2-wave
    // windows of Aztec 4096 heavy-first was slower (1/4 window 4.3 -> 7.1 us)
    const bool full = h->win_m0 == 0 && h->win_mn == h->nmtiles;
    return h->m_order && h->m_adapt && h->m_wpl == 2 && !h->coupled && h->win_mn > 0 && !pipe_launch(h, n) &&
           h->win_mn <= kOrderThreads * kOrderPer && (full || h->win_mn >= 12 * h->num_sms);
}

// kMK sweeps (temporally blocked) of chains [chain0, chain0+n); graph mode only.
int launch_multi(tsb_domino *h, int chain0, int n, uint64_t step_off, cudaStream_t stream, bool compact) {
    SweepCtx c;
    const size_t off = (size_t)chain0 * h->chain_stride + h->pitch + kPad;
    c.src = h->buf[h->cur] + off;
    c.dst = h->buf[h->cur ^ 1] + off;
    c.seedinfo = h->seedinfo;
    c.tgrid = h->tgrid;
    c.step_dev = h->step_dev;
    c.colors = h->colors;
    c.tiles = h->mtiles + h->win_m0;
    c.ntiles = h->win_mn;
    c.t0 = h->t0;
    c.t1 = h->t1;
    c.chain_stride = h->chain_stride;
    c.side = h->side;
    c.pitch = h->pitch;
    c.step = step_off;
    c.color_override = -1;
    c.xlist = compact ? h->xlist : nullptr;
    c.xcnt = compact ? h->xcnt : nullptr;
    c.xbase = compact ? h->step_dev + 2 : nullptr;
    c.xpitch = (int)h->xpitch;
    const bool adapt = adaptive_order(h, n);
    // adaptive order over the launched window: indices relative to its first tile
    c.order = adapt ? h->m_order + h->win_m0 : nullptr;
    c.cost = adapt ? h->m_cost + h->win_m0 : nullptr;
    if (adapt) c.tiles = h->m_perm + h->win_m0;
    h->cur ^= 1;
    if (h->win_mn == 0) return TSB_OK;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(h->win_mn, 1, n);
    cfg.blockDim = dim3(32 * kMRows);
    cfg.dynamicSmemBytes = kMSmem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    // The coupled-pair kernel runs without programmatic dependent launch: with
    // PDL, back-to-back launches of it in run-collapsed CFTP walks (a sweeping
    // launch followed by a tile-copy launch) intermittently produced wrong top
    // chains (tools/dbg_cftp_rounds.py: 3 of 6 runs; 0 of 12 without PDL for
    // this kernel or outside graphs; the other kernels are unaffected).
    cfg.numAttrs = (h->m_wpl == 1 && h->coupled) ? 0 : 1;
    const int mode = compact ? kSelList : (h->collapse ? kSelSkip : kSelPlain);
#define TSB_DOM_LAUNCH(kern)                                                              \
    switch (h->tmode * 3 + mode) {                                                        \
        case 0: TSB_CUDA(cudaLaunchKernelEx(&cfg, kern<0, kSelPlain>, c)); break;         \
        case 1: TSB_CUDA(cudaLaunchKernelEx(&cfg, kern<0, kSelSkip>, c)); break;          \
        case 2: TSB_CUDA(cudaLaunchKernelEx(&cfg, kern<0, kSelList>, c)); break;          \
        case 3: TSB_CUDA(cudaLaunchKernelEx(&cfg, kern<1, kSelPlain>, c)); break;         \
        case 4: TSB_CUDA(cudaLaunchKernelEx(&cfg, kern<1, kSelSkip>, c)); break;          \
        case 5: TSB_CUDA(cudaLaunchKernelEx(&cfg, kern<1, kSelList>, c)); break;          \
        case 6: TSB_CUDA(cudaLaunchKernelEx(&cfg, kern<2, kSelPlain>, c)); break;         \
        case 7: TSB_CUDA(cudaLaunchKernelEx(&cfg, kern<2, kSelSkip>, c)); break;          \
        default: TSB_CUDA(cudaLaunchKernelEx(&cfg, kern<2, kSelList>, c)); break;         \
    }
    if (h->m_wpl == 1 && h->coupled && (n & 1) == 0) {
        cfg.gridDim.z = n / 2;  // one block per tile and coupled pair
        TSB_DOM_LAUNCH(domino_multi1c_kernel);
        return TSB_OK;
    }
    if (h->m_wpl == 1) {
        TSB_DOM_LAUNCH(domino_multi1_kernel);
        return TSB_OK;
    }
    // HBM-streaming launches: the persistent cp.async-pipelined kernel (pipe_launch)
    if (pipe_launch(h, n)) {
        cfg.gridDim.x = std::min(h->win_mn, kMBlocks * h->num_sms);
        cfg.dynamicSmemBytes = kPipeSmem;
        TSB_DOM_LAUNCH(domino_multi_pipe_kernel);
        return TSB_OK;
    }
    TSB_DOM_LAUNCH(domino_multi_kernel);
#undef TSB_DOM_LAUNCH
    return TSB_OK;
}

__global__ void set_step_kernel(uint64_t *step_dev, uint64_t v) { *step_dev = v; }
// step_dev = {step0, end}; with a colour table, also the table of the
// first kGraphSweeps steps (launched <<<chains, kGraphSweeps>>>)
__global__ void set_walk_kernel(uint64_t *step_dev, uint64_t step0, uint64_t end, const uint64_t *seedinfo = nullptr,
                                uint8_t *colors = nullptr, int collapse = 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        step_dev[0] = step0;
        step_dev[1] = end;
    }
    if (colors)
        colors[blockIdx.x * kGraphSweeps + threadIdx.x] =
            color_entry(seedinfo[2 * blockIdx.x + 1], step0 + threadIdx.x, end, collapse);
}

// canonical (band-major) order of a window's tiles [0, n): reorder_tiles input state
__global__ void order_reset_kernel(const int2 *tiles, int n, int *order, int2 *perm, unsigned *cost) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    order[i] = i;
    perm[i] = tiles[i];
    cost[i] = 0u;
}

// Adaptive dispatch order of whole-domain multi-sweep launches (end of every
// 4th graph replay: the heavy tiles move slowly).  Each block records how long its tile took (cycles, thread
// 0, after the last barrier); tiles are then dispatched by cost class --
// more than 3x the mean duration, 1.5x, 1x, the rest --
// and in band-major order within a class.  The slow tiles are those whose
// rows hold many rotateable sites (long coin queues: the melting seam of an
// Aztec diamond started from T_max, the disordered disk of a mixed state);
// dispatched first they no longer start mid-launch and set its end, while
// band-major order within a class keeps neighbouring bands together.
// Results do not depend on the order.

__device__ __forceinline__ int cost_class(unsigned cost, int n, unsigned long long tot) {
    const unsigned long long x = 2ull * (unsigned long long)cost * (unsigned long long)n;  // 2 * cost / mean * tot
    return x > 6ull * tot ? 3 : x > 3ull * tot ? 2 : x > 2ull * tot ? 1 : 0;
}

__device__ __forceinline__ void reorder_tiles(const unsigned *cost, const int2 *tiles, int n, int *order, int2 *perm) {
    typedef cub::BlockReduce<unsigned long long, kOrderThreads> Reduce;
    typedef cub::BlockScan<int, kOrderThreads> Scan;
    __shared__ union {
        typename Reduce::TempStorage r;
        typename Scan::TempStorage s;
    } tmp;
    __shared__ unsigned long long tot_s;
    // thread t owns tiles kOrderPer * t .. kOrderPer * t + kOrderPer - 1 (one load each)
    const int i0 = kOrderPer * threadIdx.x;
    unsigned c[kOrderPer];
    unsigned long long part = 0;
#pragma unroll
    for (int j = 0; j < kOrderPer; ++j) {
        c[j] = i0 + j < n ? cost[i0 + j] : 0u;
        part += c[j];
    }
    const unsigned long long tot = Reduce(tmp.r).Sum(part);
    if (threadIdx.x == 0) tot_s = tot;
    __syncthreads();
    int cls[kOrderPer];
    bool hot = false;
#pragma unroll
    for (int j = 0; j < kOrderPer; ++j) {
        cls[j] = i0 + j < n ? cost_class(c[j], n, tot_s) : -1;
        hot |= cls[j] == kOrderClasses - 1;
    }
    // heavy-first pays only with a few hot tiles (a melting seam: some tile
    // above 3x the mean); with a broad load (an equilibrium state) the
    // band-major order interleaves heavy and light tiles on every SM
    if (!__syncthreads_or(hot)) {
#pragma unroll
        for (int j = 0; j < kOrderPer; ++j) cls[j] = i0 + j < n ? 0 : -1;
    }
    int pos = 0;  // block-uniform
    for (int k = kOrderClasses - 1; k >= 0; --k) {
        int cnt = 0;
#pragma unroll
        for (int j = 0; j < kOrderPer; ++j) cnt += cls[j] == k;
        int o, t;
        __syncthreads();
        Scan(tmp.s).ExclusiveSum(cnt, o, t);
#pragma unroll
        for (int j = 0; j < kOrderPer; ++j)
            if (cls[j] == k) {
                order[pos + o] = i0 + j;
                perm[pos + o] = tiles[i0 + j];
                ++o;
            }
        pos += t;
    }
}

// Bookkeeping between graph replays, one launch instead of three: the
// adaptive tile reorder when it is due (the heavy tiles move slowly: every
// `every`-th replay), the replay counter advance, and the colour table of
// the next replay (colour-table walks; set_walk_kernel fills the first).
struct ReplayTail {
    const unsigned *cost;  // adaptive order (nullptr: none)
    const int2 *tiles;
    int ntiles, every;
    int *order;
    int2 *perm;
    uint64_t *counter;          // step_dev[0] (colour tables) or step_dev[2] (executed-sweep lists)
    const uint64_t *step_dev;   // step_dev[1] = end of the walk
    const uint64_t *seedinfo;
    uint8_t *colors;            // nullptr for list replays
    int nchains, collapse;
};

__global__ void __launch_bounds__(kOrderThreads) replay_tail_kernel(ReplayTail t) {
    const uint64_t base = *t.counter;
    if (t.cost && (base / kGraphSweeps) % (uint64_t)t.every == 0)  // block-uniform
        reorder_tiles(t.cost, t.tiles, t.ntiles, t.order, t.perm);
    if (threadIdx.x == 0) *t.counter = base + kGraphSweeps;
    if (t.colors) {
        const uint64_t end = t.step_dev[1];
        for (int i = threadIdx.x; i < t.nchains * kGraphSweeps; i += blockDim.x) {
            const int z = i / kGraphSweeps, j = i - z * kGraphSweeps;
            t.colors[i] = color_entry(t.seedinfo[2 * z + 1], base + kGraphSweeps + (uint64_t)j, end, t.collapse);
        }
    }
}

// A CUDA graph of kGraphSweeps sweeps (even, so the buffers end where they
// started) followed by `step += kGraphSweeps`; long walks replay it, which
// removes the per-launch host overhead (the kernels read the step base from
// device memory).
int ensure_graph(tsb_domino *h, int chain0, int n, bool compact) {
    const bool same = h->graph_exec && h->g_chain0 == chain0 && h->g_n == n && h->g_cur == h->cur &&
                      h->g_compact == (int)compact &&
                      h->g_tmode == h->tmode && h->g_t0 == h->t0 && h->g_t1 == h->t1 &&
                      h->g_win0 == h->win_t0 && h->g_winn == h->win_tn && h->g_winm == h->win_m0 &&
                      h->g_tail == h->graph_tail && h->g_coupled == h->coupled && h->g_collapse == h->collapse;
    if (same) return TSB_OK;
    if (h->graph_exec) {
        cudaGraphExecDestroy(h->graph_exec);
        h->graph_exec = nullptr;
    }
    if (!h->cap_stream) TSB_CUDA(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    TSB_CUDA(cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal));
    int rc = TSB_OK;
    // compact replays take the next kGraphSweeps entries of the executed-sweep
    // lists (step_dev[2] advances); colour-table replays the next kGraphSweeps
    // steps (step_dev[0] advances)
    // (the colour table of a replay is written by the previous replay's
    // tail or by set_walk_kernel)
    static_assert(kGraphSweeps % (2 * kMK) == 0, "graph replays must end in the starting buffer");
    for (int i = 0; i < kGraphSweeps / kMK && !rc; ++i)
        rc = launch_multi(h, chain0, n, (uint64_t)(i * kMK), h->cap_stream, compact);
    ReplayTail tail;
    const bool adapt = adaptive_order(h, n);
    tail.cost = adapt ? h->m_cost + h->win_m0 : nullptr;
    tail.tiles = h->mtiles + h->win_m0;
    tail.ntiles = h->win_mn;
    tail.every = h->m_order_every;
    tail.order = h->m_order + h->win_m0;
    tail.perm = h->m_perm + h->win_m0;
    tail.counter = compact ? h->step_dev + 2 : h->step_dev;
    tail.step_dev = h->step_dev;
    tail.seedinfo = h->seedinfo;
    tail.colors = compact ? nullptr : h->colors;
    tail.nchains = n;
    tail.collapse = h->collapse;
    if (!rc) replay_tail_kernel<<<1, kOrderThreads, 0, h->cap_stream>>>(tail);
    if (!rc && h->graph_tail) rc = h->graph_tail(h, h->cap_stream);
    cudaError_t e = cudaStreamEndCapture(h->cap_stream, &g);
    if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    if (e != cudaSuccess) return cuda_fail(e, "graph capture");
    e = cudaGraphInstantiate(&h->graph_exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
        h->graph_exec = nullptr;
        return cuda_fail(e, "graph instantiate");
    }
    h->g_chain0 = chain0;
    h->g_n = n;
    h->g_cur = h->cur;
    h->g_tmode = h->tmode;
    h->g_t0 = h->t0;
    h->g_t1 = h->t1;
    h->g_win0 = h->win_t0;
    h->g_winn = h->win_tn;
    h->g_winm = h->win_m0;
    h->g_tail = h->graph_tail;
    h->g_coupled = h->coupled;
    h->g_collapse = h->collapse;
    h->g_compact = (int)compact;
    return TSB_OK;
}

// After an odd number of sweeps the walked chains live in the other buffer;
// copy them back so the handle keeps one canonical buffer for all chains.
int settle(tsb_domino *h, int chain0, int n, int cur0) {
    if (h->cur == cur0 || n == h->nchains) return TSB_OK;
    const size_t off = (size_t)chain0 * h->chain_stride;
    TSB_CUDA(cudaMemcpyAsync(h->buf_alloc[h->cur ^ 1] + off, h->buf_alloc[h->cur] + off,
                             sizeof(uint2) * h->chain_stride * n, cudaMemcpyDeviceToDevice, h->stream));
    h->cur ^= 1;
    return TSB_OK;
}

}  // namespace tsb

extern "C" {

static int create_impl(int device, int side, int nchains, const uint8_t *faces, int row_lo, int row_hi,
                       tsb_domino **out);

int tsb_domino_create(int device, int side, int nchains, const uint8_t *faces, tsb_domino **out) {
    return create_impl(device, side, nchains, faces, 0, side, out);
}

int tsb_domino_create_window(int device, int side, int row_lo, int row_hi, const uint8_t *faces, tsb_domino **out) {
    if (row_lo < 0 || row_hi > side || row_hi <= row_lo) return fail(TSB_E_VALUE, "window rows out of range");
    return create_impl(device, side, 1, faces, row_lo, row_hi, out);
}

// Rows beyond a window that its tiles may load or store: a multi-sweep tile
// reaches kMK + kMOut - 1 rows past the window edge, a single-sweep tile
// kTileRows (zero there: the stale halo a strip never reads back).
constexpr int kWinMargin = kMK + kMOut - 1 > 16 ? kMK + kMOut - 1 : 16;

static int create_impl(int device, int side, int nchains, const uint8_t *faces, int row_lo, int row_hi,
                       tsb_domino **out) {
    if (!out) return fail(TSB_E_VALUE, "null output pointer");
    *out = nullptr;
    if (side < 1 || nchains < 1) return fail(TSB_E_VALUE, "side and nchains must be positive");
    if ((uint64_t)side * (uint64_t)side >= kCapacity)
        return fail(TSB_E_CAPACITY, "grid of %lld sites exceeds capacity", (long long)side * side);
    int rc = ensure_device(device);
    if (rc) return rc;
    tsb_domino *h = new tsb_domino();
    h->device = device;
    h->side = side;
    h->nchains = nchains;
    h->W = (side + 31) / 32;
    // rows: kPad zero words, W words, zero padding up to the last tile's halo;
    // 256-byte aligned
    // right padding: the single-sweep tiles (multiples of kTileWords) and the
    // band-aligned multi-sweep tiles (any even start <= W - 2, 64 words) both
    // load and store inside the row
    const int nchunks_ = (h->W + 1 + kTileWords - 1) / kTileWords;
    h->pitch = (std::max(kPad + nchunks_ * kTileWords + 2, kPad + h->W + 64) + 31) / 32 * 32;
    h->windowed = row_lo > 0 || row_hi < side;
    h->row_a = h->windowed ? std::max(-1, row_lo - kWinMargin) : -1;
    h->row_b = h->windowed ? std::min(side + 1, row_hi + kWinMargin) : side + 1;
    h->chain_stride = (size_t)(h->row_b - h->row_a) * h->pitch;
    const int da = std::max(0, h->row_a), db = std::min(side, h->row_b);  // allocated rows of the domain planes
    cudaError_t e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) { delete h; return cuda_fail(e, "cudaStreamCreate"); }
    h->own_stream = true;
    auto bail = [&](cudaError_t err, const char *what) {
        int code = cuda_fail(err, what);
        tsb_domino_destroy(h);
        return code;
    };
    const size_t sbytes = sizeof(uint2) * h->chain_stride * nchains;
    for (int i = 0; i < 2; ++i) {
        if ((e = cudaMalloc(&h->buf_alloc[i], sbytes)) != cudaSuccess) return bail(e, "cudaMalloc state");
        if ((e = cudaMemsetAsync(h->buf_alloc[i], 0, sbytes, h->stream)) != cudaSuccess) return bail(e, "memset");
        h->buf[i] = h->buf_alloc[i] - (ptrdiff_t)(h->row_a + 1) * h->pitch;  // global row indexing
    }
    if ((e = cudaMalloc(&h->dom_alloc, sizeof(uint4) * (size_t)(db - da) * h->pitch)) != cudaSuccess)
        return bail(e, "cudaMalloc dom");
    if ((e = cudaMalloc(&h->fbits_alloc, sizeof(uint32_t) * (size_t)(db - da) * h->pitch)) != cudaSuccess)
        return bail(e, "cudaMalloc fbits");
    h->dom = h->dom_alloc - (ptrdiff_t)da * h->pitch;
    h->fbits = h->fbits_alloc - (ptrdiff_t)da * h->pitch;
    if ((e = cudaMalloc(&h->range, sizeof(int2) * side)) != cudaSuccess) return bail(e, "cudaMalloc range");
    if ((e = cudaMalloc(&h->seedinfo, sizeof(uint64_t) * 2 * nchains)) != cudaSuccess)
        return bail(e, "cudaMalloc seeds");
    if ((e = cudaMallocHost(&h->seed_pinned, sizeof(uint64_t) * 2 * nchains)) != cudaSuccess)
        return bail(e, "cudaMallocHost seeds");
    if ((e = cudaMalloc(&h->bad, sizeof(int))) != cudaSuccess) return bail(e, "cudaMalloc flag");
    if ((e = cudaMalloc(&h->step_dev, 3 * sizeof(uint64_t))) != cudaSuccess) return bail(e, "cudaMalloc step");
    if ((e = cudaMalloc(&h->colors, (size_t)kGraphSweeps * nchains)) != cudaSuccess) return bail(e, "cudaMalloc colors");
    if ((e = cudaEventCreateWithFlags(&h->seed_ev, cudaEventDisableTiming)) != cudaSuccess)
        return bail(e, "cudaEventCreate");
    if ((e = cudaEventRecord(h->seed_ev, h->stream)) != cudaSuccess) return bail(e, "cudaEventRecord");

    // domain -> crossable planes and row ranges
    const int nf = side - 1;
    uint8_t *dfaces = nullptr;
    const size_t fbytes = std::max<size_t>(1, (size_t)nf * nf);
    if ((e = cudaMalloc(&dfaces, fbytes)) != cudaSuccess) return bail(e, "cudaMalloc faces");
    if (faces && nf > 0) e = cudaMemcpyAsync(dfaces, faces, (size_t)nf * nf, cudaMemcpyHostToDevice, h->stream);
    else e = cudaMemsetAsync(dfaces, 1, fbytes, h->stream);
    if (e != cudaSuccess) { cudaFree(dfaces); return bail(e, "faces upload"); }
    std::vector<int2> init(side, make_int2(INT_MAX, INT_MIN));
    cudaMemcpyAsync(h->range, init.data(), sizeof(int2) * side, cudaMemcpyHostToDevice, h->stream);
    domain_planes_kernel<<<dim3((h->W + 127) / 128, db - da), 128, 0, h->stream>>>(
        dfaces, side, h->W, h->pitch, h->dom, h->fbits, h->range, da, h->windowed ? row_lo : 0,
        h->windowed ? row_hi : side);
    fix_ranges_kernel<<<(side + 255) / 256, 256, 0, h->stream>>>(h->range, side);
    e = cudaStreamSynchronize(h->stream);
    cudaFree(dfaces);
    if (e != cudaSuccess) return bail(e, "domain planes");
    // non-empty sweep tiles (kTileRows rows x kTileWords output words)
    std::vector<int2> rg(side);
    if ((e = cudaMemcpy(rg.data(), h->range, sizeof(int2) * side, cudaMemcpyDeviceToHost)) != cudaSuccess)
        return bail(e, "ranges");
    const int nchunks = (h->W + 1 + kTileWords - 1) / kTileWords;
    // non-empty tiles of `band` output rows x kTileWords output words,
    // band-major, plus the first tile of every band (row windows)
    auto make_tiles = [&](int band, std::vector<int2> &tl, std::vector<int> &bstart) {
        const int nb = (side + band - 1) / band;
        bstart.assign(nb + 1, 0);
        for (int y = 0; y < nb; ++y) {
            bstart[y] = (int)tl.size();
            int lo = INT_MAX, hi = INT_MIN;
            for (int r = y * band; r < std::min(side, (y + 1) * band); ++r)
                if (rg[r].y > rg[r].x) { lo = std::min(lo, rg[r].x); hi = std::max(hi, rg[r].y); }
            for (int x = 0; x < nchunks; ++x) {
                const int w0 = x * kTileWords - 1;
                if (hi > w0 && lo < w0 + kTileWords) tl.push_back(make_int2(x, y));
            }
        }
        bstart[nb] = (int)tl.size();
    };
    std::vector<int2> tiles, mtiles;
    make_tiles(kTileRows, tiles, h->band_start);
    {
        // multi-sweep tiles are aligned to each band's own word range: tile.x
        // = first loaded word wa0 (even, for 16-byte loads), outputs words
        // wa0+1 .. wa0+kTileWords; a band [wl, wh) starts at (wl-1) & ~1
        // Two widths: 2 words per lane (62 output words, 16-byte loads) or 1
        // (30 output words) -- whichever covers the domain with fewer word
        // slots (TSB_DOM_WPL=1|2 forces one).
        const int nb = (side + kMOut - 1) / kMOut;
        auto build = [&](int wpl, std::vector<int2> &tl, std::vector<int> &bs) {
            const int out_words = 32 * wpl - 2;
            bs.assign(nb + 1, 0);
            for (int y = 0; y < nb; ++y) {
                bs[y] = (int)tl.size();
                int lo = INT_MAX, hi = INT_MIN;
                for (int r = y * kMOut; r < std::min(side, (y + 1) * kMOut); ++r)
                    if (rg[r].y > rg[r].x) { lo = std::min(lo, rg[r].x); hi = std::max(hi, rg[r].y); }
                if (hi <= lo) continue;
                for (int wa0 = wpl == 2 ? ((lo - 1) & ~1) : lo - 1; wa0 + 1 < hi; wa0 += out_words)
                    tl.push_back(make_int2(wa0, y));
            }
            bs[nb] = (int)tl.size();
        };
        std::vector<int2> t1;
        std::vector<int> b1, b2;
        build(2, mtiles, b2);
        build(1, t1, b1);
        int wpl = (size_t)t1.size() * 32 < mtiles.size() * 64 * 9 / 10 ? 1 : 2;  // 1 only when clearly cheaper
        if (const char *ev = getenv("TSB_DOM_WPL")) wpl = atoi(ev) == 1 ? 1 : 2;
        h->m_wpl = wpl;
        if (const char *ev = getenv("TSB_DOM_PIPE")) h->m_pipe = atoi(ev) ? 1 : 0;  // force the pipelined kernel on / off
        if (wpl == 1) {
            mtiles.swap(t1);
            h->mband_start.swap(b1);
        } else {
            h->mband_start.swap(b2);
        }
    }
    h->ntiles = (int)tiles.size();
    h->nmtiles = (int)mtiles.size();
    h->win_t0 = 0;
    h->win_tn = h->ntiles;
    h->win_m0 = 0;
    h->win_mn = h->nmtiles;
    h->win_rows = side;
    if ((e = cudaMalloc(&h->mtiles, sizeof(int2) * std::max<size_t>(1, mtiles.size()))) != cudaSuccess)
        return bail(e, "cudaMalloc mtiles");
    if (!mtiles.empty() &&
        (e = cudaMemcpy(h->mtiles, mtiles.data(), sizeof(int2) * mtiles.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
        return bail(e, "mtiles");
    {
        std::vector<int> iota(std::max<size_t>(1, mtiles.size()));
        for (size_t i = 0; i < iota.size(); ++i) iota[i] = (int)i;
        if ((e = cudaMalloc(&h->m_order, sizeof(int) * iota.size())) != cudaSuccess) return bail(e, "cudaMalloc order");
        if ((e = cudaMemcpy(h->m_order, iota.data(), sizeof(int) * iota.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
            return bail(e, "order");
        if ((e = cudaMalloc(&h->m_perm, sizeof(int2) * iota.size())) != cudaSuccess) return bail(e, "cudaMalloc perm");
        if (!mtiles.empty() &&
            (e = cudaMemcpy(h->m_perm, mtiles.data(), sizeof(int2) * mtiles.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
            return bail(e, "perm");
        if ((e = cudaMalloc(&h->m_cost, sizeof(unsigned) * iota.size())) != cudaSuccess) return bail(e, "cudaMalloc cost");
        if ((e = cudaMemset(h->m_cost, 0, sizeof(unsigned) * iota.size())) != cudaSuccess) return bail(e, "cost");
        if (const char *ev = getenv("TSB_DOM_ADAPT")) h->m_adapt = atoi(ev) != 0;
        if (const char *ev = getenv("TSB_DOM_COLLAPSE")) h->collapse = atoi(ev) != 0;
        if (const char *ev = getenv("TSB_DOM_ORDER_EVERY")) h->m_order_every = std::max(1, atoi(ev));
    }
#define TSB_ALL_MODES(kern)                                                                            \
    (const void *)kern<0, kSelPlain>, (const void *)kern<0, kSelSkip>, (const void *)kern<0, kSelList>,     \
        (const void *)kern<1, kSelPlain>, (const void *)kern<1, kSelSkip>, (const void *)kern<1, kSelList>, \
        (const void *)kern<2, kSelPlain>, (const void *)kern<2, kSelSkip>, (const void *)kern<2, kSelList>
    for (const void *fn : {TSB_ALL_MODES(domino_multi_kernel), TSB_ALL_MODES(domino_multi1_kernel),
                           TSB_ALL_MODES(domino_multi1c_kernel)})
        if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMSmem)) != cudaSuccess)
            return bail(e, "smem attribute");
    for (const void *fn : {TSB_ALL_MODES(domino_multi_pipe_kernel)})
        if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPipeSmem)) != cudaSuccess)
            return bail(e, "smem attribute");
#undef TSB_ALL_MODES
    cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
    if ((e = cudaMalloc(&h->tiles, sizeof(int2) * std::max<size_t>(1, tiles.size()))) != cudaSuccess)
        return bail(e, "cudaMalloc tiles");
    if (!tiles.empty() &&
        (e = cudaMemcpy(h->tiles, tiles.data(), sizeof(int2) * tiles.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
        return bail(e, "tiles");
    *out = h;
    return TSB_OK;
}

int tsb_domino_destroy(tsb_domino *h) {
    if (!h) return TSB_OK;
    cudaSetDevice(h->device);
    strip_free(h);
    if (h->stream) cudaStreamSynchronize(h->stream);
    cudaFree(h->buf_alloc[0]);
    cudaFree(h->buf_alloc[1]);
    cudaFree(h->dom_alloc);
    cudaFree(h->fbits_alloc);
    cudaFree(h->range);
    cudaFree(h->xlist);
    cudaFree(h->xcnt);
    for (int i = 0; i < 2; ++i) {
        if (h->xpin[i]) cudaFreeHost(h->xpin[i]);
        if (h->xev[i]) cudaEventDestroy(h->xev[i]);
    }
    cudaFree(h->hx_h);
    cudaFree(h->hx_flags);
    cudaFree(h->hx_rows);
    cudaFree(h->hx_off);
    cudaFree(h->tiles);
    cudaFree(h->mtiles);
    cudaFree(h->m_order);
    cudaFree(h->m_perm);
    cudaFree(h->m_cost);
    cudaFree(h->tgrid);
    cudaFree(h->seedinfo);
    cudaFree(h->bytes);
    cudaFree(h->bad);
    cudaFree(h->step_dev);
    cudaFree(h->colors);
    if (h->graph_exec) cudaGraphExecDestroy(h->graph_exec);
    if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
    if (h->seed_pinned) cudaFreeHost(h->seed_pinned);
    if (h->seed_ev) cudaEventDestroy(h->seed_ev);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    delete h;
    return TSB_OK;
}

int tsb_domino_set_stream(tsb_domino *h, void *stream) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    TSB_CUDA(cudaSetDevice(h->device));
    TSB_CUDA(cudaStreamSynchronize(h->stream));
    if (h->own_stream) cudaStreamDestroy(h->stream);
    h->stream = (cudaStream_t)stream;
    h->own_stream = false;
    return TSB_OK;
}

int tsb_domino_set_p_up(tsb_domino *h, const double *p_up) {
    if (!h || !p_up) return fail(TSB_E_VALUE, "null argument");
    TSB_CUDA(cudaSetDevice(h->device));
    const int64_t s = h->side;
    // pass 1: uniform or parity-only thresholds need no grid on the device
    uint64_t par[2] = {threshold_of(p_up[0]), s > 1 ? threshold_of(p_up[1]) : threshold_of(p_up[0])};
    bool parity_ok = true;
    for (int64_t r = 0; r < s && parity_ok; ++r)
        for (int64_t c = 0; c < s; ++c)
            if (threshold_of(p_up[r * s + c]) != par[(r + c) & 1]) {
                parity_ok = false;
                break;
            }
    if (parity_ok) return tsb_domino_set_p_up_parity(h, p_up[0], s > 1 ? p_up[1] : p_up[0]);
    // pass 2: per-site thresholds
    std::vector<uint64_t> t((size_t)(s * s));
    for (int64_t i = 0; i < s * s; ++i) t[(size_t)i] = threshold_of(p_up[i]);
    h->tmode = 2;
    if (!h->tgrid) TSB_CUDA(cudaMalloc(&h->tgrid, sizeof(uint64_t) * t.size()));
    TSB_CUDA(cudaMemcpyAsync(h->tgrid, t.data(), sizeof(uint64_t) * t.size(), cudaMemcpyHostToDevice, h->stream));
    TSB_CUDA(cudaStreamSynchronize(h->stream));
    return TSB_OK;
}

int tsb_domino_set_p_up_parity(tsb_domino *h, double p_even, double p_odd) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    const uint64_t t0 = threshold_of(p_even), t1 = threshold_of(p_odd);
    h->tmode = t0 == t1 ? 0 : 1;
    h->t0 = t0;
    h->t1 = t1;
    return TSB_OK;
}

int tsb_domino_upload(tsb_domino *h, int chain0, int n, const uint8_t *states) {
    TSB_FULL_ONLY(h);
    int rc = check_range(h, chain0, n);
    if (rc || n == 0) return rc;
    TSB_CUDA(cudaSetDevice(h->device));
    const size_t grid = (size_t)h->side * h->side;
    if ((rc = ensure_bytes(h, grid * n))) return rc;
    if ((rc = staged_h2d(h->bytes, states, grid * n, h->stream))) return rc;
    TSB_CUDA(cudaMemsetAsync(h->bad, 0, sizeof(int), h->stream));
    pack_kernel<<<dim3((h->W + 127) / 128, h->side, n), 128, 0, h->stream>>>(
        h->bytes, h->side, h->W, h->pitch, h->chain_stride, h->dom,
        h->buf[h->cur] + (size_t)chain0 * h->chain_stride + kPad, h->bad);
    TSB_CUDA(cudaGetLastError());
    int bad = 0;
    TSB_CUDA(cudaMemcpyAsync(&bad, h->bad, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    TSB_CUDA(cudaStreamSynchronize(h->stream));
    if (bad & 1) return fail(TSB_E_INCONSISTENT, "tilestate values must be < 16");
    if (bad & 2) return fail(TSB_E_INCONSISTENT, "edge bit not mirrored by the neighbouring vertex");
    if (bad & 4) return fail(TSB_E_INCONSISTENT, "crossed edge leaves the grid or the domain");
    return TSB_OK;
}

int tsb_domino_download(tsb_domino *h, int chain0, int n, uint8_t *states) {
    TSB_FULL_ONLY(h);
    int rc = check_range(h, chain0, n);
    if (rc || n == 0) return rc;
    TSB_CUDA(cudaSetDevice(h->device));
    const size_t grid = (size_t)h->side * h->side;
    if ((rc = ensure_bytes(h, grid * n))) return rc;
    unpack_kernel<<<dim3((h->side + 127) / 128, h->side, n), 128, 0, h->stream>>>(
        h->buf[h->cur] + (size_t)chain0 * h->chain_stride + kPad, h->side, h->pitch, h->chain_stride, h->bytes);
    TSB_CUDA(cudaGetLastError());
    return staged_d2h(states, h->bytes, grid * n, h->stream);
}

static int rows_range(tsb_domino *h, int r0, int nrows) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    const int lo = std::max(0, h->row_a), hi = std::min(h->side, h->row_b);
    if (nrows < 0 || r0 < lo || r0 + nrows > hi)
        return fail(TSB_E_VALUE, "rows [%d, %d) outside the handle's rows [%d, %d)", r0, r0 + nrows, lo, hi);
    return TSB_OK;
}

int tsb_domino_upload_rows(tsb_domino *h, int r0, int nrows, const uint8_t *rows) {
    int rc = rows_range(h, r0, nrows);
    if (rc || nrows == 0) return rc;
    if (!rows) return fail(TSB_E_VALUE, "null rows");
    TSB_CUDA(cudaSetDevice(h->device));
    const size_t bytes = (size_t)nrows * h->side;
    if ((rc = ensure_bytes(h, bytes))) return rc;
    if ((rc = staged_h2d(h->bytes, rows, bytes, h->stream))) return rc;
    TSB_CUDA(cudaMemsetAsync(h->bad, 0, sizeof(int), h->stream));
    pack_rows_kernel<<<dim3((h->W + 127) / 128, nrows), 128, 0, h->stream>>>(h->bytes, r0, h->side, h->W, h->pitch,
                                                                              h->dom, h->buf[h->cur] + kPad, h->bad);
    TSB_CUDA(cudaGetLastError());
    int bad = 0;
    TSB_CUDA(cudaMemcpyAsync(&bad, h->bad, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    TSB_CUDA(cudaStreamSynchronize(h->stream));
    if (bad & 1) return fail(TSB_E_INCONSISTENT, "tilestate values must be < 16");
    if (bad & 2) return fail(TSB_E_INCONSISTENT, "edge bit not mirrored by the neighbouring vertex");
    if (bad & 4) return fail(TSB_E_INCONSISTENT, "crossed edge leaves the grid or the domain");
    return TSB_OK;
}

int tsb_domino_download_rows(tsb_domino *h, int r0, int nrows, uint8_t *rows) {
    int rc = rows_range(h, r0, nrows);
    if (rc || nrows == 0) return rc;
    if (!rows) return fail(TSB_E_VALUE, "null rows");
    TSB_CUDA(cudaSetDevice(h->device));
    const size_t bytes = (size_t)nrows * h->side;
    if ((rc = ensure_bytes(h, bytes))) return rc;
    unpack_rows_kernel<<<dim3((h->side + 127) / 128, nrows), 128, 0, h->stream>>>(h->buf[h->cur] + kPad, r0, h->side,
                                                                                   h->pitch, h->bytes);
    TSB_CUDA(cudaGetLastError());
    return staged_d2h(rows, h->bytes, bytes, h->stream);
}

int tsb_domino_walk(tsb_domino *h, int chain0, int n, const uint64_t *seeds, uint64_t step0,
                    uint64_t n_steps) {
    int rc = check_range(h, chain0, n);
    if (rc || n == 0 || n_steps == 0) return rc;
    if (!seeds) return fail(TSB_E_VALUE, "null seeds");
    TSB_CUDA(cudaSetDevice(h->device));
    if ((rc = push_seeds(h, n, seeds))) return rc;
    return walk_steps(h, chain0, n, step0, n_steps);
}

}  // extern "C"

// n_steps sweeps of chains [chain0, chain0+n) whose seeds are already on the
// device: graph replays, direct multi-sweep launches, single sweeps; the
// walked chains end in the handle's canonical buffer.  Stream-ordered, no
// host synchronisation.
// Shared-memory bytes of a resident walk, 0 when the lattice is not eligible.
// Default: tiny lattices (<= kResMaxItems words: a tiled launch is a few
// blocks of pure latency) or batches of >= kResMinChains chains (the tiled
// launches then queue many waves of small tiles while one resident block per
// chain stays within about one wave; Aztec 128 x 128 chains: 8.2 -> 3.2 us
// per sweep, Aztec 256: 13.4 -> 6.8).  A single chain of a larger lattice
// keeps the tiled kernels (Aztec 128: 1.85 vs 3.1 us).
static size_t resident_smem(const tsb_domino *h, int n) {
    const char *ev = getenv("TSB_DOM_RESIDENT");  // 0: never, 1: whenever it fits (read per walk)
    const int mode = ev ? atoi(ev) : -1;
    if (mode == 0 || h->strip || h->windowed || h->win_mn != h->nmtiles || h->win_tn != h->ntiles) return 0;
    const size_t items = (size_t)h->side * h->W;
    if (mode < 0 && items > (size_t)kResMaxItems && n < kResMinChains) return 0;
    const size_t bytes = kResScratch + sizeof(uint2) * (size_t)(h->side + 2) * h->W +
                         sizeof(uint32_t) * (size_t)(h->side + 1) * (h->W + 1);
    return bytes <= 200u * 1024u ? bytes : 0;
}

static int launch_resident(tsb_domino *h, int chain0, int n, uint64_t step0, uint64_t n_steps, size_t smem) {
    ResCtx c;
    c.state = h->buf[h->cur] + (size_t)chain0 * h->chain_stride + h->pitch + kPad;
    c.seedinfo = h->seedinfo;
    c.tgrid = h->tgrid;
    c.t0 = h->t0;
    c.t1 = h->t1;
    c.chain_stride = h->chain_stride;
    c.side = h->side;
    c.pitch = h->pitch;
    c.W = h->W;
    c.step0 = step0;
    c.n_steps = n_steps;
    c.collapse = h->collapse;
    const size_t items = (size_t)h->side * h->W;
    const int threads = (int)std::min<size_t>(kResThreads, (items + 31) / 32 * 32);
    const void *fn = h->tmode == 0 ? (const void *)domino_resident_kernel<0>
                   : h->tmode == 1 ? (const void *)domino_resident_kernel<1> : (const void *)domino_resident_kernel<2>;
    TSB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    switch (h->tmode) {
        case 0: domino_resident_kernel<0><<<n, threads, smem, h->stream>>>(c); break;
        case 1: domino_resident_kernel<1><<<n, threads, smem, h->stream>>>(c); break;
        default: domino_resident_kernel<2><<<n, threads, smem, h->stream>>>(c); break;
    }
    TSB_CUDA(cudaGetLastError());
    return TSB_OK;
}

__global__ void set_segment_kernel(uint64_t *step_dev, uint64_t step) {
    step_dev[0] = step;  // base of the executed-sweep offsets
    step_dev[2] = 0;     // list cursor of the replays
}

// Executed-sweep lists of a walk segment (run collapsing, host side): sweep i
// of the segment is executed unless sweep i+1 of the same walk has the same
// colour (color_entry's comment explains why that is exact).  Entry = i | colour << 31.
static int build_lists(tsb_domino *h, int n, uint64_t seg_step, uint64_t len, bool walk_end, uint32_t *list,
                       int *cnt) {
    const size_t pitch = h->xpitch;
    auto one = [&](int z) {
        const uint64_t g = h->gkeys[z];
        uint32_t *o = list + (size_t)z * pitch;
        int m = 0;
        int col = (int)(mix64(g + (seg_step + 1ull) * kGold) >> 63);
        for (uint64_t i = 0; i < len; ++i) {
            const bool last = i + 1 == len;
            const int nxt = (last && walk_end) ? -1 : (int)(mix64(g + (seg_step + i + 2ull) * kGold) >> 63);
            if (nxt != col) o[m++] = (uint32_t)i | ((uint32_t)col << 31);
            col = nxt;
        }
        cnt[z] = m;
    };
    host_parallel_for(n, [&](int z) {
        if (h->coupled && (z & 1)) return;  // CFTP pairs share their seeds: the pair's second list is a copy
        one(z);
    });
    if (h->coupled)
        for (int z = 1; z < n; z += 2) {
            std::memcpy(list + (size_t)z * pitch, list + (size_t)(z - 1) * pitch, sizeof(uint32_t) * cnt[z - 1]);
            cnt[z] = cnt[z - 1];
        }
    return TSB_OK;
}

constexpr uint64_t kSegSweeps = 16384;  // raw sweeps per list segment

static int xlist_alloc(tsb_domino *h) {
    if (h->xlist) return TSB_OK;
    h->xpitch = kSegSweeps;
    const size_t entries = (size_t)h->nchains * h->xpitch;
    TSB_CUDA(cudaMalloc(&h->xlist, sizeof(uint32_t) * entries));
    TSB_CUDA(cudaMalloc(&h->xcnt, sizeof(int) * h->nchains));
    for (int i = 0; i < 2; ++i) {
        TSB_CUDA(cudaMallocHost(&h->xpin[i], sizeof(uint32_t) * entries + sizeof(int) * h->nchains));
        TSB_CUDA(cudaEventCreateWithFlags(&h->xev[i], cudaEventDisableTiming));
        TSB_CUDA(cudaEventRecord(h->xev[i], h->stream));
    }
    return TSB_OK;
}

// Run-collapsed walk: per segment, the executed sweeps of every chain are
// listed on the host and uploaded; graph replays then sweep kGraphSweeps
// listed sweeps each (two per multi-sweep launch) and the remainder runs as
// direct launches.  A launch past a chain's list copies its tiles, so every
// chain ends each segment in the canonical buffer.
static int walk_compact(tsb_domino *h, int chain0, int n, uint64_t step0, uint64_t n_steps) {
    int rc = xlist_alloc(h);
    if (rc) return rc;
    const int cur0 = h->cur;
    for (uint64_t seg = 0; seg < n_steps; seg += kSegSweeps) {
        const uint64_t len = std::min<uint64_t>(kSegSweeps, n_steps - seg);
        const int slot = h->xslot;
        h->xslot ^= 1;
        TSB_CUDA(cudaEventSynchronize(h->xev[slot]));  // the slot's previous upload has been consumed
        uint32_t *list = h->xpin[slot];
        int *cnt = reinterpret_cast<int *>(list + (size_t)h->nchains * h->xpitch);
        if ((rc = build_lists(h, n, step0 + seg, len, seg + len == n_steps, list, cnt))) return rc;
        int maxe = 0;
        for (int z = 0; z < n; ++z) maxe = std::max(maxe, cnt[z]);
        TSB_CUDA(cudaMemcpy2DAsync(h->xlist, sizeof(uint32_t) * h->xpitch, list, sizeof(uint32_t) * h->xpitch,
                                   sizeof(uint32_t) * std::max(1, maxe), n, cudaMemcpyHostToDevice, h->stream));
        TSB_CUDA(cudaMemcpyAsync(h->xcnt, cnt, sizeof(int) * n, cudaMemcpyHostToDevice, h->stream));
        TSB_CUDA(cudaEventRecord(h->xev[slot], h->stream));
        set_segment_kernel<<<1, 1, 0, h->stream>>>(h->step_dev, step0 + seg);
        TSB_CUDA(cudaGetLastError());
        const int replays = maxe / kGraphSweeps;
        if (replays) {
            if ((rc = ensure_graph(h, chain0, n, true))) return rc;
            for (int r = 0; r < replays; ++r) TSB_CUDA(cudaGraphLaunch(h->graph_exec, h->stream));
        }
        int launches = (maxe - replays * kGraphSweeps + kMK - 1) / kMK;
        launches += launches & 1;  // even: the chains end where they started
        for (int i = 0; i < launches; ++i)
            if ((rc = launch_multi(h, chain0, n, (uint64_t)(i * kMK), h->stream, true))) return rc;
    }
    return settle(h, chain0, n, cur0);
}

int tsb::walk_steps(tsb_domino *h, int chain0, int n, uint64_t step0, uint64_t n_steps) {
    int rc;
    const int cur0 = h->cur;
    uint64_t s = 0;
    if (n_steps >= 2) {
        if (const size_t smem = resident_smem(h, n)) return launch_resident(h, chain0, n, step0, n_steps, smem);
    }
    if (h->collapse && !h->strip && n_steps >= 2 && (int)h->gkeys.size() >= n)
        return walk_compact(h, chain0, n, step0, n_steps);
    if (n_steps >= kGraphSweeps) {
        if ((rc = ensure_graph(h, chain0, n, false))) return rc;
        set_walk_kernel<<<n, kGraphSweeps, 0, h->stream>>>(h->step_dev, step0, step0 + n_steps, h->seedinfo,
                                                         h->colors, h->collapse);
        TSB_CUDA(cudaGetLastError());
        for (; s + kGraphSweeps <= n_steps; s += kGraphSweeps) TSB_CUDA(cudaGraphLaunch(h->graph_exec, h->stream));
    }
    if (n_steps - s >= (uint64_t)kMK) {  // remainder: direct multi-sweep launches (step_dev = step0 + s)
        // after replays the last replay's tail wrote this table
        if (s == 0)
            set_walk_kernel<<<n, kGraphSweeps, 0, h->stream>>>(h->step_dev, step0, step0 + n_steps, h->seedinfo,
                                                             h->colors, h->collapse);
        TSB_CUDA(cudaGetLastError());
        for (uint64_t i = 0; s + kMK <= n_steps; s += kMK, i += kMK)
            if ((rc = launch_multi(h, chain0, n, i, h->stream, false))) return rc;
    }
    for (; s < n_steps; ++s)
        if ((rc = launch_sweep(h, chain0, n, step0 + s, -1, h->stream, nullptr))) return rc;
    return settle(h, chain0, n, cur0);
}

extern "C" {

int tsb_domino_sweep(tsb_domino *h, int chain0, int n, const uint64_t *seeds, uint64_t step, int color) {
    int rc = check_range(h, chain0, n);
    if (rc || n == 0) return rc;
    if (color != 0 && color != 1) return fail(TSB_E_VALUE, "colour must be 0 (BLACK) or 1 (WHITE)");
    TSB_CUDA(cudaSetDevice(h->device));
    if ((rc = push_seeds(h, n, seeds))) return rc;
    const int cur0 = h->cur;
    if ((rc = launch_sweep(h, chain0, n, step, color, h->stream, nullptr))) return rc;
    return settle(h, chain0, n, cur0);
}

int tsb_domino_set_window(tsb_domino *h, int row_lo, int row_hi) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    if (row_hi < 0) row_hi = h->side;
    row_lo = std::max(0, row_lo);
    row_hi = std::min(h->side, row_hi);
    if (row_hi <= row_lo) {
        h->win_t0 = h->win_tn = h->win_m0 = h->win_mn = 0;
        h->win_rows = 0;
        return TSB_OK;
    }
    h->win_rows = row_hi - row_lo;
    int y0 = row_lo / kTileRows, y1 = (row_hi - 1) / kTileRows;
    h->win_t0 = h->band_start[y0];
    h->win_tn = h->band_start[y1 + 1] - h->win_t0;
    y0 = row_lo / kMOut;
    y1 = (row_hi - 1) / kMOut;
    h->win_m0 = h->mband_start[y0];
    h->win_mn = h->mband_start[y1 + 1] - h->win_m0;
    if (h->m_order && h->win_mn > 0) {  // the window's adaptive order starts band-major
        TSB_CUDA(cudaSetDevice(h->device));
        order_reset_kernel<<<(h->win_mn + 255) / 256, 256, 0, h->stream>>>(h->mtiles + h->win_m0, h->win_mn,
                                                                            h->m_order + h->win_m0,
                                                                            h->m_perm + h->win_m0, h->m_cost + h->win_m0);
        TSB_CUDA(cudaGetLastError());
    }
    return TSB_OK;
}

static int row_copy(tsb_domino *h, int chain, int r0, int nrows, void *dev, bool get) {
    if (!h || !dev) return fail(TSB_E_VALUE, "null argument");
    if (chain < 0 || chain >= h->nchains || r0 < -1 || nrows < 0 || r0 + nrows > h->side + 1)
        return fail(TSB_E_VALUE, "rows [%d, %d) of chain %d out of range", r0, r0 + nrows, chain);
    TSB_CUDA(cudaSetDevice(h->device));
    uint2 *base = h->buf[h->cur] + (size_t)chain * h->chain_stride + (size_t)(r0 + 1) * h->pitch;
    const size_t bytes = sizeof(uint2) * (size_t)nrows * h->pitch;
    TSB_CUDA(cudaMemcpyAsync(get ? dev : (void *)base, get ? (const void *)base : dev, bytes, cudaMemcpyDeviceToDevice,
                             h->stream));
    return TSB_OK;
}

int tsb_domino_row_bytes(tsb_domino *h, int64_t *bytes) {
    if (!h || !bytes) return fail(TSB_E_VALUE, "null argument");
    *bytes = (int64_t)sizeof(uint2) * h->pitch;
    return TSB_OK;
}

int tsb_domino_set_collapse(tsb_domino *h, int on) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    h->collapse = on ? 1 : 0;
    return TSB_OK;
}

int tsb_domino_get_rows(tsb_domino *h, int chain, int r0, int nrows, void *dev_dst) {
    return row_copy(h, chain, r0, nrows, dev_dst, true);
}

int tsb_domino_set_rows(tsb_domino *h, int chain, int r0, int nrows, const void *dev_src) {
    return row_copy(h, chain, r0, nrows, const_cast<void *>(dev_src), false);
}

#ifdef TSB_TIMING
int tsb_debug_timing(unsigned long long *out) {
    TSB_CUDA(cudaDeviceSynchronize());
    TSB_CUDA(cudaMemcpyFromSymbol(out, g_tt, sizeof(g_tt)));
    return TSB_OK;
}
#endif

int tsb_domino_sync(tsb_domino *h) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    TSB_CUDA(cudaSetDevice(h->device));
    TSB_CUDA(cudaStreamSynchronize(h->stream));
    return TSB_OK;
}

int tsb_domino_walk_host(int device, uint8_t *states, int nchains, int side, const uint64_t *seeds,
                         const double *p_up, const uint8_t *faces, uint64_t n_steps) {
    tsb_domino *h = nullptr;
    int rc = tsb_domino_create(device, side, nchains, faces, &h);
    if (rc) return rc;
    if (!rc && p_up) rc = tsb_domino_set_p_up(h, p_up);
    if (!rc) rc = tsb_domino_upload(h, 0, nchains, states);
    if (!rc) rc = tsb_domino_walk(h, 0, nchains, seeds, 0, n_steps);
    if (!rc) rc = tsb_domino_download(h, 0, nchains, states);
    tsb_domino_destroy(h);
    return rc;
}

}  // extern "C"
