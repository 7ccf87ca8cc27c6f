// Lozenge tilings of triangular-lattice domains: three edge bit-planes,
// 3-colour Glauber sweep, heights, Thurston extremal tilings, CFTP.
//
// Reference (relative to /root/reference/pkg/src/tilesampler/):
//   lozenge.py:43-141    DIRS, _STEPS, _edge_at, ROT_HIGH / ROT_LOW
//   lozenge.py:285-330   LozengeTiling.edges (3, sx+1, sy+1) bool
//   lozenge.py:414-447   loz_heights;  453-622 states_grid_batch, _apply_fire,
//                        loz_sweep_batch, loz_random_walk_batch
//   lozenge.py:674-775   _loz_relax, _tiling_from_loz_heights, loz_extremal; 778-827 loz_cftp
//
// State: planes A, B, C over the (X = sx+1) x (Y = sy+1) vertex grid, row x,
// 32 columns y per word.  The 6-bit state of vertex (x,y) is
//   d0 = A[x]y, d1 = B[x]y, d2 = C[x-1]y+1, d3 = A[x-1]y, d4 = B[x]y-1, d5 = C[x]y.
// ROT_LOW = {d1,d3,d5}, ROT_HIGH = {d0,d2,d4}; a rotation of either toggles all
// six star edges (ROT_HIGH ^ ROT_LOW == 63).  Class (x - y) mod 3 is chosen by
// min(int(u*3), 2) of the global draw.  Same-class stars are disjoint, so a
// sweep is a pure function of the previous state, applied in pull form:
//   A[x] ^= F[x] ^ F[x+1];  B[x] ^= F[x] ^ F[x] >> 1;  C[x] ^= F[x] ^ F[x+1] << 1.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <vector>

#include "tsb_fire.cuh"

namespace tsb {
constexpr int kLzRows = 15;   // output rows per tile (+1 halo fire row)
constexpr int kLzWords = 62;  // output words per tile
constexpr int kLzGraph = 128;  // sweeps per CUDA graph
constexpr int kLzMRows = 16;  // rows per temporally blocked tile (warps per block)
constexpr size_t kLzMSmem = sizeof(uint4) * kLzMRows * 32 + sizeof(uint2) * kLzMRows * 32 +
                            sizeof(uint32_t) * kLzMRows * 64 + sizeof(uint16_t) * kLzMRows * 1024;
}  // namespace tsb

struct tsb_loz {
    int device = 0, sx = 0, sy = 0, X = 0, Y = 0, nchains = 0, W = 0, pitch = 0;
    int m_sms = 148, m_dense = -1;  // SM count; 3-blocks-per-SM kernel: -1 auto (multi-wave batches), 0/1 (TSB_LZ_DENSE)
    size_t plane = 0;        // u32 per plane (incl. guard rows)
    size_t chain_words = 0;  // 3 planes
    uint32_t *buf[2] = {nullptr, nullptr};
    int cur = 0;
    uint32_t *dom = nullptr;  // 6 planes (X rows x pitch): crA crB crC exA exB exC
    uint8_t *tri = nullptr;   // up / down triangle grids (2, sx, sy)
    int2 *range = nullptr;
    int2 *tiles = nullptr;
    int ntiles = 0;
    int tmode = 0;
    uint64_t t0 = 1ull << 52;
    uint64_t *tgrid = nullptr;
    uint64_t *seedinfo = nullptr;
    uint64_t *seed_pinned = nullptr;
    cudaEvent_t seed_ev = nullptr;
    uint8_t *bytes = nullptr;
    size_t bytes_cap = 0;
    int *flag = nullptr;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    uint64_t *step_dev = nullptr;
    cudaStream_t cap_stream = nullptr;
    cudaGraphExec_t graph_exec = nullptr;
    int g_chain0 = -1, g_n = -1, g_cur = -1, g_tmode = -1;
    uint64_t g_t0 = 0;
    int2 *mtiles = nullptr;  // tiles of the temporally blocked kernel (m_out-row bands)
    int nmtiles = 0;
    int m_K = 4, m_out = 8;
    int collapse = 1, g_collapse = -1;  // run collapsing (TSB_LZ_COLLAPSE, tsb_loz_set_collapse)
    // height export scratch, allocated on first use (no cudaMalloc per call)
    int *hx_h = nullptr, *hx_flags = nullptr, *hx_off = nullptr;
    int4 *hx_rows = nullptr;
    int hx_scan = -1, hx_r0 = 0, hx_r1 = -1;  // row-scan classification (-1: not yet)
};

namespace tsb {

struct LzCtx {
    const uint32_t *src;
    uint32_t *dst;
    const int2 *range;
    const int2 *tiles;
    const uint64_t *seedinfo;
    const uint64_t *tgrid;
    const uint64_t *step_dev;
    uint64_t t0;
    size_t plane, chain_words;
    int X, Y, W, pitch;
    uint64_t step;
    int class_override;
};

// bits b of a word with b == k (mod 3)
__device__ __forceinline__ uint32_t mod3_mask(int k) {
    return k == 0 ? 0x49249249u : (k == 1 ? 0x92492492u : 0x24924924u);
}

template <int TM>
__device__ __noinline__ uint32_t lz_rng(uint32_t rot, uint32_t low, uint64_t row_idx, int w, uint64_t base,
                                        uint64_t salt, uint64_t t, const uint64_t *__restrict__ tgrid) {
    uint32_t fire = 0;
    do {
        const int b = __ffs(rot) - 1;
        rot &= rot - 1;
        const uint64_t idx = row_idx + (uint64_t)(w * 32 + b);  // x * Y + y
        const uint64_t x = mix64(mix64(base + (idx + 1ull) * kGold) + salt);
        const uint64_t tt = TM == 2 ? __ldg(tgrid + idx) : t;
        const bool go_high = (x >> 11) < tt;
        // fire_high: class & u < p & state == ROT_LOW; fire_low: u >= p & ROT_HIGH
        if (go_high == (bool)((low >> b) & 1u)) fire |= 1u << b;
    } while (rot);
    return fire;
}

struct Words2 {
    uint32_t a, b;
};

__device__ __forceinline__ Words2 ld2(const uint32_t *row, int wa, bool ina, bool inb) {
    Words2 r{0u, 0u};
    if (ina && inb) {
        const uint2 q = __ldg(reinterpret_cast<const uint2 *>(row + wa));
        r.a = q.x;
        r.b = q.y;
    } else {
        if (ina) r.a = __ldg(row + wa);
        if (inb) r.b = __ldg(row + wa + 1);
    }
    return r;
}

// Same tile scheme as the domino kernel: warp k owns row x0+k, lane owns
// words (wa, wa+1), lanes 0/31 hold one halo word each.
template <int TM>
__global__ void __launch_bounds__(32 * (kLzRows + 1)) loz_sweep_kernel(LzCtx c) {
    __shared__ uint2 fs[kLzRows + 1][32];
    const int lane = threadIdx.x & 31;
    const int k = threadIdx.x >> 5;
    const int2 tile = c.tiles[blockIdx.x];
    const int x = tile.y * kLzRows + k;
    const int wout0 = tile.x * kLzWords - 1;
    const int wa = wout0 - 1 + 2 * lane, wb = wa + 1;
    const int z = blockIdx.z;
    const uint32_t *src = c.src + (size_t)z * c.chain_words + c.pitch;  // row 0 of plane A
    const uint64_t step = c.step + (c.step_dev ? *c.step_dev : 0ull);
    const uint64_t salt = (step + 1ull) * kGold;
    const uint64_t base = c.seedinfo[2 * z];
    int cls = c.class_override;
    if (cls < 0) {
        const double coin = (double)(mix64(c.seedinfo[2 * z + 1] + salt) >> 11) * 0x1p-53;
        cls = min((int)__dmul_rn(coin, 3.0), 2);  // min(int(coin * 3), 2)
    }
    const bool live = x < c.X;
    const int2 g = live ? __ldg(c.range + x) : make_int2(0, 0);
    const int2 gm = (live && x > 0) ? __ldg(c.range + x - 1) : make_int2(0, 0);
    const bool ina = wa >= g.x && wa < g.y, inb = wb >= g.x && wb < g.y;
    const bool inma = wa >= gm.x && wa < gm.y, inmb = wb >= gm.x && wb < gm.y;
    const uint32_t *rA = src + (ptrdiff_t)x * c.pitch;
    const uint32_t *rB = rA + c.plane, *rC = rB + c.plane;
    const Words2 A = ld2(rA, wa, ina, inb), B = ld2(rB, wa, ina, inb), C = ld2(rC, wa, ina, inb);
    const Words2 Am = ld2(rA - c.pitch, wa, inma, inmb), Cm = ld2(rC - c.pitch, wa, inma, inmb);
    // neighbour words: B[x] of word wa-1 (lane-1's b), C[x-1] of word wb+1 (lane+1's a)
    const uint32_t bprev = __shfl_up_sync(0xffffffffu, B.b, 1);
    const uint32_t cmnext = __shfl_down_sync(0xffffffffu, Cm.a, 1);
    // d2 = C[x-1] >> 1 (carry bit 0 of the next word), d4 = B[x] << 1 (carry bit 31 of the previous)
    const uint32_t d2a = (Cm.a >> 1) | (Cm.b << 31), d2b = (Cm.b >> 1) | (cmnext << 31);
    const uint32_t d4a = (B.a << 1) | (bprev >> 31), d4b = (B.b << 1) | (B.a >> 31);
    const uint32_t lowa = B.a & Am.a & C.a & ~A.a & ~d2a & ~d4a, lowb = B.b & Am.b & C.b & ~A.b & ~d2b & ~d4b;
    const uint32_t higha = A.a & d2a & d4a & ~B.a & ~Am.a & ~C.a, highb = A.b & d2b & d4b & ~B.b & ~Am.b & ~C.b;
    // class columns: y == x - cls (mod 3); y = 32w + b, 32 == 2 (mod 3)
    const int ra = (((x - cls - 2 * wa) % 3) + 3) % 3, rb = (((x - cls - 2 * wb) % 3) + 3) % 3;
    // lane 0's first word: only bit 31 feeds an output (C carry); lane 31's
    // second word: only bit 0 feeds an output (B carry).
    const uint32_t acta = mod3_mask(ra) & (lane == 0 ? 0x80000000u : 0xFFFFFFFFu);
    const uint32_t actb = mod3_mask(rb) & (lane == 31 ? 1u : 0xFFFFFFFFu);
    const uint64_t ridx = (uint64_t)x * (uint64_t)c.Y;
    const uint32_t rota = (lowa | higha) & acta, rotb = (lowb | highb) & actb;
    const uint32_t fa = rota ? lz_rng<TM>(rota, lowa, ridx, wa, base, salt, c.t0, c.tgrid) : 0u;
    const uint32_t fb = rotb ? lz_rng<TM>(rotb, lowb, ridx, wb, base, salt, c.t0, c.tgrid) : 0u;
    fs[k][lane] = make_uint2(fa, fb);
    __syncthreads();
    if (k == kLzRows || !live) return;
    const uint2 fn = fs[k + 1][lane];                                  // F[x+1]
    const uint32_t fnprev = __shfl_up_sync(0xffffffffu, fn.y, 1);       // F[x+1] of word wa-1
    const uint32_t fnext = __shfl_down_sync(0xffffffffu, fa, 1);        // F[x] of word wb+1
    const uint32_t nAa = A.a ^ fa ^ fn.x, nAb = A.b ^ fb ^ fn.y;
    const uint32_t nBa = B.a ^ fa ^ ((fa >> 1) | (fb << 31)), nBb = B.b ^ fb ^ ((fb >> 1) | (fnext << 31));
    const uint32_t nCa = C.a ^ fa ^ ((fn.x << 1) | (fnprev >> 31)), nCb = C.b ^ fb ^ ((fn.y << 1) | (fn.x >> 31));
    uint32_t *oA = c.dst + (size_t)z * c.chain_words + c.pitch + (ptrdiff_t)x * c.pitch;
    uint32_t *oB = oA + c.plane, *oC = oB + c.plane;
    const bool sa = lane > 0 && ina, sb = lane < 31 && inb;
    if (sa && sb) {
        *reinterpret_cast<uint2 *>(oA + wa) = make_uint2(nAa, nAb);
        *reinterpret_cast<uint2 *>(oB + wa) = make_uint2(nBa, nBb);
        *reinterpret_cast<uint2 *>(oC + wa) = make_uint2(nCa, nCb);
    } else {
        if (sa) { oA[wa] = nAa; oB[wa] = nBa; oC[wa] = nCa; }
        if (sb) { oA[wb] = nAb; oB[wb] = nBb; oC[wb] = nCb; }
    }
}

struct LzMCtx {
    const uint32_t *src;  // chain 0, plane A, row 0
    uint32_t *dst;
    const int2 *tiles;
    const uint64_t *seedinfo;
    const uint64_t *tgrid;
    const uint64_t *step_dev;
    uint64_t t0;
    size_t plane, chain_words;
    int X, Y, W, pitch;
    int K, out_rows;
    uint64_t step;  // offset of this launch inside the graph replay
    int collapse;   // skip sweeps followed by a sweep of the same class
};

// Temporal blocking: K sweeps per launch (graph replays), the domino
// multi-sweep scheme on three planes.  Warp k owns row x0 - K + k, lane owns
// words (wa, wa+1) of A, B and C in registers; per sweep the A/C words go to
// shared memory for the row below (d2, d3), the fire words for the row above
// (pull-form updates).  Rows / bits next to the unloaded outside go stale by
// one per sweep, so the central kLzMRows - 2K rows and the 62 interior words
// are exact and are the only ones stored.  Coins exactly as loz_sweep_kernel.
template <int TM, int MINB = 2>
__global__ void __launch_bounds__(32 * kLzMRows, MINB) lz_multi_kernel(LzMCtx c) {
    extern __shared__ __align__(16) unsigned char dsm[];
    uint4(*acs)[32] = reinterpret_cast<uint4(*)[32]>(dsm);
    uint2(*fs)[32] = reinterpret_cast<uint2(*)[32]>(dsm + sizeof(uint4) * kLzMRows * 32);
    uint32_t(*fres)[64] =
        reinterpret_cast<uint32_t(*)[64]>(dsm + sizeof(uint4) * kLzMRows * 32 + sizeof(uint2) * kLzMRows * 32);
    uint16_t(*queue)[1024] = reinterpret_cast<uint16_t(*)[1024]>(
        dsm + sizeof(uint4) * kLzMRows * 32 + sizeof(uint2) * kLzMRows * 32 + sizeof(uint32_t) * kLzMRows * 64);
    const int lane = threadIdx.x & 31;
    const int k = threadIdx.x >> 5;
    const int2 tile = c.tiles[blockIdx.x];
    const int x = tile.y * c.out_rows - c.K + k;
    const int wa = tile.x + 2 * lane, wb = wa + 1;  // band-aligned tile: tile.x = first loaded word (even)
    // a halo word whose outer neighbour lies beyond the grid reads the true
    // (zero) neighbour and stays exact: a tile starting at word 0 also owns
    // word 0, one reaching the grid's last word also owns word tile.x + 63
    const bool lclosed = tile.x == 0, rclosed = tile.x + 63 >= c.W - 1;
    const int z = blockIdx.z;
    const uint64_t gkey = c.seedinfo[2 * z + 1];
    const bool in_grid = x >= 0 && x < c.X;
    const bool ina = in_grid && wa >= 0 && wa < c.pitch, inb = in_grid && wb >= 0 && wb < c.pitch;
    // class residues: y = 32w + b == x - cls (mod 3), 32 == 2 (mod 3)
    const int b3a = (((x - 2 * wa) % 3) + 3) % 3, b3b = (((x - 2 * wb) % 3) + 3) % 3;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint32_t *rA = c.src + (size_t)z * c.chain_words + (ptrdiff_t)x * c.pitch;
    const uint32_t *rB = rA + c.plane, *rC = rB + c.plane;
    Words2 A = ld2(rA, wa, ina, inb), B = ld2(rB, wa, ina, inb), C = ld2(rC, wa, ina, inb);
    const uint64_t step0 = c.step_dev[0] + c.step, walk_end = c.step_dev[1];
    int mycls;
    {
        const double coin = (double)(mix64(gkey + (step0 + (uint64_t)lane + 1ull) * kGold) >> 11) * 0x1p-53;
        mycls = min((int)__dmul_rn(coin, 3.0), 2);  // min(int(coin * 3), 2)
    }
#pragma unroll 1
    for (int s = 0; s < c.K; ++s) {
        const int cls = __shfl_sync(0xffffffffu, mycls, s);
        // run collapsing: heat-bath move (a rotateable star ends high iff
        // u < p, lozenge.py:575-597) and same-class stars are disjoint, so
        // within a run of one class only its last sweep decides
        if (c.collapse && step0 + (uint64_t)s + 1ull < walk_end && __shfl_sync(0xffffffffu, mycls, s + 1) == cls)
            continue;
        acs[k][lane] = make_uint4(A.a, A.b, C.a, C.b);
        __syncthreads();
        const uint4 m = k > 0 ? acs[k - 1][lane] : make_uint4(0u, 0u, 0u, 0u);  // A, C of row x-1
        uint32_t bprev = __shfl_up_sync(0xffffffffu, B.b, 1);
        uint32_t cmnext = __shfl_down_sync(0xffffffffu, m.z, 1);
        if (lane == 0) bprev = 0u;
        if (lane == 31) cmnext = 0u;
        const uint32_t d2a = (m.z >> 1) | (m.w << 31), d2b = (m.w >> 1) | (cmnext << 31);
        const uint32_t d4a = (B.a << 1) | (bprev >> 31), d4b = (B.b << 1) | (B.a >> 31);
        // a rotateable star has (B, C, row-above A) all set and (A, d2, d4) all
        // clear (low) or the reverse (high): the six bits agree once A, d2
        // and d4 are inverted; low = rotateable with B set
        const uint32_t stara = ~((B.a ^ m.x) | (B.a ^ C.a) | (B.a ^ ~A.a) | (B.a ^ ~d2a) | (B.a ^ ~d4a));
        const uint32_t starb = ~((B.b ^ m.y) | (B.b ^ C.b) | (B.b ^ ~A.b) | (B.b ^ ~d2b) | (B.b ^ ~d4b));
        const uint32_t lowa = stara & B.a, lowb = starb & B.b;
        // coins that cannot reach a stored bit are not drawn (as the domino
        // tiles): fire row x touches rows x-1 and x, so sweep s needs fire rows
        // s+1 .. kLzMRows-1-s, and a fire moves about one column per sweep, so
        // the halo words (lane 0 word a, lane 31 word b) need only the bits
        // within K-s (+1) columns of the interior
        const bool need = k >= s + 1 && k <= kLzMRows - 1 - s;
        const int reach = c.K - s;
        // (a tile side closed by the grid edge has no stale halo: all its bits count)
        const uint32_t hl = lane == 0 && !lclosed ? (reach >= 32 ? ~0u : ~0u << (32 - reach)) : ~0u;
        const uint32_t hr = lane == 31 && !rclosed ? (reach >= 31 ? ~0u : (1u << (reach + 1)) - 1u) : ~0u;
        // bits b == k (mod 3) of a word: 0x49249249 << k (k = 0, 1, 2)
        int ka = b3a - cls, kb = b3b - cls;
        ka += ka < 0 ? 3 : 0;
        kb += kb < 0 ? 3 : 0;
        const uint32_t rota = need ? stara & (0x49249249u << ka) & hl : 0u;
        const uint32_t rotb = need ? starb & (0x49249249u << kb) & hr : 0u;
        uint2 f = make_uint2(0u, 0u);
        if (__any_sync(0xffffffffu, (rota | rotb) != 0u))
            f = warp_fire_body<TM>(rota, rotb, lowa, lowb, queue[k], fres[k], c.seedinfo, c.tgrid, c.t0, c.Y, z, x, wa,
                              step0 + (uint64_t)s);
        fs[k][lane] = f;
        __syncthreads();
        const uint2 fn = k + 1 < kLzMRows ? fs[k + 1][lane] : make_uint2(0u, 0u);  // F[x+1]
        uint32_t fnprev = __shfl_up_sync(0xffffffffu, fn.y, 1);
        uint32_t fnext = __shfl_down_sync(0xffffffffu, f.x, 1);
        if (lane == 0) fnprev = 0u;
        if (lane == 31) fnext = 0u;
        if (in_grid) {
            A.a ^= f.x ^ fn.x;
            A.b ^= f.y ^ fn.y;
            B.a ^= f.x ^ ((f.x >> 1) | (f.y << 31));
            B.b ^= f.y ^ ((f.y >> 1) | (fnext << 31));
            C.a ^= f.x ^ ((fn.x << 1) | (fnprev >> 31));
            C.b ^= f.y ^ ((fn.y << 1) | (fn.x >> 31));
        }
    }
    if (k >= c.K && k < kLzMRows - c.K && in_grid) {  // warp-uniform
        uint32_t *oA = c.dst + (size_t)z * c.chain_words + (ptrdiff_t)x * c.pitch;
        uint32_t *oB = oA + c.plane, *oC = oB + c.plane;
        const bool sa = (lane > 0 || lclosed) && wa >= 0 && wa < c.W, sb = (lane < 31 || rclosed) && wb >= 0 && wb < c.W;
        if (sa && sb) {
            *reinterpret_cast<uint2 *>(oA + wa) = make_uint2(A.a, A.b);
            *reinterpret_cast<uint2 *>(oB + wa) = make_uint2(B.a, B.b);
            *reinterpret_cast<uint2 *>(oC + wa) = make_uint2(C.a, C.b);
        } else {
            if (sa) { oA[wa] = A.a; oB[wa] = B.a; oC[wa] = C.a; }
            if (sb) { oA[wb] = A.b; oB[wb] = B.b; oC[wb] = C.b; }
        }
    }
}

__global__ void lz_set_step(uint64_t *p, uint64_t v, uint64_t end) {  // p[0] = step, p[1] = end of the walk
    p[0] = v;
    p[1] = end;
}
__global__ void lz_advance_step(uint64_t *p, uint64_t by) { *p += by; }

__device__ __forceinline__ bool tri_in(const uint8_t *t, int sx, int sy, int x, int y) {
    return x >= 0 && y >= 0 && x < sx && y < sy && t[(size_t)x * sy + y] != 0;
}

// crossable / existing edge planes, vertex mask ranges (lozenge.py:73-82, 674-692)
__global__ void lz_domain_kernel(const uint8_t *tri, int sx, int sy, int X, int Y, int W, int pitch, uint32_t *dom,
                                 int2 *range) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    const int x = blockIdx.y;
    if (w >= W) return;
    const uint8_t *up = tri, *dn = tri + (size_t)sx * sy;
    uint32_t cr[3] = {0, 0, 0}, ex[3] = {0, 0, 0};
    bool any = false;
    for (int b = 0; b < 32; ++b) {
        const int y = w * 32 + b;
        if (y >= Y) break;
        // a[x,y]: up(x,y) | down(x,y-1);  b[x,y]: up(x,y) | down(x-1,y);  c[x,y]: up(x,y-1) | down(x,y-1)
        const bool u0 = tri_in(up, sx, sy, x, y), ua = tri_in(dn, sx, sy, x, y - 1);
        const bool ub = tri_in(dn, sx, sy, x - 1, y), uc = tri_in(up, sx, sy, x, y - 1);
        const bool pa[3][2] = {{u0, ua}, {u0, ub}, {uc, ua}};
        for (int e = 0; e < 3; ++e) {
            if (pa[e][0] && pa[e][1]) cr[e] |= 1u << b;
            if (pa[e][0] || pa[e][1]) ex[e] |= 1u << b;
        }
        // vertex mask: corner of an up triangle (x,y),(x-1,y),(x,y-1) or of a
        // down triangle (x-1,y),(x,y-1),(x-1,y-1)
        if (tri_in(up, sx, sy, x, y) || tri_in(up, sx, sy, x - 1, y) || tri_in(up, sx, sy, x, y - 1) ||
            tri_in(dn, sx, sy, x - 1, y) || tri_in(dn, sx, sy, x, y - 1) || tri_in(dn, sx, sy, x - 1, y - 1))
            any = true;
    }
    for (int e = 0; e < 3; ++e) {
        dom[(size_t)e * X * pitch + (size_t)x * pitch + w] = cr[e];
        dom[(size_t)(3 + e) * X * pitch + (size_t)x * pitch + w] = ex[e];
    }
    if (any) {
        atomicMin(&range[x].x, w);
        atomicMax(&range[x].y, w + 1);
    }
}

__global__ void lz_fix_ranges(int2 *range, int X) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x < X && range[x].x >= range[x].y) range[x] = make_int2(0, 0);
}

// edges (n, 3, X, Y) uint8 -> planes; crossed edges must be crossable.
__global__ void lz_pack_kernel(const uint8_t *bytes, int X, int Y, int W, int pitch, size_t plane, size_t chain_words,
                               const uint32_t *dom, uint32_t *state, int *bad) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    const int x = blockIdx.y, z = blockIdx.z;
    if (w >= W) return;
    const uint8_t *g = bytes + (size_t)z * 3 * X * Y;
    int err = 0;
    for (int e = 0; e < 3; ++e) {
        uint32_t word = 0;
        const uint32_t cr = dom[(size_t)e * X * pitch + (size_t)x * pitch + w];
        for (int b = 0; b < 32; ++b) {
            const int y = w * 32 + b;
            if (y >= Y) break;
            const uint8_t v = g[(size_t)e * X * Y + (size_t)x * Y + y];
            if (v > 1) err = 1;
            if (v) {
                word |= 1u << b;
                if (!((cr >> b) & 1u)) err |= 2;
            }
        }
        state[(size_t)z * chain_words + (size_t)e * plane + (size_t)(x + 1) * pitch + w] = word;
    }
    if (err) atomicOr(bad, err);
}

__global__ void lz_unpack_kernel(const uint32_t *state, int X, int Y, int pitch, size_t plane, size_t chain_words,
                                 uint8_t *bytes) {
    const int y = blockIdx.x * blockDim.x + threadIdx.x;
    const int x = blockIdx.y, z = blockIdx.z;
    if (y >= Y) return;
    for (int e = 0; e < 3; ++e) {
        const uint32_t word = state[(size_t)z * chain_words + (size_t)e * plane + (size_t)(x + 1) * pitch + (y >> 5)];
        bytes[(size_t)z * 3 * X * Y + (size_t)e * X * Y + (size_t)x * Y + y] = (word >> (y & 31)) & 1u;
    }
}

// ------------------------------------------------------------ heights, extremal
constexpr int kLzT = 32;
constexpr int kLzInf = 0x3FFFFFFF;
constexpr int8_t kLzNo = 127;

__device__ __forceinline__ bool pbit(const uint32_t *p, int pitch, int x, int y) {
    return (p[(size_t)x * pitch + (y >> 5)] >> (y & 31)) & 1u;
}

// MODE 0: exact steps; 1: upper bounds (h_max, min-relax); 2: lower bounds.
template <int MODE>
__device__ __forceinline__ int8_t lz_w(bool exists, bool crossable, bool crossed, bool even) {
    if (!exists) return kLzNo;
    const int unc = even ? 1 : -1, cr = even ? -2 : 2;  // _STEPS (lozenge.py:47)
    if (MODE == 0) return (int8_t)(crossed ? cr : unc);
    if (MODE == 1) return (int8_t)(crossable ? max(unc, cr) : unc);
    return (int8_t)(crossable ? min(unc, cr) : unc);
}

// incoming neighbours of v = (x, y): u = v - DIRS[k] reaches v in direction k
//   k0 u=(x-1,y) a[x-1,y]  k1 u=(x,y-1) b[x,y-1]  k2 u=(x+1,y-1) c[x,y]
//   k3 u=(x+1,y) a[x,y]    k4 u=(x,y+1) b[x,y]    k5 u=(x-1,y+1) c[x-1,y+1]
template <int MODE>
__global__ void __launch_bounds__(256) lz_relax_kernel(int *h, const uint32_t *st, size_t plane, const uint32_t *dom,
                                                       int X, int Y, int pitch, int limit, int *flags) {
    __shared__ int s[kLzT + 2][kLzT + 2];
    __shared__ int8_t wt[6][kLzT][kLzT];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int y0 = blockIdx.x * kLzT, x0 = blockIdx.y * kLzT;
    const int sentinel = MODE == 2 ? -kLzInf : kLzInf;
    for (int i = ty * 32 + tx; i < (kLzT + 2) * (kLzT + 2); i += 256) {
        const int lx = i / (kLzT + 2), ly = i % (kLzT + 2);
        const int x = x0 + lx - 1, y = y0 + ly - 1;
        s[lx][ly] = (x >= 0 && y >= 0 && x < X && y < Y) ? h[(size_t)x * Y + y] : sentinel;
    }
    const size_t dp = (size_t)X * pitch;  // dom plane stride
    const uint32_t *crA = dom, *crB = dom + dp, *crC = dom + 2 * dp, *exA = dom + 3 * dp, *exB = dom + 4 * dp,
                   *exC = dom + 5 * dp;
    const uint32_t *sA = st, *sB = st ? st + plane : nullptr, *sC = st ? st + 2 * plane : nullptr;
    int orig[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int lx = ty + 8 * q, x = x0 + lx, y = y0 + tx;
        int8_t w[6] = {kLzNo, kLzNo, kLzNo, kLzNo, kLzNo, kLzNo};
        if (x < X && y < Y) {
            // each: (plane set, edge x, edge y, even direction)
            const int ex_[6] = {x - 1, x, x, x, x, x - 1};
            const int ey_[6] = {y, y - 1, y, y, y, y + 1};
            const int kind[6] = {0, 1, 2, 0, 1, 2};
            const int ux[6] = {x - 1, x, x + 1, x + 1, x, x - 1};
            const int uy[6] = {y, y - 1, y - 1, y, y + 1, y + 1};
#pragma unroll
            for (int d = 0; d < 6; ++d) {
                if (ux[d] < 0 || uy[d] < 0 || ux[d] >= X || uy[d] >= Y) continue;
                const int xx = ex_[d], yy = ey_[d];
                if (xx < 0 || yy < 0 || xx >= X || yy >= Y) continue;
                const uint32_t *cr = kind[d] == 0 ? crA : (kind[d] == 1 ? crB : crC);
                const uint32_t *exs = kind[d] == 0 ? exA : (kind[d] == 1 ? exB : exC);
                const uint32_t *ss = kind[d] == 0 ? sA : (kind[d] == 1 ? sB : sC);
                const bool crossed = MODE == 0 ? (pbit(ss + pitch, pitch, xx, yy)) : false;
                w[d] = lz_w<MODE>(pbit(exs, pitch, xx, yy), pbit(cr, pitch, xx, yy), crossed, (d & 1) == 0);
            }
        }
#pragma unroll
        for (int d = 0; d < 6; ++d) wt[d][lx][tx] = w[d];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) orig[q] = s[ty + 8 * q + 1][tx + 1];
    // Jacobi rounds (read, barrier, write): race-free, same unique fixpoint
    bool over = false;
    for (int it = 0; it < 4 * kLzT; ++it) {
        bool ch = false;
        int nv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int lx = ty + 8 * q, ly = tx;
            const int cur = s[lx + 1][ly + 1];
            int best = cur;
            const int nb[6] = {s[lx][ly + 1], s[lx + 1][ly], s[lx + 2][ly], s[lx + 2][ly + 1], s[lx + 1][ly + 2],
                               s[lx][ly + 2]};
#pragma unroll
            for (int d = 0; d < 6; ++d) {
                const int8_t w = wt[d][lx][ly];
                if (w == kLzNo || nb[d] == sentinel) continue;
                const int cand = nb[d] + w;
                best = MODE == 2 ? max(best, cand) : min(best, cand);
            }
            if (best != cur && (MODE == 2 ? best > limit : best < -limit)) {
                over = true;
                best = MODE == 2 ? limit : -limit;
            }
            nv[q] = best;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int lx = ty + 8 * q, ly = tx;
            if (nv[q] != s[lx + 1][ly + 1]) {
                s[lx + 1][ly + 1] = nv[q];
                ch = true;
            }
        }
        if (!__syncthreads_or(ch)) break;
    }
    bool changed = false;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int lx = ty + 8 * q, x = x0 + lx, y = y0 + tx;
        const int v = s[lx + 1][tx + 1];
        if (x < X && y < Y && v != orig[q]) {
            h[(size_t)x * Y + y] = v;
            changed = true;
        }
    }
    if (__syncthreads_or(changed) && tx == 0 && ty == 0) atomicExch(flags, 1);
    if (over) atomicExch(flags + 1, 1);
}

__global__ void lz_fill(int *h, size_t n, int v, size_t ref) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n) h[i] = i == ref ? 0 : v;
}

// output heights: 0 outside the vertex mask (any incident existing edge);
// flags[0] set if a mask vertex was never reached.
__global__ void lz_finish(const int *h, const uint32_t *dom, int X, int Y, int pitch, int32_t *out, int sentinel,
                          int *flags) {
    const int y = blockIdx.x * blockDim.x + threadIdx.x;
    const int x = blockIdx.y;
    if (y >= Y) return;
    const size_t dp = (size_t)X * pitch;
    const uint32_t *exA = dom + 3 * dp, *exB = dom + 4 * dp, *exC = dom + 5 * dp;
    bool in = pbit(exA, pitch, x, y) || pbit(exB, pitch, x, y) || pbit(exC, pitch, x, y);
    if (x > 0) in = in || pbit(exA, pitch, x - 1, y);
    if (y > 0) in = in || pbit(exB, pitch, x, y - 1);
    if (x > 0 && y + 1 < Y) in = in || pbit(exC, pitch, x - 1, y + 1);
    const int v = h[(size_t)x * Y + y];
    if (in && v == sentinel) atomicExch(flags, 1);
    out[(size_t)x * Y + y] = in ? v : 0;
}

// extremal heights -> edge planes (_tiling_from_loz_heights, lozenge.py:739-759):
// crossed iff crossable and h(v2) - h(v1) equals the crossed step
// (a: v2 = (x+1,y), -2;  b: v2 = (x,y+1), +2;  c: v2 = (x+1,y-1), +2).
__global__ void lz_decode(const int32_t *hh, const uint32_t *dom, int X, int Y, int W, int pitch, size_t plane,
                          uint32_t *state) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    const int x = blockIdx.y;
    if (w >= W) return;
    const size_t dp = (size_t)X * pitch;
    uint32_t pa = 0, pb = 0, pc = 0;
    for (int b = 0; b < 32; ++b) {
        const int y = w * 32 + b;
        if (y >= Y) break;
        const int h0 = hh[(size_t)x * Y + y];
        if (pbit(dom, pitch, x, y) && x + 1 < X && hh[(size_t)(x + 1) * Y + y] - h0 == -2) pa |= 1u << b;
        if (pbit(dom + dp, pitch, x, y) && y + 1 < Y && hh[(size_t)x * Y + y + 1] - h0 == 2) pb |= 1u << b;
        if (pbit(dom + 2 * dp, pitch, x, y) && x + 1 < X && y > 0 && hh[(size_t)(x + 1) * Y + y - 1] - h0 == 2)
            pc |= 1u << b;
    }
    state[(size_t)(x + 1) * pitch + w] = pa;
    state[plane + (size_t)(x + 1) * pitch + w] = pb;
    state[2 * plane + (size_t)(x + 1) * pitch + w] = pc;
}

// lozenges_from_tiling validation (lozenge.py:356-378): every domain triangle
// is covered exactly once.  up(x,y): a[x,y], b[x,y], c[x,y+1];
// down(x,y): b[x+1,y], a[x,y+1], c[x,y+1].
__global__ void lz_cover_check(const uint8_t *tri, int sx, int sy, const uint32_t *st, int pitch, size_t plane,
                               int *bad) {
    const int y = blockIdx.x * blockDim.x + threadIdx.x;
    const int x = blockIdx.y;
    if (y >= sy) return;
    const uint32_t *A = st + pitch, *B = A + plane, *C = B + plane;  // row 0
    const uint8_t *up = tri, *dn = tri + (size_t)sx * sy;
    if (up[(size_t)x * sy + y]) {
        const int n = pbit(A, pitch, x, y) + pbit(B, pitch, x, y) + pbit(C, pitch, x, y + 1);
        if (n != 1) atomicOr(bad, 1);
    }
    if (dn[(size_t)x * sy + y]) {
        const int n = pbit(B, pitch, x + 1, y) + pbit(A, pitch, x, y + 1) + pbit(C, pitch, x, y + 1);
        if (n != 1) atomicOr(bad, 1);
    }
}

__global__ void lz_replicate(uint4 *base, size_t chain_u4, int src, int dst0, int step, int n) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= chain_u4) return;
    const uint4 v = base[(size_t)src * chain_u4 + i];
    for (int k = 0; k < n; ++k) base[(size_t)(dst0 + (size_t)k * step) * chain_u4 + i] = v;
}

__global__ void __launch_bounds__(256) lz_coalesced(const uint4 *base, size_t chain_u4, int chain0, uint8_t *flags) {
    const int j = blockIdx.x;
    const uint4 *a = base + (size_t)(chain0 + 2 * j) * chain_u4;
    const uint4 *b = a + chain_u4;
    uint32_t diff = 0;
    for (size_t i = threadIdx.x; i < chain_u4; i += blockDim.x) {
        const uint4 p = __ldg(a + i), q = __ldg(b + i);
        diff |= (p.x ^ q.x) | (p.y ^ q.y) | (p.z ^ q.z) | (p.w ^ q.w);
    }
    const int any = __syncthreads_or(diff != 0);
    if (threadIdx.x == 0) flags[j] = any ? 0 : 1;
}

// Archive record (stats.py:146-153): LozengeTiling.edges (3, X, Y) ravelled
// as '0'/'1'; thread per (plane, row, 32-column word).
__global__ void lz_serialize_kernel(const uint32_t *st, int X, int Y, int pitch, size_t plane, char *out) {
    const int e = blockIdx.z, x = blockIdx.y, w = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= X || w * 32 >= Y) return;
    const uint32_t m = st[(size_t)e * plane + (size_t)(x + 1) * pitch + w];
    char *o = out + ((size_t)e * X + x) * Y + (size_t)w * 32;
    const int lim = min(32, Y - w * 32);
    for (int b = 0; b < lim; ++b) o[b] = ((m >> b) & 1u) ? '1' : '0';
}

// ----------------------------------------------------------------- host helpers
int lz_check(tsb_loz *h, int chain0, int n) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    if (chain0 < 0 || n < 0 || chain0 + n > h->nchains)
        return fail(TSB_E_VALUE, "chains [%d, %d) outside the handle's %d chains", chain0, chain0 + n, h->nchains);
    return TSB_OK;
}

int lz_bytes(tsb_loz *h, size_t need) {
    if (h->bytes_cap >= need) return TSB_OK;
    TSB_CUDA(cudaStreamSynchronize(h->stream));
    cudaFree(h->bytes);
    h->bytes = nullptr;
    TSB_CUDA(cudaMalloc(&h->bytes, need));
    h->bytes_cap = need;
    return TSB_OK;
}

int lz_launch(tsb_loz *h, int chain0, int n, uint64_t step, int cls, cudaStream_t stream, const uint64_t *step_dev) {
    LzCtx c;
    c.src = h->buf[h->cur] + (size_t)chain0 * h->chain_words;
    c.dst = h->buf[h->cur ^ 1] + (size_t)chain0 * h->chain_words;
    c.range = h->range;
    c.tiles = h->tiles;
    c.seedinfo = h->seedinfo;
    c.tgrid = h->tgrid;
    c.step_dev = step_dev;
    c.t0 = h->t0;
    c.plane = h->plane;
    c.chain_words = h->chain_words;
    c.X = h->X;
    c.Y = h->Y;
    c.W = h->W;
    c.pitch = h->pitch;
    c.step = step;
    c.class_override = cls;
    h->cur ^= 1;
    if (h->ntiles == 0) return TSB_OK;
    dim3 grid(h->ntiles, 1, n), block(32 * (kLzRows + 1));
    if (h->tmode == 0) loz_sweep_kernel<0><<<grid, block, 0, stream>>>(c);
    else loz_sweep_kernel<2><<<grid, block, 0, stream>>>(c);
    TSB_CUDA(cudaGetLastError());
    return TSB_OK;
}

// One temporally blocked launch (m_K sweeps); graph mode only.
int lz_launch_multi(tsb_loz *h, int chain0, int n, uint64_t step_off, cudaStream_t stream) {
    LzMCtx c;
    c.src = h->buf[h->cur] + (size_t)chain0 * h->chain_words + h->pitch;
    c.dst = h->buf[h->cur ^ 1] + (size_t)chain0 * h->chain_words + h->pitch;
    c.tiles = h->mtiles;
    c.seedinfo = h->seedinfo;
    c.tgrid = h->tgrid;
    c.step_dev = h->step_dev;
    c.t0 = h->t0;
    c.plane = h->plane;
    c.chain_words = h->chain_words;
    c.X = h->X;
    c.Y = h->Y;
    c.W = h->W;
    c.pitch = h->pitch;
    c.K = h->m_K;
    c.collapse = h->collapse;
    c.out_rows = h->m_out;
    c.step = step_off;
    h->cur ^= 1;
    if (h->nmtiles == 0) return TSB_OK;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(h->nmtiles, 1, n);
    cfg.blockDim = dim3(32 * kLzMRows);
    cfg.dynamicSmemBytes = kLzMSmem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // batches of several waves: the 3-blocks-per-SM build (register cap 40)
    const bool dense = h->m_dense >= 0 ? h->m_dense == 1 : (int64_t)h->nmtiles * n > 4 * (int64_t)h->m_sms;
    if (dense) {
        if (h->tmode == 0) TSB_CUDA(cudaLaunchKernelEx(&cfg, lz_multi_kernel<0, 3>, c));
        else TSB_CUDA(cudaLaunchKernelEx(&cfg, lz_multi_kernel<2, 3>, c));
        return TSB_OK;
    }
    if (h->tmode == 0) TSB_CUDA(cudaLaunchKernelEx(&cfg, lz_multi_kernel<0>, c));
    else TSB_CUDA(cudaLaunchKernelEx(&cfg, lz_multi_kernel<2>, c));
    return TSB_OK;
}

int lz_graph(tsb_loz *h, int chain0, int n) {
    if (h->graph_exec && h->g_chain0 == chain0 && h->g_n == n && h->g_cur == h->cur && h->g_tmode == h->tmode &&
        h->g_t0 == h->t0 && h->g_collapse == h->collapse)
        return TSB_OK;
    if (h->graph_exec) {
        cudaGraphExecDestroy(h->graph_exec);
        h->graph_exec = nullptr;
    }
    if (!h->cap_stream) TSB_CUDA(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    TSB_CUDA(cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal));
    int rc = TSB_OK;
    // kLzGraph / m_K launches (even, so the buffers end where they started)
    for (int i = 0; i < kLzGraph / h->m_K && !rc; ++i)
        rc = lz_launch_multi(h, chain0, n, (uint64_t)i * h->m_K, h->cap_stream);
    lz_advance_step<<<1, 1, 0, h->cap_stream>>>(h->step_dev, (uint64_t)kLzGraph);
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
    h->g_collapse = h->collapse;
    return TSB_OK;
}

// After a walk the walked chains live in buf[cur]; when that is not the
// buffer the other chains live in (cur0), copy them back.
int lz_settle(tsb_loz *h, int chain0, int n, int cur0) {
    if (h->cur == cur0 || n == h->nchains) return TSB_OK;
    const size_t off = (size_t)chain0 * h->chain_words;
    TSB_CUDA(cudaMemcpyAsync(h->buf[h->cur ^ 1] + off, h->buf[h->cur] + off, sizeof(uint32_t) * h->chain_words * n,
                             cudaMemcpyDeviceToDevice, h->stream));
    h->cur ^= 1;
    return TSB_OK;
}

template <int MODE>
int lz_relax(tsb_loz *h, int *dh, size_t ref, const uint32_t *st, int *dflags, bool *overflow) {
    const size_t nv = (size_t)h->X * h->Y;
    lz_fill<<<(unsigned)((nv + 255) / 256), 256, 0, h->stream>>>(dh, nv, MODE == 2 ? -kLzInf : kLzInf, ref);
    const int64_t lim64 = 3 * (int64_t)nv + 8;
    const int limit = (int)std::min<int64_t>(lim64, (int64_t)1 << 30);
    const dim3 grid((h->Y + kLzT - 1) / kLzT, (h->X + kLzT - 1) / kLzT), block(32, 8);
    int hf[2];
    for (int64_t it = 0; it < lim64 + 16; ++it) {
        TSB_CUDA(cudaMemsetAsync(dflags, 0, 2 * sizeof(int), h->stream));
        lz_relax_kernel<MODE><<<grid, block, 0, h->stream>>>(dh, st, h->plane, h->dom, h->X, h->Y, h->pitch, limit,
                                                              dflags);
        TSB_CUDA(cudaGetLastError());
        TSB_CUDA(cudaMemcpyAsync(hf, dflags, 2 * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        TSB_CUDA(cudaStreamSynchronize(h->stream));
        if (hf[1]) { *overflow = true; return TSB_OK; }
        if (!hf[0]) { *overflow = false; return TSB_OK; }
    }
    *overflow = true;
    return TSB_OK;
}

// ------------------------------------------------------------ row-scan heights
// Exact loz_heights (lozenge.py:414-447) for domains whose vertex rows x are
// intervals of existing b-edges (direction d1, step +2 crossed / -1 not,
// _STEPS lozenge.py:47) with consecutive rows linked by an a-edge (d0,
// -2 / +1): h(x, y) = off[x] + local(x, y), then every a- and c-edge is
// checked against its step, so inconsistent states still raise.  The same
// construction as the domino row scan (heights.cu).

__device__ __forceinline__ uint32_t lz_word(const uint32_t *p, int pitch, int x, int w) {
    return p[(size_t)x * pitch + w];
}

// vertex_mask word: any of the six incident edges exists (lz_finish)
__device__ __forceinline__ uint32_t lz_in_mask(const uint32_t *dom, int X, int W, int pitch, int x, int w) {
    const size_t dp = (size_t)X * pitch;
    const uint32_t *exA = dom + 3 * dp, *exB = dom + 4 * dp, *exC = dom + 5 * dp;
    uint32_t m = lz_word(exA, pitch, x, w) | lz_word(exB, pitch, x, w) | lz_word(exC, pitch, x, w);
    m |= lz_word(exB, pitch, x, w) << 1;
    if (w > 0) m |= lz_word(exB, pitch, x, w - 1) >> 31;
    if (x > 0) {
        m |= lz_word(exA, pitch, x - 1, w) | (lz_word(exC, pitch, x - 1, w) >> 1);
        if (w + 1 < W) m |= lz_word(exC, pitch, x - 1, w + 1) << 31;
    }
    return m;
}

__global__ void __launch_bounds__(256) lz_hx_rows_kernel(const uint32_t *dom, int X, int W, int pitch, int4 *rows) {
    __shared__ int sh[8];
    const int x = blockIdx.x;
    const size_t dp = (size_t)X * pitch;
    const uint32_t *exA = dom + 3 * dp, *exB = dom + 4 * dp;
    int a = INT_MAX, b = -1, link = INT_MAX;
    for (int w = threadIdx.x; w < W; w += blockDim.x) {
        const uint32_t m = lz_in_mask(dom, X, W, pitch, x, w);
        if (m) {
            a = min(a, w * 32 + __ffs(m) - 1);
            b = max(b, w * 32 + 31 - __clz(m));
        }
        if (x > 0) {
            const uint32_t up = lz_word(exA, pitch, x - 1, w);
            if (up) link = min(link, w * 32 + __ffs(up) - 1);
        }
    }
    a = block_reduce(a, [](int p, int q) { return min(p, q); }, sh);
    b = block_reduce(b, [](int p, int q) { return max(p, q); }, sh);
    link = block_reduce(link, [](int p, int q) { return min(p, q); }, sh);
    int missing = 0;
    if (a < b) {
        for (int w = (a >> 5) + threadIdx.x; w <= ((b - 1) >> 5); w += blockDim.x) {
            uint32_t e = 0xffffffffu;  // b-edges y in [a, b)
            if (w == (a >> 5)) e &= 0xffffffffu << (a & 31);
            if (w == ((b - 1) >> 5)) e &= 0xffffffffu >> (31 - ((b - 1) & 31));
            missing += __popc(e & ~lz_word(exB, pitch, x, w));
        }
    }
    missing = block_reduce(missing, [](int p, int q) { return p + q; }, sh);
    if (threadIdx.x == 0) rows[x] = make_int4(a, b, link == INT_MAX ? -1 : link, missing == 0);
}

__global__ void __launch_bounds__(256) lz_hx_local_kernel(const uint32_t *st, size_t plane, int pitch, int Y, int r0,
                                                         const int4 *rows, int *loc) {
    __shared__ int sh[8];
    const int x = r0 + blockIdx.x;
    const int4 ri = rows[x];
    const int a = ri.x, b = ri.y;
    if (a > b) return;
    const int w0 = a >> 5, w1 = b >> 5, nw = w1 - w0 + 1;
    const int per = (nw + blockDim.x - 1) / blockDim.x;
    const int wa = w0 + threadIdx.x * per, wb = min(w1, wa + per - 1);
    const uint32_t *rowB = st + plane + (size_t)(x + 1) * pitch;  // plane B, after the guard row
    int sum = 0;
    for (int w = wa; w <= wb; ++w) {
        uint32_t e = 0xffffffffu;
        if (w == w0) e &= 0xffffffffu << (a & 31);
        if (w == w1) e = (b & 31) ? (e & (0xffffffffu >> (32 - (b & 31)))) : 0u;
        const uint32_t cr = rowB[w];
        sum += 2 * __popc(e & cr) - __popc(e & ~cr);
    }
    int acc = block_exclusive_sum(sum, sh);
    int *out = loc + (size_t)x * Y;
    for (int w = wa; w <= wb; ++w) {
        const uint32_t cr = rowB[w];
        const int cb = max(a, w * 32), ce = min(b, w * 32 + 31);
        for (int y = cb; y <= ce; ++y) {
            out[y] = acc;
            acc += ((cr >> (y & 31)) & 1u) ? 2 : -1;
        }
    }
}

__global__ void __launch_bounds__(1024) lz_hx_offsets_kernel(const uint32_t *st, int pitch, int Y, int r0, int r1,
                                                            const int4 *rows, const int *loc, int *off, int ref_x,
                                                            int ref_y) {
    __shared__ int sh[32];
    const int nr = r1 - r0 + 1;
    const int per = (nr + blockDim.x - 1) / blockDim.x;
    const int xa = r0 + threadIdx.x * per, xb = min(r1, xa + per - 1);
    int sum = 0;
    for (int x = xa; x <= xb; ++x) {
        if (x > r0) {
            const int y = rows[x].z;
            const bool cr = (st[(size_t)x * pitch + (y >> 5)] >> (y & 31)) & 1u;  // A[x-1] y
            sum += loc[(size_t)(x - 1) * Y + y] + (cr ? -2 : 1) - loc[(size_t)x * Y + y];
        }
        off[x] = sum;
    }
    const int excl = block_exclusive_sum(sum, sh);
    for (int x = xa; x <= xb; ++x) off[x] += excl;
    __syncthreads();
    const int shift = off[ref_x] + loc[(size_t)ref_x * Y + ref_y];
    __syncthreads();
    for (int x = xa; x <= xb; ++x) off[x] -= shift;
}

template <bool SUM>
__global__ void __launch_bounds__(256) lz_hx_finish_kernel(const uint32_t *st, size_t plane, const uint32_t *dom, int X,
                                                          int Y, int W, int pitch, int r0, int r1, const int *loc,
                                                          const int *off, int32_t *out, long long *acc, int *flags) {
    const int y = blockIdx.x * blockDim.x + threadIdx.x;
    const int x = blockIdx.y;
    if (y >= Y) return;
    const int w = y >> 5;
    const uint32_t bit = 1u << (y & 31);
    const bool in = x >= r0 && x <= r1 && (lz_in_mask(dom, X, W, pitch, x, w) & bit);
    int v = 0;
    if (in) {
        const size_t dp = (size_t)X * pitch;
        const uint32_t *exA = dom + 3 * dp, *exC = dom + 5 * dp;
        v = off[x] + loc[(size_t)x * Y + y];
        if (x > 0 && (lz_word(exA, pitch, x - 1, w) & bit)) {  // a[x-1, y]: (x-1, y) -> (x, y)
            const bool cr = st[(size_t)x * pitch + w] & bit;
            if (v - (off[x - 1] + loc[(size_t)(x - 1) * Y + y]) != (cr ? -2 : 1)) atomicExch(flags, 1);
        }
        if (lz_word(exC, pitch, x, w) & bit) {  // c[x, y]: (x+1, y-1) -> (x, y)
            const bool cr = st[2 * plane + (size_t)(x + 1) * pitch + w] & bit;
            if (v - (off[x + 1] + loc[(size_t)(x + 1) * Y + y - 1]) != (cr ? -2 : 1)) atomicExch(flags, 1);
        }
    }
    if (SUM) acc[(size_t)x * Y + y] += v;
    else out[(size_t)x * Y + y] = v;
}

__global__ void lz_add_heights(const int32_t *h, size_t n, long long *acc) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n) acc[i] += h[i];
}

int lz_hx_scratch(tsb_loz *h) {
    if (h->hx_h) return TSB_OK;
    const size_t nv = (size_t)h->X * h->Y;
    TSB_CUDA(cudaMalloc(&h->hx_h, nv * sizeof(int)));
    TSB_CUDA(cudaMalloc(&h->hx_flags, 4 * sizeof(int)));
    TSB_CUDA(cudaMalloc(&h->hx_off, h->X * sizeof(int)));
    TSB_CUDA(cudaMalloc(&h->hx_rows, h->X * sizeof(int4)));
    return TSB_OK;
}


int lz_hx_classify(tsb_loz *h) {
    if (h->hx_scan >= 0) return TSB_OK;
    int rc = lz_hx_scratch(h);
    if (rc) return rc;
    lz_hx_rows_kernel<<<h->X, 256, 0, h->stream>>>(h->dom, h->X, h->W, h->pitch, h->hx_rows);
    TSB_CUDA(cudaGetLastError());
    std::vector<int4> rows(h->X);
    TSB_CUDA(cudaMemcpyAsync(rows.data(), h->hx_rows, sizeof(int4) * h->X, cudaMemcpyDeviceToHost, h->stream));
    TSB_CUDA(cudaStreamSynchronize(h->stream));
    int r0 = -1, r1 = -1;
    bool ok = true;
    for (int x = 0; x < h->X; ++x) {
        if (rows[x].x > rows[x].y) continue;
        if (r0 < 0) r0 = x;
        else if (r1 != x - 1 || rows[x].z < 0) ok = false;
        if (!rows[x].w) ok = false;
        r1 = x;
    }
    h->hx_r0 = r0 < 0 ? 0 : r0;
    h->hx_r1 = r0 < 0 ? -1 : r1;
    h->hx_scan = (ok && r0 >= 0) ? 1 : 0;
    const char *env = getenv("TSB_HEIGHTS_RELAX");  // test knob: force the relaxation path
    if (env && env[0] == '1') h->hx_scan = 0;
    return TSB_OK;
}


// heights of one chain into dout (device) or added to acc
int lz_heights_dev(tsb_loz *h, int chain, int ref_x, int ref_y, int32_t *dout, long long *acc) {
    int rc = lz_hx_classify(h);
    if (rc) return rc;
    const size_t nv = (size_t)h->X * h->Y;
    const uint32_t *st = h->buf[h->cur] + (size_t)chain * h->chain_words;
    int hf = 0;
    if (h->hx_scan == 1 && ref_x >= h->hx_r0 && ref_x <= h->hx_r1) {
        TSB_CUDA(cudaMemsetAsync(h->hx_flags, 0, sizeof(int), h->stream));
        lz_hx_local_kernel<<<h->hx_r1 - h->hx_r0 + 1, 256, 0, h->stream>>>(st, h->plane, h->pitch, h->Y, h->hx_r0,
                                                                           h->hx_rows, h->hx_h);
        lz_hx_offsets_kernel<<<1, 1024, 0, h->stream>>>(st, h->pitch, h->Y, h->hx_r0, h->hx_r1, h->hx_rows, h->hx_h,
                                                        h->hx_off, ref_x, ref_y);
        const dim3 g((h->Y + 255) / 256, h->X);
        if (acc)
            lz_hx_finish_kernel<true><<<g, 256, 0, h->stream>>>(st, h->plane, h->dom, h->X, h->Y, h->W, h->pitch,
                                                                h->hx_r0, h->hx_r1, h->hx_h, h->hx_off, nullptr, acc,
                                                                h->hx_flags);
        else
            lz_hx_finish_kernel<false><<<g, 256, 0, h->stream>>>(st, h->plane, h->dom, h->X, h->Y, h->W, h->pitch,
                                                                 h->hx_r0, h->hx_r1, h->hx_h, h->hx_off, dout, nullptr,
                                                                 h->hx_flags);
        TSB_CUDA(cudaGetLastError());
        TSB_CUDA(cudaMemcpyAsync(&hf, h->hx_flags, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        TSB_CUDA(cudaStreamSynchronize(h->stream));
        if (hf) return fail(TSB_E_INCONSISTENT, "height propagation inconsistent");
        return TSB_OK;
    }
    bool overflow = false;
    if ((rc = lz_relax<0>(h, h->hx_h, (size_t)ref_x * h->Y + ref_y, st, h->hx_flags, &overflow))) return rc;
    if (overflow) return fail(TSB_E_INCONSISTENT, "height propagation inconsistent");
    int32_t *o = dout;
    if (acc) {
        if ((rc = lz_bytes(h, nv * sizeof(int32_t)))) return rc;
        o = reinterpret_cast<int32_t *>(h->bytes);
    }
    TSB_CUDA(cudaMemsetAsync(h->hx_flags, 0, sizeof(int), h->stream));
    lz_finish<<<dim3((h->Y + 127) / 128, h->X), 128, 0, h->stream>>>(h->hx_h, h->dom, h->X, h->Y, h->pitch, o, kLzInf,
                                                                   h->hx_flags);
    if (acc) lz_add_heights<<<(unsigned)((nv + 255) / 256), 256, 0, h->stream>>>(o, nv, acc);
    TSB_CUDA(cudaGetLastError());
    TSB_CUDA(cudaMemcpyAsync(&hf, h->hx_flags, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    TSB_CUDA(cudaStreamSynchronize(h->stream));
    if (hf) return fail(TSB_E_INCONSISTENT, "height propagation inconsistent");
    return TSB_OK;
}

}  // namespace tsb

using namespace tsb;

extern "C" {

int tsb_loz_destroy(tsb_loz *h);

int tsb_loz_create(int device, int sx, int sy, int nchains, const uint8_t *up, const uint8_t *down, tsb_loz **out) {
    if (!out || !up || !down) return fail(TSB_E_VALUE, "null argument");
    *out = nullptr;
    if (sx < 1 || sy < 1 || nchains < 1) return fail(TSB_E_VALUE, "sizes must be positive");
    if ((uint64_t)(sx + 1) * (uint64_t)(sy + 1) >= kCapacity) return fail(TSB_E_CAPACITY, "grid exceeds capacity");
    int rc = ensure_device(device);
    if (rc) return rc;
    tsb_loz *h = new tsb_loz();
    h->device = device;
    h->sx = sx;
    h->sy = sy;
    h->X = sx + 1;
    h->Y = sy + 1;
    h->nchains = nchains;
    h->W = (h->Y + 31) / 32;
    h->pitch = (h->W + 31) / 32 * 32;
    h->plane = (size_t)(h->X + 2) * h->pitch;
    h->chain_words = 3 * h->plane;
    cudaError_t e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
    h->own_stream = true;
    auto bail = [&](cudaError_t err, const char *what) {
        int code = cuda_fail(err, what);
        tsb_loz_destroy(h);
        return code;
    };
    if (e != cudaSuccess) return bail(e, "stream");
    const size_t sbytes = sizeof(uint32_t) * h->chain_words * nchains;
    for (int i = 0; i < 2; ++i) {
        if ((e = cudaMalloc(&h->buf[i], sbytes)) != cudaSuccess) return bail(e, "state");
        if ((e = cudaMemset(h->buf[i], 0, sbytes)) != cudaSuccess) return bail(e, "memset");
    }
    const size_t tb = (size_t)sx * sy;
    if ((e = cudaMalloc(&h->tri, 2 * tb)) != cudaSuccess) return bail(e, "tri");
    cudaMemcpy(h->tri, up, tb, cudaMemcpyHostToDevice);
    cudaMemcpy(h->tri + tb, down, tb, cudaMemcpyHostToDevice);
    if ((e = cudaMalloc(&h->dom, sizeof(uint32_t) * 6 * (size_t)h->X * h->pitch)) != cudaSuccess) return bail(e, "dom");
    if ((e = cudaMalloc(&h->range, sizeof(int2) * h->X)) != cudaSuccess) return bail(e, "range");
    std::vector<int2> init(h->X, make_int2(INT_MAX, INT_MIN));
    cudaMemcpy(h->range, init.data(), sizeof(int2) * h->X, cudaMemcpyHostToDevice);
    lz_domain_kernel<<<dim3((h->W + 127) / 128, h->X), 128>>>(h->tri, sx, sy, h->X, h->Y, h->W, h->pitch, h->dom,
                                                            h->range);
    lz_fix_ranges<<<(h->X + 255) / 256, 256>>>(h->range, h->X);
    std::vector<int2> rg(h->X);
    if ((e = cudaMemcpy(rg.data(), h->range, sizeof(int2) * h->X, cudaMemcpyDeviceToHost)) != cudaSuccess)
        return bail(e, "domain");
    std::vector<int2> tiles;
    const int nchunks = (h->W + 1 + kLzWords - 1) / kLzWords;
    for (int y = 0; y * kLzRows < h->X; ++y) {
        int lo = INT_MAX, hi = INT_MIN;
        for (int x = y * kLzRows; x < std::min(h->X, (y + 1) * kLzRows); ++x)
            if (rg[x].y > rg[x].x) { lo = std::min(lo, rg[x].x); hi = std::max(hi, rg[x].y); }
        for (int cx = 0; cx < nchunks; ++cx) {
            const int w0 = cx * kLzWords - 1;
            if (hi > w0 && lo < w0 + kLzWords) tiles.push_back(make_int2(cx, y));
        }
    }
    h->ntiles = (int)tiles.size();
    if ((e = cudaMalloc(&h->tiles, sizeof(int2) * std::max<size_t>(1, tiles.size()))) != cudaSuccess)
        return bail(e, "tiles");
    if (!tiles.empty()) cudaMemcpy(h->tiles, tiles.data(), sizeof(int2) * tiles.size(), cudaMemcpyHostToDevice);
    // temporally blocked tiles: K sweeps per launch (TSB_LZ_K overrides; K | kLzGraph, even launch count)
    {
        int K = 4;
        if (const char *ev = getenv("TSB_LZ_K")) K = atoi(ev);
        if (K != 2 && K != 4 && K != 8 && K != 16) K = 4;
        while (kLzMRows - 2 * K < 2) K /= 2;
        h->m_K = K;
        h->m_out = kLzMRows - 2 * K;
        // tiles aligned to each band's own word range: tile.x = first loaded
        // word wa0 (even; loads are predicated to the row), outputs wa0+1 .. wa0+kLzWords
        std::vector<int2> mt;
        for (int y = 0; y * h->m_out < h->X; ++y) {
            int lo = INT_MAX, hi = INT_MIN;
            for (int x = y * h->m_out; x < std::min(h->X, (y + 1) * h->m_out); ++x)
                if (rg[x].y > rg[x].x) { lo = std::min(lo, rg[x].x); hi = std::max(hi, rg[x].y); }
            if (hi <= lo) continue;
            // first tile from word 0 when the band starts there (it owns word 0);
            // a tile reaching the grid's last word owns it (lz_multi_kernel)
            for (int wa0 = lo == 0 ? 0 : (lo - 1) & ~1;; wa0 += kLzWords) {
                mt.push_back(make_int2(wa0, y));
                const int last = wa0 + kLzWords + (wa0 + 63 >= h->W - 1 ? 1 : 0);  // last owned word
                if (last >= hi - 1) break;
            }
        }
        h->nmtiles = (int)mt.size();
        if ((e = cudaMalloc(&h->mtiles, sizeof(int2) * std::max<size_t>(1, mt.size()))) != cudaSuccess)
            return bail(e, "tiles");
        if (!mt.empty()) cudaMemcpy(h->mtiles, mt.data(), sizeof(int2) * mt.size(), cudaMemcpyHostToDevice);
        for (const void *fn : {(const void *)lz_multi_kernel<0, 3>, (const void *)lz_multi_kernel<2, 3>})
            if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLzMSmem)) != cudaSuccess)
                return bail(e, "smem attribute");
        cudaDeviceGetAttribute(&h->m_sms, cudaDevAttrMultiProcessorCount, h->device);
        if (const char *ev = getenv("TSB_LZ_DENSE")) h->m_dense = atoi(ev) ? 1 : 0;
        if (const char *ev = getenv("TSB_LZ_COLLAPSE")) h->collapse = atoi(ev) != 0;
        if ((e = cudaFuncSetAttribute(lz_multi_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kLzMSmem)) != cudaSuccess ||
            (e = cudaFuncSetAttribute(lz_multi_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kLzMSmem)) != cudaSuccess)
            return bail(e, "smem attribute");
    }
    if ((e = cudaMalloc(&h->seedinfo, sizeof(uint64_t) * 2 * nchains)) != cudaSuccess) return bail(e, "seeds");
    if ((e = cudaMallocHost(&h->seed_pinned, sizeof(uint64_t) * 2 * nchains)) != cudaSuccess) return bail(e, "seeds");
    if ((e = cudaMalloc(&h->flag, 2 * sizeof(int))) != cudaSuccess) return bail(e, "flag");
    if ((e = cudaMalloc(&h->step_dev, 2 * sizeof(uint64_t))) != cudaSuccess) return bail(e, "step");
    if ((e = cudaEventCreateWithFlags(&h->seed_ev, cudaEventDisableTiming)) != cudaSuccess) return bail(e, "event");
    if ((e = cudaEventRecord(h->seed_ev, h->stream)) != cudaSuccess) return bail(e, "event");
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return bail(e, "create");
    *out = h;
    return TSB_OK;
}

int tsb_loz_destroy(tsb_loz *h) {
    if (!h) return TSB_OK;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    cudaFree(h->buf[0]);
    cudaFree(h->buf[1]);
    cudaFree(h->dom);
    cudaFree(h->tri);
    cudaFree(h->range);
    cudaFree(h->tiles);
    cudaFree(h->mtiles);
    cudaFree(h->tgrid);
    cudaFree(h->seedinfo);
    cudaFree(h->bytes);
    cudaFree(h->flag);
    cudaFree(h->step_dev);
    cudaFree(h->hx_h);
    cudaFree(h->hx_flags);
    cudaFree(h->hx_off);
    cudaFree(h->hx_rows);
    if (h->graph_exec) cudaGraphExecDestroy(h->graph_exec);
    if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
    if (h->seed_pinned) cudaFreeHost(h->seed_pinned);
    if (h->seed_ev) cudaEventDestroy(h->seed_ev);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    delete h;
    return TSB_OK;
}

int tsb_loz_set_stream(tsb_loz *h, void *stream) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    TSB_CUDA(cudaSetDevice(h->device));
    TSB_CUDA(cudaStreamSynchronize(h->stream));
    if (h->own_stream) cudaStreamDestroy(h->stream);
    h->stream = (cudaStream_t)stream;
    h->own_stream = false;
    return TSB_OK;
}

int tsb_loz_set_p_up(tsb_loz *h, const double *p_up) {
    if (!h || !p_up) return fail(TSB_E_VALUE, "null argument");
    TSB_CUDA(cudaSetDevice(h->device));
    const size_t nv = (size_t)h->X * h->Y;
    std::vector<uint64_t> t(nv);
    bool uniform = true;
    for (size_t i = 0; i < nv; ++i) {
        t[i] = threshold_of(p_up[i]);
        if (t[i] != t[0]) uniform = false;
    }
    if (uniform) {
        h->tmode = 0;
        h->t0 = t[0];
    } else {
        h->tmode = 2;
        if (!h->tgrid) TSB_CUDA(cudaMalloc(&h->tgrid, sizeof(uint64_t) * nv));
        TSB_CUDA(cudaMemcpy(h->tgrid, t.data(), sizeof(uint64_t) * nv, cudaMemcpyHostToDevice));
    }
    return TSB_OK;
}

int tsb_loz_upload(tsb_loz *h, int chain0, int n, const uint8_t *edges) {
    int rc = lz_check(h, chain0, n);
    if (rc || n == 0) return rc;
    TSB_CUDA(cudaSetDevice(h->device));
    const size_t need = (size_t)n * 3 * h->X * h->Y;
    if ((rc = lz_bytes(h, need))) return rc;
    if ((rc = staged_h2d(h->bytes, edges, need, h->stream))) return rc;
    TSB_CUDA(cudaMemsetAsync(h->flag, 0, sizeof(int), h->stream));
    lz_pack_kernel<<<dim3((h->W + 127) / 128, h->X, n), 128, 0, h->stream>>>(
        h->bytes, h->X, h->Y, h->W, h->pitch, h->plane, h->chain_words, h->dom,
        h->buf[h->cur] + (size_t)chain0 * h->chain_words, h->flag);
    TSB_CUDA(cudaGetLastError());
    int bad = 0;
    TSB_CUDA(cudaMemcpyAsync(&bad, h->flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    TSB_CUDA(cudaStreamSynchronize(h->stream));
    if (bad & 1) return fail(TSB_E_INCONSISTENT, "edge grids must be boolean");
    if (bad & 2) return fail(TSB_E_INCONSISTENT, "crossed edge leaves the domain");
    return TSB_OK;
}

int tsb_loz_download(tsb_loz *h, int chain0, int n, uint8_t *edges) {
    int rc = lz_check(h, chain0, n);
    if (rc || n == 0) return rc;
    TSB_CUDA(cudaSetDevice(h->device));
    const size_t need = (size_t)n * 3 * h->X * h->Y;
    if ((rc = lz_bytes(h, need))) return rc;
    lz_unpack_kernel<<<dim3((h->Y + 127) / 128, h->X, n), 128, 0, h->stream>>>(
        h->buf[h->cur] + (size_t)chain0 * h->chain_words, h->X, h->Y, h->pitch, h->plane, h->chain_words, h->bytes);
    TSB_CUDA(cudaGetLastError());
    return staged_d2h(edges, h->bytes, need, h->stream);
}

static int lz_push_seeds(tsb_loz *h, int n, const uint64_t *seeds) {
    TSB_CUDA(cudaEventSynchronize(h->seed_ev));
    for (int i = 0; i < n; ++i) {
        const uint64_t b = family_base(seeds[i]);
        h->seed_pinned[2 * i] = b;
        h->seed_pinned[2 * i + 1] = global_key(b);
    }
    TSB_CUDA(cudaMemcpyAsync(h->seedinfo, h->seed_pinned, sizeof(uint64_t) * 2 * n, cudaMemcpyHostToDevice,
                             h->stream));
    TSB_CUDA(cudaEventRecord(h->seed_ev, h->stream));
    return TSB_OK;
}

int tsb_loz_walk(tsb_loz *h, int chain0, int n, const uint64_t *seeds, uint64_t step0, uint64_t n_steps) {
    int rc = lz_check(h, chain0, n);
    if (rc || n == 0 || n_steps == 0) return rc;
    if (!seeds) return fail(TSB_E_VALUE, "null seeds");
    TSB_CUDA(cudaSetDevice(h->device));
    if ((rc = lz_push_seeds(h, n, seeds))) return rc;
    const int cur0 = h->cur;
    uint64_t s = 0;
    if (n_steps >= 2 * kLzGraph) {
        if ((rc = lz_graph(h, chain0, n))) return rc;
        lz_set_step<<<1, 1, 0, h->stream>>>(h->step_dev, step0, step0 + n_steps);
        TSB_CUDA(cudaGetLastError());
        for (; s + kLzGraph <= n_steps; s += kLzGraph) TSB_CUDA(cudaGraphLaunch(h->graph_exec, h->stream));
    }
    if (n_steps - s >= (uint64_t)h->m_K) {  // remainder: direct multi-sweep launches (step_dev = step0 + s)
        if (s == 0) lz_set_step<<<1, 1, 0, h->stream>>>(h->step_dev, step0, step0 + n_steps);
        TSB_CUDA(cudaGetLastError());
        for (uint64_t i = 0; s + h->m_K <= n_steps; s += h->m_K, i += h->m_K)
            if ((rc = lz_launch_multi(h, chain0, n, i, h->stream))) return rc;
    }
    for (; s < n_steps; ++s)
        if ((rc = lz_launch(h, chain0, n, step0 + s, -1, h->stream, nullptr))) return rc;
    return lz_settle(h, chain0, n, cur0);
}

int tsb_loz_sweep(tsb_loz *h, int chain0, int n, const uint64_t *seeds, uint64_t step, int color) {
    int rc = lz_check(h, chain0, n);
    if (rc || n == 0) return rc;
    if (color < 0 || color > 2) return fail(TSB_E_VALUE, "colour class must be 0, 1 or 2");
    TSB_CUDA(cudaSetDevice(h->device));
    if ((rc = lz_push_seeds(h, n, seeds))) return rc;
    const int cur0 = h->cur;
    if ((rc = lz_launch(h, chain0, n, step, color, h->stream, nullptr))) return rc;
    return lz_settle(h, chain0, n, cur0);
}

int tsb_loz_sync(tsb_loz *h) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    TSB_CUDA(cudaSetDevice(h->device));
    TSB_CUDA(cudaStreamSynchronize(h->stream));
    return TSB_OK;
}

int tsb_loz_heights(tsb_loz *h, int chain, int ref_x, int ref_y, int32_t *out) {
    if (!h || !out) return fail(TSB_E_VALUE, "null argument");
    if (chain < 0 || chain >= h->nchains) return fail(TSB_E_VALUE, "chain out of range");
    if (ref_x < 0 || ref_y < 0 || ref_x >= h->X || ref_y >= h->Y) return fail(TSB_E_VALUE, "reference vertex outside");
    TSB_CUDA(cudaSetDevice(h->device));
    const size_t nv = (size_t)h->X * h->Y;
    int rc = lz_bytes(h, nv * sizeof(int32_t));  // handle staging: no allocation per call
    if (rc) return rc;
    int32_t *dout = reinterpret_cast<int32_t *>(h->bytes);
    if ((rc = lz_heights_dev(h, chain, ref_x, ref_y, dout, nullptr))) return rc;
    return staged_d2h(out, dout, nv * sizeof(int32_t), h->stream);  // pinned staging, returns complete
}

int tsb_loz_height_sum_add(tsb_loz *h, int chain0, int n, int ref_x, int ref_y, long long *acc_dev) {
    int rc = lz_check(h, chain0, n);
    if (rc || n == 0) return rc;
    if (!acc_dev) return fail(TSB_E_VALUE, "null accumulator");
    if (ref_x < 0 || ref_y < 0 || ref_x >= h->X || ref_y >= h->Y) return fail(TSB_E_VALUE, "reference vertex outside");
    TSB_CUDA(cudaSetDevice(h->device));
    for (int k = 0; k < n && !rc; ++k) rc = lz_heights_dev(h, chain0 + k, ref_x, ref_y, nullptr, acc_dev);
    return rc;
}

int tsb_loz_extremal(tsb_loz *h, int chain_max, int chain_min, int ref_x, int ref_y) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    if (chain_max < 0 || chain_max >= h->nchains || chain_min < 0 || chain_min >= h->nchains)
        return fail(TSB_E_VALUE, "chain out of range");
    TSB_CUDA(cudaSetDevice(h->device));
    const size_t nv = (size_t)h->X * h->Y;
    int rc = lz_hx_scratch(h);
    if (!rc) rc = lz_bytes(h, nv * sizeof(int32_t));
    if (rc) return rc;
    int *dh = h->hx_h, *df = h->hx_flags;
    int32_t *dout = reinterpret_cast<int32_t *>(h->bytes);
    bool untileable = false;
    for (int pass = 0; pass < 2 && !rc && !untileable; ++pass) {
        bool overflow = false;
        const size_t ref = (size_t)ref_x * h->Y + ref_y;
        rc = pass == 0 ? lz_relax<1>(h, dh, ref, nullptr, df, &overflow) : lz_relax<2>(h, dh, ref, nullptr, df, &overflow);
        if (rc) break;
        if (overflow) { untileable = true; break; }
        int hf[2] = {0, 0};
        cudaMemsetAsync(df, 0, 2 * sizeof(int), h->stream);
        lz_finish<<<dim3((h->Y + 127) / 128, h->X), 128, 0, h->stream>>>(dh, h->dom, h->X, h->Y, h->pitch, dout,
                                                                       pass == 0 ? kLzInf : -kLzInf, df);
        uint32_t *st = h->buf[h->cur] + (size_t)(pass == 0 ? chain_max : chain_min) * h->chain_words;
        lz_decode<<<dim3((h->W + 127) / 128, h->X), 128, 0, h->stream>>>(dout, h->dom, h->X, h->Y, h->W, h->pitch,
                                                                       h->plane, st);
        lz_cover_check<<<dim3((h->sy + 127) / 128, h->sx), 128, 0, h->stream>>>(h->tri, h->sx, h->sy, st, h->pitch,
                                                                               h->plane, df + 1);
        cudaMemcpyAsync(hf, df, 2 * sizeof(int), cudaMemcpyDeviceToHost, h->stream);
        cudaError_t e = cudaStreamSynchronize(h->stream);
        if (e != cudaSuccess) { rc = cuda_fail(e, "loz extremal"); break; }
        if (hf[0] || hf[1]) untileable = true;
    }
    if (rc) return rc;
    if (untileable) return fail(TSB_E_UNTILEABLE, "triangle domain is not tileable");
    return TSB_OK;
}

int tsb_loz_set_collapse(tsb_loz *h, int on) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    h->collapse = on ? 1 : 0;
    return TSB_OK;
}

int tsb_loz_serialize(tsb_loz *h, int chain, char *out, size_t cap, size_t *len) {
    if (!h || !len) return fail(TSB_E_VALUE, "null argument");
    int rc = lz_check(h, chain, 1);
    if (rc) return rc;
    const size_t total = 3 * (size_t)h->X * h->Y;
    *len = total;
    if (!out || cap < total) return TSB_OK;  // size query
    TSB_CUDA(cudaSetDevice(h->device));
    if ((rc = lz_bytes(h, total))) return rc;  // handle scratch: no allocation per record
    char *d = reinterpret_cast<char *>(h->bytes);
    lz_serialize_kernel<<<dim3((h->W + 63) / 64, h->X, 3), 64, 0, h->stream>>>(
        h->buf[h->cur] + (size_t)chain * h->chain_words, h->X, h->Y, h->pitch, h->plane, d);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, total, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "loz serialize");
    return TSB_OK;
}

int tsb_loz_coalesced(tsb_loz *h, int chain0, int npairs, uint8_t *flags) {
    int rc = lz_check(h, chain0, 2 * npairs);
    if (rc || npairs == 0) return rc;
    TSB_CUDA(cudaSetDevice(h->device));
    if ((rc = lz_bytes(h, npairs))) return rc;
    uint8_t *d = reinterpret_cast<uint8_t *>(h->bytes);
    lz_coalesced<<<npairs, 256, 0, h->stream>>>(reinterpret_cast<const uint4 *>(h->buf[h->cur]), h->chain_words / 4,
                                               chain0, d);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(flags, d, npairs, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "loz coalesced");
    return TSB_OK;
}

int tsb_loz_replicate(tsb_loz *h, int src, int dst0, int step, int n) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    if (n <= 0) return TSB_OK;
    if (src < 0 || src >= h->nchains || dst0 < 0 || step < 1 || dst0 + (int64_t)(n - 1) * step >= h->nchains)
        return fail(TSB_E_VALUE, "replicate chains out of range");
    TSB_CUDA(cudaSetDevice(h->device));
    const size_t u4 = h->chain_words / 4;
    lz_replicate<<<(unsigned)((u4 + 255) / 256), 256, 0, h->stream>>>(reinterpret_cast<uint4 *>(h->buf[h->cur]), u4,
                                                                      src, dst0, step, n);
    TSB_CUDA(cudaGetLastError());
    return TSB_OK;
}

int tsb_loz_cftp(tsb_loz *h, const uint8_t *top0, const uint8_t *bot0, const uint64_t *masters, int count,
                 int max_doublings, uint8_t *out_edges, int32_t *collapsed_round, tsb_progress_fn progress,
                 void *user) {
    if (!h || !top0 || !bot0 || !masters || !out_edges) return fail(TSB_E_VALUE, "null argument");
    if (count <= 0) return TSB_OK;
    if (h->nchains < 2 * count + 2)
        return fail(TSB_E_VALUE, "handle needs >= %d chains for %d samples", 2 * count + 2, count);
    const int T = 2 * count, B = 2 * count + 1;
    int rc;
    if ((rc = tsb_loz_upload(h, T, 1, top0))) return rc;
    if ((rc = tsb_loz_upload(h, B, 1, bot0))) return rc;
    const size_t grid = (size_t)3 * h->X * h->Y;
    std::vector<int> active(count);
    for (int k = 0; k < count; ++k) {
        active[k] = k;
        if (collapsed_round) collapsed_round[k] = 0;
    }
    std::vector<uint64_t> seeds;
    std::vector<uint8_t> flags;
    uint64_t steps_total = 0;
    const uint64_t kSalt = 0x51ED2701ull, kMul = 0xD6E8FEB86659FD93ull;
    for (int round_no = 1; round_no <= max_doublings; ++round_no) {
        steps_total += 1ull << round_no;
        const int na = (int)active.size();
        if ((rc = tsb_loz_replicate(h, T, 0, 2, na))) return rc;
        if ((rc = tsb_loz_replicate(h, B, 1, 2, na))) return rc;
        for (int i = round_no; i >= 1; --i) {
            seeds.assign(2 * na, 0);
            for (int j = 0; j < na; ++j)
                seeds[2 * j] = seeds[2 * j + 1] =
                    mix64(mix64(masters[active[j]] ^ (kSalt * kMul)) + ((uint64_t)i + 1ull) * kGold);
            if ((rc = tsb_loz_walk(h, 0, 2 * na, seeds.data(), 0, 1ull << i))) return rc;
        }
        flags.assign(na, 0);
        if ((rc = tsb_loz_coalesced(h, 0, na, flags.data()))) return rc;
        std::vector<int> still;
        for (int j = 0; j < na; ++j) {
            if (flags[j]) {
                const int k = active[j];
                if ((rc = tsb_loz_download(h, 2 * j + 1, 1, out_edges + (size_t)k * grid))) return rc;
                if (collapsed_round) collapsed_round[k] = round_no;
            } else {
                still.push_back(active[j]);
            }
        }
        active.swap(still);
        if (progress) progress(round_no, steps_total, count - (int)active.size(), count, user);
        if (active.empty()) return TSB_OK;
    }
    return fail(TSB_E_CONVERGENCE, "no coalescence after %d doublings", max_doublings);
}

}  // extern "C"
