// Six-vertex model with fixed boundary: 1-bit face-height state, 4-class
// heat-bath c-flip sweep, height codec, extremal heights, CFTP.
//
// Reference (relative to /root/reference/pkg/src/tilesampler/):
//   sixvertex.py:199-277  FaceHeights / heights_from_config / config_from_heights
//   sixvertex.py:343-467  _interior_class_masks, _vertex_weight_grid, sv_sweep_batch,
//                         sv_random_walk_batch
//   sixvertex.py:508-562  _ring_heights, sv_extremal;  565-622 sv_cftp
//
// State.  Face heights step by exactly 1 across every edge, so with
// p0 = h(0,0) mod 2 every face has h = 2u + ((R+C+p0) & 1) for an integer u,
// and one bit per face, b = u & 1 (h mod 4), determines every edge of the
// configuration: between adjacent faces X -> Y,  Y = X + 1  iff
// (bit X == bit Y) xor (X has odd parity).  A c-flip (h -> h +- 2) toggles
// the bit.  Absolute heights are restored by integrating from h(0,0).
//
// Sweep.  Class k = x >> 62 of the global draw (min(int(u*4),3),
// sixvertex.py:463-464) selects interior faces with (R%2, C%2) = (k>>1, k&1).
// Same-class faces share no edge or corner vertex, so a sweep reads only
// other-class bits and updates in place.  A candidate is a local minimum (all
// four neighbours = h+1, moves +2 iff u < p_high) or maximum (all = h-1,
// moves -2 iff u >= p_high).  p_high depends only on the direction and on the
// four diagonal faces (the corner vertices' types); the host evaluates the
// reference's float64 expression ((w00*w01)*w10)*w11 ratio on those 32
// patches and passes p_high, converted here to exact integer thresholds.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <vector>

#include "tsb_internal.cuh"

struct tsb_sv {
    int device = 0, n = 0, f = 0, nchains = 0, W = 0, pitch = 0;
    size_t chain_words = 0;  // uint32 words per chain (incl. guard rows)
    uint32_t *bits = nullptr;
    int32_t *h00 = nullptr;  // per chain h(0,0) (device)
    uint64_t lut[32] = {};
    uint64_t *seedinfo = nullptr;
    uint64_t *seed_pinned = nullptr;
    cudaEvent_t seed_ev = nullptr;
    int32_t *hbuf = nullptr;  // device staging (count, f, f) int32
    size_t hbuf_cap = 0;
    int *flag = nullptr;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // temporally blocked walks (sv_multi_kernel) replayed from a CUDA graph
    uint32_t *bits2 = nullptr;  // second buffer (out-of-place launches)
    uint64_t *step_dev = nullptr;
    int m_wpl = 1, m_nw = 8, m_K = 4, m_out = 8, m_stride = 32, m_woff = 0, m_gx = 1, m_gy = 1;
    int m_xw = 0;  // tiles of 32 * m_wpl words plus the read-only east boundary word
    bool m_k_fixed = false;  // TSB_SV_K given: no per-batch choice of K
    int m_sms = 148;
    size_t m_smem = 0;
    cudaStream_t cap_stream = nullptr;
    cudaGraphExec_t graph_exec = nullptr;
    int g_chain0 = -1, g_n = -1;
    uint64_t lut_version = 0, g_lut_version = ~0ull;
    int collapse = 1, g_collapse = -1;  // run collapsing (TSB_SV_COLLAPSE, tsb_sv_set_collapse)
};

namespace tsb {

struct SvCtx {
    uint32_t *bits;
    const int32_t *h00;
    const uint64_t *seedinfo;
    size_t chain_words;
    int n, f, W, pitch;
    uint64_t step;
    int class_override;  // -1: class from the global coin
    uint64_t lut[32];
};

template <typename T>
__device__ __forceinline__ T shfl_up(T v) { return __shfl_up_sync(0xffffffffu, v, 1); }
template <typename T>
__device__ __forceinline__ T shfl_dn(T v) { return __shfl_down_sync(0xffffffffu, v, 1); }

__device__ __noinline__ uint32_t sv_rng(uint32_t cand, uint32_t is_min, uint32_t dnw, uint32_t dne, uint32_t dsw,
                                        uint32_t dse, uint64_t row_idx, int w, uint64_t base, uint64_t salt,
                                        const uint64_t *lut) {
    uint32_t flip = 0;
    do {
        const int b = __ffs(cand) - 1;
        cand &= cand - 1;
        const uint64_t idx = row_idx + (uint64_t)(w * 32 + b);
        const uint64_t x = mix64(mix64(base + (idx + 1ull) * kGold) + salt);
        const uint32_t up = (is_min >> b) & 1u;
        const int li = (up ? 0 : 16) | (((dnw >> b) & 1) << 3) | (((dne >> b) & 1) << 2) | (((dsw >> b) & 1) << 1) |
                       ((dse >> b) & 1);
        const bool high = (x >> 11) < lut[li];
        if (high == (bool)up) flip |= 1u << b;
    } while (cand);
    return flip;
}

// One class sweep; warp = 32 consecutive words of one class row.
__global__ void __launch_bounds__(256) sv_sweep_kernel(SvCtx c) {
    const int lane = threadIdx.x & 31;
    const int w = blockIdx.x * 32 + lane;
    const int z = blockIdx.z;
    const uint64_t base = c.seedinfo[2 * z];
    const uint64_t gkey = c.seedinfo[2 * z + 1];
    const uint64_t salt = (c.step + 1ull) * kGold;
    const int cls = c.class_override >= 0 ? c.class_override : (int)(mix64(gkey + salt) >> 62);  // min(int(u*4),3)
    const int pr = cls >> 1, pc = cls & 1;
    const int R = 2 * (blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5)) + pr;
    if (R < 1 || R > c.n - 1) return;  // warp-uniform
    uint32_t *P = c.bits + (size_t)z * c.chain_words + c.pitch;  // row 0
    const uint32_t *ru = P + (size_t)(R - 1) * c.pitch;
    uint32_t *rc = P + (size_t)R * c.pitch;
    const uint32_t *rd = P + (size_t)(R + 1) * c.pitch;
    const bool inw = w < c.W;
    const uint32_t u = inw ? __ldcg(ru + w) : 0u, b = inw ? __ldcg(rc + w) : 0u, d = inw ? __ldcg(rd + w) : 0u;
    uint32_t ul = shfl_up(u), bl = shfl_up(b), dl = shfl_up(d);
    uint32_t ur = shfl_dn(u), br = shfl_dn(b), dr = shfl_dn(d);
    if (lane == 0) {
        ul = w > 0 ? __ldcg(ru + w - 1) : 0u;
        bl = w > 0 ? __ldcg(rc + w - 1) : 0u;
        dl = w > 0 ? __ldcg(rd + w - 1) : 0u;
    }
    if (lane == 31) {
        ur = w + 1 < c.W ? __ldcg(ru + w + 1) : 0u;
        br = w + 1 < c.W ? __ldcg(rc + w + 1) : 0u;
        dr = w + 1 < c.W ? __ldcg(rd + w + 1) : 0u;
    }
    // class columns C = 32w+b with C % 2 == pc and 1 <= C <= n-1
    uint32_t act = pc ? 0xAAAAAAAAu : 0x55555555u;
    const int c0 = w * 32;
    if (c0 < 1) act &= ~1u;
    const int hi = c.n - 1 - c0;  // last allowed bit
    if (hi < 31) act &= hi < 0 ? 0u : (0xFFFFFFFFu >> (31 - hi));
    if (!inw) act = 0;
    const uint32_t left = (b << 1) | (bl >> 31), right = (b >> 1) | (br << 31);
    const uint32_t eq_u = ~(u ^ b), eq_d = ~(d ^ b), eq_l = ~(left ^ b), eq_r = ~(right ^ b);
    const int odd = (pr + pc + (c.h00[z] & 1)) & 1;  // parity of the class faces
    const uint32_t all_eq = eq_u & eq_d & eq_l & eq_r;
    const uint32_t all_ne = ~eq_u & ~eq_d & ~eq_l & ~eq_r;
    const uint32_t is_min = (odd ? all_ne : all_eq) & act;  // neighbours all h+1
    const uint32_t is_max = (odd ? all_eq : all_ne) & act;  // neighbours all h-1
    const uint32_t cand = is_min | is_max;
    if (!cand) return;
    // diagonal faces differ from the centre (by +-2) iff their bit differs
    const uint32_t dnw = ((u << 1) | (ul >> 31)) ^ b, dne = ((u >> 1) | (ur << 31)) ^ b;
    const uint32_t dsw = ((d << 1) | (dl >> 31)) ^ b, dse = ((d >> 1) | (dr << 31)) ^ b;
    const uint32_t flip = sv_rng(cand, is_min, dnw, dne, dsw, dse, (uint64_t)R * (uint64_t)c.f, w, base, salt, c.lut);
    if (flip) rc[w] = b ^ flip;
}

// ---------------------------------------------------------------------------
// Temporal blocking: K class sweeps per launch (sv_multi_kernel).
//
// A block of NW warps holds a tile of 2*NW rows x 32*WPL words in registers
// (warp k owns tile rows 2k and 2k+1; lane l owns words l*WPL .. l*WPL+WPL-1)
// with a shared-memory copy of every row for the vertical neighbours.  In a
// sweep of class (pr, pc) every warp updates exactly one of its rows (the one
// with R % 2 == pr) and reads only rows of the other parity, which no warp
// writes in that sweep, so one block barrier per sweep suffices.  Rows and
// words next to the unloaded outside go stale by one row / bit per sweep, so
// after K sweeps the central 2*NW - 2K rows (and, for tiles with word halos,
// all but the first and last word) are exact and are the only ones stored.
// Out of place (double buffer): neighbouring tiles read each other's rows.
// Class coins, site coins and the heat-bath LUT are exactly those of
// sv_sweep_kernel, so the result is bit-identical for any tiling.
struct SvMCtx {
    const uint32_t *src;  // chain 0, row 0 (after the guard row)
    uint32_t *dst;
    const int32_t *h00;
    const uint64_t *seedinfo;
    const uint64_t *step_dev;
    size_t chain_words;
    int n, f, W, pitch;
    int K, out_rows;      // sweeps per launch, exact rows per tile (2*NW - 2K)
    int collapse;         // skip sweeps followed by a sweep of the same class
    int half;             // every LUT entry is 2^52 (p_high = 1/2: a = b = c)
    int xw;               // word 32 * WPL holds only the east boundary column: lane 31 keeps it read-only
    int stride, woff;     // column tiles: first word of tile x = x*stride + woff
    uint64_t step;        // offset of this launch inside the graph replay
    uint64_t lut[32];
};

template <int WPL, int NW>
constexpr size_t sv_multi_smem() {
    return sizeof(uint32_t) * (2 * NW) * (32 * WPL + 1)  // rows (+ the east boundary word, XW tiles)
           + sizeof(uint64_t) * 32                      // lut
           + sizeof(uint32_t) * NW * (32 * WPL)         // per-warp flip words
           + sizeof(uint16_t) * NW * (32 * WPL) * 16    // per-warp job queues
           + sizeof(uint4) * NW * (32 * WPL)            // per-warp diagonal masks (nw, ne, sw, se)
           + sizeof(uint32_t) * NW * (32 * WPL)         // per-warp local-minimum masks
           + 16;                                        // alignment of the mask arrays
}

// XW: tiles of 32 * WPL words plus the read-only east boundary word (c.xw)
template <int WPL, int NW, int MINB = 1, bool XW = false>
__global__ void __launch_bounds__(32 * NW, MINB) sv_multi_kernel(SvMCtx c) {
    constexpr int TW = 32 * WPL, TR = 2 * NW, RS = TW + (XW ? 1 : 0);  // RS: smem row stride
    extern __shared__ __align__(16) unsigned char dsm[];
    uint32_t(*rows)[RS] = reinterpret_cast<uint32_t(*)[RS]>(dsm);
    uint64_t *lut = reinterpret_cast<uint64_t *>(dsm + sizeof(uint32_t) * TR * RS);
    uint32_t *fres = reinterpret_cast<uint32_t *>(dsm + sizeof(uint32_t) * TR * RS + sizeof(uint64_t) * 32) +
                     (threadIdx.x >> 5) * TW;
    uint16_t *queue = reinterpret_cast<uint16_t *>(dsm + sizeof(uint32_t) * TR * RS + sizeof(uint64_t) * 32 +
                                                   sizeof(uint32_t) * NW * TW) +
                      (threadIdx.x >> 5) * TW * 16;
    unsigned char *mbase = dsm + sizeof(uint32_t) * TR * RS + sizeof(uint64_t) * 32 + sizeof(uint32_t) * NW * TW +
                           sizeof(uint16_t) * NW * TW * 16;
    mbase += (16 - (size_t)(mbase - dsm) % 16) % 16;  // uint4 alignment
    uint4 *dmask = reinterpret_cast<uint4 *>(mbase) + (threadIdx.x >> 5) * TW;
    uint32_t *mnv = reinterpret_cast<uint32_t *>(mbase + sizeof(uint4) * NW * TW) + (threadIdx.x >> 5) * TW;
    const int lane = threadIdx.x & 31, k = threadIdx.x >> 5;
    const int z = blockIdx.z;
    const int r0 = (int)blockIdx.y * c.out_rows - c.K;  // even
    const int wl = (int)blockIdx.x * c.stride + c.woff + lane * WPL;  // first word of this lane
    if (threadIdx.x < 32) lut[threadIdx.x] = c.lut[threadIdx.x];
    const uint64_t base = c.seedinfo[2 * z], gkey = c.seedinfo[2 * z + 1];
    const int p0 = c.h00[z] & 1;
    // interior columns 1..n-1 of this lane's words
    uint32_t cm[WPL];
#pragma unroll
    for (int j = 0; j < WPL; ++j) {
        const int w = wl + j, c0 = w * 32;
        uint32_t m = (w >= 0 && w < c.W) ? 0xFFFFFFFFu : 0u;
        if (c0 < 1) m &= ~1u;
        const int hi = c.n - 1 - c0;
        if (hi < 31) m &= hi < 0 ? 0u : (0xFFFFFFFFu >> (31 - hi));
        cm[j] = m;
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint64_t step0 = c.step_dev[0] + c.step, walk_end = c.step_dev[1];
    // class of sweep s is computed by lane s: min(int(u*4),3) = x >> 62
    const int mycls = (int)(mix64(gkey + (step0 + (uint64_t)lane + 1ull) * kGold) >> 62);
    const uint32_t *src = c.src + (size_t)z * c.chain_words;
    const int Ra = r0 + 2 * k;
    uint32_t ra[WPL], rb[WPL];  // rows Ra, Ra + 1
#pragma unroll
    for (int j = 0; j < WPL; ++j) {
        const int w = wl + j;
        const bool inw = w >= 0 && w < c.W;
        ra[j] = (inw && Ra >= 0 && Ra < c.f) ? __ldcg(src + (size_t)Ra * c.pitch + w) : 0u;
        rb[j] = (inw && Ra + 1 >= 0 && Ra + 1 < c.f) ? __ldcg(src + (size_t)(Ra + 1) * c.pitch + w) : 0u;
        rows[2 * k][lane * WPL + j] = ra[j];
        rows[2 * k + 1][lane * WPL + j] = rb[j];
    }
    // the east boundary word (tiles of W = 32 * WPL + 1 words whose last word
    // holds only column n): never updated, read as the right neighbour of
    // lane 31's last word and stored back unchanged
    uint32_t xa = 0u, xb = 0u;
    if (XW && lane == 31) {
        xa = (Ra >= 0 && Ra < c.f) ? __ldcg(src + (size_t)Ra * c.pitch + TW) : 0u;
        xb = (Ra + 1 >= 0 && Ra + 1 < c.f) ? __ldcg(src + (size_t)(Ra + 1) * c.pitch + TW) : 0u;
        rows[2 * k][RS - 1] = xa;
        rows[2 * k + 1][RS - 1] = xb;
    }
    __syncthreads();
#pragma unroll 1
    for (int s = 0; s < c.K; ++s) {
        const int cls = __shfl_sync(0xffffffffu, mycls, s);
        // run collapsing: the move is a heat-bath update (after it a candidate
        // is a local maximum iff u < p_high, whatever it was, sixvertex.py:
        // 420-441) and within a run of one class nothing else moves, so only
        // the run's last sweep decides (bit-identical; block-uniform skip)
        if (c.collapse && step0 + (uint64_t)s + 1ull < walk_end && __shfl_sync(0xffffffffu, mycls, s + 1) == cls)
            continue;
        const int pr = cls >> 1, pc = cls & 1;
        const int i = 2 * k + pr, R = r0 + i;
        uint32_t u[WPL], b[WPL], d[WPL];
#pragma unroll
        for (int j = 0; j < WPL; ++j) {
            if (pr == 0) {
                b[j] = ra[j];
                d[j] = rb[j];
                u[j] = i > 0 ? rows[i - 1][lane * WPL + j] : 0u;
            } else {
                b[j] = rb[j];
                u[j] = ra[j];
                d[j] = i + 1 < TR ? rows[i + 1][lane * WPL + j] : 0u;
            }
        }
        uint32_t bL = __shfl_up_sync(0xffffffffu, b[WPL - 1], 1), bR = __shfl_down_sync(0xffffffffu, b[0], 1);
        if (lane == 0) bL = 0u;
        if (lane == 31) bR = XW ? (pr == 0 ? xa : xb) : 0u;
        // coins that cannot reach a stored face are not drawn: a flip moves
        // one row / column per sweep, so sweep s only needs tile rows
        // s+1 .. TR-2-s and, in tiles with word halos, the halo bits within
        // K-1-s columns of the interior (one column of slack each side)
        const bool rowok = R >= 1 && R <= c.n - 1 && i >= s + 1 && i <= TR - 2 - s;
        const int reach = c.K - s;  // K-1-s plus one column of slack
        const uint32_t hmask_l = c.woff < 0 && lane == 0 ? (reach >= 32 ? ~0u : ~0u << (32 - reach)) : ~0u;
        const uint32_t hmask_r = c.woff < 0 && lane == 31 ? (reach >= 32 ? ~0u : (1u << reach) - 1u) : ~0u;
        const int odd = (pr + pc + p0) & 1;  // parity of the class faces
        const uint32_t pcm = pc ? 0xAAAAAAAAu : 0x55555555u;
        // candidates (local minima and maxima) first; the rest of the fire
        // test -- which kind, the diagonal faces -- only in warps that have
        // candidates (the frozen bulk of an early state pays the masks alone)
        // a candidate's four neighbours are all equal to the centre or all
        // different from it, i.e. equal to each other (the centre drops out)
        uint32_t cand[WPL];
        int cnt = 0;
#pragma unroll
        for (int j = 0; j < WPL; ++j) {
            const uint32_t pb = j > 0 ? b[j - 1] : bL, nb = j < WPL - 1 ? b[j + 1] : bR;
            const uint32_t left = (b[j] << 1) | (pb >> 31), right = (b[j] >> 1) | (nb << 31);
            const uint32_t act = rowok ? (cm[j] & pcm & (j == 0 ? hmask_l : ~0u) & (j == WPL - 1 ? hmask_r : ~0u)) : 0u;
            cand[j] = ~((u[j] ^ d[j]) | (u[j] ^ left) | (u[j] ^ right)) & act;
            cnt += __popc(cand[j]);
        }
        if (__any_sync(0xffffffffu, cnt != 0)) {
            uint32_t uL = __shfl_up_sync(0xffffffffu, u[WPL - 1], 1), dL = __shfl_up_sync(0xffffffffu, d[WPL - 1], 1);
            uint32_t uR = __shfl_down_sync(0xffffffffu, u[0], 1), dR = __shfl_down_sync(0xffffffffu, d[0], 1);
            if (lane == 0) uL = dL = 0u;
            if (lane == 31) {
                uR = XW && i > 0 ? rows[i - 1][RS - 1] : 0u;
                dR = XW && i + 1 < TR ? rows[i + 1][RS - 1] : 0u;
            }
            // local minima (all four neighbours one up): all equal for odd-parity
            // class faces, all different for even ones; diagonal faces differ
            // from the centre (by +-2) iff their bit differs
            uint32_t mn[WPL], nw[WPL], ne[WPL], sw[WPL], se[WPL];
#pragma unroll
            for (int j = 0; j < WPL; ++j) {
                const uint32_t pu = j > 0 ? u[j - 1] : uL, nu = j < WPL - 1 ? u[j + 1] : uR;
                const uint32_t pd = j > 0 ? d[j - 1] : dL, nd = j < WPL - 1 ? d[j + 1] : dR;
                mn[j] = cand[j] & (odd ? u[j] ^ b[j] : ~(u[j] ^ b[j]));  // neighbours one up
                nw[j] = ((u[j] << 1) | (pu >> 31)) ^ b[j];
                ne[j] = ((u[j] >> 1) | (nu << 31)) ^ b[j];
                sw[j] = ((d[j] << 1) | (pd >> 31)) ^ b[j];
                se[j] = ((d[j] >> 1) | (nd << 31)) ^ b[j];
            }
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            int pos = incl - cnt;
            // job = lane << 6 | j << 4 | bit >> 1 (a class sweep's sites all have bit
            // parity pc); the site's kind and LUT index are read from the warp's
            // masks in shared memory by whichever lane draws its coin, so the
            // serial per-lane queue loop stays short
            const uint32_t head = (uint32_t)lane << 6;
#pragma unroll
            for (int j = 0; j < WPL; ++j) {
                dmask[lane * WPL + j] = make_uint4(nw[j], ne[j], sw[j], se[j]);
                mnv[lane * WPL + j] = mn[j];
                for (uint32_t m = cand[j]; m; m &= m - 1)
                    queue[pos++] = (uint16_t)(head | ((uint32_t)j << 4) | ((uint32_t)(__ffs(m) - 1) >> 1));
                fres[lane * WPL + j] = 0u;
            }
            __syncwarp();
            const uint64_t salt = (step0 + (uint64_t)s + 1ull) * kGold;
            // site index R * f + 32 * (word) + bit, word = wl(lane 0) + lane' * WPL + j
            const uint64_t row_idx = (uint64_t)R * (uint64_t)c.f + (uint64_t)(int64_t)((wl - lane * WPL) * 32);
            __syncwarp();
            // high(x, w, b, up): u < p_high for site bit b of word w (up: a local minimum)
            auto deal = [&](auto high) {
                for (int q = lane; q < total; q += 64) {
                    const bool two = q + 32 < total;
                    const uint32_t j0 = queue[q], j1 = two ? queue[q + 32] : j0;
                    const uint32_t w0 = ((j0 >> 6) & 31u) * WPL + ((j0 >> 4) & 3u), b0 = ((j0 & 15u) << 1) | (uint32_t)pc;
                    const uint32_t w1 = ((j1 >> 6) & 31u) * WPL + ((j1 >> 4) & 3u), b1 = ((j1 & 15u) << 1) | (uint32_t)pc;
                    const uint32_t up0 = (mnv[w0] >> b0) & 1u, up1 = (mnv[w1] >> b1) & 1u;
                    const uint64_t i0 = row_idx + (uint64_t)(w0 * 32u + b0);
                    const uint64_t i1 = row_idx + (uint64_t)(w1 * 32u + b1);
                    const uint64_t x0 = mix64(mix64(base + (i0 + 1ull) * kGold) + salt);
                    const uint64_t x1 = mix64(mix64(base + (i1 + 1ull) * kGold) + salt);
                    // local min (up) moves iff u < p_high; local max moves iff u >= p_high
                    if (high(x0, w0, b0, up0) == (bool)up0) atomicOr(&fres[w0], 1u << b0);
                    if (two && high(x1, w1, b1, up1) == (bool)up1) atomicOr(&fres[w1], 1u << b1);
                }
            };
            if (c.half) {  // p_high = 1/2: (x >> 11) < 2^52 iff bit 63 of x is 0
                deal([](uint64_t x, uint32_t, uint32_t, uint32_t) { return (int32_t)(uint32_t)(x >> 32) >= 0; });
            } else {
                // LUT index (up ? 0 : 16) | nw << 3 | ne << 2 | sw << 1 | se of the site
                deal([&](uint64_t x, uint32_t w, uint32_t b, uint32_t up) {
                    const uint4 dm = dmask[w];
                    const uint32_t li = (up ? 0u : 16u) | (((dm.x >> b) & 1u) << 3) | (((dm.y >> b) & 1u) << 2) |
                                        (((dm.z >> b) & 1u) << 1) | ((dm.w >> b) & 1u);
                    return (x >> 11) < lut[li];
                });
            }
            __syncwarp();
#pragma unroll
            for (int j = 0; j < WPL; ++j) {
                const uint32_t nb = b[j] ^ fres[lane * WPL + j];
                if (pr == 0) ra[j] = nb;
                else rb[j] = nb;
                rows[i][lane * WPL + j] = nb;
            }
        }
        __syncthreads();
    }
    // store the exact rows / words
    uint32_t *dst = c.dst + (size_t)z * c.chain_words;
    const bool halo = c.woff < 0;
#pragma unroll
    for (int j = 0; j < WPL; ++j) {
        const int w = wl + j;
        bool ok = w >= 0 && w < c.W;
        if (halo && ((lane == 0 && j == 0) || (lane == 31 && j == WPL - 1))) ok = false;
        if (!ok) continue;
        if (2 * k >= c.K && 2 * k < TR - c.K && Ra < c.f && Ra >= 0) dst[(size_t)Ra * c.pitch + w] = ra[j];
        if (2 * k + 1 >= c.K && 2 * k + 1 < TR - c.K && Ra + 1 < c.f && Ra + 1 >= 0)
            dst[(size_t)(Ra + 1) * c.pitch + w] = rb[j];
    }
    if (XW && lane == 31) {
        if (2 * k >= c.K && 2 * k < TR - c.K && Ra < c.f && Ra >= 0) dst[(size_t)Ra * c.pitch + TW] = xa;
        if (2 * k + 1 >= c.K && 2 * k + 1 < TR - c.K && Ra + 1 < c.f && Ra + 1 >= 0)
            dst[(size_t)(Ra + 1) * c.pitch + TW] = xb;
    }
}

__global__ void sv_set_step(uint64_t *p, uint64_t v, uint64_t end) {  // p[0] = step, p[1] = end of the walk
    p[0] = v;
    p[1] = end;
}
__global__ void sv_advance_step(uint64_t *p, uint64_t by) { *p += by; }

// int32 heights (count, f, f) -> bits; validates |dh| == 1 across every edge.
__global__ void sv_pack_kernel(const int32_t *h, int f, int W, int pitch, size_t chain_words, uint32_t *bits,
                               int32_t *h00, int *bad) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    const int R = blockIdx.y, z = blockIdx.z;
    if (w >= W) return;
    const int32_t *g = h + (size_t)z * f * f;
    const int p0 = g[0] & 1;
    uint32_t word = 0;
    int err = 0;
    for (int b = 0; b < 32; ++b) {
        const int C = w * 32 + b;
        if (C >= f) break;
        const int32_t x = g[(size_t)R * f + C];
        if (C + 1 < f && abs(g[(size_t)R * f + C + 1] - x) != 1) err = 1;
        if (R + 1 < f && abs(g[(size_t)(R + 1) * f + C] - x) != 1) err = 1;
        const int32_t q = (x - ((R + C + p0) & 1)) >> 1;
        word |= (uint32_t)(q & 1) << b;
    }
    bits[(size_t)z * chain_words + (size_t)(R + 1) * pitch + w] = word;
    if (R == 0 && w == 0) h00[z] = g[0];
    if (err) atomicOr(bad, 1);
}

__device__ __forceinline__ int bit_of(const uint32_t *row, int C) { return (row[C >> 5] >> (C & 31)) & 1; }

// West column heights by a serial walk down column 0 (one thread per chain).
__global__ void sv_col0_kernel(const uint32_t *bits, const int32_t *h00, int f, int pitch, size_t chain_words,
                               int32_t *out) {
    const int z = blockIdx.x;
    if (threadIdx.x) return;
    const uint32_t *P = bits + (size_t)z * chain_words + pitch;
    const int p0 = h00[z] & 1;
    int32_t h = h00[z];
    int prev = bit_of(P, 0);
    out[(size_t)z * f * f] = h;
    for (int R = 1; R < f; ++R) {
        const int cur = bit_of(P + (size_t)R * pitch, 0);
        const int par = (R - 1 + p0) & 1;  // parity of face (R-1, 0)
        h += ((prev == cur) ^ par) ? 1 : -1;
        out[(size_t)z * f * f + (size_t)R * f] = h;
        prev = cur;
    }
}

// Row scan: h(R, C) = h(R, 0) + 2 * #(+1 steps before C) - C.
__global__ void sv_rows_kernel(const uint32_t *bits, const int32_t *h00, int f, int W, int pitch, size_t chain_words,
                               int32_t *out) {
    const int R = blockIdx.x, z = blockIdx.y;
    const uint32_t *row = bits + (size_t)z * chain_words + (size_t)(R + 1) * pitch;
    const int p0 = h00[z] & 1;
    int32_t *o = out + (size_t)z * f * f + (size_t)R * f;
    const int32_t h0 = o[0];
    int carry = 0;  // +1 steps in earlier chunks
    for (int w0 = 0; w0 < W; w0 += 32) {
        const int w = w0 + threadIdx.x;
        const uint32_t b = w < W ? row[w] : 0u;
        uint32_t nxt = __shfl_down_sync(0xffffffffu, b, 1);
        if (threadIdx.x == 31) nxt = w + 1 < W ? row[w + 1] : 0u;
        const uint32_t e = b ^ ((b >> 1) | (nxt << 31));               // bit C: faces C, C+1 differ
        const uint32_t par = ((R + w * 32 + p0) & 1) ? 0x55555555u : 0xAAAAAAAAu;  // odd-parity faces
        const uint32_t plus = ~(e ^ par);  // +1 step iff (bits equal) xor (odd parity)
        int cnt = 0;
        const int ncol = min(32, f - w * 32);
        uint32_t valid = ncol >= 32 ? 0xFFFFFFFFu : (ncol <= 0 ? 0u : ((1u << ncol) - 1u));
        // steps from column C to C+1 exist for C <= f-2
        const int nstep = min(32, f - 1 - w * 32);
        const uint32_t svalid = nstep >= 32 ? 0xFFFFFFFFu : (nstep <= 0 ? 0u : ((1u << nstep) - 1u));
        cnt = __popc(plus & svalid);
        int incl = cnt;
        for (int o2 = 1; o2 < 32; o2 <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o2);
            if ((int)threadIdx.x >= o2) incl += y;
        }
        const int excl = carry + incl - cnt;
        int run = excl;
        for (int b2 = 0; b2 < 32; ++b2) {
            if (!((valid >> b2) & 1u)) break;
            const int C = w * 32 + b2;
            o[C] = h0 + 2 * run - C;
            run += (plus & svalid) >> b2 & 1u;
        }
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
}

// L1 distance transform of the ring heights (sixvertex.py:534-562):
// maximal: min over ring faces of ring + |dR| + |dC|; minimal: max of ring - dist.
// Separable: columns then rows.  `ring` holds ring values, +-INF elsewhere.
__global__ void sv_dt_cols(int32_t *g, int f, int maximal) {
    const int C = blockIdx.x * blockDim.x + threadIdx.x;
    if (C >= f) return;
    const int s = maximal ? 1 : -1;
    for (int R = 1; R < f; ++R) {
        const int32_t a = g[(size_t)(R - 1) * f + C] + s, x = g[(size_t)R * f + C];
        g[(size_t)R * f + C] = maximal ? min(x, a) : max(x, a);
    }
    for (int R = f - 2; R >= 0; --R) {
        const int32_t a = g[(size_t)(R + 1) * f + C] + s, x = g[(size_t)R * f + C];
        g[(size_t)R * f + C] = maximal ? min(x, a) : max(x, a);
    }
}
__global__ void sv_dt_rows(int32_t *g, int f, int maximal) {
    const int R = blockIdx.x * blockDim.x + threadIdx.x;
    if (R >= f) return;
    const int s = maximal ? 1 : -1;
    int32_t *row = g + (size_t)R * f;
    for (int C = 1; C < f; ++C) row[C] = maximal ? min(row[C], row[C - 1] + s) : max(row[C], row[C - 1] + s);
    for (int C = f - 2; C >= 0; --C) row[C] = maximal ? min(row[C], row[C + 1] + s) : max(row[C], row[C + 1] + s);
}

__global__ void sv_replicate_kernel(uint32_t *bits, int32_t *h00, size_t chain_words, int src, int dst0, int step,
                                    int n) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= chain_words) return;
    const uint32_t v = bits[(size_t)src * chain_words + i];
    for (int k = 0; k < n; ++k) bits[(size_t)(dst0 + (size_t)k * step) * chain_words + i] = v;
    if (i == 0)
        for (int k = 0; k < n; ++k) h00[dst0 + k * step] = h00[src];
}

__global__ void __launch_bounds__(256) sv_coalesced_kernel(const uint32_t *bits, const int32_t *h00,
                                                           size_t chain_words, int chain0, uint8_t *flags) {
    const int j = blockIdx.x;
    const uint32_t *a = bits + (size_t)(chain0 + 2 * j) * chain_words;
    const uint32_t *b = a + chain_words;
    uint32_t diff = 0;
    for (size_t i = threadIdx.x; i < chain_words; i += blockDim.x) diff |= a[i] ^ b[i];
    const int any = __syncthreads_or(diff != 0);
    if (threadIdx.x == 0) flags[j] = (any || h00[chain0 + 2 * j] != h00[chain0 + 2 * j + 1]) ? 0 : 1;
}

constexpr int kSvGraphSweeps = 128;  // sweeps per graph replay

// Tile geometry of sv_multi_kernel: rows of W <= 128 words fit one column
// tile (WPL = ceil(W/32) words per lane, no word halo); wider grids use
// 4 words per lane with a one-word halo on each side.  K sweeps per launch
// (even, dividing kSvGraphSweeps with an even number of launches per replay)
// and NW warps per block; TSB_SV_K / TSB_SV_NW override them for tuning.
static int getenv_int(const char *name, int dflt) {
    const char *e = getenv(name);
    return e ? atoi(e) : dflt;
}

void sv_multi_config(tsb_sv *h) {
    int force = 0;
    if (const char *e = getenv("TSB_SV_WPL")) force = atoi(e);
    if (force >= 1 && force <= 4) {
        h->m_wpl = force;
        h->m_woff = -1;
        h->m_stride = 32 * force - 2;
        h->m_gx = (h->W + h->m_stride - 1) / h->m_stride;
    } else if (h->W <= 129 && h->W % 32 == 1 && h->n % 32 == 0 && getenv_int("TSB_SV_XW", 1)) {
        // the last word holds only the east boundary column n (bit 0 of word
        // n / 32): 32 * WPL words per row on 32 lanes, the boundary word read-only
        // (DWBC 2048: 2 words per lane instead of 3 on 22 lanes)
        h->m_wpl = (h->W - 1) / 32;
        h->m_xw = 1;
        h->m_woff = 0;
        h->m_stride = 32 * h->m_wpl;
        h->m_gx = 1;
    } else if (h->W <= 128) {
        h->m_wpl = (h->W + 31) / 32;
        h->m_woff = 0;
        h->m_stride = 32 * h->m_wpl;
        h->m_gx = 1;
    } else {
        h->m_wpl = 4;
        h->m_woff = -1;
        h->m_stride = 32 * 4 - 2;
        h->m_gx = (h->W + h->m_stride - 1) / h->m_stride;
    }
    int nw = 16, K = 8;
    cudaDeviceGetAttribute(&h->m_sms, cudaDevAttrMultiProcessorCount, h->device);
    // a single chain that fits one wave either way: 15 warps (14 exact rows per
    // tile at K = 8) spread it over more SMs than 16 (DWBC 2048: 147 instead of
    // 129 blocks; 1.83 -> 1.78 us per sweep at Delta = 1/2, 2.24 -> 2.16 at -3)
    if (h->nchains == 1) {
        const int b16 = h->m_gx * ((h->f + 15) / 16), b15 = h->m_gx * ((h->f + 13) / 14);
        if (b15 <= h->m_sms && b15 > b16) nw = 15;
    }
    if (const char *e = getenv("TSB_SV_NW")) nw = atoi(e) == 16 ? 16 : atoi(e) == 15 ? 15 : 8;
    if (const char *e = getenv("TSB_SV_K")) {
        K = atoi(e);
        h->m_k_fixed = true;
    }
    if (K != 2 && K != 4 && K != 8 && K != 16) K = 4;
    while (2 * nw - 2 * K < 2) K /= 2;
    h->m_nw = nw;
    h->m_K = K;
    h->m_out = 2 * nw - 2 * K;
    h->m_gy = (h->f + h->m_out - 1) / h->m_out;
}

// Sweeps per launch for a batch of n chains: a single lattice is latency
// bound and takes K = 8 (fewer launches); once the batch fills two waves
// with K = 4 tiles the halo redundancy dominates and K = 4 (24 of 32 rows
// exact) is faster (DWBC 2048 x 32 chains: 0.20 -> 0.27 of the roofline).
static int sv_k(const tsb_sv *h, int n) {
    if (h->m_k_fixed || h->m_K != 8 || 2 * h->m_nw - 8 < 2) return h->m_K;
    const int out4 = 2 * h->m_nw - 8;
    const int64_t blocks = (int64_t)n * h->m_gx * ((h->f + out4 - 1) / out4);
    return blocks >= 2 * (int64_t)h->m_sms ? 4 : 8;
}

// A launch of at most one block per SM reserves more than half an SM's
// shared memory per block, so the scheduler spreads the blocks over all SMs
// instead of packing two onto one (single chains of the DWBC 2048 lattice:
// 129 blocks); larger launches pack as tightly as registers allow.
constexpr size_t kSvSpreadSmem = 116 * 1024;

template <int WPL, int NW>
static int sv_launch_multi_t(const cudaLaunchConfig_t &cfg0, const SvMCtx &c, int sms) {
    constexpr size_t smem = sv_multi_smem<WPL, NW>();
    const size_t blocks = (size_t)cfg0.gridDim.x * cfg0.gridDim.y * cfg0.gridDim.z;
    const size_t use = blocks <= (size_t)sms ? std::max(smem, kSvSpreadSmem) : smem;
    cudaLaunchConfig_t cfg = cfg0;
    cfg.blockDim = dim3(32 * NW);
    cfg.dynamicSmemBytes = use;
    static const int dense_env = [] {
        const char *ev = getenv("TSB_SV_DENSE");  // 0 / 1: force the 1- / 2-blocks-per-SM build
        return ev ? atoi(ev) : -1;
    }();
    const bool dense = NW == 16 && (dense_env >= 0 ? dense_env == 1 : blocks > 4 * (size_t)sms);
    auto go = [&](auto kern) -> int {
        TSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)use));
        TSB_CUDA(cudaLaunchKernelEx(&cfg, kern, c));
        return TSB_OK;
    };
    if (c.xw) return dense ? go(sv_multi_kernel<WPL, NW, 2, true>) : go(sv_multi_kernel<WPL, NW, 1, true>);
    return dense ? go(sv_multi_kernel<WPL, NW, 2>) : go(sv_multi_kernel<WPL, NW>);
}

// One temporally blocked launch (m_K sweeps) of chains [chain0, chain0+n).
static int sv_launch_multi(tsb_sv *h, int chain0, int n, uint64_t step_off, const uint32_t *src, uint32_t *dst,
                           cudaStream_t stream) {
    SvMCtx c;
    c.src = src + (size_t)chain0 * h->chain_words + h->pitch;
    c.dst = dst + (size_t)chain0 * h->chain_words + h->pitch;
    c.h00 = h->h00 + chain0;
    c.seedinfo = h->seedinfo;
    c.step_dev = h->step_dev;
    c.chain_words = h->chain_words;
    c.n = h->n;
    c.f = h->f;
    c.W = h->W;
    c.pitch = h->pitch;
    c.K = sv_k(h, n);
    c.collapse = h->collapse;
    c.out_rows = 2 * h->m_nw - 2 * c.K;
    c.stride = h->m_stride;
    c.woff = h->m_woff;
    c.xw = h->m_xw;
    c.step = step_off;
    c.half = 1;
    for (int i = 0; i < 32; ++i) {
        c.lut[i] = h->lut[i];
        c.half &= h->lut[i] == (1ull << 52);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(h->m_gx, (h->f + c.out_rows - 1) / c.out_rows, n);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const int key = h->m_wpl * 100 + h->m_nw;
    switch (key) {
        case 108: return sv_launch_multi_t<1, 8>(cfg, c, h->m_sms);
        case 208: return sv_launch_multi_t<2, 8>(cfg, c, h->m_sms);
        case 308: return sv_launch_multi_t<3, 8>(cfg, c, h->m_sms);
        case 408: return sv_launch_multi_t<4, 8>(cfg, c, h->m_sms);
        case 116: return sv_launch_multi_t<1, 16>(cfg, c, h->m_sms);
        case 216: return sv_launch_multi_t<2, 16>(cfg, c, h->m_sms);
        case 316: return sv_launch_multi_t<3, 16>(cfg, c, h->m_sms);
        case 315: return sv_launch_multi_t<3, 15>(cfg, c, h->m_sms);
        case 215: return sv_launch_multi_t<2, 15>(cfg, c, h->m_sms);
        case 115: return sv_launch_multi_t<1, 15>(cfg, c, h->m_sms);
        default: return sv_launch_multi_t<4, 16>(cfg, c, h->m_sms);
    }
}

// Graph of kSvGraphSweeps sweeps: an even number of out-of-place launches
// (bits -> bits2 -> bits ...), then step += kSvGraphSweeps.
static int sv_ensure_graph(tsb_sv *h, int chain0, int n) {
    if (h->graph_exec && h->g_chain0 == chain0 && h->g_n == n && h->g_lut_version == h->lut_version &&
        h->g_collapse == h->collapse)
        return TSB_OK;
    if (h->graph_exec) {
        cudaGraphExecDestroy(h->graph_exec);
        h->graph_exec = nullptr;
    }
    if (!h->cap_stream) TSB_CUDA(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    TSB_CUDA(cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal));
    int rc = TSB_OK;
    const int K = sv_k(h, n), launches = kSvGraphSweeps / K;
    for (int i = 0; i < launches && !rc; ++i)
        rc = sv_launch_multi(h, chain0, n, (uint64_t)i * K, (i & 1) ? h->bits2 : h->bits,
                             (i & 1) ? h->bits : h->bits2, h->cap_stream);
    sv_advance_step<<<1, 1, 0, h->cap_stream>>>(h->step_dev, (uint64_t)kSvGraphSweeps);
    cudaError_t e = cudaStreamEndCapture(h->cap_stream, &g);
    if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    if (e != cudaSuccess) return cuda_fail(e, "sv graph capture");
    e = cudaGraphInstantiate(&h->graph_exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
        h->graph_exec = nullptr;
        return cuda_fail(e, "sv graph instantiate");
    }
    h->g_chain0 = chain0;
    h->g_n = n;
    h->g_lut_version = h->lut_version;
    h->g_collapse = h->collapse;
    return TSB_OK;
}

// On-device observables (stats.py:213-245 density_map of "h-edge", "v-edge",
// "c-vertex").  Edge occupancies from the 1-bit state: between faces X -> Y,
// Y = X + 1 iff (bit X == bit Y) xor (X has odd parity);
//   v_edges[r, c] = h(r, c+1) - h(r, c) == 1          (sixvertex.py:270-277)
//   h_edges[r, c] = h(r, c) - h(r+1, c) == 1
//   c-vertex (r, c): code W + 2E + 4N + 8S in {0b1001, 0b0110} with
//   W = h_edges[r, c], E = h_edges[r, c+1], N = v_edges[r, c], S = v_edges[r+1, c]
//   (vertex_type_codes, sixvertex.py:236-239; stats.py:225-228).
__device__ __forceinline__ uint32_t sv_odd_mask(int r, int p0) {  // bit b: (r + b + p0) odd (32w is even)
    return ((r + p0) & 1) ? 0x55555555u : 0xAAAAAAAAu;
}
__device__ __forceinline__ uint32_t sv_vedge(const uint32_t *row, int w, int r, int p0) {
    const uint32_t b = row[w], bn = (b >> 1) | (row[w + 1] << 31);
    return ~(b ^ bn) ^ sv_odd_mask(r, p0);
}
__device__ __forceinline__ uint32_t sv_hedge(const uint32_t *row, const uint32_t *below, int w, int r, int p0) {
    return ~(row[w] ^ below[w]) ^ sv_odd_mask(r + 1, p0);
}

// obs 0: h-edge (n, n+1); 1: v-edge (n+1, n); 2: c-vertex (n, n).  One thread
// per (row, 32-site word), chains summed in registers.
__global__ void sv_observe_kernel(const uint32_t *bits, const int32_t *h00, size_t chain_words, int pitch, int nchains,
                                  int n, int obs, uint32_t *acc) {
    const int rows = obs == 1 ? n + 1 : n, cols = obs == 0 ? n + 1 : n;
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y;
    if (r >= rows || w * 32 >= cols) return;
    uint32_t cnt[32];
#pragma unroll
    for (int b = 0; b < 32; ++b) cnt[b] = 0;
    for (int z = 0; z < nchains; ++z) {
        const uint32_t *P = bits + (size_t)z * chain_words + pitch;  // face row 0
        const uint32_t *row = P + (size_t)r * pitch;
        const int p0 = h00[z] & 1;
        uint32_t m;
        if (obs == 0) {
            m = sv_hedge(row, row + pitch, w, r, p0);
        } else if (obs == 1) {
            m = sv_vedge(row, w, r, p0);
        } else {
            const uint32_t hw = sv_hedge(row, row + pitch, w, r, p0);
            const uint32_t he = (hw >> 1) | (sv_hedge(row, row + pitch, w + 1, r, p0) << 31);
            const uint32_t vn = sv_vedge(row, w, r, p0), vs = sv_vedge(row + pitch, w, r + 1, p0);
            m = (hw & ~he & ~vn & vs) | (~hw & he & vn & ~vs);
        }
#pragma unroll
        for (int b = 0; b < 32; ++b) cnt[b] += (m >> b) & 1u;
    }
    uint32_t *a = acc + (size_t)r * cols + (size_t)w * 32;
    const int lim = min(32, cols - w * 32);
#pragma unroll
    for (int b = 0; b < 32; ++b)
        if (b < lim) a[b] += cnt[b];
}

// Sum of face heights over chains (mean height function), int64 per face.
__global__ void sv_height_sum_kernel(const int32_t *h, int nchains, size_t nf, long long *acc) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= nf) return;
    long long s = 0;
    for (int z = 0; z < nchains; ++z) s += h[(size_t)z * nf + i];
    acc[i] += s;
}

// Archive record (stats.py:146-153): h_edges (n, n+1) then v_edges (n+1, n)
// ravelled as '0'/'1' characters; thread per (row, 32-site word).
__global__ void sv_serialize_kernel(const uint32_t *bits, int p0, int pitch, int n, char *out) {
    const int part = blockIdx.z;  // 0: h_edges, 1: v_edges
    const int rows = part ? n + 1 : n, cols = part ? n : n + 1;
    const int w = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y;
    if (r >= rows || w * 32 >= cols) return;
    const uint32_t *row = bits + pitch + (size_t)r * pitch;  // face row r (after the guard row)
    const uint32_t m = part ? sv_vedge(row, w, r, p0) : sv_hedge(row, row + pitch, w, r, p0);
    char *o = out + (part ? (size_t)n * (n + 1) : 0) + (size_t)r * cols + (size_t)w * 32;
    const int lim = min(32, cols - w * 32);
    for (int b = 0; b < lim; ++b) o[b] = ((m >> b) & 1u) ? '1' : '0';
}

int sv_check(tsb_sv *h, int chain0, int n) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    if (chain0 < 0 || n < 0 || chain0 + n > h->nchains)
        return fail(TSB_E_VALUE, "chains [%d, %d) outside the handle's %d chains", chain0, chain0 + n, h->nchains);
    return TSB_OK;
}

int sv_hbuf(tsb_sv *h, size_t count) {
    const size_t need = count * (size_t)h->f * h->f * sizeof(int32_t);
    if (h->hbuf_cap >= need) return TSB_OK;
    TSB_CUDA(cudaStreamSynchronize(h->stream));
    cudaFree(h->hbuf);
    h->hbuf = nullptr;
    TSB_CUDA(cudaMalloc(&h->hbuf, need));
    h->hbuf_cap = need;
    return TSB_OK;
}

int sv_pack_dev(tsb_sv *h, int chain0, int n, const int32_t *dsrc) {
    TSB_CUDA(cudaMemsetAsync(h->flag, 0, sizeof(int), h->stream));
    sv_pack_kernel<<<dim3((h->W + 127) / 128, h->f, n), 128, 0, h->stream>>>(
        dsrc, h->f, h->W, h->pitch, h->chain_words, h->bits + (size_t)chain0 * h->chain_words, h->h00 + chain0,
        h->flag);
    TSB_CUDA(cudaGetLastError());
    int bad = 0;
    TSB_CUDA(cudaMemcpyAsync(&bad, h->flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    TSB_CUDA(cudaStreamSynchronize(h->stream));
    if (bad) return fail(TSB_E_INCONSISTENT, "adjacent faces must differ by exactly 1");
    return TSB_OK;
}

int sv_unpack_dev(tsb_sv *h, int chain0, int n, int32_t *dout) {
    const uint32_t *b = h->bits + (size_t)chain0 * h->chain_words;
    sv_col0_kernel<<<n, 32, 0, h->stream>>>(b, h->h00 + chain0, h->f, h->pitch, h->chain_words, dout);
    sv_rows_kernel<<<dim3(h->f, n), 32, 0, h->stream>>>(b, h->h00 + chain0, h->f, h->W, h->pitch, h->chain_words,
                                                       dout);
    TSB_CUDA(cudaGetLastError());
    return TSB_OK;
}

}  // namespace tsb

using namespace tsb;

extern "C" {

int tsb_sv_create(int device, int n, int nchains, tsb_sv **out) {
    if (!out) return fail(TSB_E_VALUE, "null output pointer");
    *out = nullptr;
    if (n < 1 || nchains < 1) return fail(TSB_E_VALUE, "n and nchains must be positive");
    if ((uint64_t)(n + 1) * (uint64_t)(n + 1) >= kCapacity) return fail(TSB_E_CAPACITY, "grid exceeds capacity");
    int rc = ensure_device(device);
    if (rc) return rc;
    tsb_sv *h = new tsb_sv();
    h->device = device;
    h->n = n;
    h->f = n + 1;
    h->nchains = nchains;
    h->W = (h->f + 31) / 32;
    h->pitch = (h->W + 31) / 32 * 32;
    h->chain_words = (size_t)(h->f + 2) * h->pitch;
    cudaError_t e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
    h->own_stream = true;
    if (e == cudaSuccess) e = cudaMalloc(&h->bits, sizeof(uint32_t) * h->chain_words * nchains);
    if (e == cudaSuccess) e = cudaMemset(h->bits, 0, sizeof(uint32_t) * h->chain_words * nchains);
    if (e == cudaSuccess) e = cudaMalloc(&h->h00, sizeof(int32_t) * nchains);
    if (e == cudaSuccess) e = cudaMemset(h->h00, 0, sizeof(int32_t) * nchains);
    if (e == cudaSuccess) e = cudaMalloc(&h->seedinfo, sizeof(uint64_t) * 2 * nchains);
    if (e == cudaSuccess) e = cudaMallocHost(&h->seed_pinned, sizeof(uint64_t) * 2 * nchains);
    if (e == cudaSuccess) e = cudaMalloc(&h->flag, sizeof(int));
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->seed_ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(h->seed_ev, h->stream);
    if (e == cudaSuccess) e = cudaMalloc(&h->bits2, sizeof(uint32_t) * h->chain_words * nchains);
    if (e == cudaSuccess) e = cudaMemset(h->bits2, 0, sizeof(uint32_t) * h->chain_words * nchains);
    if (e == cudaSuccess) e = cudaMalloc(&h->step_dev, 2 * sizeof(uint64_t));
    for (int i = 0; i < 32; ++i) h->lut[i] = 1ull << 52;
    sv_multi_config(h);
    if (const char *ev = getenv("TSB_SV_COLLAPSE")) h->collapse = atoi(ev) != 0;
    if (e != cudaSuccess) {
        int code = cuda_fail(e, "tsb_sv_create");
        tsb_sv_destroy(h);
        return code;
    }
    *out = h;
    return TSB_OK;
}

int tsb_sv_destroy(tsb_sv *h) {
    if (!h) return TSB_OK;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    cudaFree(h->bits);
    cudaFree(h->h00);
    cudaFree(h->seedinfo);
    cudaFree(h->hbuf);
    cudaFree(h->flag);
    cudaFree(h->bits2);
    cudaFree(h->step_dev);
    if (h->graph_exec) cudaGraphExecDestroy(h->graph_exec);
    if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
    if (h->seed_pinned) cudaFreeHost(h->seed_pinned);
    if (h->seed_ev) cudaEventDestroy(h->seed_ev);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    delete h;
    return TSB_OK;
}

int tsb_sv_set_stream(tsb_sv *h, void *stream) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    TSB_CUDA(cudaSetDevice(h->device));
    TSB_CUDA(cudaStreamSynchronize(h->stream));
    if (h->own_stream) cudaStreamDestroy(h->stream);
    h->stream = (cudaStream_t)stream;
    h->own_stream = false;
    return TSB_OK;
}

int tsb_sv_set_p_high(tsb_sv *h, const double *p_high) {
    if (!h || !p_high) return fail(TSB_E_VALUE, "null argument");
    for (int i = 0; i < 32; ++i) h->lut[i] = threshold_of(p_high[i]);
    ++h->lut_version;
    return TSB_OK;
}

int tsb_sv_upload(tsb_sv *h, int chain0, int n, const int32_t *heights) {
    int rc = sv_check(h, chain0, n);
    if (rc || n == 0) return rc;
    TSB_CUDA(cudaSetDevice(h->device));
    if ((rc = sv_hbuf(h, n))) return rc;
    if ((rc = staged_h2d(h->hbuf, heights, sizeof(int32_t) * (size_t)n * h->f * h->f, h->stream))) return rc;
    return sv_pack_dev(h, chain0, n, h->hbuf);
}

int tsb_sv_download(tsb_sv *h, int chain0, int n, int32_t *heights) {
    int rc = sv_check(h, chain0, n);
    if (rc || n == 0) return rc;
    TSB_CUDA(cudaSetDevice(h->device));
    if ((rc = sv_hbuf(h, n))) return rc;
    if ((rc = sv_unpack_dev(h, chain0, n, h->hbuf))) return rc;
    return staged_d2h(heights, h->hbuf, sizeof(int32_t) * (size_t)n * h->f * h->f, h->stream);
}

static int sv_walk_impl(tsb_sv *h, int chain0, int n, const uint64_t *seeds, uint64_t step0, uint64_t n_steps,
                        int class_override) {
    int rc = sv_check(h, chain0, n);
    if (rc || n == 0 || n_steps == 0) return rc;
    if (!seeds) return fail(TSB_E_VALUE, "null seeds");
    TSB_CUDA(cudaSetDevice(h->device));
    TSB_CUDA(cudaEventSynchronize(h->seed_ev));
    for (int i = 0; i < n; ++i) {
        const uint64_t b = family_base(seeds[i]);
        h->seed_pinned[2 * i] = b;
        h->seed_pinned[2 * i + 1] = global_key(b);
    }
    TSB_CUDA(cudaMemcpyAsync(h->seedinfo, h->seed_pinned, sizeof(uint64_t) * 2 * n, cudaMemcpyHostToDevice,
                             h->stream));
    TSB_CUDA(cudaEventRecord(h->seed_ev, h->stream));
    if (h->n < 2) return TSB_OK;  // no interior faces
    SvCtx c;
    c.bits = h->bits + (size_t)chain0 * h->chain_words;
    c.h00 = h->h00 + chain0;
    c.seedinfo = h->seedinfo;
    c.chain_words = h->chain_words;
    c.n = h->n;
    c.f = h->f;
    c.W = h->W;
    c.pitch = h->pitch;
    c.class_override = class_override;
    for (int i = 0; i < 32; ++i) c.lut[i] = h->lut[i];
    const int class_rows = (h->f + 1) / 2;
    const int warps = 8;
    dim3 grid((h->W + 31) / 32, (class_rows + warps - 1) / warps, n);
    uint64_t done = 0;
    const uint64_t replays = class_override < 0 ? n_steps / kSvGraphSweeps : 0;
    if (replays) {
        if ((rc = sv_ensure_graph(h, chain0, n))) return rc;
        sv_set_step<<<1, 1, 0, h->stream>>>(h->step_dev, step0, step0 + n_steps);
        for (uint64_t r = 0; r < replays; ++r) TSB_CUDA(cudaGraphLaunch(h->graph_exec, h->stream));
        done = replays * kSvGraphSweeps;
    }
    const uint64_t Kn = (uint64_t)sv_k(h, n);
    if (class_override < 0 && n_steps - done >= Kn) {
        // remainder: direct multi-sweep launches bits -> bits2 -> ..., step_dev = step0 + done
        if (done == 0) sv_set_step<<<1, 1, 0, h->stream>>>(h->step_dev, step0, step0 + n_steps);
        int launches = 0;
        for (uint64_t i = 0; done + Kn <= n_steps; done += Kn, i += Kn, ++launches)
            if ((rc = sv_launch_multi(h, chain0, n, i, (launches & 1) ? h->bits2 : h->bits,
                                      (launches & 1) ? h->bits : h->bits2, h->stream)))
                return rc;
        if (launches & 1)
            TSB_CUDA(cudaMemcpyAsync(h->bits + (size_t)chain0 * h->chain_words,
                                     h->bits2 + (size_t)chain0 * h->chain_words,
                                     sizeof(uint32_t) * h->chain_words * n, cudaMemcpyDeviceToDevice, h->stream));
    }
    for (uint64_t s = done; s < n_steps; ++s) {
        c.step = step0 + s;
        sv_sweep_kernel<<<grid, 32 * warps, 0, h->stream>>>(c);
    }
    TSB_CUDA(cudaGetLastError());
    return TSB_OK;
}

int tsb_sv_walk(tsb_sv *h, int chain0, int n, const uint64_t *seeds, uint64_t step0, uint64_t n_steps) {
    return sv_walk_impl(h, chain0, n, seeds, step0, n_steps, -1);
}

int tsb_sv_sweep(tsb_sv *h, int chain0, int n, const uint64_t *seeds, uint64_t step, int face_class) {
    if (face_class < 0 || face_class > 3) return fail(TSB_E_VALUE, "face class must be in 0..3");
    return sv_walk_impl(h, chain0, n, seeds, step, 1, face_class);
}

int tsb_sv_sync(tsb_sv *h) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    TSB_CUDA(cudaSetDevice(h->device));
    TSB_CUDA(cudaStreamSynchronize(h->stream));
    return TSB_OK;
}

// Extremal heights from the boundary ring (`ring`: (f, f) int32 with the ring
// heights of _ring_heights, interior ignored) into chains chain_max/chain_min;
// heights also returned through hmax/hmin (nullable).  TSB_E_INFEASIBLE when
// the ring heights are mutually incompatible (InfeasibleBoundary).
int tsb_sv_extremal(tsb_sv *h, const int32_t *ring, int chain_max, int chain_min, int32_t *hmax, int32_t *hmin) {
    if (!h || !ring) return fail(TSB_E_VALUE, "null argument");
    int rc = sv_check(h, chain_max, 1);
    if (!rc) rc = sv_check(h, chain_min, 1);
    if (rc) return rc;
    TSB_CUDA(cudaSetDevice(h->device));
    const int f = h->f;
    const size_t nf = (size_t)f * f;
    std::vector<int32_t> g(nf);
    int32_t *dg = nullptr;
    TSB_CUDA(cudaMalloc(&dg, nf * sizeof(int32_t)));
    for (int pass = 0; pass < 2; ++pass) {
        const int maximal = pass == 0;
        const int32_t inf = maximal ? (1 << 29) : -(1 << 29);
        for (int R = 0; R < f; ++R)
            for (int C = 0; C < f; ++C) {
                const bool on = R == 0 || C == 0 || R == f - 1 || C == f - 1;
                g[(size_t)R * f + C] = on ? ring[(size_t)R * f + C] : inf;
            }
        cudaMemcpyAsync(dg, g.data(), nf * sizeof(int32_t), cudaMemcpyHostToDevice, h->stream);
        sv_dt_cols<<<(f + 127) / 128, 128, 0, h->stream>>>(dg, f, maximal);
        sv_dt_rows<<<(f + 127) / 128, 128, 0, h->stream>>>(dg, f, maximal);
        cudaMemcpyAsync(g.data(), dg, nf * sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream);
        cudaError_t e = cudaStreamSynchronize(h->stream);
        if (e != cudaSuccess) {
            cudaFree(dg);
            return cuda_fail(e, "sv extremal");
        }
        for (int R = 0; R < f; ++R)
            for (int C = 0; C < f; ++C)
                if ((R == 0 || C == 0 || R == f - 1 || C == f - 1) && g[(size_t)R * f + C] != ring[(size_t)R * f + C]) {
                    cudaFree(dg);
                    return fail(TSB_E_INFEASIBLE, "ring heights are mutually incompatible");
                }
        if ((rc = sv_pack_dev(h, maximal ? chain_max : chain_min, 1, dg))) {
            cudaFree(dg);
            return rc;
        }
        int32_t *dst = maximal ? hmax : hmin;
        if (dst) std::copy(g.begin(), g.end(), dst);
    }
    cudaFree(dg);
    return TSB_OK;
}

int tsb_sv_set_collapse(tsb_sv *h, int on) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    h->collapse = on ? 1 : 0;
    return TSB_OK;
}

int tsb_sv_observe_add(tsb_sv *h, int chain0, int n, int observable, uint32_t *acc_dev) {
    int rc = sv_check(h, chain0, n);
    if (rc || n == 0) return rc;
    if (!acc_dev) return fail(TSB_E_VALUE, "null accumulator");
    if (observable < 0 || observable > 2) return fail(TSB_E_VALUE, "observable must be 0 (h-edge), 1 (v-edge), 2 (c-vertex)");
    TSB_CUDA(cudaSetDevice(h->device));
    const int rows = observable == 1 ? h->n + 1 : h->n, cols = observable == 0 ? h->n + 1 : h->n;
    const int W = (cols + 31) / 32;
    sv_observe_kernel<<<dim3((W + 63) / 64, rows), 64, 0, h->stream>>>(h->bits + (size_t)chain0 * h->chain_words,
                                                                       h->h00 + chain0, h->chain_words, h->pitch, n,
                                                                       h->n, observable, acc_dev);
    TSB_CUDA(cudaGetLastError());
    return TSB_OK;
}

int tsb_sv_height_sum_add(tsb_sv *h, int chain0, int n, long long *acc_dev) {
    int rc = sv_check(h, chain0, n);
    if (rc || n == 0) return rc;
    if (!acc_dev) return fail(TSB_E_VALUE, "null accumulator");
    TSB_CUDA(cudaSetDevice(h->device));
    if ((rc = sv_hbuf(h, n))) return rc;
    if ((rc = sv_unpack_dev(h, chain0, n, h->hbuf))) return rc;
    const size_t nf = (size_t)h->f * h->f;
    sv_height_sum_kernel<<<(unsigned)((nf + 255) / 256), 256, 0, h->stream>>>(h->hbuf, n, nf, acc_dev);
    TSB_CUDA(cudaGetLastError());
    return TSB_OK;
}

int tsb_sv_serialize(tsb_sv *h, int chain, char *out, size_t cap, size_t *len) {
    if (!h || !len) return fail(TSB_E_VALUE, "null argument");
    int rc = sv_check(h, chain, 1);
    if (rc) return rc;
    const size_t total = 2 * (size_t)h->n * (h->n + 1);
    *len = total;
    if (!out || cap < total) return TSB_OK;  // size query
    TSB_CUDA(cudaSetDevice(h->device));
    int32_t p00 = 0;
    TSB_CUDA(cudaMemcpyAsync(&p00, h->h00 + chain, sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream));
    TSB_CUDA(cudaStreamSynchronize(h->stream));
    if ((rc = sv_hbuf(h, 1))) return rc;  // handle scratch (f^2 int32 >= total bytes): no allocation per record
    char *d = reinterpret_cast<char *>(h->hbuf);
    const int W = (h->n + 1 + 31) / 32;
    sv_serialize_kernel<<<dim3((W + 63) / 64, h->n + 1, 2), 64, 0, h->stream>>>(
        h->bits + (size_t)chain * h->chain_words, p00 & 1, h->pitch, h->n, d);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, total, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "sv serialize");
    return TSB_OK;
}

int tsb_sv_coalesced(tsb_sv *h, int chain0, int npairs, uint8_t *flags) {
    int rc = sv_check(h, chain0, 2 * npairs);
    if (rc || npairs == 0) return rc;
    TSB_CUDA(cudaSetDevice(h->device));
    if ((rc = sv_hbuf(h, ((size_t)npairs + 4 * (size_t)h->f * h->f - 1) / (4 * (size_t)h->f * h->f)))) return rc;
    uint8_t *d = reinterpret_cast<uint8_t *>(h->hbuf);
    sv_coalesced_kernel<<<npairs, 256, 0, h->stream>>>(h->bits, h->h00, h->chain_words, chain0, d);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(flags, d, npairs, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "sv coalesced");
    return TSB_OK;
}

int tsb_sv_replicate(tsb_sv *h, int src, int dst0, int step, int n) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    if (n <= 0) return TSB_OK;
    if (src < 0 || src >= h->nchains || dst0 < 0 || step < 1 || dst0 + (int64_t)(n - 1) * step >= h->nchains)
        return fail(TSB_E_VALUE, "replicate chains out of range");
    TSB_CUDA(cudaSetDevice(h->device));
    sv_replicate_kernel<<<(unsigned)((h->chain_words + 255) / 256), 256, 0, h->stream>>>(h->bits, h->h00,
                                                                                       h->chain_words, src, dst0,
                                                                                       step, n);
    TSB_CUDA(cudaGetLastError());
    return TSB_OK;
}

// sv_cftp (sixvertex.py:565-622) on the device; same layout and schedule as
// tsb_domino_cftp.  Templates: chain 2*count = h_max, 2*count+1 = h_min.
int tsb_sv_cftp(tsb_sv *h, const int32_t *top0, const int32_t *bot0, const uint64_t *masters, int count,
                int max_doublings, int32_t *out_heights, int32_t *collapsed_round, tsb_progress_fn progress,
                void *user) {
    if (!h || !top0 || !bot0 || !masters || !out_heights) return fail(TSB_E_VALUE, "null argument");
    if (count <= 0) return TSB_OK;
    if (h->nchains < 2 * count + 2)
        return fail(TSB_E_VALUE, "handle needs >= %d chains for %d samples", 2 * count + 2, count);
    const int T = 2 * count, B = 2 * count + 1;
    int rc;
    if ((rc = tsb_sv_upload(h, T, 1, top0))) return rc;
    if ((rc = tsb_sv_upload(h, B, 1, bot0))) return rc;
    const size_t grid = (size_t)h->f * h->f;
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
        if ((rc = tsb_sv_replicate(h, T, 0, 2, na))) return rc;
        if ((rc = tsb_sv_replicate(h, B, 1, 2, na))) return rc;
        for (int i = round_no; i >= 1; --i) {
            seeds.assign(2 * na, 0);
            for (int j = 0; j < na; ++j)
                seeds[2 * j] = seeds[2 * j + 1] =
                    mix64(mix64(masters[active[j]] ^ (kSalt * kMul)) + ((uint64_t)i + 1ull) * kGold);
            if ((rc = tsb_sv_walk(h, 0, 2 * na, seeds.data(), 0, 1ull << i))) return rc;
        }
        flags.assign(na, 0);
        if ((rc = tsb_sv_coalesced(h, 0, na, flags.data()))) return rc;
        std::vector<int> still;
        for (int j = 0; j < na; ++j) {
            if (flags[j]) {
                const int k = active[j];
                if ((rc = tsb_sv_download(h, 2 * j + 1, 1, out_heights + (size_t)k * grid))) return rc;
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
