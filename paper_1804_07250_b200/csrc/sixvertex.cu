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
    for (int i = 0; i < 32; ++i) h->lut[i] = 1ull << 52;
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
    return TSB_OK;
}

int tsb_sv_upload(tsb_sv *h, int chain0, int n, const int32_t *heights) {
    int rc = sv_check(h, chain0, n);
    if (rc || n == 0) return rc;
    TSB_CUDA(cudaSetDevice(h->device));
    if ((rc = sv_hbuf(h, n))) return rc;
    TSB_CUDA(cudaMemcpyAsync(h->hbuf, heights, sizeof(int32_t) * (size_t)n * h->f * h->f, cudaMemcpyHostToDevice,
                             h->stream));
    return sv_pack_dev(h, chain0, n, h->hbuf);
}

int tsb_sv_download(tsb_sv *h, int chain0, int n, int32_t *heights) {
    int rc = sv_check(h, chain0, n);
    if (rc || n == 0) return rc;
    TSB_CUDA(cudaSetDevice(h->device));
    if ((rc = sv_hbuf(h, n))) return rc;
    if ((rc = sv_unpack_dev(h, chain0, n, h->hbuf))) return rc;
    TSB_CUDA(cudaMemcpyAsync(heights, h->hbuf, sizeof(int32_t) * (size_t)n * h->f * h->f, cudaMemcpyDeviceToHost,
                             h->stream));
    TSB_CUDA(cudaStreamSynchronize(h->stream));
    return TSB_OK;
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
    for (uint64_t s = 0; s < n_steps; ++s) {
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

int tsb_sv_coalesced(tsb_sv *h, int chain0, int npairs, uint8_t *flags) {
    int rc = sv_check(h, chain0, 2 * npairs);
    if (rc || npairs == 0) return rc;
    TSB_CUDA(cudaSetDevice(h->device));
    uint8_t *d = nullptr;
    TSB_CUDA(cudaMalloc(&d, npairs));
    sv_coalesced_kernel<<<npairs, 256, 0, h->stream>>>(h->bits, h->h00, h->chain_words, chain0, d);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(flags, d, npairs, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    cudaFree(d);
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
