// Domino height export (K6) and Thurston extremal tilings (K8).
//
// Both are shortest-path fixpoints on the vertex graph rooted at the domain's
// reference vertex, solved by a tiled min-plus (max-plus) relaxation:
//   K6  height_function   (lattice.py:537-580): exact edge steps; for a
//       consistent state every path gives the same sum, so the fixpoint IS the
//       height function; an inconsistent state has a negative cycle, detected
//       by the value bound -> InconsistencyError.
//   K8  extremal_tilings  (lattice.py:639-754, _relax/_edge_bound_grids): the
//       upper (lower) step bounds; the unique fixpoint is h_max (h_min), decoded
//       by "|dh| == 3 on an edge => crossed" (tiling_from_heights 598-620).
// Any correct relaxation order reaches the same unique fixpoint, so the result
// is bit-identical to the reference's Bellman-Ford iteration.
//
// Step rule (lattice.py:17-20, 524-534): along an edge with the dark face
// ((r+c) odd) on the left, +1 uncrossed / -3 crossed; mirrored otherwise.
// For the edge entering vertex (r,c) from its vertical neighbours the left
// face is dark iff (r+c) is even; from its horizontal neighbours iff odd.
#include "domino.cuh"

namespace tsb {

constexpr int kTile = 32;
constexpr int kInf = 0x3FFFFFFF;
constexpr int8_t kNoEdge = 127;

// MODE 0: exact steps of a tiling (min-relax); 1: upper bounds (min-relax, h_max);
// 2: lower bounds (max-relax, h_min).
template <int MODE>
__device__ __forceinline__ int8_t edge_weight(bool exists, bool crossable, bool crossed, bool dark) {
    if (!exists) return kNoEdge;
    const int unc = dark ? 1 : -1, cr = dark ? -3 : 3;
    if (MODE == 0) return (int8_t)(crossed ? cr : unc);
    if (MODE == 1) return (int8_t)(crossable ? max(unc, cr) : unc);
    return (int8_t)(crossable ? min(unc, cr) : unc);
}

__device__ __forceinline__ bool bit_at(uint32_t word, int c) { return (word >> (c & 31)) & 1u; }

// One global relaxation round: each 32x32 tile relaxes to a local fixpoint in
// shared memory against its halo, then writes back.  Values only move in one
// direction, so reading a neighbour tile mid-update is harmless.
template <int MODE>
__global__ void __launch_bounds__(256) relax_kernel(int *h, const uint2 *st, const uint4 *dom, int side,
                                                    int pitch, int limit, int *flags) {
    __shared__ int s[kTile + 2][kTile + 2];
    __shared__ int8_t wt[4][kTile][kTile];  // incoming weights: up, down, left, right
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int c0 = blockIdx.x * kTile, r0 = blockIdx.y * kTile;
    const int sentinel = MODE == 2 ? -kInf : kInf;
    // load tile + halo
    for (int i = ty * 32 + tx; i < (kTile + 2) * (kTile + 2); i += 256) {
        const int lr = i / (kTile + 2), lc = i % (kTile + 2);
        const int r = r0 + lr - 1, c = c0 + lc - 1;
        s[lr][lc] = (r >= 0 && c >= 0 && r < side && c < side) ? h[(size_t)r * side + c] : sentinel;
    }
    int orig[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int lr = ty + 8 * k;
        const int r = r0 + lr, c = c0 + tx;
        int8_t wu = kNoEdge, wd = kNoEdge, wl = kNoEdge, wr = kNoEdge;
        if (r < side && c < side) {
            const bool even = ((r + c) & 1) == 0;
            const int w = c >> 5;
            if (r > 0) {
                const uint4 d = dom[(size_t)(r - 1) * pitch + w];
                const bool x = MODE == 0 ? bit_at(st[(size_t)r * pitch + w].x, c) : false;  // V[r-1]
                wu = edge_weight<MODE>(bit_at(d.z, c), bit_at(d.x, c), x, even);
            }
            {
                const uint4 d = dom[(size_t)r * pitch + w];
                const uint2 sv = MODE == 0 ? st[(size_t)(r + 1) * pitch + w] : make_uint2(0, 0);  // row r
                wd = edge_weight<MODE>(bit_at(d.z, c), bit_at(d.x, c), bit_at(sv.x, c), even);
                wr = edge_weight<MODE>(bit_at(d.w, c), bit_at(d.y, c), bit_at(sv.y, c), !even);
            }
            if (c > 0) {
                const int wl_ = (c - 1) >> 5;
                const uint4 d = dom[(size_t)r * pitch + wl_];
                const bool x = MODE == 0 ? bit_at(st[(size_t)(r + 1) * pitch + wl_].y, c - 1) : false;
                wl = edge_weight<MODE>(bit_at(d.w, c - 1), bit_at(d.y, c - 1), x, !even);
            }
        }
        wt[0][lr][tx] = wu;
        wt[1][lr][tx] = wd;
        wt[2][lr][tx] = wl;
        wt[3][lr][tx] = wr;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; ++k) orig[k] = s[ty + 8 * k + 1][tx + 1];
    volatile int(*vs)[kTile + 2] = s;
    bool over = false;
    for (int it = 0; it < 4 * kTile; ++it) {
        bool ch = false;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int lr = ty + 8 * k;
            const int cur = vs[lr + 1][tx + 1];
            int best = cur;
            const int nb[4] = {vs[lr][tx + 1], vs[lr + 2][tx + 1], vs[lr + 1][tx], vs[lr + 1][tx + 2]};
#pragma unroll
            for (int d = 0; d < 4; ++d) {
                const int8_t w = wt[d][lr][tx];
                if (w == kNoEdge || nb[d] == sentinel) continue;
                const int cand = nb[d] + w;
                best = MODE == 2 ? max(best, cand) : min(best, cand);
            }
            if (best != cur) {
                if (MODE == 2 ? best > limit : best < -limit) {
                    over = true;
                    best = MODE == 2 ? limit : -limit;  // clamp; the run is abandoned
                }
                if (best != cur) {
                    vs[lr + 1][tx + 1] = best;
                    ch = true;
                }
            }
        }
        if (!__syncthreads_or(ch)) break;
    }
    bool changed = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int lr = ty + 8 * k;
        const int r = r0 + lr, c = c0 + tx;
        const int v = s[lr + 1][tx + 1];
        if (r < side && c < side && v != orig[k]) {
            h[(size_t)r * side + c] = v;
            changed = true;
        }
    }
    if (__syncthreads_or(changed) && tx == 0 && ty == 0) atomicExch(flags, 1);
    if (over) atomicExch(flags + 1, 1);
}

__global__ void fill_kernel(int *h, size_t n, int v, int ref) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n) h[i] = (int)i == ref ? 0 : v;
}

// Heights -> int32 output: 0 outside vertex_mask; flags[0] set when a mask
// vertex is unreachable.
__global__ void finish_heights_kernel(const int *h, const uint4 *dom, int side, int pitch, int32_t *out,
                                      int sentinel, int *flags) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y;
    if (c >= side) return;
    const int w = c >> 5;
    const uint4 d = dom[(size_t)r * pitch + w];
    bool in = bit_at(d.z, c) || bit_at(d.w, c);
    if (r > 0) in |= bit_at(dom[(size_t)(r - 1) * pitch + w].z, c);
    if (c > 0) in |= bit_at(dom[(size_t)r * pitch + ((c - 1) >> 5)].w, c - 1);
    const int v = h[(size_t)r * side + c];
    if (in && v == sentinel) atomicExch(flags, 1);
    out[(size_t)r * side + c] = in ? v : 0;
}

// Extremal heights -> {V, H} planes of a chain: crossed iff crossable and
// |dh| == 3.  Also validates tiling_from_heights: every domain face has
// exactly one side with |dh| == 3 and its partner face lies in the domain.
__global__ void decode_extremal_kernel(const int32_t *hh, const uint4 *dom, const uint32_t *fbits, int side,
                                       int W, int pitch, uint2 *state, int *bad) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y;
    if (w >= W) return;
    const uint4 d = dom[(size_t)r * pitch + w];
    const uint32_t fb = r + 1 < side ? fbits[(size_t)r * pitch + w] : 0u;
    uint32_t v = 0, hz = 0;
    int err = 0;
    for (int b = 0; b < 32; ++b) {
        const int c = w * 32 + b;
        if (c >= side) break;
        const int h00 = hh[(size_t)r * side + c];
        const bool right = c + 1 < side, down = r + 1 < side;
        const int h01 = right ? hh[(size_t)r * side + c + 1] : 0;
        const int h10 = down ? hh[(size_t)(r + 1) * side + c] : 0;
        if (down && bit_at(d.x, c) && abs(h10 - h00) == 3) v |= 1u << b;
        if (right && bit_at(d.y, c) && abs(h01 - h00) == 3) hz |= 1u << b;
        if ((fb >> b) & 1u) {  // face (r, c): corners (r,c) (r,c+1) (r+1,c) (r+1,c+1)
            const int h11 = hh[(size_t)(r + 1) * side + c + 1];
            const int n3 = (abs(h01 - h00) == 3) + (abs(h11 - h10) == 3) + (abs(h10 - h00) == 3) +
                           (abs(h11 - h01) == 3);
            const uint4 dd = dom[(size_t)(r + 1) * pitch + w];
            const uint4 dr = dom[(size_t)r * pitch + ((c + 1) >> 5)];
            const int n3c = (abs(h01 - h00) == 3 && bit_at(d.y, c)) +       // top edge H(r,c)
                            (abs(h11 - h10) == 3 && bit_at(dd.y, c)) +      // bottom edge H(r+1,c)
                            (abs(h10 - h00) == 3 && bit_at(d.x, c)) +       // left edge V(r,c)
                            (abs(h11 - h01) == 3 && bit_at(dr.x, c + 1));   // right edge V(r,c+1)
            if (n3 != 1 || n3c != 1) err = 1;
        }
    }
    state[(size_t)(r + 1) * pitch + w] = make_uint2(v, hz);
    if (err) atomicOr(bad, 1);
}

template <int MODE>
int relax(tsb_domino *h, int *dh, int ref, const uint2 *st, int *dflags, bool *overflow) {
    const size_t nv = (size_t)h->side * h->side;
    const int sentinel = MODE == 2 ? -kInf : kInf;
    fill_kernel<<<(unsigned)((nv + 255) / 256), 256, 0, h->stream>>>(dh, nv, sentinel, ref);
    const int64_t lim64 = 3 * (int64_t)nv + 8;
    const int limit = (int)std::min<int64_t>(lim64, (int64_t)1 << 30);
    const dim3 grid((h->side + kTile - 1) / kTile, (h->side + kTile - 1) / kTile);
    const dim3 block(32, 8);
    int hf[2];
    const int64_t cap = lim64 + 16;
    for (int64_t it = 0; it < cap; ++it) {
        TSB_CUDA(cudaMemsetAsync(dflags, 0, 2 * sizeof(int), h->stream));
        relax_kernel<MODE><<<grid, block, 0, h->stream>>>(dh, st, h->dom, h->side, h->pitch, limit, dflags);
        TSB_CUDA(cudaGetLastError());
        TSB_CUDA(cudaMemcpyAsync(hf, dflags, 2 * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        TSB_CUDA(cudaStreamSynchronize(h->stream));
        if (hf[1]) { *overflow = true; return TSB_OK; }
        if (!hf[0]) { *overflow = false; return TSB_OK; }
    }
    *overflow = true;
    return TSB_OK;
}

}  // namespace tsb

using namespace tsb;

extern "C" {

int tsb_domino_heights(tsb_domino *h, int chain, int ref_r, int ref_c, int32_t *out) {
    if (!h || !out) return fail(TSB_E_VALUE, "null argument");
    if (chain < 0 || chain >= h->nchains) return fail(TSB_E_VALUE, "chain %d out of range", chain);
    if (ref_r < 0 || ref_c < 0 || ref_r >= h->side || ref_c >= h->side)
        return fail(TSB_E_VALUE, "reference vertex outside the grid");
    TSB_CUDA(cudaSetDevice(h->device));
    const size_t nv = (size_t)h->side * h->side;
    int *dh = nullptr, *dflags = nullptr;
    int32_t *dout = nullptr;
    TSB_CUDA(cudaMalloc(&dh, nv * sizeof(int)));
    TSB_CUDA(cudaMalloc(&dout, nv * sizeof(int32_t)));
    TSB_CUDA(cudaMalloc(&dflags, 2 * sizeof(int)));
    bool overflow = false;
    const uint2 *st = h->buf[h->cur] + (size_t)chain * h->chain_stride + kStatePad;
    int rc = relax<0>(h, dh, ref_r * h->side + ref_c, st, dflags, &overflow);
    int hf = 0;
    if (!rc && !overflow) {
        cudaMemsetAsync(dflags, 0, sizeof(int), h->stream);
        finish_heights_kernel<<<dim3((h->side + 127) / 128, h->side), 128, 0, h->stream>>>(
            dh, h->dom, h->side, h->pitch, dout, kInf, dflags);
        cudaMemcpyAsync(out, dout, nv * sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream);
        cudaMemcpyAsync(&hf, dflags, sizeof(int), cudaMemcpyDeviceToHost, h->stream);
        cudaError_t e = cudaStreamSynchronize(h->stream);
        if (e != cudaSuccess) rc = cuda_fail(e, "heights");
    }
    cudaFree(dh);
    cudaFree(dout);
    cudaFree(dflags);
    if (rc) return rc;
    if (overflow || hf) return fail(TSB_E_INCONSISTENT, "height propagation is cyclically inconsistent");
    return TSB_OK;
}

// Thurston extremal tilings into chains `chain_max` / `chain_min`.
// Returns TSB_E_UNTILEABLE (no exception message needed) when the domain has
// no tiling, mirroring extremal_tilings() -> None.
int tsb_domino_extremal(tsb_domino *h, int chain_max, int chain_min, int ref_r, int ref_c) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    if (chain_max < 0 || chain_max >= h->nchains || chain_min < 0 || chain_min >= h->nchains)
        return fail(TSB_E_VALUE, "chain out of range");
    TSB_CUDA(cudaSetDevice(h->device));
    const size_t nv = (size_t)h->side * h->side;
    int *dh = nullptr, *dflags = nullptr;
    int32_t *dout = nullptr;
    TSB_CUDA(cudaMalloc(&dh, nv * sizeof(int)));
    TSB_CUDA(cudaMalloc(&dout, nv * sizeof(int32_t)));
    TSB_CUDA(cudaMalloc(&dflags, 2 * sizeof(int)));
    int rc = TSB_OK;
    bool untileable = false;
    for (int pass = 0; pass < 2 && !rc && !untileable; ++pass) {
        bool overflow = false;
        const int ref = ref_r * h->side + ref_c;
        rc = pass == 0 ? relax<1>(h, dh, ref, nullptr, dflags, &overflow)
                       : relax<2>(h, dh, ref, nullptr, dflags, &overflow);
        if (rc) break;
        if (overflow) { untileable = true; break; }
        int hf[2] = {0, 0};
        cudaMemsetAsync(dflags, 0, 2 * sizeof(int), h->stream);
        finish_heights_kernel<<<dim3((h->side + 127) / 128, h->side), 128, 0, h->stream>>>(
            dh, h->dom, h->side, h->pitch, dout, pass == 0 ? kInf : -kInf, dflags);
        uint2 *st = h->buf[h->cur] + (size_t)(pass == 0 ? chain_max : chain_min) * h->chain_stride + kStatePad;
        decode_extremal_kernel<<<dim3((h->W + 127) / 128, h->side), 128, 0, h->stream>>>(
            dout, h->dom, h->fbits, h->side, h->W, h->pitch, st, dflags + 1);
        cudaMemcpyAsync(hf, dflags, 2 * sizeof(int), cudaMemcpyDeviceToHost, h->stream);
        cudaError_t e = cudaStreamSynchronize(h->stream);
        if (e != cudaSuccess) { rc = cuda_fail(e, "extremal"); break; }
        if (hf[0] || hf[1]) untileable = true;
    }
    cudaFree(dh);
    cudaFree(dout);
    cudaFree(dflags);
    if (rc) return rc;
    if (untileable) return fail(TSB_E_UNTILEABLE, "domain is not tileable");
    return TSB_OK;
}

}  // extern "C"
