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
#include <climits>
#include <cstdlib>
#include <vector>

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
    // Jacobi rounds: every thread reads its neighbours, a barrier, then the
    // improved values are written (race-free; the fixpoint is unique, so the
    // update order does not change the result)
    bool over = false;
    for (int it = 0; it < 4 * kTile; ++it) {
        bool ch = false;
        int nv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int lr = ty + 8 * k;
            const int cur = s[lr + 1][tx + 1];
            int best = cur;
            const int nb[4] = {s[lr][tx + 1], s[lr + 2][tx + 1], s[lr + 1][tx], s[lr + 1][tx + 2]};
#pragma unroll
            for (int d = 0; d < 4; ++d) {
                const int8_t w = wt[d][lr][tx];
                if (w == kNoEdge || nb[d] == sentinel) continue;
                const int cand = nb[d] + w;
                best = MODE == 2 ? max(best, cand) : min(best, cand);
            }
            if (best != cur && (MODE == 2 ? best > limit : best < -limit)) {
                over = true;
                best = MODE == 2 ? limit : -limit;  // clamp; the run is abandoned
            }
            nv[k] = best;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int lr = ty + 8 * k;
            if (nv[k] != s[lr + 1][tx + 1]) {
                s[lr + 1][tx + 1] = nv[k];
                ch = true;
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

// ---------------------------------------------------------------- row scan
// Fast exact height export for domains whose vertex rows are intervals joined
// by horizontal domain edges, with consecutive rows linked by a vertical
// domain edge (every convex-row domain: Aztec diamonds, rectangles, ...).
// A consistent state's heights are path-independent, so
//   h(r, c) = off[r] + local(r, c),  local(r, c) = sum of the horizontal steps
//   from the row's first vertex, off[r] chained through one vertical link
// per row and shifted so h(reference vertex) = 0.  Every vertical domain edge
// is then checked against its step (lattice.py:554-580
// _check_height_consistency), so inconsistent states still raise.  Three
// passes over the int32 grid instead of ~2·side/31 relaxation rounds.

// step of edge a -> b whose "left face dark" flag is `dark` (lattice.py:17-20)
__device__ __forceinline__ int hstep(bool crossed, bool dark) {
    return dark ? (crossed ? -3 : 1) : (crossed ? 3 : -1);
}

// vertex (r, c) of word w lies in vertex_mask iff one of its edges exists
__device__ __forceinline__ uint32_t in_mask(const uint4 *dom, int r, int w, int pitch) {
    const uint4 d = dom[(size_t)r * pitch + w];
    uint32_t m = d.z | d.w | (d.w << 1);
    if (w > 0) m |= dom[(size_t)r * pitch + w - 1].w >> 31;
    if (r > 0) m |= dom[(size_t)(r - 1) * pitch + w].z;
    return m;
}

// Row classification, once per handle: {first, last} in-domain vertex,
// link = first column with a vertical domain edge to the row above (-1:
// none), ok = every horizontal edge between first and last exists.
__global__ void __launch_bounds__(256) hx_rows_kernel(const uint4 *dom, int side, int pitch, int W, int4 *rows) {
    __shared__ int sh[8];
    const int r = blockIdx.x;
    int a = INT_MAX, b = -1, link = INT_MAX;
    for (int w = threadIdx.x; w < W; w += blockDim.x) {
        const uint32_t m = in_mask(dom, r, w, pitch);
        if (m) {
            a = min(a, w * 32 + __ffs(m) - 1);
            b = max(b, w * 32 + 31 - __clz(m));
        }
        if (r > 0) {
            const uint32_t up = dom[(size_t)(r - 1) * pitch + w].z;
            if (up) link = min(link, w * 32 + __ffs(up) - 1);
        }
    }
    a = block_reduce(a, [](int x, int y) { return min(x, y); }, sh);
    b = block_reduce(b, [](int x, int y) { return max(x, y); }, sh);
    link = block_reduce(link, [](int x, int y) { return min(x, y); }, sh);
    int missing = 0;
    if (a <= b) {
        for (int w = (a >> 5) + threadIdx.x; w <= ((b - 1) >> 5) && b > a; w += blockDim.x) {
            uint32_t e = 0xffffffffu;  // edges c in [a, b)
            if (w == (a >> 5)) e &= 0xffffffffu << (a & 31);
            if (w == ((b - 1) >> 5)) e &= 0xffffffffu >> (31 - ((b - 1) & 31));
            missing += __popc(e & ~dom[(size_t)r * pitch + w].w);
        }
    }
    missing = block_reduce(missing, [](int x, int y) { return x + y; }, sh);
    if (threadIdx.x == 0) rows[r] = make_int4(a, b, link == INT_MAX ? -1 : link, missing == 0);
}

// local(r, c) for c in [first, last] of row r: one block per row, thread t
// owns consecutive words; word sums by popcount, block exclusive scan, then
// the per-vertex prefix within the word.
__global__ void __launch_bounds__(256) hx_local_kernel(const uint2 *st, int pitch, int side, int r0,
                                                      const int4 *rows, int *loc) {
    __shared__ int sh[8];
    const int r = r0 + blockIdx.x;
    const int4 ri = rows[r];
    const int a = ri.x, b = ri.y;
    if (a > b) return;
    const int w0 = a >> 5, w1 = b >> 5, nw = w1 - w0 + 1;
    const int per = (nw + blockDim.x - 1) / blockDim.x;
    const int wa = w0 + threadIdx.x * per, wb = min(w1, wa + per - 1);
    const uint32_t D = (r & 1) ? 0xAAAAAAAAu : 0x55555555u;  // dark: (r + c) even
    const uint2 *row = st + (size_t)(r + 1) * pitch;
    int sum = 0;
    for (int w = wa; w <= wb; ++w) {
        uint32_t e = 0xffffffffu;  // edges c in [a, b)
        if (w == w0) e &= 0xffffffffu << (a & 31);
        if (w == w1) e = (b & 31) ? (e & (0xffffffffu >> (32 - (b & 31)))) : 0u;
        const uint32_t x = row[w].y;
        sum += __popc(e & D & ~x) - 3 * __popc(e & D & x) - __popc(e & ~D & ~x) + 3 * __popc(e & ~D & x);
    }
    int acc = block_exclusive_sum(sum, sh);
    int *out = loc + (size_t)r * side;
    for (int w = wa; w <= wb; ++w) {
        const uint32_t x = row[w].y;
        const int cb = max(a, w * 32), ce = min(b, w * 32 + 31);
        for (int c = cb; c <= ce; ++c) {
            out[c] = acc;
            acc += hstep((x >> (c & 31)) & 1u, ((r + c) & 1) == 0);
        }
    }
}

// Row offsets: delta[r] through the vertical link edge, block scan over the
// rows r0..r1 (one block, 1024 threads, consecutive rows per thread), then
// the shift that puts the reference vertex at 0.  flags[0]: a row without a
// link (cannot happen for a classified domain).
__global__ void __launch_bounds__(1024) hx_offsets_kernel(const uint2 *st, int pitch, int side, int r0, int r1,
                                                         const int4 *rows, const int *loc, int *off, int ref_r,
                                                         int ref_c) {
    __shared__ int sh[32];
    const int nr = r1 - r0 + 1;
    const int per = (nr + blockDim.x - 1) / blockDim.x;
    const int ra = r0 + threadIdx.x * per, rb = min(r1, ra + per - 1);
    int sum = 0;
    for (int r = ra; r <= rb; ++r) {
        int d = 0;
        if (r > r0) {
            const int c = rows[r].z;
            const bool x = (st[(size_t)r * pitch + (c >> 5)].x >> (c & 31)) & 1u;  // V(r-1, c)
            d = loc[(size_t)(r - 1) * side + c] + hstep(x, ((r + c) & 1) == 0) - loc[(size_t)r * side + c];
        }
        sum += d;
        off[r] = sum;  // partial within the thread's run
    }
    const int excl = block_exclusive_sum(sum, sh);
    for (int r = ra; r <= rb; ++r) off[r] += excl;
    __syncthreads();
    const int shift = off[ref_r] + loc[(size_t)ref_r * side + ref_c];
    __syncthreads();
    for (int r = ra; r <= rb; ++r) off[r] -= shift;
}

// h = off[r] + local inside vertex_mask, 0 outside; every vertical domain
// edge checked (flags[0] on a violation).  SUM: add into an int64
// accumulator instead of writing the grid.
template <bool SUM>
__global__ void __launch_bounds__(256) hx_finish_kernel(const uint2 *st, const uint4 *dom, int pitch, int side, int r0,
                                                       int r1, const int *loc, const int *off, int32_t *out,
                                                       long long *acc, int *flags) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y;
    if (c >= side) return;
    const int w = c >> 5;
    const bool in = r >= r0 && r <= r1 && ((in_mask(dom, r, w, pitch) >> (c & 31)) & 1u);
    int v = 0;
    if (in) {
        v = off[r] + loc[(size_t)r * side + c];
        if (r > 0 && ((dom[(size_t)(r - 1) * pitch + w].z >> (c & 31)) & 1u)) {
            const bool x = (st[(size_t)r * pitch + w].x >> (c & 31)) & 1u;
            const int up = off[r - 1] + loc[(size_t)(r - 1) * side + c];
            if (v - up != hstep(x, ((r + c) & 1) == 0)) atomicExch(flags, 1);
        }
    }
    if (SUM) acc[(size_t)r * side + c] += v;
    else out[(size_t)r * side + c] = v;
}

__global__ void add_heights_kernel(const int32_t *h, size_t n, long long *acc) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n) acc[i] += h[i];
}

int hx_scratch(tsb_domino *h) {
    if (h->hx_h) return TSB_OK;
    const size_t nv = (size_t)h->side * h->side;
    TSB_CUDA(cudaMalloc(&h->hx_h, nv * sizeof(int)));
    TSB_CUDA(cudaMalloc(&h->hx_flags, 4 * sizeof(int)));
    TSB_CUDA(cudaMalloc(&h->hx_rows, h->side * sizeof(int4)));
    TSB_CUDA(cudaMalloc(&h->hx_off, h->side * sizeof(int)));
    return TSB_OK;
}

// classify the domain once: row scan when every non-empty row is an interval
// of horizontal domain edges and every row after the first has a link
int hx_classify(tsb_domino *h) {
    if (h->hx_scan >= 0) return TSB_OK;
    int rc = hx_scratch(h);
    if (rc) return rc;
    hx_rows_kernel<<<h->side, 256, 0, h->stream>>>(h->dom, h->side, h->pitch, h->W, h->hx_rows);
    TSB_CUDA(cudaGetLastError());
    std::vector<int4> rows(h->side);
    TSB_CUDA(cudaMemcpyAsync(rows.data(), h->hx_rows, sizeof(int4) * h->side, cudaMemcpyDeviceToHost, h->stream));
    TSB_CUDA(cudaStreamSynchronize(h->stream));
    int r0 = -1, r1 = -1;
    bool ok = true;
    for (int r = 0; r < h->side; ++r) {
        if (rows[r].x > rows[r].y) continue;
        if (r0 < 0) r0 = r;
        else if (r1 != r - 1 || rows[r].z < 0) ok = false;  // a gap row, or no vertical link
        if (!rows[r].w) ok = false;
        r1 = r;
    }
    h->hx_r0 = r0 < 0 ? 0 : r0;
    h->hx_r1 = r0 < 0 ? -1 : r1;
    h->hx_scan = (ok && r0 >= 0) ? 1 : 0;
    const char *env = getenv("TSB_HEIGHTS_RELAX");  // test knob: force the relaxation path
    if (env && env[0] == '1') h->hx_scan = 0;
    return TSB_OK;
}

// Heights of one chain into dout (device, side^2 int32) or added to acc.
// Returns TSB_E_INCONSISTENT for an inconsistent state.
int domino_heights_dev(tsb_domino *h, int chain, int ref_r, int ref_c, int32_t *dout, long long *acc) {
    int rc = hx_classify(h);
    if (rc) return rc;
    const size_t nv = (size_t)h->side * h->side;
    const uint2 *st = h->buf[h->cur] + (size_t)chain * h->chain_stride + kStatePad;
    int hf[2] = {0, 0};
    const int ref = ref_r * h->side + ref_c;
    const dim3 fgrid((h->side + 255) / 256, h->side);
    if (h->hx_scan == 1 && ref_r >= h->hx_r0 && ref_r <= h->hx_r1) {
        TSB_CUDA(cudaMemsetAsync(h->hx_flags, 0, 2 * sizeof(int), h->stream));
        hx_local_kernel<<<h->hx_r1 - h->hx_r0 + 1, 256, 0, h->stream>>>(st, h->pitch, h->side, h->hx_r0, h->hx_rows,
                                                                        h->hx_h);
        hx_offsets_kernel<<<1, 1024, 0, h->stream>>>(st, h->pitch, h->side, h->hx_r0, h->hx_r1, h->hx_rows, h->hx_h,
                                                     h->hx_off, ref_r, ref_c);
        if (acc)
            hx_finish_kernel<true><<<fgrid, 256, 0, h->stream>>>(st, h->dom, h->pitch, h->side, h->hx_r0, h->hx_r1,
                                                                 h->hx_h, h->hx_off, nullptr, acc, h->hx_flags);
        else
            hx_finish_kernel<false><<<fgrid, 256, 0, h->stream>>>(st, h->dom, h->pitch, h->side, h->hx_r0, h->hx_r1,
                                                                  h->hx_h, h->hx_off, dout, nullptr, h->hx_flags);
        TSB_CUDA(cudaGetLastError());
        TSB_CUDA(cudaMemcpyAsync(hf, h->hx_flags, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        TSB_CUDA(cudaStreamSynchronize(h->stream));
        if (hf[0]) return fail(TSB_E_INCONSISTENT, "height propagation is cyclically inconsistent");
        return TSB_OK;
    }
    bool overflow = false;
    if ((rc = relax<0>(h, h->hx_h, ref, st, h->hx_flags, &overflow))) return rc;
    if (overflow) return fail(TSB_E_INCONSISTENT, "height propagation is cyclically inconsistent");
    int32_t *o = dout;
    if (acc) {
        if ((rc = ensure_bytes(h, nv * sizeof(int32_t)))) return rc;
        o = reinterpret_cast<int32_t *>(h->bytes);
    }
    TSB_CUDA(cudaMemsetAsync(h->hx_flags, 0, sizeof(int), h->stream));
    finish_heights_kernel<<<dim3((h->side + 127) / 128, h->side), 128, 0, h->stream>>>(
        h->hx_h, h->dom, h->side, h->pitch, o, kInf, h->hx_flags);
    if (acc) add_heights_kernel<<<(unsigned)((nv + 255) / 256), 256, 0, h->stream>>>(o, nv, acc);
    TSB_CUDA(cudaGetLastError());
    TSB_CUDA(cudaMemcpyAsync(hf, h->hx_flags, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    TSB_CUDA(cudaStreamSynchronize(h->stream));
    if (hf[0]) return fail(TSB_E_INCONSISTENT, "height propagation is cyclically inconsistent");
    return TSB_OK;
}

}  // namespace tsb

using namespace tsb;

extern "C" {

int tsb_domino_heights(tsb_domino *h, int chain, int ref_r, int ref_c, int32_t *out) {
    TSB_FULL_ONLY(h);
    if (!h || !out) return fail(TSB_E_VALUE, "null argument");
    if (chain < 0 || chain >= h->nchains) return fail(TSB_E_VALUE, "chain %d out of range", chain);
    if (ref_r < 0 || ref_c < 0 || ref_r >= h->side || ref_c >= h->side)
        return fail(TSB_E_VALUE, "reference vertex outside the grid");
    TSB_CUDA(cudaSetDevice(h->device));
    const size_t nv = (size_t)h->side * h->side;
    int rc = ensure_bytes(h, nv * sizeof(int32_t));  // handle staging: no allocation per call
    if (rc) return rc;
    int32_t *dout = reinterpret_cast<int32_t *>(h->bytes);
    if ((rc = domino_heights_dev(h, chain, ref_r, ref_c, dout, nullptr))) return rc;
    return staged_d2h(out, dout, nv * sizeof(int32_t), h->stream);  // pinned staging, returns complete
}

int tsb_domino_height_sum_add(tsb_domino *h, int chain0, int n, int ref_r, int ref_c, long long *acc_dev) {
    TSB_FULL_ONLY(h);
    int rc = check_range(h, chain0, n);
    if (rc || n == 0) return rc;
    if (!acc_dev) return fail(TSB_E_VALUE, "null accumulator");
    if (ref_r < 0 || ref_c < 0 || ref_r >= h->side || ref_c >= h->side)
        return fail(TSB_E_VALUE, "reference vertex outside the grid");
    TSB_CUDA(cudaSetDevice(h->device));
    for (int k = 0; k < n && !rc; ++k) rc = domino_heights_dev(h, chain0 + k, ref_r, ref_c, nullptr, acc_dev);
    return rc;
}

// Thurston extremal tilings into chains `chain_max` / `chain_min`.
// Returns TSB_E_UNTILEABLE (no exception message needed) when the domain has
// no tiling, mirroring extremal_tilings() -> None.
int tsb_domino_extremal(tsb_domino *h, int chain_max, int chain_min, int ref_r, int ref_c) {
    TSB_FULL_ONLY(h);
    if (!h) return fail(TSB_E_VALUE, "null handle");
    if (chain_max < 0 || chain_max >= h->nchains || chain_min < 0 || chain_min >= h->nchains)
        return fail(TSB_E_VALUE, "chain out of range");
    TSB_CUDA(cudaSetDevice(h->device));
    const size_t nv = (size_t)h->side * h->side;
    int rc = hx_scratch(h);
    if (!rc) rc = ensure_bytes(h, nv * sizeof(int32_t));
    if (rc) return rc;
    int *dh = h->hx_h, *dflags = h->hx_flags;
    int32_t *dout = reinterpret_cast<int32_t *>(h->bytes);
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
    if (rc) return rc;
    if (untileable) return fail(TSB_E_UNTILEABLE, "domain is not tileable");
    return TSB_OK;
}

}  // extern "C"
