// On-device observables: the reference's indicator
// observables accumulated over chains and samples without downloading states.
//
// Reference (relative to /root/reference/pkg/src/tilesampler/):
//   stats.py:187-200  domino_orientation_grid (1 horizontal, 0 vertical per face)
//   stats.py:213-245  density_map over an archive: per-site mean of an indicator
// The caller owns a device accumulator of uint32 counts; every call adds the
// indicator of each listed chain's current state, so after S calls over B
// chains acc / (S*B) is the reference's density_map of those S*B states.
#include "domino.cuh"

namespace tsb {

// Face (r, c) is covered by a horizontal domino iff the vertical edge on its
// left ((r,c)-(r+1,c), plane V[r] bit c) or on its right (V[r] bit c+1) is
// crossed.  One thread per (face row, 32-face word); chains summed in
// registers, one read-modify-write of the accumulator per face.
__global__ void domino_orientation_kernel(const uint2 *state, size_t chain_stride, int pitch, int nchains, int nf,
                                          int W, uint32_t *acc) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y;
    if (w >= W || r >= nf) return;
    uint32_t cnt[32];
#pragma unroll
    for (int b = 0; b < 32; ++b) cnt[b] = 0;
    for (int z = 0; z < nchains; ++z) {
        const uint2 *row = state + (size_t)z * chain_stride + (size_t)(r + 1) * pitch;  // after the guard row
        const uint32_t v = row[w].x, vn = row[w + 1].x;  // rows are zero-padded on the right
        const uint32_t hm = v | (v >> 1) | (vn << 31);
#pragma unroll
        for (int b = 0; b < 32; ++b) cnt[b] += (hm >> b) & 1u;
    }
    uint32_t *a = acc + (size_t)r * nf + (size_t)w * 32;
    const int lim = min(32, nf - w * 32);
#pragma unroll
    for (int b = 0; b < 32; ++b)
        if (b < lim) a[b] += cnt[b];
}

}  // namespace tsb

using namespace tsb;

extern "C" {

int tsb_domino_orientation_add(tsb_domino *h, int chain0, int n, uint32_t *acc_dev) {
    TSB_FULL_ONLY(h);
    int rc = check_range(h, chain0, n);
    if (rc || n == 0) return rc;
    if (!acc_dev) return fail(TSB_E_VALUE, "null accumulator");
    const int nf = h->side - 1;
    if (nf < 1) return TSB_OK;
    TSB_CUDA(cudaSetDevice(h->device));
    const int W = (nf + 31) / 32;
    const uint2 *st = h->buf[h->cur] + (size_t)chain0 * h->chain_stride + kStatePad;
    domino_orientation_kernel<<<dim3((W + 63) / 64, nf), 64, 0, h->stream>>>(st, h->chain_stride, h->pitch, n, nf,
                                                                             W, acc_dev);
    TSB_CUDA(cudaGetLastError());
    return TSB_OK;
}

}  // extern "C"
