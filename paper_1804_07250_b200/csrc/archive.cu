// Sample-archive records straight from device states.
//
// Reference (relative to /root/reference/pkg/src/tilesampler/):
//   stats.py:146-153  _serialize_state: a domino Tiling is its tilestates
//                     (V, V) uint8 ravelled and joined by single spaces in
//                     decimal ("3 0 12 ..."), one line per sample.
// The record is produced on the device from the bit planes -- the host only
// receives the finished text -- in two passes: per-row lengths (a tilestate
// >= 10 takes two digits), a host prefix over the rows, then one block per
// row scans its columns and writes digits and separators.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include <vector>

#include "domino.cuh"

namespace tsb {

constexpr int kSerThreads = 256;

// Tilestate of vertex (r, c) from the planes (see domino.cu):
// V[r-1]c | V[r]c << 1 | H[r]c-1 << 2 | H[r]c << 3.
__device__ __forceinline__ uint32_t tilestate_at(const uint2 *row, int pitch, int c) {
    const uint2 w = row[c >> 5], wu = row[(c >> 5) - pitch];
    const uint32_t b = c & 31;
    const uint32_t hl = c > 0 ? (row[(c - 1) >> 5].y >> ((c - 1) & 31)) & 1u : 0u;
    return ((wu.x >> b) & 1u) | (((w.x >> b) & 1u) << 1) | (hl << 2) | (((w.y >> b) & 1u) << 3);
}

// pass 1: characters of row r ("d " or "dd " per vertex)
__global__ void dser_count_kernel(const uint2 *state, int side, int pitch, unsigned long long *row_len) {
    typedef cub::BlockReduce<int, kSerThreads> Reduce;
    __shared__ typename Reduce::TempStorage tmp;
    const int r = blockIdx.x;
    const uint2 *row = state + (size_t)(r + 1) * pitch;  // after the guard row
    int two = 0;
    for (int c = threadIdx.x; c < side; c += blockDim.x) two += tilestate_at(row, pitch, c) >= 10u;
    const int tot = Reduce(tmp).Sum(two);
    if (threadIdx.x == 0) row_len[r] = 2ull * (unsigned long long)side + (unsigned long long)tot;
}

// pass 2: digits and separators of row r at row_off[r]; the very last
// separator (after the final vertex) is not written
__global__ void dser_write_kernel(const uint2 *state, int side, int pitch, const unsigned long long *row_off,
                                  unsigned long long total, char *out) {
    typedef cub::BlockScan<int, kSerThreads> Scan;
    __shared__ typename Scan::TempStorage tmp;
    const int r = blockIdx.x;
    const uint2 *row = state + (size_t)(r + 1) * pitch;
    unsigned long long pos = row_off[r];
    for (int c0 = 0; c0 < side; c0 += kSerThreads) {
        const int c = c0 + threadIdx.x;
        const uint32_t v = c < side ? tilestate_at(row, pitch, c) : 0u;
        const int len = c < side ? (v >= 10u ? 3 : 2) : 0;
        int off, chunk;
        Scan(tmp).ExclusiveSum(len, off, chunk);
        if (c < side) {
            char *p = out + pos + off;
            if (v >= 10u) {
                p[0] = '1';
                p[1] = (char)('0' + v - 10u);
            } else {
                p[0] = (char)('0' + v);
            }
            if (pos + off + len - 1 < total) p[len - 1] = ' ';
        }
        pos += (unsigned long long)chunk;
        __syncthreads();  // temp storage reuse
    }
}

}  // namespace tsb

using namespace tsb;

extern "C" {

int tsb_domino_serialize(tsb_domino *h, int chain, char *out, size_t cap, size_t *len) {
    TSB_FULL_ONLY(h);
    if (!h || !len) return fail(TSB_E_VALUE, "null argument");
    if (chain < 0 || chain >= h->nchains) return fail(TSB_E_VALUE, "chain %d out of range", chain);
    TSB_CUDA(cudaSetDevice(h->device));
    const int side = h->side;
    const uint2 *st = h->buf[h->cur] + (size_t)chain * h->chain_stride + kStatePad;
    // scratch: the handle's staging buffer (row lengths, then offsets + text)
    const size_t len_bytes = sizeof(unsigned long long) * (size_t)side;
    int rc = ensure_bytes(h, len_bytes);
    if (rc) return rc;
    unsigned long long *d_len = reinterpret_cast<unsigned long long *>(h->bytes);
    dser_count_kernel<<<side, kSerThreads, 0, h->stream>>>(st, side, h->pitch, d_len);
    std::vector<unsigned long long> rl(side);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(rl.data(), d_len, len_bytes, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "serialize count");
    unsigned long long acc = 0;
    for (int r = 0; r < side; ++r) {
        const unsigned long long l = rl[r];
        rl[r] = acc;
        acc += l;
    }
    const unsigned long long total = acc - 1;  // no separator after the last vertex
    *len = (size_t)total;
    if (!out || cap < total) return TSB_OK;  // size query
    if ((rc = ensure_bytes(h, len_bytes + acc))) return rc;
    d_len = reinterpret_cast<unsigned long long *>(h->bytes);
    char *d_out = reinterpret_cast<char *>(h->bytes) + len_bytes;
    e = cudaMemcpyAsync(d_len, rl.data(), len_bytes, cudaMemcpyHostToDevice, h->stream);
    if (e == cudaSuccess) {
        dser_write_kernel<<<side, kSerThreads, 0, h->stream>>>(st, side, h->pitch, d_len, total, d_out);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, d_out, total, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "serialize");
    return TSB_OK;
}

}  // extern "C"
