// Coupling-from-the-past for dominoes on the device (K7 + the round driver).
//
// Reference: cftp.py:86-139 (run_cftp_batch), 161-213 (cftp_sample_many).
// Layout inside a handle with nchains >= 2*count + 2:
//   chain 2j / 2j+1   top / bottom chain of the j-th still-active sample
//   chain 2*count     T_max template,  chain 2*count+1  T_min template
// Every round restarts from the templates (cftp.py:113-114), so active
// samples are simply re-packed at the front each round; no state crosses
// rounds.  The coalescence check (cftp.py:120) is a per-pair device
// reduction; one byte per active sample returns to the host per round.
#include <vector>

#include "domino.cuh"

namespace tsb {

constexpr uint64_t kSeedSalt = 0x51ED2701ull;   // cftp.py:30
constexpr uint64_t kDeriveMul = 0xD6E8FEB86659FD93ull;  // rng.py:59

// rng.py:53-59
inline uint64_t derive_seed(uint64_t seed, uint64_t index, uint64_t salt) {
    return mix64(mix64(seed ^ (salt * kDeriveMul)) + (index + 1ull) * kGold);
}

// Copy chain `src` into chains dst0, dst0 + step, ... (n copies).
__global__ void replicate_kernel(uint4 *base, size_t chain_u4, int src, int dst0, int step, int n) {
    const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i >= chain_u4) return;
    const uint4 v = base[(size_t)src * chain_u4 + i];
    for (int k = 0; k < n; ++k) base[(size_t)(dst0 + (size_t)k * step) * chain_u4 + i] = v;
}

// K7: flags[j] = 1 iff chains chain0+2j and chain0+2j+1 are identical.
__global__ void __launch_bounds__(256) coalesced_kernel(const uint4 *base, size_t chain_u4, int chain0,
                                                        uint8_t *flags) {
    const int j = blockIdx.x;
    const uint4 *a = base + (size_t)(chain0 + 2 * j) * chain_u4;
    const uint4 *b = a + chain_u4;
    uint32_t diff = 0;
    for (size_t i = threadIdx.x; i < chain_u4; i += blockDim.x) {
        const uint4 x = __ldg(a + i), y = __ldg(b + i);
        diff |= (x.x ^ y.x) | (x.y ^ y.y) | (x.z ^ y.z) | (x.w ^ y.w);
    }
    const int any = __syncthreads_or(diff != 0);
    if (threadIdx.x == 0) flags[j] = any ? 0 : 1;
}

}  // namespace tsb

using namespace tsb;

extern "C" {

int tsb_domino_coalesced(tsb_domino *h, int chain0, int npairs, uint8_t *flags) {
    TSB_FULL_ONLY(h);
    int rc = check_range(h, chain0, 2 * npairs);
    if (rc || npairs == 0) return rc;
    TSB_CUDA(cudaSetDevice(h->device));
    if ((rc = ensure_bytes(h, npairs))) return rc;  // handle scratch: no allocation per round
    uint8_t *d = h->bytes;
    const size_t chain_u4 = h->chain_stride / 2;  // chain_stride is even (pitch % 32 == 0)
    coalesced_kernel<<<npairs, 256, 0, h->stream>>>(reinterpret_cast<const uint4 *>(h->buf[h->cur]),
                                                   chain_u4, chain0, d);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(flags, d, npairs, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "coalesced");
    return TSB_OK;
}

int tsb_domino_replicate(tsb_domino *h, int src, int dst0, int step, int n) {
    TSB_FULL_ONLY(h);
    if (!h) return fail(TSB_E_VALUE, "null handle");
    if (n <= 0) return TSB_OK;
    if (src < 0 || src >= h->nchains || dst0 < 0 || step < 1 || dst0 + (int64_t)(n - 1) * step >= h->nchains)
        return fail(TSB_E_VALUE, "replicate chains out of range");
    TSB_CUDA(cudaSetDevice(h->device));
    const size_t chain_u4 = h->chain_stride / 2;
    replicate_kernel<<<(unsigned)((chain_u4 + 255) / 256), 256, 0, h->stream>>>(
        reinterpret_cast<uint4 *>(h->buf[h->cur]), chain_u4, src, dst0, step, n);
    TSB_CUDA(cudaGetLastError());
    return TSB_OK;
}

int tsb_domino_cftp(tsb_domino *h, const uint8_t *top0, const uint8_t *bot0, const uint64_t *masters,
                    int count, int max_doublings, uint8_t *out_states, int32_t *collapsed_round,
                    tsb_progress_fn progress, void *user) {
    if (!h || !top0 || !bot0 || !masters || !out_states) return fail(TSB_E_VALUE, "null argument");
    TSB_FULL_ONLY(h);
    if (count <= 0) return TSB_OK;
    if (h->nchains < 2 * count + 2)
        return fail(TSB_E_VALUE, "handle needs >= %d chains for %d samples", 2 * count + 2, count);
    const int T = 2 * count, B = 2 * count + 1;
    int rc;
    if ((rc = tsb_domino_upload(h, T, 1, top0))) return rc;
    if ((rc = tsb_domino_upload(h, B, 1, bot0))) return rc;
    const size_t grid = (size_t)h->side * h->side;
    std::vector<int> active(count);
    for (int k = 0; k < count; ++k) {
        active[k] = k;
        if (collapsed_round) collapsed_round[k] = 0;
    }
    std::vector<uint64_t> seeds;
    std::vector<uint8_t> flags;
    uint64_t steps_total = 0;
    for (int round_no = 1; round_no <= max_doublings; ++round_no) {
        steps_total += 1ull << round_no;
        const int na = (int)active.size();
        if ((rc = tsb_domino_replicate(h, T, 0, 2, na))) return rc;
        if ((rc = tsb_domino_replicate(h, B, 1, 2, na))) return rc;
        // newest pair first: pair i runs 2**i sweeps (cftp.py:115-119)
        for (int i = round_no; i >= 1; --i) {
            seeds.assign(2 * na, 0);
            for (int j = 0; j < na; ++j)
                seeds[2 * j] = seeds[2 * j + 1] = derive_seed(masters[active[j]], (uint64_t)i, kSeedSalt);
            h->coupled = true;  // pairs share seeds: draw each coin once per pair
            rc = tsb_domino_walk(h, 0, 2 * na, seeds.data(), 0, 1ull << i);
            h->coupled = false;
            if (rc) return rc;
        }
        flags.assign(na, 0);
        if ((rc = tsb_domino_coalesced(h, 0, na, flags.data()))) return rc;
        std::vector<int> still;
        for (int j = 0; j < na; ++j) {
            if (flags[j]) {
                const int k = active[j];
                if ((rc = tsb_domino_download(h, 2 * j + 1, 1, out_states + (size_t)k * grid))) return rc;
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
