// Device-driven strip exchange over peer memory.
//
// One lattice is split into row strips, one per GPU (one process per GPU on
// one node).  Every rank sweeps its strip plus `halo` rows on each side
// (tsb_domino_set_window); after `halo` sweeps the strip rows are still exact
// and the halo rows are refreshed from the neighbours.  The host-driven
// version (strips.py StripWalker) does that refresh with NCCL send/recv from
// Python; here it is a pair of kernels in the walk's own stream:
//
//   push:  my rows [lo, lo+halo)  -> up neighbour's staging "from_dn"[e & 1]
//          my rows [hi-halo, hi)  -> down neighbour's staging "from_up"[e & 1]
//          (stores into the peer's memory over NVLink / NVSwitch), then the
//          last block raises the peer's flag to epoch e (system-scope release)
//   pull:  wait until my flags from both neighbours reach e, then copy the
//          staging slots into my halo rows [lo-halo, lo) and [hi, hi+halo)
//
// so a multi-GPU walk is enqueued once and runs without any host round trip.
// Staging is double-buffered by epoch parity: a neighbour can only push epoch
// e+2 into slot e&1 after it pulled my epoch e+1 push, which I issue after my
// own pull of epoch e, so a slot is never overwritten before it was consumed.
// Every coin is pure in (seed, site, step), so the result is bit-identical to
// the single-GPU walk (tests/test_strips_gpu.py).
//
// Exchange regions are plain cudaMalloc allocations exported with CUDA IPC
// (cudaIpcGetMemHandle / cudaIpcOpenMemHandle); handles in one process (the
// single-GPU tests) are connected directly.
#include <algorithm>

#include "domino.cuh"

struct tsb_strip {
    int lo = 0, hi = 0, halo = 0;
    size_t slot = 0;                 // uint2 per staging slot (halo rows x pitch)
    uint2 *region = nullptr;         // own: [from_up 0][from_up 1][from_dn 0][from_dn 1], then 2 flags
    uint2 *peer_up = nullptr, *peer_dn = nullptr;  // neighbours' regions
    bool up_ipc = false, dn_ipc = false;
    unsigned int *counter = nullptr;  // push-kernel completion counter (own)
    uint64_t *epoch_dev = nullptr;    // rounds completed (device; read by push / pull)
    uint64_t epoch = 0;               // rounds enqueued (host)
};

namespace tsb {

constexpr int kStripBlocks = 64;

__device__ __forceinline__ uint64_t *region_flags(uint2 *region, size_t slot) {
    return reinterpret_cast<uint64_t *>(region + 4 * slot);
}

__device__ __forceinline__ void copy_rows(uint2 *dst, const uint2 *src, size_t n) {
    const size_t i0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x, step = (size_t)gridDim.x * blockDim.x;
    for (size_t i = i0; i < n; i += step) dst[i] = src[i];
}

// push epoch e: own boundary rows into the neighbours' staging slots
__global__ void strip_push_kernel(const uint2 *rows_top, const uint2 *rows_bot, uint2 *peer_up, uint2 *peer_dn,
                                  size_t slot, const uint64_t *epoch_dev, unsigned int *counter) {
    const uint64_t e = *epoch_dev + 1;  // this round's epoch (advanced after the pull)
    const int par = (int)(e & 1);
    if (peer_up) copy_rows(peer_up + (2 + par) * slot, rows_top, slot);  // up's from_dn[par]
    if (peer_dn) copy_rows(peer_dn + par * slot, rows_bot, slot);        // down's from_up[par]
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int done = atomicAdd(counter, 1u);
        if (done == gridDim.x - 1) {  // last block: every block's stores are visible system-wide
            *counter = 0u;
            __threadfence_system();
            if (peer_up) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(region_flags(peer_up, slot) + 1), "l"(e) : "memory");
            if (peer_dn) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(region_flags(peer_dn, slot) + 0), "l"(e) : "memory");
        }
    }
}

// pull epoch e: wait for both neighbours' pushes, then staging -> halo rows
__global__ void strip_pull_kernel(uint2 *halo_top, uint2 *halo_bot, uint2 *region, size_t slot,
                                  const uint64_t *epoch_dev, int has_up, int has_dn) {
    const uint64_t e = *epoch_dev + 1;
    __shared__ int timed_out;
    if (threadIdx.x == 0) {
        uint64_t *fl = region_flags(region, slot);
        timed_out = 0;
        // bounded spin (~20 s): a neighbour that never pushes is reported
        // through flag word 2 (tsb_domino_strip_status) instead of hanging
        for (int side = 0; side < 2; ++side) {
            if (!(side == 0 ? has_up : has_dn)) continue;
            uint64_t v;
            long long spins = 0;
            for (;;) {
                asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(fl + side) : "memory");
                if (v >= e) break;
                if (++spins > (1ll << 26)) {
                    timed_out = 1;
                    atomicMax((unsigned long long *)(fl + 2), (unsigned long long)e);
                    break;
                }
                __nanosleep(256);
            }
        }
    }
    __syncthreads();
    if (timed_out) return;
    const int par = (int)(e & 1);
    const size_t i0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x, step = (size_t)gridDim.x * blockDim.x;
    if (has_up) {
        const uint2 *src = region + par * slot;
        for (size_t i = i0; i < slot; i += step) halo_top[i] = __ldcv(src + i);
    }
    if (has_dn) {
        const uint2 *src = region + (2 + par) * slot;
        for (size_t i = i0; i < slot; i += step) halo_bot[i] = __ldcv(src + i);
    }
}

__global__ void strip_epoch_advance(uint64_t *epoch_dev) { *epoch_dev += 1; }

// Enqueue push, pull and epoch advance of one round on `stream` (also used
// while capturing the walk graph: the round then replays with the sweeps).
int strip_exchange(tsb_domino *h, cudaStream_t stream) {
    tsb_strip *s = h->strip;
    if (!s || (!s->peer_up && !s->peer_dn)) return TSB_OK;
    uint2 *rows = h->buf[h->cur] + h->pitch;  // chain 0, row 0 (after the guard row)
    strip_push_kernel<<<kStripBlocks, 256, 0, stream>>>(rows + (size_t)s->lo * h->pitch,
                                                        rows + (size_t)(s->hi - s->halo) * h->pitch, s->peer_up,
                                                        s->peer_dn, s->slot, s->epoch_dev, s->counter);
    strip_pull_kernel<<<kStripBlocks, 256, 0, stream>>>(rows + (size_t)(s->lo - s->halo) * h->pitch,
                                                        rows + (size_t)s->hi * h->pitch, s->region, s->slot,
                                                        s->epoch_dev, s->peer_up != nullptr, s->peer_dn != nullptr);
    strip_epoch_advance<<<1, 1, 0, stream>>>(s->epoch_dev);
    TSB_CUDA(cudaGetLastError());
    return TSB_OK;
}

void strip_free(tsb_domino *h) {
    tsb_strip *s = h->strip;
    if (!s) return;
    if (h->stream) cudaStreamSynchronize(h->stream);
    if (s->up_ipc && s->peer_up) cudaIpcCloseMemHandle(s->peer_up);
    if (s->dn_ipc && s->peer_dn) cudaIpcCloseMemHandle(s->peer_dn);
    cudaFree(s->region);
    cudaFree(s->counter);
    cudaFree(s->epoch_dev);
    delete s;
    h->strip = nullptr;
    h->graph_tail = nullptr;
}

}  // namespace tsb

using namespace tsb;

extern "C" {

int tsb_domino_strip_init(tsb_domino *h, int lo, int hi, int halo, void *ipc_handle_out) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    if (lo < 0 || hi > h->side || lo >= hi || halo < 1 || halo > hi - lo)
        return fail(TSB_E_VALUE, "strip [%d, %d) with halo %d is invalid", lo, hi, halo);
    TSB_CUDA(cudaSetDevice(h->device));
    strip_free(h);
    tsb_strip *s = new tsb_strip();
    s->lo = lo;
    s->hi = hi;
    s->halo = halo;
    s->slot = (size_t)halo * h->pitch;
    const size_t bytes = 4 * s->slot * sizeof(uint2) + 3 * sizeof(uint64_t);  // + flags {from_up, from_dn, timeout}
    cudaError_t e = cudaMalloc(&s->region, bytes);
    if (e == cudaSuccess) e = cudaMemset(s->region, 0, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&s->counter, sizeof(unsigned int));
    if (e == cudaSuccess) e = cudaMemset(s->counter, 0, sizeof(unsigned int));
    if (e == cudaSuccess) e = cudaMalloc(&s->epoch_dev, sizeof(uint64_t));
    if (e == cudaSuccess) e = cudaMemset(s->epoch_dev, 0, sizeof(uint64_t));
    if (e == cudaSuccess && ipc_handle_out) e = cudaIpcGetMemHandle((cudaIpcMemHandle_t *)ipc_handle_out, s->region);
    if (e != cudaSuccess) {
        cudaFree(s->region);
        cudaFree(s->counter);
        cudaFree(s->epoch_dev);
        delete s;
        return cuda_fail(e, "strip init");
    }
    h->strip = s;
    int rc = tsb_domino_set_window(h, lo - halo, hi + halo);
    return rc;
}

int tsb_domino_strip_connect(tsb_domino *h, const void *up_handle, const void *dn_handle) {
    if (!h || !h->strip) return fail(TSB_E_VALUE, "strip not initialised");
    TSB_CUDA(cudaSetDevice(h->device));
    tsb_strip *s = h->strip;
    void *p = nullptr;
    if (up_handle) {
        TSB_CUDA(cudaIpcOpenMemHandle(&p, *(const cudaIpcMemHandle_t *)up_handle, cudaIpcMemLazyEnablePeerAccess));
        s->peer_up = (uint2 *)p;
        s->up_ipc = true;
    }
    if (dn_handle) {
        TSB_CUDA(cudaIpcOpenMemHandle(&p, *(const cudaIpcMemHandle_t *)dn_handle, cudaIpcMemLazyEnablePeerAccess));
        s->peer_dn = (uint2 *)p;
        s->dn_ipc = true;
    }
    return TSB_OK;
}

int tsb_domino_strip_connect_local(tsb_domino *h, tsb_domino *up, tsb_domino *dn) {
    if (!h || !h->strip) return fail(TSB_E_VALUE, "strip not initialised");
    if ((up && !up->strip) || (dn && !dn->strip)) return fail(TSB_E_VALUE, "neighbour strip not initialised");
    h->strip->peer_up = up ? up->strip->region : nullptr;
    h->strip->peer_dn = dn ? dn->strip->region : nullptr;
    return TSB_OK;
}

// One exchange round, split in its two stream-ordered halves: phase 0 walks
// k sweeps from step0 and pushes this rank's boundary rows to the neighbours
// (epoch += 1); phase 1 waits for the neighbours' pushes of that epoch and
// pulls them into the halo rows.  tsb_domino_strip_walk enqueues both phases
// for every round; running phase 0 on every rank before phase 1 (host lockstep)
// lets several handles share one GPU without relying on concurrent streams.
int tsb_domino_strip_step(tsb_domino *h, uint64_t step0, uint64_t k, int phase) {
    if (!h || !h->strip) return fail(TSB_E_VALUE, "strip not initialised");
    tsb_strip *s = h->strip;
    TSB_CUDA(cudaSetDevice(h->device));
    if (!s->peer_up && !s->peer_dn) return phase == 0 && k ? walk_steps(h, 0, 1, step0, k) : TSB_OK;
    uint2 *rows = h->buf[h->cur] + h->pitch;  // chain 0, row 0 (after the guard row)
    int rc;
    if (phase == 0) {
        if (k && (rc = walk_steps(h, 0, 1, step0, k))) return rc;
        rows = h->buf[h->cur] + h->pitch;
        ++s->epoch;
        strip_push_kernel<<<kStripBlocks, 256, 0, h->stream>>>(rows + (size_t)s->lo * h->pitch,
                                                              rows + (size_t)(s->hi - s->halo) * h->pitch,
                                                              s->peer_up, s->peer_dn, s->slot, s->epoch_dev, s->counter);
    } else {
        strip_pull_kernel<<<kStripBlocks, 256, 0, h->stream>>>(rows + (size_t)(s->lo - s->halo) * h->pitch,
                                                              rows + (size_t)s->hi * h->pitch, s->region, s->slot,
                                                              s->epoch_dev, s->peer_up != nullptr, s->peer_dn != nullptr);
        strip_epoch_advance<<<1, 1, 0, h->stream>>>(s->epoch_dev);
    }
    TSB_CUDA(cudaGetLastError());
    return TSB_OK;
}

int tsb_domino_strip_seed(tsb_domino *h, uint64_t seed) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    TSB_CUDA(cudaSetDevice(h->device));
    return push_seeds(h, 1, &seed);
}

int tsb_domino_strip_walk(tsb_domino *h, uint64_t seed, uint64_t step0, uint64_t n_steps) {
    if (!h || !h->strip) return fail(TSB_E_VALUE, "strip not initialised");
    tsb_strip *s = h->strip;
    int rc = tsb_domino_strip_seed(h, seed);
    uint64_t done = 0;
    if (!rc && s->halo == kGraphSweeps && n_steps >= (uint64_t)kGraphSweeps && (s->peer_up || s->peer_dn)) {
        // full rounds: the walk graph's replay carries the exchange as its tail
        // (push, pull, epoch advance), so one graph launch per round
        h->graph_tail = strip_exchange;
        const uint64_t rounds = n_steps / kGraphSweeps;
        rc = walk_steps(h, 0, 1, step0, rounds * kGraphSweeps);
        h->graph_tail = nullptr;
        s->epoch += rounds;
        done = rounds * kGraphSweeps;
    }
    for (; !rc && done < n_steps;) {
        const uint64_t k = std::min<uint64_t>((uint64_t)s->halo, n_steps - done);
        rc = tsb_domino_strip_step(h, step0 + done, k, 0);
        if (!rc) rc = tsb_domino_strip_step(h, 0, 0, 1);
        done += k;
    }
    return rc;
}

int tsb_domino_strip_status(tsb_domino *h, uint64_t *epoch, uint64_t *timed_out_epoch) {
    if (!h || !h->strip) return fail(TSB_E_VALUE, "strip not initialised");
    TSB_CUDA(cudaSetDevice(h->device));
    TSB_CUDA(cudaStreamSynchronize(h->stream));
    uint64_t fl[3];
    TSB_CUDA(cudaMemcpy(fl, h->strip->region + 4 * h->strip->slot, sizeof fl, cudaMemcpyDeviceToHost));
    if (epoch) *epoch = h->strip->epoch;
    if (timed_out_epoch) *timed_out_epoch = fl[2];
    if (fl[2]) return fail(TSB_E_CUDA, "strip exchange timed out waiting for a neighbour at epoch %llu",
                           (unsigned long long)fl[2]);
    return TSB_OK;
}

int tsb_domino_strip_close(tsb_domino *h) {
    if (!h) return fail(TSB_E_VALUE, "null handle");
    TSB_CUDA(cudaSetDevice(h->device));
    strip_free(h);
    return tsb_domino_set_window(h, 0, -1);
}

}  // extern "C"
