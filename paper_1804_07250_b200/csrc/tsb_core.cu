// Library-wide plumbing: error channel, device checks, the device RNG grid.
#include "tsb_internal.cuh"

namespace tsb {

static thread_local std::string g_err;

void set_error(const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
}

int fail(int code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char *what) {
    return fail(TSB_E_CUDA, "CUDA error %s (%s) in %s", cudaGetErrorName(e), cudaGetErrorString(e),
                what);
}

int ensure_device(int device) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return fail(TSB_E_NODEVICE, "no CUDA device available (%s); libtsb has no CPU fallback",
                    e == cudaSuccess ? "0 devices" : cudaGetErrorString(e));
    if (device < 0 || device >= n) return fail(TSB_E_VALUE, "device %d out of range [0,%d)", device, n);
    cudaDeviceProp prop;
    TSB_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0)
        return fail(TSB_E_NODEVICE, "device %d is sm_%d%d; libtsb is built for sm_100a only", device,
                    prop.major, prop.minor);
    TSB_CUDA(cudaSetDevice(device));
    return TSB_OK;
}

// K1: StreamFamily.uniform_grid (rng.py:105-123) on the device.
__global__ void uniform_grid_kernel(uint64_t base, int64_t count, uint64_t tag, uint64_t step,
                                    double *out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= count) return;
    uint64_t key = mix64(base + (((tag << 48) + (uint64_t)i) + 1ull) * kGold);
    out[i] = (double)(draw(key, step) >> 11) * 0x1p-53;
}

}  // namespace tsb

using namespace tsb;

extern "C" {

const char *tsb_last_error(void) { return g_err.c_str(); }

int tsb_abi_version(void) { return 1; }

int tsb_device_info(int device, int *sm_count, int *cc_major, int *cc_minor, int64_t *l2_bytes) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        return fail(TSB_E_NODEVICE, "no CUDA device available");
    if (device < 0 || device >= n) return fail(TSB_E_VALUE, "device %d out of range", device);
    cudaDeviceProp p;
    TSB_CUDA(cudaGetDeviceProperties(&p, device));
    if (sm_count) *sm_count = p.multiProcessorCount;
    if (cc_major) *cc_major = p.major;
    if (cc_minor) *cc_minor = p.minor;
    if (l2_bytes) *l2_bytes = p.l2CacheSize;
    return TSB_OK;
}

int tsb_uniform_grid(int device, uint64_t seed, int rows, int cols, uint64_t step, int tag,
                     double *out) {
    if (rows <= 0 || cols <= 0) return fail(TSB_E_VALUE, "grid shape must be positive");
    if ((uint64_t)rows * (uint64_t)cols >= kCapacity)
        return fail(TSB_E_CAPACITY, "grid of %lld sites exceeds the 2^48 stream capacity",
                    (long long)rows * cols);
    int rc = ensure_device(device);
    if (rc) return rc;
    int64_t count = (int64_t)rows * cols;
    double *d = nullptr;
    TSB_CUDA(cudaMalloc(&d, sizeof(double) * count));
    uniform_grid_kernel<<<(unsigned)((count + 255) / 256), 256>>>(family_base(seed), count,
                                                                 (uint64_t)tag, step, d);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(out, d, sizeof(double) * count, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return cuda_fail(e, "uniform_grid");
    return TSB_OK;
}

}  // extern "C"
