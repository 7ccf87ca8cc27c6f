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

// Connected components of a cell grid (4-neighbourhood) by lock-free
// union-find (Domain validation, lattice.py:99-132,
// whose DFS is O(n^2) pure Python).  label[i] = parent index, -1 outside.
__device__ __forceinline__ int uf_find(const int *L, int x) {
    int p = L[x];
    while (p != x) {
        x = p;
        p = L[x];
    }
    return x;
}

__device__ void uf_unite(int *L, int a, int b) {
    for (;;) {
        a = uf_find(L, a);
        b = uf_find(L, b);
        if (a == b) return;
        if (a > b) {
            const int t = a;
            a = b;
            b = t;
        }
        // link the larger root under the smaller one; retry if b was re-linked meanwhile
        const int old = atomicCAS(&L[b], b, a);
        if (old == b) return;
        b = old;
    }
}

__global__ void cc_init(const uint8_t *grid, int64_t n, int *L) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) L[i] = grid[i] ? (int)i : -1;
}

__global__ void cc_merge(int rows, int cols, int *L) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= (int64_t)rows * cols || L[i] < 0) return;
    const int c = (int)(i % cols);
    if (c + 1 < cols && L[i + 1] >= 0) uf_unite(L, (int)i, (int)(i + 1));
    if (i + cols < (int64_t)rows * cols && L[i + cols] >= 0) uf_unite(L, (int)i, (int)(i + cols));
}

__global__ void cc_count_roots(const int *L, int64_t n, unsigned long long *count) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int root = i < n && L[i] == (int)i;
    const unsigned long long k = __popc(__ballot_sync(0xffffffffu, root));
    if ((threadIdx.x & 31) == 0 && k) atomicAdd(count, k);
}

// TriDomain checks (lozenge.py:185-210): triangle ids up(x,y) = x*sy + y,
// down(x,y) = n + x*sy + y; up(x,y) is edge-adjacent to down(x,y),
// down(x-1,y) and down(x,y-1) (lozenge.py:172-178 _neighbors).
__global__ void tri_init(const uint8_t *up, const uint8_t *down, int64_t n, int *L) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        L[i] = up[i] ? (int)i : -1;
        L[n + i] = down[i] ? (int)(n + i) : -1;
    }
}

__global__ void tri_merge(int sx, int sy, int *L) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t n = (int64_t)sx * sy;
    if (i >= n || L[i] < 0) return;
    const int x = (int)(i / sy), y = (int)(i % sy);
    if (L[n + i] >= 0) uf_unite(L, (int)i, (int)(n + i));
    if (x > 0 && L[n + i - sy] >= 0) uf_unite(L, (int)i, (int)(n + i - sy));
    if (y > 0 && L[n + i - 1] >= 0) uf_unite(L, (int)i, (int)(n + i - 1));
}

// Euler characteristic V - E + F over the (sx+1) x (sy+1) vertex grid, the
// same edge sets as lozenge.py:197-210: a(x,y) = up(x,y) | down(x,y-1),
// b(x,y) = up(x,y) | down(x-1,y), c(x,y) = up(x,y-1) | down(x,y-1).
__global__ void tri_euler(const uint8_t *up, const uint8_t *down, int sx, int sy, long long *chi) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int Y = sy + 1;
    int v = 0;
    if (i < (int64_t)(sx + 1) * Y) {
        const int x = (int)(i / Y), y = (int)(i % Y);
        auto U = [&](int a, int b) { return a >= 0 && b >= 0 && a < sx && b < sy && up[(size_t)a * sy + b]; };
        auto D = [&](int a, int b) { return a >= 0 && b >= 0 && a < sx && b < sy && down[(size_t)a * sy + b]; };
        const bool vert = U(x, y) || U(x - 1, y) || U(x, y - 1) || D(x - 1, y) || D(x, y - 1) || D(x - 1, y - 1);
        const int e = (U(x, y) || D(x, y - 1)) + (U(x, y) || D(x - 1, y)) + (U(x, y - 1) || D(x, y - 1));
        const int f = U(x, y) + D(x, y);
        v = (int)vert - e + f;
    }
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(reinterpret_cast<unsigned long long *>(chi), (unsigned long long)(long long)v);
}

}  // namespace tsb

using namespace tsb;

extern "C" {

const char *tsb_last_error(void) { return g_err.c_str(); }

int tsb_abi_version(void) { return 1; }

int tsb_grid_components(int device, const uint8_t *grid, int rows, int cols, int64_t *ncomp) {
    if (!grid || !ncomp || rows < 1 || cols < 1) return fail(TSB_E_VALUE, "bad grid arguments");
    const int64_t n = (int64_t)rows * cols;
    if (n >= (1ll << 31)) return fail(TSB_E_CAPACITY, "grid of %lld cells exceeds 2^31", (long long)n);
    int rc = ensure_device(device);
    if (rc) return rc;
    uint8_t *dg = nullptr;
    int *L = nullptr;
    unsigned long long *dc = nullptr;
    cudaError_t e = cudaMalloc(&dg, n);
    if (e == cudaSuccess) e = cudaMalloc(&L, sizeof(int) * n);
    if (e == cudaSuccess) e = cudaMalloc(&dc, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemcpy(dg, grid, n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(dc, 0, sizeof(unsigned long long));
    const unsigned blocks = (unsigned)((n + 255) / 256);
    if (e == cudaSuccess) {
        cc_init<<<blocks, 256>>>(dg, n, L);
        cc_merge<<<blocks, 256>>>(rows, cols, L);
        cc_count_roots<<<blocks, 256>>>(L, n, dc);
        e = cudaGetLastError();
    }
    unsigned long long k = 0;
    if (e == cudaSuccess) e = cudaMemcpy(&k, dc, sizeof k, cudaMemcpyDeviceToHost);
    cudaFree(dg);
    cudaFree(L);
    cudaFree(dc);
    if (e != cudaSuccess) return cuda_fail(e, "grid components");
    *ncomp = (int64_t)k;
    return TSB_OK;
}

int tsb_tri_check(int device, const uint8_t *up, const uint8_t *down, int sx, int sy, int64_t *ncomp,
                  int64_t *euler) {
    if (!up || !down || !ncomp || !euler || sx < 1 || sy < 1) return fail(TSB_E_VALUE, "bad triangle grids");
    const int64_t n = (int64_t)sx * sy;
    if (2 * n >= (1ll << 31)) return fail(TSB_E_CAPACITY, "%lld triangles exceed 2^31", (long long)(2 * n));
    int rc = ensure_device(device);
    if (rc) return rc;
    uint8_t *du = nullptr;
    int *L = nullptr;
    unsigned long long *dc = nullptr;
    long long *dchi = nullptr;
    cudaError_t e = cudaMalloc(&du, 2 * n);
    if (e == cudaSuccess) e = cudaMalloc(&L, sizeof(int) * 2 * n);
    if (e == cudaSuccess) e = cudaMalloc(&dc, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMalloc(&dchi, sizeof(long long));
    if (e == cudaSuccess) e = cudaMemcpy(du, up, n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(du + n, down, n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(dc, 0, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(dchi, 0, sizeof(long long));
    if (e == cudaSuccess) {
        const unsigned b1 = (unsigned)((n + 255) / 256), b2 = (unsigned)((2 * n + 255) / 256);
        const int64_t nv = (int64_t)(sx + 1) * (sy + 1);
        tri_init<<<b1, 256>>>(du, du + n, n, L);
        tri_merge<<<b1, 256>>>(sx, sy, L);
        cc_count_roots<<<b2, 256>>>(L, 2 * n, dc);
        tri_euler<<<(unsigned)((nv + 255) / 256), 256>>>(du, du + n, sx, sy, dchi);
        e = cudaGetLastError();
    }
    unsigned long long k = 0;
    long long chi = 0;
    if (e == cudaSuccess) e = cudaMemcpy(&k, dc, sizeof k, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(&chi, dchi, sizeof chi, cudaMemcpyDeviceToHost);
    cudaFree(du);
    cudaFree(L);
    cudaFree(dc);
    cudaFree(dchi);
    if (e != cudaSuccess) return cuda_fail(e, "triangle domain check");
    *ncomp = (int64_t)k;
    *euler = (int64_t)chi;
    return TSB_OK;
}

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
