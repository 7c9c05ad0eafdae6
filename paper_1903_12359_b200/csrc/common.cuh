// common.cuh -- shared device utilities for libpgcp_b200 (sm_100a).
//
// Errors, stream-ordered scratch, device-wide scans and a deterministic
// stable counting sort (the "segmented sort-by-key" primitive the partition
// and CSR builders are made of).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/pgcp_b200.h"

namespace pgcp {

// ---------------------------------------------------------------------------
// error plumbing

void set_error(const char* fmt, ...);
const char* get_error();

struct Status {
    int code = PGCP_OK;
};

#define PGCP_TRY_CUDA(expr)                                                        \
    do {                                                                           \
        cudaError_t _e = (expr);                                                   \
        if (_e != cudaSuccess) {                                                   \
            ::pgcp::set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e),  \
                              __FILE__, __LINE__, cudaGetErrorString(_e));         \
            return PGCP_E_CUDA;                                                    \
        }                                                                          \
    } while (0)

#define PGCP_TRY(expr)            \
    do {                          \
        int _s = (expr);          \
        if (_s != PGCP_OK) return _s; \
    } while (0)

// every kernel launch site is followed by PGCP_LAUNCH_CHECK(), which also
// counts the launch (pgcp_launch_count, bench.py's gpu_launches)
void count_launch();
#define PGCP_LAUNCH_CHECK()          \
    do {                             \
        ::pgcp::count_launch();      \
        PGCP_TRY_CUDA(cudaGetLastError()); \
    } while (0)

// Device-side error record: the first (lowest index) failure wins so that the
// reported item is deterministic.
struct DevErr {
    int code;
    int pad;
    unsigned long long index;  // atomicMin target
    long long aux;
};

__device__ __forceinline__ void dev_fail(DevErr* e, int code, long long index, long long aux = 0) {
    unsigned long long idx = (unsigned long long)index;
    unsigned long long old = atomicMin(&e->index, idx);
    if (idx < old) {
        e->code = code;  // benign race between equal-priority writers
        e->aux = aux;
    }
    __threadfence();
}

// ---------------------------------------------------------------------------
// stream-ordered scratch (freed by the owner on the same stream)

template <class T>
struct DevBuf {
    T* p = nullptr;
    int64_t n = 0;
    cudaStream_t s = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        release();
        p = o.p; n = o.n; s = o.s;
        o.p = nullptr; o.n = 0;
        return *this;
    }
    ~DevBuf() { release(); }
    int alloc(int64_t count, cudaStream_t stream) {
        release();
        s = stream;
        n = count;
        size_t bytes = (size_t)(count > 0 ? count : 1) * sizeof(T);
        PGCP_TRY_CUDA(cudaMallocAsync((void**)&p, bytes, stream));
        return PGCP_OK;
    }
    int zero(cudaStream_t stream) {
        if (n > 0) PGCP_TRY_CUDA(cudaMemsetAsync(p, 0, (size_t)n * sizeof(T), stream));
        return PGCP_OK;
    }
    int fill_bytes(int byte, cudaStream_t stream) {
        if (n > 0) PGCP_TRY_CUDA(cudaMemsetAsync(p, byte, (size_t)n * sizeof(T), stream));
        return PGCP_OK;
    }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
};

inline int grid_for(int64_t n, int block, int cap = 148 * 16) {
    int64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (int)g;
}

#define GRID_STRIDE(i, n) \
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// ---------------------------------------------------------------------------
// warp / block reductions

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ---------------------------------------------------------------------------
// device-wide exclusive scan: out[i] = sum_{j<i} f(j), out[n] = total.
// Three passes (tile sums, scan of tile sums, tile-local scan + offset);
// deterministic (integer).

int exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t s);
int exclusive_scan_i32_to_i64(const int32_t* in, int64_t* out, int64_t n, cudaStream_t s);

// Stable counting sort by small key: for keys[i] in [0, nkeys), produces
// perm (position -> original index, stable) and key_off[nkeys+1].
int stable_counting_sort(const int32_t* keys, int64_t n, int32_t nkeys, int32_t* perm,
                         int64_t* key_off, cudaStream_t s);

// Device -> host reads through a per-thread pinned staging buffer. A copy
// into pageable memory is staged by the driver synchronously and can wait
// for unrelated work (e.g. a weld running on the legacy default stream while
// the Dirichlet systems are prepared on another thread); a pinned
// destination is a plain DMA on `s`. d2h_async queues a copy, d2h_flush
// synchronises `s` and delivers every queued copy to its destination.
int d2h_async(void* host, const void* dev, size_t bytes, cudaStream_t s);
int d2h_flush(cudaStream_t s);

// copy one scalar back (synchronises the stream)
template <class T>
int fetch_scalar(const T* dptr, T* host, cudaStream_t s) {
    PGCP_TRY(d2h_async(host, dptr, sizeof(T), s));
    return d2h_flush(s);
}

}  // namespace pgcp
