// probe.cu -- bandwidth probe for bench.py's roofline denominators.
//
// k_l2_probe streams a buffer that fits in L2 (bench.py uses 48 MiB of the
// 126 MB) `reps` times with 16-byte L2-only loads (ld.global.cg: no L1
// allocation), four loads in flight per thread, a persistent grid of 4
// CTAs x 512 threads per SM. bytes x reps / time is the L2 -> SM read
// bandwidth a streaming kernel can reach on this part; the PCG kernel's
// working set is served from there.
#include <cstdlib>

#include "batch.cuh"

namespace pgcp {
namespace {

template <int U>
__global__ void __launch_bounds__(512) k_l2_probe(const int4* __restrict__ buf, int64_t n16, int reps,
                                                  unsigned long long* __restrict__ sink) {
    // one continuous stream of reps x n16 loads per grid (the index wraps at
    // the buffer end), U independent loads in flight per thread
    int acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t total = (int64_t)reps * n16;
    int64_t idx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) idx[u] = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x + u * stride) % n16;
    const int64_t step = (U * stride) % n16;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v + (U - 1) * stride < total; v += U * stride) {
        int4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = __ldcg(buf + idx[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            acc ^= x[u].x ^ x[u].w ^ x[u].y ^ x[u].z;
            idx[u] += step;
            if (idx[u] >= n16) idx[u] -= n16;
        }
    }
    if (acc == 0x7f3a5c11) atomicAdd(sink, 1ull);  // keeps the loads live
}

// FP64 FMA throughput: 8 independent chains per thread, no memory traffic
__global__ void __launch_bounds__(256) k_fp64_probe(int iters, double seed, double* __restrict__ sink) {
    double a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = seed + 1e-3 * (threadIdx.x + u);
    const double m = 0.999999, c = 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] = fma(a[u], m, c);
    }
    double t = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) t += a[u];
    if (t == 12345.678) sink[0] = t;  // keeps the chains live
}

}  // namespace
}  // namespace pgcp

using namespace pgcp;

extern "C" {

// Streams buf[0, bytes) reps times through L2 (see above). Not part of the
// PGCP path: a measurement kernel for the roofline's L2 denominator.
PGCP_API int pgcp_l2_probe(const void* buf, int64_t bytes, int32_t reps, unsigned long long* sink, void* stream) {
    if (!buf || bytes < 16 || reps < 1 || !sink) {
        set_error("pgcp_l2_probe: invalid arguments");
        return PGCP_E_INVALID;
    }
    int dev = 0, sms = 148;
    PGCP_TRY_CUDA(cudaGetDevice(&dev));
    PGCP_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // 4 independent 16-byte loads per thread in flight (8 with PGCP_L2_PROBE_U=8;
    // tools/l2_probe_sweep.py: 4 reaches the higher rate)
    const char* eu = getenv("PGCP_L2_PROBE_U");
    if (!(eu && atoi(eu) == 8))
        k_l2_probe<4><<<4 * sms, 512, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
            reinterpret_cast<const int4*>(buf), bytes / 16, reps, sink);
    else
        k_l2_probe<8><<<4 * sms, 512, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
            reinterpret_cast<const int4*>(buf), bytes / 16, reps, sink);
    PGCP_LAUNCH_CHECK();
    return PGCP_OK;
}

// FP64 peak probe for the direct solver's roofline: grid 8 CTAs x 256
// threads per SM, 8 FMA chains per thread; flops = 2 * 8 * iters * threads.
PGCP_API int pgcp_fp64_probe(int32_t iters, double* sink, int64_t* threads_out, void* stream) {
    if (iters < 1 || !sink || !threads_out) {
        set_error("pgcp_fp64_probe: invalid arguments");
        return PGCP_E_INVALID;
    }
    int dev = 0, sms = 148;
    PGCP_TRY_CUDA(cudaGetDevice(&dev));
    PGCP_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    k_fp64_probe<<<8 * sms, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(iters, 1.0, sink);
    PGCP_LAUNCH_CHECK();
    *threads_out = (int64_t)8 * sms * 256;
    return PGCP_OK;
}

}  // extern "C"
