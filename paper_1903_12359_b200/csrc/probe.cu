// probe.cu -- bandwidth probe for bench.py's roofline denominators.
//
// k_l2_probe streams a buffer that fits in L2 (bench.py uses 48 MiB of the
// 126 MB) `reps` times with 16-byte L2-only loads (ld.global.cg: no L1
// allocation), eight loads in flight per thread, a persistent grid of 4
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
    int acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int r = 0; r < reps; ++r) {
        int64_t i = t0;
        for (; i + (U - 1) * stride < n16; i += U * stride) {
            int4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = __ldcg(buf + i + u * stride);
#pragma unroll
            for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].w ^ v[u].y ^ v[u].z;
        }
        for (; i < n16; i += stride) {
            int4 a = __ldcg(buf + i);
            acc ^= a.x ^ a.w;
        }
    }
    if (acc == 0x7f3a5c11) atomicAdd(sink, 1ull);  // keeps the loads live
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
    // 8 independent 16-byte loads per thread in flight (4 with PGCP_L2_PROBE_U=4)
    const char* eu = getenv("PGCP_L2_PROBE_U");
    if (eu && atoi(eu) == 4)
        k_l2_probe<4><<<4 * sms, 512, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
            reinterpret_cast<const int4*>(buf), bytes / 16, reps, sink);
    else
        k_l2_probe<8><<<4 * sms, 512, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
            reinterpret_cast<const int4*>(buf), bytes / 16, reps, sink);
    PGCP_LAUNCH_CHECK();
    return PGCP_OK;
}

}  // extern "C"
