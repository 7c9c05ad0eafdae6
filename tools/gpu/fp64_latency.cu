// FP64 dependent-chain latencies on the B200 (one thread): the costs that
// bound the weld's serial record chain (weld.cu k_phase1w).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/gpu/fp64_latency.cu -o /tmp/fp64_lat && /tmp/fp64_lat
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k_chain(double x0, int n, double* out, long long* cyc) {
    double x = x0, y = 1.000001;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (OP == 0) x = fma(x, y, 1e-300);                 // DFMA
        if (OP == 1) x = 1.0 / x + 1e-300;                   // IEEE division (reciprocal form)
        if (OP == 2) x = sqrt(x) + 1.5;                      // IEEE sqrt
        if (OP == 3) x = rsqrt(x) + 1.5;                     // rsqrt
        if (OP == 4) x = __drcp_rn(x) + 1e-300;              // correctly rounded reciprocal
        if (OP == 5) x = y / x + 1e-300;                     // general division
        if (OP == 6) x = hypot(x, y);                        // hypot
    }
    long long t1 = clock64();
    out[0] = x;
    cyc[OP] = (t1 - t0) / n;
}

int main() {
    double* d;
    long long* c;
    cudaMalloc(&d, 8);
    cudaMalloc(&c, 16 * 8);
    const int n = 4096;
    for (int rep = 0; rep < 2; ++rep) {
        k_chain<0><<<1, 1>>>(1.1, n, d, c);
        k_chain<1><<<1, 1>>>(1.1, n, d, c);
        k_chain<2><<<1, 1>>>(1.1, n, d, c);
        k_chain<3><<<1, 1>>>(1.1, n, d, c);
        k_chain<4><<<1, 1>>>(1.1, n, d, c);
        k_chain<5><<<1, 1>>>(1.1, n, d, c);
        k_chain<6><<<1, 1>>>(1.1, n, d, c);
        cudaDeviceSynchronize();
    }
    long long h[7];
    cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    const char* names[7] = {"dfma", "1/x", "sqrt", "rsqrt", "__drcp_rn", "y/x", "hypot"};
    for (int i = 0; i < 7; ++i) printf("%-10s %lld cycles (incl. the add)\n", names[i], h[i]);
    return 0;
}
