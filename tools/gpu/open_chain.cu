// Latency of the weld's Open-record chain on one thread (weld.cu k_phase1w):
// record j's parameter is point j after record j-1, so the chain is
// open_params -> apply_open -> open_params -> ...  Variants of the arithmetic
// are timed side by side, and their results compared.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/gpu/open_chain.cu -o /tmp/oc && /tmp/oc
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double2 C(double x, double y) { return make_double2(x, y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) { return C(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ double2 cdiv(double2 a, double2 b) {
    double abr = fabs(b.x), abi = fabs(b.y);
    if (abr >= abi) {
        double rat = b.y / b.x;
        double scl = 1.0 / (b.x + b.y * rat);
        return C((a.x + a.y * rat) * scl, (a.y - a.x * rat) * scl);
    }
    double rat = b.x / b.y;
    double scl = 1.0 / (b.y + b.x * rat);
    return C((a.x * rat + a.y) * scl, (a.y * rat - a.x) * scl);
}
__device__ __forceinline__ double fast_hypot(double x, double y) {
    const double ax = fabs(x), ay = fabs(y);
    const double m = fmax(ax, ay), n = fmin(ax, ay);
    if (m < 1e150 && (n > 1e-150 || n == 0.0) && m > 1e-150) return sqrt(fma(ax, ax, ay * ay));
    return hypot(x, y);
}
__device__ double2 csqrt_(double2 z) {
    double re = z.x, im = z.y;
    if (im == 0.0 || re == 0.0) return C(sqrt(fabs(re)), 0.0);
    double d = fast_hypot(re, im);
    double r, s;
    if (re > 0) {
        r = sqrt(0.5 * (d + re));
        s = 0.5 * (im / r);
    } else {
        s = sqrt(0.5 * (d - re));
        r = fabs(0.5 * (im / s));
    }
    return C(r, copysign(s, im));
}
// variant: one rsqrt instead of sqrt + division
__device__ double2 csqrt_r(double2 z) {
    double re = z.x, im = z.y;
    if (im == 0.0 || re == 0.0) return C(sqrt(fabs(re)), 0.0);
    double d = fast_hypot(re, im);
    double h = 0.5 * (d + fabs(re));
    double rs = rsqrt(h);
    double big = h * rs, small = fabs(0.5 * im * rs);
    double r = re > 0 ? big : small, s = re > 0 ? 0.5 * im * rs : big;
    return C(r, copysign(fabs(s), im));
}
__device__ __forceinline__ void open_params(double2 xi, double& pp, double& qq) {
    const double s2 = fma(xi.x, xi.x, xi.y * xi.y);
    const double inv = 1.0 / s2;
    pp = xi.x * inv;
    qq = xi.y * inv;
}

template <int V>
__global__ void k_chain(const double2* pts, int n, double2* out, long long* cyc) {
    const int off = threadIdx.x;
    double2 z = pts[off];
    long long t0 = clock64();
    for (int i = 1; i < n; ++i) {
        const double2 p = pts[(i + off) % n];  // independent of the chain (prefetchable)
        double2 L;
        if (V == 0) {  // current: params, numpy division, glibc csqrt
            double pp, qq;
            open_params(z, pp, qq);
            L = cdiv(C(pp * p.x, pp * p.y), C(1.0 - qq * p.y, qq * p.x));
            z = csqrt_(C(fma(L.x, L.x, -L.y * L.y) - 1.0, 2 * L.x * L.y));
        } else if (V == 1) {  // L = x z / (|xi|^2 + i y z), one reciprocal; csqrt with rsqrt
            const double s2 = fma(z.x, z.x, z.y * z.y);
            const double2 D = C(fma(-z.y, p.y, s2), z.y * p.x);
            const double inv = 1.0 / fma(D.x, D.x, D.y * D.y);
            const double2 num = C(z.x * p.x, z.x * p.y);
            L = C((num.x * D.x + num.y * D.y) * inv, (num.y * D.x - num.x * D.y) * inv);
            z = csqrt_r(C(fma(L.x, L.x, -L.y * L.y) - 1.0, 2 * L.x * L.y));
        } else {  // params kept, division by |den|^2 reciprocal, rsqrt csqrt
            double pp, qq;
            open_params(z, pp, qq);
            const double2 D = C(1.0 - qq * p.y, qq * p.x);
            const double inv = 1.0 / fma(D.x, D.x, D.y * D.y);
            const double2 num = C(pp * p.x, pp * p.y);
            L = C((num.x * D.x + num.y * D.y) * inv, (num.y * D.x - num.x * D.y) * inv);
            z = csqrt_r(C(fma(L.x, L.x, -L.y * L.y) - 1.0, 2 * L.x * L.y));
        }
        if (threadIdx.x == 0) out[i] = z;
    }
    if (threadIdx.x == 0) cyc[V] = (clock64() - t0) / n;
}

int main() {
    const int n = 2048;
    double2* h = new double2[n];
    unsigned s = 12345;
    for (int i = 0; i < n; ++i) {
        s = s * 1664525u + 1013904223u;
        double a = (s >> 8) / 16777216.0;
        s = s * 1664525u + 1013904223u;
        double b = (s >> 8) / 16777216.0;
        h[i] = make_double2(0.2 + a, 0.5 + b);
    }
    double2 *d, *o;
    long long* c;
    cudaMalloc(&d, n * 16);
    cudaMalloc(&o, 3 * n * 16);
    cudaMalloc(&c, 64);
    cudaMemcpy(d, h, n * 16, cudaMemcpyHostToDevice);
    for (int lanes : {1, 4, 32}) {
        for (int r = 0; r < 2; ++r) {
            k_chain<0><<<1, lanes>>>(d, n, o, c);
            k_chain<1><<<1, lanes>>>(d, n, o + n, c);
            k_chain<2><<<1, lanes>>>(d, n, o + 2 * n, c);
            cudaDeviceSynchronize();
        }
        long long cy[3];
        cudaMemcpy(cy, c, sizeof(cy), cudaMemcpyDeviceToHost);
        printf("%d lanes: %lld / %lld / %lld cycles per record (variants 0/1/2)\n", lanes, cy[0], cy[1], cy[2]);
    }
    long long cy[3];
    cudaMemcpy(cy, c, sizeof(cy), cudaMemcpyDeviceToHost);
    double2* ho = new double2[3 * n];
    cudaMemcpy(ho, o, 3 * n * 16, cudaMemcpyDeviceToHost);
    for (int v = 0; v < 3; ++v) {
        double md = 0;
        for (int i = 1; i < n; ++i) {
            double dx = ho[v * n + i].x - ho[i].x, dy = ho[v * n + i].y - ho[i].y;
            double m = std::hypot(ho[i].x, ho[i].y);
            md = std::fmax(md, std::hypot(dx, dy) / m);
        }
        printf("variant %d: %lld cycles/record, max rel diff vs variant 0 %.3e\n", v, cy[v], md);
    }
    printf("sample z[100] = %.17g %.17g\n", ho[100].x, ho[100].y);
    return 0;
}
