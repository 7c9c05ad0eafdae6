// metrics.cu -- stitch and K5 (angle distortion, flips, distortion report).
//
// Replaces
//   assemble.py:286-337  stitch_global: average seam copies in submesh order,
//                        spread/scale checks, sphere stereographic finish,
//                        disk circle check, flips (assemble.py:97-102,259-263)
//   metrics.py:22-176    corner angles (planar / spherical tangent plane),
//                        per-corner distortion, per-face area log ratio,
//                        summarize (mean, population sd, linear-interpolated
//                        median and IQR), 0.1-degree histogram of |d|
// Order statistics are exact (radix select on the IEEE bits of |d|), and the
// percentile interpolation is numpy's _lerp, so median/IQR equal numpy's for
// equal inputs; mean/sd are deterministic fixed-order reductions.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "batch.cuh"

namespace pgcp {
namespace {

__device__ __forceinline__ void atomic_max_pos(unsigned long long* p, double v) {
    if (v > 0) atomicMax(p, (unsigned long long)__double_as_longlong(v));
}
__device__ __forceinline__ double2 cdiv_np(double2 a, double2 b) {
    double abr = fabs(b.x), abi = fabs(b.y);
    if (abr >= abi) {
        if (abr == 0.0 && abi == 0.0) return make_double2(a.x / abr, a.y / abi);
        double rat = b.y / b.x;
        double scl = 1.0 / (b.x + b.y * rat);
        return make_double2((a.x + a.y * rat) * scl, (a.y - a.x * rat) * scl);
    }
    double rat = b.x / b.y;
    double scl = 1.0 / (b.y + b.x * rat);
    return make_double2((a.x * rat + a.y) * scl, (a.y * rat - a.x) * scl);
}

// per parent vertex: average of its copies in submesh order
__global__ void k_stitch(int64_t n, const int64_t* __restrict__ lv_off, const int32_t* __restrict__ lv_gid,
                         const double2* __restrict__ z, double2* __restrict__ coords, int32_t* __restrict__ prov,
                         const int32_t* __restrict__ lv_comp, unsigned long long* spread_bits,
                         unsigned long long* scale_bits, int* missing) {
    double tsp = 0, tsc = 0;  // this thread's maxima (reduced per warp: max is order-free)
    GRID_STRIDE(v, n) {
        int64_t lo = lv_off[v], hi = lv_off[v + 1];
        if (lo == hi) {
            atomicExch(missing, 1);
            coords[v] = make_double2(NAN, NAN);
            prov[v] = -1;
            continue;
        }
        double2 first = z[lv_gid[lo]];
        double2 acc = make_double2(0.0, 0.0);
        double sp = 0, sc = 0;
        for (int64_t e = lo; e < hi; ++e) {
            double2 w = z[lv_gid[e]];
            acc.x += w.x;
            acc.y += w.y;
            sp = fmax(sp, hypot(w.x - first.x, w.y - first.y));
            sc = fmax(sc, hypot(w.x, w.y));
        }
        double cnt = (double)(hi - lo);
        coords[v] = cdiv_np(acc, make_double2(cnt, 0.0));
        prov[v] = lv_comp[lo];
        tsp = fmax(tsp, sp);
        tsc = fmax(tsc, sc);
    }
    tsp = warp_max(tsp);
    tsc = warp_max(tsc);
    if ((threadIdx.x & 31) == 0) {
        atomic_max_pos(spread_bits, tsp);
        atomic_max_pos(scale_bits, tsc);
    }
}

// sphere finish: stereographic_inverse(conj(z)) normalised (assemble.py:322-329)
__global__ void k_sphere_finish(int64_t n, const double2* __restrict__ coords, double* __restrict__ P) {
    GRID_STRIDE(v, n) {
        double2 z = coords[v];
        z.y = -z.y;
        double x, y, w;
        if (isinf(z.x) || isinf(z.y)) {
            x = 0; y = 0; w = 1;
        } else if (hypot(z.x, z.y) > 1.0) {
            double2 q = cdiv_np(make_double2(1.0, 0.0), z);
            double h = hypot(q.x, q.y);
            double s = h * h;
            x = 2 * q.x / (1 + s);
            y = -2 * q.y / (1 + s);
            w = (1 - s) / (1 + s);
        } else {
            double h = hypot(z.x, z.y);
            double s = h * h;
            x = 2 * z.x / (1 + s);
            y = 2 * z.y / (1 + s);
            w = (s - 1) / (1 + s);
        }
        double nr = sqrt((x * x + y * y) + w * w);
        P[3 * v] = x / nr;
        P[3 * v + 1] = y / nr;
        P[3 * v + 2] = w / nr;
    }
}

// max | |z| - 1 | over parent boundary vertices (twin-less half-edge origins)
__global__ void k_circle_dev(const int32_t* __restrict__ F, const int32_t* __restrict__ twin, int64_t m,
                             const double2* __restrict__ coords, unsigned long long* dev_bits) {
    GRID_STRIDE(h, 3 * m) {
        if (twin[h] >= 0) continue;
        double2 z = coords[F[h]];
        atomic_max_pos(dev_bits, fabs(hypot(z.x, z.y) - 1.0));
    }
}

__global__ void k_flips(const int32_t* __restrict__ F, int64_t m, const double2* __restrict__ zc,
                        const double* __restrict__ P, int mode_sphere, const uint8_t* __restrict__ fmask,
                        uint8_t* __restrict__ flip, unsigned long long* count) {
    GRID_STRIDE(f, m) {
        if (fmask && !fmask[f]) {  // a face another rank owns (sharded run)
            flip[f] = 0;
            continue;
        }
        int a = F[3 * f], b = F[3 * f + 1], c = F[3 * f + 2];
        bool fl;
        if (mode_sphere) {
            double ax = P[3 * a], ay = P[3 * a + 1], az = P[3 * a + 2];
            double bx = P[3 * b], by = P[3 * b + 1], bz = P[3 * b + 2];
            double cx = P[3 * c], cy = P[3 * c + 1], cz = P[3 * c + 2];
            double x = by * cz - bz * cy, y = bz * cx - bx * cz, z = bx * cy - by * cx;
            fl = (ax * x + ay * y + az * z) < 0;
        } else {
            double2 p0 = zc[a], p1 = zc[b], p2 = zc[c];
            double d1x = p1.x - p0.x, d1y = p1.y - p0.y, d2x = p2.x - p0.x, d2y = p2.y - p0.y;
            fl = 0.5 * (d1x * d2y - d1y * d2x) <= 0;
        }
        flip[f] = fl;
        if (fl) atomicAdd(count, 1ull);
    }
}

// ---------------------------------------------------------------------------
// distortion

__device__ __forceinline__ void corner_angle3(const double* pi, const double* pj, const double* pk, double* ang,
                                              bool* bad) {
    double ux = pj[0] - pi[0], uy = pj[1] - pi[1], uz = pj[2] - pi[2];
    double vx = pk[0] - pi[0], vy = pk[1] - pi[1], vz = pk[2] - pi[2];
    double nu = sqrt((ux * ux + uy * uy) + uz * uz);
    double nv = sqrt((vx * vx + vy * vy) + vz * vz);
    double c = ((ux * vx + uz * vz) + uy * vy) / (nu * nv);
    *ang = acos(fmin(fmax(c, -1.0), 1.0));
    *bad = (nu == 0) || (nv == 0);
}
__device__ __forceinline__ void corner_angle2(double2 pi, double2 pj, double2 pk, double* ang, bool* bad) {
    double ux = pj.x - pi.x, uy = pj.y - pi.y, vx = pk.x - pi.x, vy = pk.y - pi.y;
    double nu = sqrt(ux * ux + uy * uy), nv = sqrt(vx * vx + vy * vy);
    double c = (ux * vx + uy * vy) / (nu * nv);
    *ang = acos(fmin(fmax(c, -1.0), 1.0));
    *bad = (nu == 0) || (nv == 0);
}

__global__ void k_distortion(const double* __restrict__ V, const int32_t* __restrict__ F, int64_t m,
                             const double* __restrict__ coords, int mode_sphere, const uint8_t* __restrict__ fmask,
                             double* __restrict__ d, uint8_t* __restrict__ valid, double* __restrict__ absd,
                             double* __restrict__ a_new, double* __restrict__ a_ref) {
    GRID_STRIDE(f, m) {
        if (fmask && !fmask[f]) {  // counted by the rank that owns the face (sharded run)
            for (int c = 0; c < 3; ++c) {
                d[3 * f + c] = 0.0;
                valid[3 * f + c] = 0;
                absd[3 * f + c] = -1.0;
            }
            a_new[f] = 0.0;
            a_ref[f] = 0.0;
            continue;
        }
        int id[3] = {F[3 * f], F[3 * f + 1], F[3 * f + 2]};
        for (int c = 0; c < 3; ++c) {
            int i = id[c], j = id[(c + 1) % 3], k = id[(c + 2) % 3];
            double ar, an;
            bool br, bn;
            corner_angle3(V + 3 * i, V + 3 * j, V + 3 * k, &ar, &br);
            if (mode_sphere) {
                const double* P = coords;
                double a0 = P[3 * i], a1 = P[3 * i + 1], a2 = P[3 * i + 2];
                double tb[3], tc[3];
                double db = (P[3 * j] * a0 + P[3 * j + 2] * a2) + P[3 * j + 1] * a1;
                double dc = (P[3 * k] * a0 + P[3 * k + 2] * a2) + P[3 * k + 1] * a1;
                for (int q = 0; q < 3; ++q) {
                    tb[q] = P[3 * j + q] - db * P[3 * i + q];
                    tc[q] = P[3 * k + q] - dc * P[3 * i + q];
                }
                double o[3] = {0, 0, 0};
                corner_angle3(o, tb, tc, &an, &bn);
            } else {
                const double2* Z = reinterpret_cast<const double2*>(coords);
                corner_angle2(Z[i], Z[j], Z[k], &an, &bn);
            }
            double dv = (an - ar) * (180.0 / M_PI);
            bool ok = !(br || bn);
            d[3 * f + c] = dv;
            valid[3 * f + c] = ok;
            absd[3 * f + c] = ok ? fabs(dv) : -1.0;  // -1 marks excluded
        }
        // face areas: parametric and original (metrics.py:78-86, mesh.py:128-132)
        {
            const double* p0 = V + 3 * id[0];
            const double* p1 = V + 3 * id[1];
            const double* p2 = V + 3 * id[2];
            double ux = p1[0] - p0[0], uy = p1[1] - p0[1], uz = p1[2] - p0[2];
            double vx = p2[0] - p0[0], vy = p2[1] - p0[1], vz = p2[2] - p0[2];
            double cx = uy * vz - uz * vy, cy = uz * vx - ux * vz, cz = ux * vy - uy * vx;
            a_ref[f] = 0.5 * sqrt((cx * cx + cy * cy) + cz * cz);
            if (mode_sphere) {
                const double* q0 = coords + 3 * id[0];
                const double* q1 = coords + 3 * id[1];
                const double* q2 = coords + 3 * id[2];
                ux = q1[0] - q0[0]; uy = q1[1] - q0[1]; uz = q1[2] - q0[2];
                vx = q2[0] - q0[0]; vy = q2[1] - q0[1]; vz = q2[2] - q0[2];
                cx = uy * vz - uz * vy; cy = uz * vx - ux * vz; cz = ux * vy - uy * vx;
                a_new[f] = 0.5 * sqrt((cx * cx + cy * cy) + cz * cz);
            } else {
                const double2* Z = reinterpret_cast<const double2*>(coords);
                double2 z0 = Z[id[0]], z1 = Z[id[1]], z2 = Z[id[2]];
                double d1x = z1.x - z0.x, d1y = z1.y - z0.y, d2x = z2.x - z0.x, d2y = z2.y - z0.y;
                a_new[f] = 0.5 * fabs(d1x * d2y - d1y * d2x);
            }
        }
    }
}

// corner_angles / corner_angles_sphere (metrics.py:31-58): per corner the
// angle between the two edges leaving it. kind 0: complex planar points,
// 1: real 2D, 2: real 3D, 3: unit-sphere points (edges projected on the
// tangent plane of the corner).
__global__ void k_corner_angles(const double* __restrict__ P, int kind, const int32_t* __restrict__ F, int64_t m,
                                double* __restrict__ ang, uint8_t* __restrict__ bad) {
    GRID_STRIDE(f, m) {
        const int id[3] = {F[3 * f], F[3 * f + 1], F[3 * f + 2]};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int i = id[c], j = id[(c + 1) % 3], k = id[(c + 2) % 3];
            double a;
            bool b;
            if (kind == 0) {
                const double2* Z = reinterpret_cast<const double2*>(P);
                corner_angle2(Z[i], Z[j], Z[k], &a, &b);
            } else if (kind == 1) {
                corner_angle2(make_double2(P[2 * i], P[2 * i + 1]), make_double2(P[2 * j], P[2 * j + 1]),
                              make_double2(P[2 * k], P[2 * k + 1]), &a, &b);
            } else if (kind == 2) {
                corner_angle3(P + 3 * i, P + 3 * j, P + 3 * k, &a, &b);
            } else {
                const double a0 = P[3 * i], a1 = P[3 * i + 1], a2 = P[3 * i + 2];
                const double db = (P[3 * j] * a0 + P[3 * j + 2] * a2) + P[3 * j + 1] * a1;
                const double dc = (P[3 * k] * a0 + P[3 * k + 2] * a2) + P[3 * k + 1] * a1;
                double tb[3], tc[3];
                for (int q = 0; q < 3; ++q) {
                    tb[q] = P[3 * j + q] - db * P[3 * i + q];
                    tc[q] = P[3 * k + q] - dc * P[3 * i + q];
                }
                const double o[3] = {0, 0, 0};
                corner_angle3(o, tb, tc, &a, &b);
            }
            ang[3 * f + c] = a;
            bad[3 * f + c] = b;
        }
    }
}

// deterministic block partial sums: out[block] = sum of f(i) over its range
template <class Fn>
__global__ void k_partial_sum(int64_t n, Fn fn, double* __restrict__ part) {
    __shared__ double red[32];
    double acc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc += fn(i);
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        t = warp_sum(t);
        if (threadIdx.x == 0) part[blockIdx.x] = t;
    }
}

struct AbsVal {
    const double* x;
    __device__ double operator()(int64_t i) const { return x[i] >= 0 ? x[i] : 0.0; }
};
struct Count {
    const double* x;
    __device__ double operator()(int64_t i) const { return x[i] >= 0 ? 1.0 : 0.0; }
};
struct SqDev {
    const double* x;
    double mean;
    __device__ double operator()(int64_t i) const {
        if (x[i] < 0) return 0.0;
        double t = x[i] - mean;
        return t * t;
    }
};
struct Plain {
    const double* x;
    __device__ double operator()(int64_t i) const { return x[i]; }
};

__global__ void k_area_logratio(int64_t m, const double* __restrict__ a_new, const double* __restrict__ a_ref,
                                double sum_new, double sum_ref, double* __restrict__ absd) {
    GRID_STRIDE(f, m) {
        double an = a_new[f];
        absd[f] = an > 0 ? fabs(log((an / sum_new) / (a_ref[f] / sum_ref))) : -1.0;
    }
}

// area_distortion (metrics.py:89-104): signed log of the normalised area
// ratio per face; faces of zero parametric area flagged invalid (d = 0)
__global__ void k_area_log_signed(int64_t m, const double* __restrict__ a_new, const double* __restrict__ a_ref,
                                  double sum_new, double sum_ref, double* __restrict__ d, uint8_t* __restrict__ valid) {
    GRID_STRIDE(f, m) {
        const double an = a_new[f];
        const bool ok = an > 0;
        d[f] = ok ? log((an / sum_new) / (a_ref[f] / sum_ref)) : 0.0;
        valid[f] = ok;
    }
}

// ---- radix select on non-negative doubles (bits are order-preserving)
// RB-bit digits, most significant first (RB = 12: 6 passes, shifts 52, 40,
// 28, 16, 4, then the last 4 bits; RB = 8: 8 passes, used when the
// histograms are summed over ranks, 7 KB each), block-private shared-memory
// histograms with warp-aggregated increments; selections that share their
// prefix share one histogram.
constexpr int RBITS = 12;
constexpr int NSEL = 7;
constexpr int SEL_BLOCKS = 296;

struct SelState {
    unsigned long long prefix;  // selected high bits so far
    long long rank;             // remaining rank within the prefix
};

template <int RB>
struct Digits {
    static constexpr int passes = (64 + RB - 1) / RB;
    __host__ __device__ static int width(int pass) { return 64 - RB * pass < RB ? 64 - RB * pass : RB; }
    __host__ __device__ static int shift(int pass) { return 64 - RB * pass - width(pass); }
};

// representative (first selection with the same prefix) of selection s
__device__ inline int sel_rep(const SelState* st, int s) {
    for (int t = 0; t < s; ++t)
        if (st[t].prefix == st[s].prefix) return t;
    return s;
}

template <int RB>
__global__ void __launch_bounds__(512) k_sel_hist(const double* __restrict__ x, int64_t n, int pass,
                                                  const SelState* __restrict__ st, unsigned int* __restrict__ hist,
                                                  int* __restrict__ rep_out) {
    constexpr int NB = 1 << RB;
    extern __shared__ unsigned int sh[];  // [NSEL][NB]
    __shared__ unsigned long long pre[NSEL];
    __shared__ int rep[NSEL];
    const int shift = Digits<RB>::shift(pass);
    const int width = Digits<RB>::width(pass);
    const int nb = 1 << width;
    if (threadIdx.x < NSEL) {
        pre[threadIdx.x] = st[threadIdx.x].prefix;
        rep[threadIdx.x] = sel_rep(st, threadIdx.x);
        if (blockIdx.x == 0) rep_out[threadIdx.x] = rep[threadIdx.x];
    }
    for (int i = threadIdx.x; i < NSEL * NB; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const int hs = shift + width;  // bits above the current digit
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n_round = (n + 31) & ~(int64_t)31;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_round; i += stride) {
        double v = i < n ? x[i] : -1.0;
        bool ok = v >= 0;
        unsigned long long b = ok ? (unsigned long long)__double_as_longlong(v) : 0ull;
        int digit = (int)((b >> shift) & (unsigned long long)(nb - 1));
        for (int s = 0; s < NSEL; ++s) {
            if (rep[s] != s) continue;
            bool m = ok && (hs >= 64 || (b >> hs) == (pre[s] >> hs));
            unsigned int act = __ballot_sync(0xffffffffu, m);
            if (!act) continue;
            if (m) {
                unsigned int peers = __match_any_sync(act, digit);
                if (lane == __ffs(peers) - 1) atomicAdd(&sh[s * NB + digit], (unsigned int)__popc(peers));
            }
        }
    }
    __syncthreads();
    for (int s = 0; s < NSEL; ++s) {
        if (rep[s] != s) continue;
        for (int i = threadIdx.x; i < nb; i += blockDim.x) {
            unsigned int c = sh[s * NB + i];
            if (c) atomicAdd(&hist[s * NB + i], c);
        }
    }
}

template <int RB>
__global__ void k_sel_pick(int pass, SelState* st, const unsigned int* __restrict__ hist,
                           const int* __restrict__ rep) {
    // one block per selection; chunk sums, then a serial scan by thread 0
    constexpr int NB = 1 << RB;
    __shared__ unsigned long long chunk[256];
    const int s = blockIdx.x;
    const int width = Digits<RB>::width(pass);
    const int nb = 1 << width;
    const unsigned int* h = hist + (int64_t)rep[s] * NB;
    const int per = (nb + 255) / 256;
    unsigned long long t = 0;
    for (int i = 0; i < per; ++i) {
        int j = threadIdx.x * per + i;
        if (j < nb) t += h[j];
    }
    chunk[threadIdx.x] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long r = st[s].rank;
        int c = 0;
        while (c < 255 && r >= (long long)chunk[c]) {
            r -= chunk[c];
            ++c;
        }
        int d = c * per;
        while (d < nb - 1 && r >= (long long)h[d]) {
            r -= h[d];
            ++d;
        }
        st[s].prefix |= ((unsigned long long)d) << Digits<RB>::shift(pass);
        st[s].rank = r;
    }
}

// np.histogram with explicit edges: bin j holds edges[j] <= v < edges[j+1],
// the last bin also v == edges[nb]. Edges and counts in shared memory
// (nb <= HIST_SMEM_BINS), warp-aggregated increments, one global add per
// non-empty bin per block.
constexpr int HIST_SMEM_BINS = 3072;

__device__ inline int hist_bin(const double* e, int nb, double v) {
    if (!(v >= e[0]) || v > e[nb]) return -1;
    int lo = 0, hi = nb;  // largest j with e[j] <= v
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (e[mid] <= v) lo = mid; else hi = mid - 1;
    }
    return lo >= nb ? nb - 1 : lo;
}

__global__ void __launch_bounds__(512) k_hist_bins_smem(const double* __restrict__ x, int64_t n,
                                                        const double* __restrict__ edges, int nb,
                                                        unsigned long long* __restrict__ counts) {
    __shared__ double se[HIST_SMEM_BINS + 1];
    __shared__ unsigned int sc[HIST_SMEM_BINS];
    for (int i = threadIdx.x; i <= nb; i += blockDim.x) se[i] = edges[i];
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sc[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n_round = (n + 31) & ~(int64_t)31;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_round; i += stride) {
        double v = i < n ? x[i] : -1.0;
        int bin = v >= 0 ? hist_bin(se, nb, v) : -1;
        unsigned int act = __ballot_sync(0xffffffffu, bin >= 0);
        if (bin >= 0) {
            unsigned int peers = __match_any_sync(act, bin);
            if (lane == __ffs(peers) - 1) atomicAdd(&sc[bin], (unsigned int)__popc(peers));
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nb; i += blockDim.x)
        if (sc[i]) atomicAdd(&counts[i], (unsigned long long)sc[i]);
}

__global__ void k_hist_bins(const double* __restrict__ x, int64_t n, const double* __restrict__ edges, int nb,
                            unsigned long long* __restrict__ counts) {
    GRID_STRIDE(i, n) {
        double v = x[i];
        if (v < 0) continue;
        int bin = hist_bin(edges, nb, v);
        if (bin >= 0) atomicAdd(&counts[bin], 1ull);
    }
}

// host sum of nsums consecutive groups of nblocks block partials (fixed
// order), read through the pinned staging buffer with one synchronisation
int sum_of(const double* part, int nblocks, double* out, cudaStream_t s, int nsums = 1) {
    std::vector<double> h((size_t)nblocks * nsums);
    PGCP_TRY(d2h_async(h.data(), part, h.size() * sizeof(double), s));
    PGCP_TRY(d2h_flush(s));
    for (int q = 0; q < nsums; ++q) {
        double t = 0;
        for (int i = 0; i < nblocks; ++i) t += h[(size_t)q * nblocks + i];
        out[q] = t;
    }
    return PGCP_OK;
}

constexpr int SUM_BLOCKS = 296;

template <class Fn>
int dsum(int64_t n, Fn fn, DevBuf<double>& part, double* out, cudaStream_t s) {
    k_partial_sum<Fn><<<SUM_BLOCKS, 256, 0, s>>>(n, fn, part.p);
    PGCP_LAUNCH_CHECK();
    return sum_of(part.p, SUM_BLOCKS, out, s);
}
// two independent sums, one synchronisation (part holds 2 x SUM_BLOCKS)
template <class Fa, class Fb>
int dsum2(int64_t na, Fa fa, int64_t nb, Fb fb, DevBuf<double>& part, double* out2, cudaStream_t s) {
    k_partial_sum<Fa><<<SUM_BLOCKS, 256, 0, s>>>(na, fa, part.p);
    PGCP_LAUNCH_CHECK();
    k_partial_sum<Fb><<<SUM_BLOCKS, 256, 0, s>>>(nb, fb, part.p + SUM_BLOCKS);
    PGCP_LAUNCH_CHECK();
    return sum_of(part.p, SUM_BLOCKS, out2, s, 2);
}

double lerp_np(double a, double b, double t) {
    double diff = b - a;
    if (t >= 0.5) return b - diff * (1.0 - t);
    return a + diff * t;
}

// sharded runs: faces / parent vertices belonging to this rank's submeshes
__global__ void k_shard_face_mask(int64_t m, const int32_t* __restrict__ face_comp, const uint8_t* __restrict__ own,
                                  uint8_t* __restrict__ mask) {
    GRID_STRIDE(f, m) mask[f] = own[face_comp[f]];
}
__global__ void k_shard_vert_flag(int64_t n, const int64_t* __restrict__ lv_off, const int32_t* __restrict__ lv_comp,
                                  const uint8_t* __restrict__ own, int32_t* __restrict__ flag) {
    GRID_STRIDE(v, n) {
        int f = 0;
        for (int64_t e = lv_off[v]; e < lv_off[v + 1]; ++e) f |= own[lv_comp[e]];
        flag[v] = f;
    }
}
__global__ void k_shard_compact(int64_t n, const int32_t* __restrict__ flag, const int64_t* __restrict__ pos,
                                int32_t* __restrict__ out) {
    GRID_STRIDE(v, n) if (flag[v]) out[pos[v]] = (int32_t)v;
}

// Sums / maxima over the ranks of a sharded run (pgcp_reduce_fn supplied
// by the caller, e.g. an NCCL all-reduce); a no-op for a single GPU.
struct Reducer {
    pgcp_reduce_fn fn = nullptr;
    void* user = nullptr;
    cudaStream_t s = nullptr;
    DevBuf<double> buf;
    int64_t bytes = 0;  // payload handed to the hook

    int dev(void* p, int64_t n, int dtype, int op) {
        if (!fn || n == 0) return PGCP_OK;
        bytes += n * (dtype == PGCP_RED_U32 ? 4 : 8);
        if (fn(p, n, dtype, op, user, s) != 0) {
            set_error("distributed reduction (pgcp_reduce_fn) failed");
            return PGCP_E_CUDA;
        }
        return PGCP_OK;
    }
    // in place over host doubles (staged through a small device buffer)
    int host(double* v, int n, int op) {
        if (!fn) return PGCP_OK;
        if (buf.n < n) PGCP_TRY(buf.alloc(std::max(n, 8), s));
        PGCP_TRY_CUDA(cudaMemcpyAsync(buf.p, v, n * sizeof(double), cudaMemcpyHostToDevice, s));
        PGCP_TRY(dev(buf.p, n, PGCP_RED_F64, op));
        PGCP_TRY_CUDA(cudaMemcpyAsync(v, buf.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        PGCP_TRY_CUDA(cudaStreamSynchronize(s));
        return PGCP_OK;
    }
};

// exact order statistics: NSEL selections of given ranks among the entries
// of x that are >= 0 (histograms summed over ranks between the passes)
template <int RB>
int select_ranks(const double* x, int64_t n, SelState* hs, Reducer& red, cudaStream_t s) {
    constexpr int NB = 1 << RB;
    DevBuf<SelState> st;
    DevBuf<unsigned int> hist;
    DevBuf<int> rep;
    PGCP_TRY(rep.alloc(NSEL, s));
    PGCP_TRY(st.alloc(NSEL, s));
    PGCP_TRY(hist.alloc(NSEL * (int64_t)NB, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(st.p, hs, NSEL * sizeof(SelState), cudaMemcpyHostToDevice, s));
    const size_t smem = NSEL * NB * sizeof(unsigned int);
    static bool attr = false;
    if (!attr) {
        PGCP_TRY_CUDA(cudaFuncSetAttribute(k_sel_hist<RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
    }
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(SEL_BLOCKS, (n + 511) / 512));
    for (int pass = 0; pass < Digits<RB>::passes; ++pass) {
        PGCP_TRY(hist.zero(s));
        k_sel_hist<RB><<<blocks, 512, smem, s>>>(x, n, pass, st.p, hist.p, rep.p);
        PGCP_LAUNCH_CHECK();
        PGCP_TRY(red.dev(hist.p, NSEL * (int64_t)NB, PGCP_RED_U32, PGCP_RED_SUM));
        k_sel_pick<RB><<<NSEL, 256, 0, s>>>(pass, st.p, hist.p, rep.p);
        PGCP_LAUNCH_CHECK();
    }
    PGCP_TRY(d2h_async(hs, st.p, NSEL * sizeof(SelState), s));  // pinned staging (common.cuh)
    PGCP_TRY(d2h_flush(s));
    return PGCP_OK;
}

// mean, population sd, median, IQR of the entries of x that are >= 0
// (over every rank's entries when red carries a hook)
int summarize_dev(const double* x, int64_t n, double* out4, int64_t* count, DevBuf<double>& part, cudaStream_t s,
                  Reducer& red, double* vmax = nullptr) {
    double cs[2] = {0, 0};  // count, sum
    PGCP_TRY(dsum2(n, Count{x}, n, AbsVal{x}, part, cs, s));
    PGCP_TRY(red.host(cs, 2, PGCP_RED_SUM));
    const double cnt = cs[0], sum = cs[1];
    *count = (int64_t)cnt;
    if (cnt == 0) {
        out4[0] = out4[1] = out4[2] = out4[3] = NAN;
        if (vmax) *vmax = 0.0;
        return PGCP_OK;
    }
    double mean = sum / cnt;
    double sq = 0;
    PGCP_TRY(dsum(n, SqDev{x, mean}, part, &sq, s));
    PGCP_TRY(red.host(&sq, 1, PGCP_RED_SUM));
    out4[0] = mean;
    out4[1] = sqrt(sq / cnt);
    // order statistics for q = 25, 50, 75 (numpy 'linear')
    const int64_t N = (int64_t)cnt;
    const double qs[3] = {0.25, 0.5, 0.75};
    int64_t ranks[7];
    double gam[3];
    ranks[6] = N - 1;  // maximum
    for (int q = 0; q < 3; ++q) {
        double vi = (double)(N - 1) * qs[q];
        double pv = floor(vi);
        gam[q] = vi - pv;
        ranks[2 * q] = (int64_t)pv;
        ranks[2 * q + 1] = std::min<int64_t>((int64_t)pv + 1, N - 1);
    }
    SelState hs[NSEL];
    for (int q = 0; q < NSEL; ++q) hs[q] = {0ull, (long long)ranks[q]};
    if (red.fn)
        PGCP_TRY(select_ranks<8>(x, n, hs, red, s));
    else
        PGCP_TRY(select_ranks<RBITS>(x, n, hs, red, s));
    double v[NSEL];
    for (int q = 0; q < NSEL; ++q) memcpy(&v[q], &hs[q].prefix, sizeof(double));
    if (vmax) *vmax = v[6];
    double q25 = lerp_np(v[0], v[1], gam[0]);
    double q50 = lerp_np(v[2], v[3], gam[1]);
    double q75 = lerp_np(v[4], v[5], gam[2]);
    out4[2] = q50;
    out4[3] = q75 - q25;
    return PGCP_OK;
}

}  // namespace
}  // namespace pgcp

using namespace pgcp;

extern "C" {

// stitch_global (assemble.py:286-337) over a batch's per-submesh embeddings.
//   z        device complex [sum_n]
//   mode     0 free, 1 disk, 2 sphere
//   coords   device complex [n] (averaged plane coordinates)
//   sphere   device f64 [3n] (sphere mode; may be NULL otherwise)
//   prov     device int32 [n]; flip device uint8 [m]
//   stats    host f64 [8]: seam_max, scale, circle_dev, nflip, status
PGCP_API int pgcp_batch_stitch(pgcp_batch* b, const double* z, int mode, double hard_tol, double circle_tol,
                               double* coords, double* sphere, int32_t* prov, uint8_t* flip, double* stats,
                               void* stream) {
    return pgcp_batch_stitch_ex(b, z, mode, hard_tol, circle_tol, nullptr, coords, sphere, prov, flip, stats, stream);
}

PGCP_API int pgcp_batch_stitch_ex(pgcp_batch* b, const double* z, int mode, double hard_tol, double circle_tol,
                                  const uint8_t* face_mask, double* coords, double* sphere, int32_t* prov,
                                  uint8_t* flip, double* stats, void* stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (!b || !z || !coords || !prov || !flip || !stats || (mode == 2 && !sphere)) {
        set_error("pgcp_batch_stitch: invalid arguments");
        return PGCP_E_INVALID;
    }
    PGCP_TRY_CUDA(cudaSetDevice(b->device));
    DevBuf<unsigned long long> bits;
    DevBuf<int> missing;
    PGCP_TRY(bits.alloc(4, s));
    PGCP_TRY(bits.zero(s));
    PGCP_TRY(missing.alloc(1, s));
    PGCP_TRY(missing.zero(s));
    k_stitch<<<grid_for(b->n, 256), 256, 0, s>>>(b->n, b->lv_off.p, b->lv_gid.p, reinterpret_cast<const double2*>(z),
                                                 reinterpret_cast<double2*>(coords), prov, b->lv_comp.p, bits.p,
                                                 bits.p + 1, missing.p);
    PGCP_LAUNCH_CHECK();
    if (mode == 2) {
        k_sphere_finish<<<grid_for(b->n, 256), 256, 0, s>>>(b->n, reinterpret_cast<const double2*>(coords), sphere);
        PGCP_LAUNCH_CHECK();
    }
    if (mode == 1) {
        k_circle_dev<<<grid_for(3 * b->m, 256), 256, 0, s>>>(b->F.p, b->twin.p, b->m,
                                                             reinterpret_cast<const double2*>(coords), bits.p + 2);
        PGCP_LAUNCH_CHECK();
    }
    k_flips<<<grid_for(b->m, 256), 256, 0, s>>>(b->F.p, b->m, reinterpret_cast<const double2*>(coords), sphere,
                                               mode == 2, face_mask, flip, bits.p + 3);
    PGCP_LAUNCH_CHECK();
    unsigned long long h[4];
    int hm = 0;
    PGCP_TRY(d2h_async(h, bits.p, sizeof h, s));
    PGCP_TRY(d2h_async(&hm, missing.p, sizeof hm, s));
    PGCP_TRY(d2h_flush(s));
    double seam, scale, circ;
    memcpy(&seam, &h[0], 8);
    memcpy(&scale, &h[1], 8);
    memcpy(&circ, &h[2], 8);
    stats[0] = seam;
    stats[1] = scale;
    stats[2] = circ;
    stats[3] = (double)h[3];
    stats[4] = 0;
    if (hm) {
        set_error("some parent vertices received no coordinates");
        stats[4] = PGCP_E_SOLVE;
        return PGCP_E_SOLVE;
    }
    if (scale > 0 && seam > hard_tol * scale) {
        set_error("seam disagreement %.3e exceeds %g x scale %.3e (welding bug upstream)", seam, hard_tol, scale);
        stats[4] = PGCP_E_SOLVE;
        return PGCP_E_SOLVE;
    }
    if (mode == 1 && circ > circle_tol) {
        set_error("disk boundary off the unit circle by %.3e", circ);
        stats[4] = PGCP_E_SOLVE;
        return PGCP_E_SOLVE;
    }
    return PGCP_OK;
}

// Maps of one rank's share of a batch (dist.py): face_mask[f] = 1 for the
// faces of the listed submeshes; own_vertices = the parent vertices with a
// copy in one of them, ascending (count in *n_own). Synchronises.
PGCP_API int pgcp_batch_shard_maps(pgcp_batch* b, const int32_t* comps, int32_t ncomp, uint8_t* face_mask,
                                   int32_t* own_vertices, int64_t* n_own, void* stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (!b || (ncomp > 0 && !comps) || !face_mask || !own_vertices || !n_own) {
        set_error("pgcp_batch_shard_maps: invalid arguments");
        return PGCP_E_INVALID;
    }
    PGCP_TRY_CUDA(cudaSetDevice(b->device));
    std::vector<uint8_t> h(std::max<int64_t>(b->K, 1), 0);
    for (int i = 0; i < ncomp; ++i) {
        if (comps[i] < 0 || comps[i] >= b->K) {
            set_error("pgcp_batch_shard_maps: submesh %d out of range", comps[i]);
            return PGCP_E_INVALID;
        }
        h[comps[i]] = 1;
    }
    DevBuf<uint8_t> own;
    DevBuf<int32_t> flag;
    DevBuf<int64_t> pos;
    PGCP_TRY(own.alloc((int64_t)h.size(), s));
    PGCP_TRY(flag.alloc(b->n, s));
    PGCP_TRY(pos.alloc(b->n + 1, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(own.p, h.data(), h.size(), cudaMemcpyHostToDevice, s));
    k_shard_face_mask<<<grid_for(b->m, 256), 256, 0, s>>>(b->m, b->face_comp.p, own.p, face_mask);
    PGCP_LAUNCH_CHECK();
    k_shard_vert_flag<<<grid_for(b->n, 256), 256, 0, s>>>(b->n, b->lv_off.p, b->lv_comp.p, own.p, flag.p);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY(exclusive_scan_i32_to_i64(flag.p, pos.p, b->n, s));
    k_shard_compact<<<grid_for(b->n, 256), 256, 0, s>>>(b->n, flag.p, pos.p, own_vertices);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY(fetch_scalar(pos.p + b->n, n_own, s));
    return PGCP_OK;
}

PGCP_API int pgcp_corner_angles(const double* points, int kind, const int32_t* F, int64_t m, double* ang,
                                uint8_t* bad, void* stream) {
    if (m < 0 || kind < 0 || kind > 3 || (m > 0 && (!points || !F || !ang || !bad))) {
        set_error("pgcp_corner_angles: invalid arguments");
        return PGCP_E_INVALID;
    }
    if (m == 0) return PGCP_OK;
    k_corner_angles<<<grid_for(m, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(points, kind, F, m, ang,
                                                                                          bad);
    PGCP_LAUNCH_CHECK();
    return PGCP_OK;
}

PGCP_API int pgcp_area_distortion(const double* V, const int32_t* F, int64_t n, int64_t m, const double* coords,
                                  int mode_sphere, double* d, uint8_t* valid, void* stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (!V || !F || !coords || !d || !valid || m <= 0) {
        set_error("pgcp_area_distortion: invalid arguments");
        return PGCP_E_INVALID;
    }
    DevBuf<double> dc, absd, a_new, a_ref, part;
    DevBuf<uint8_t> vc;
    PGCP_TRY(dc.alloc(3 * m, s));
    PGCP_TRY(vc.alloc(3 * m, s));
    PGCP_TRY(absd.alloc(3 * m, s));
    PGCP_TRY(a_new.alloc(m, s));
    PGCP_TRY(a_ref.alloc(m, s));
    PGCP_TRY(part.alloc(2 * SUM_BLOCKS, s));
    k_distortion<<<grid_for(m, 256), 256, 0, s>>>(V, F, m, coords, mode_sphere, nullptr, dc.p, vc.p, absd.p, a_new.p,
                                                  a_ref.p);
    PGCP_LAUNCH_CHECK();
    double sn = 0, sr = 0;
    PGCP_TRY(dsum(m, Plain{a_new.p}, part, &sn, s));
    PGCP_TRY(dsum(m, Plain{a_ref.p}, part, &sr, s));
    k_area_log_signed<<<grid_for(m, 256), 256, 0, s>>>(m, a_new.p, a_ref.p, sn, sr, d, valid);
    PGCP_LAUNCH_CHECK();
    return PGCP_OK;
}

// distortion_report (metrics.py:165-176) of a parameterization.
//   coords  device: complex [n] (planar) or f64 [3n] (mode_sphere = 1)
//   d       device f64 [3m] per-corner distortion (degrees); valid uint8 [3m]
//   summary host f64 [16]: angular mean, sd, median, iqr, area mean, sd,
//           median, iqr, excluded corners, excluded faces, max |d|, nbins,
//           valid corners, valid faces
//   hist    host uint64 [hist_cap] 0.1-degree counts (hist_cap 0: skip)
PGCP_API int pgcp_distortion(const double* V, const int32_t* F, int64_t n, int64_t m, const double* coords,
                             int mode_sphere, double* d, uint8_t* valid, double* summary, uint64_t* hist,
                             int64_t hist_cap, void* stream) {
    return pgcp_distortion_ex(V, F, n, m, coords, mode_sphere, nullptr, nullptr, nullptr, d, valid, summary, hist,
                              hist_cap, stream);
}

// Sharded form: only the faces with face_mask[f] != 0 are this rank's; every
// global quantity (sums, the radix-select histograms, the 0.1-degree counts)
// goes through `reduce` (sum / max over ranks), so every rank returns the
// summary of the whole mesh. summary[14] = bytes handed to `reduce`.
PGCP_API int pgcp_distortion_ex(const double* V, const int32_t* F, int64_t n, int64_t m, const double* coords,
                                int mode_sphere, const uint8_t* face_mask, pgcp_reduce_fn reduce, void* user,
                                double* d, uint8_t* valid, double* summary, uint64_t* hist, int64_t hist_cap,
                                void* stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (!V || !F || !coords || !d || !valid || !summary || m <= 0) {
        set_error("pgcp_distortion: invalid arguments");
        return PGCP_E_INVALID;
    }
    Reducer red;
    red.fn = reduce;
    red.user = user;
    red.s = s;
    DevBuf<double> absd, a_new, a_ref, aabs, part;
    PGCP_TRY(absd.alloc(3 * m, s));
    PGCP_TRY(a_new.alloc(m, s));
    PGCP_TRY(a_ref.alloc(m, s));
    PGCP_TRY(aabs.alloc(m, s));
    PGCP_TRY(part.alloc(2 * SUM_BLOCKS, s));
    k_distortion<<<grid_for(m, 256), 256, 0, s>>>(V, F, m, coords, mode_sphere, face_mask, d, valid, absd.p, a_new.p,
                                                  a_ref.p);
    PGCP_LAUNCH_CHECK();
    double ang[4], ar[4];
    int64_t nc = 0, nf = 0;
    double mval = 0;
    PGCP_TRY(summarize_dev(absd.p, 3 * m, ang, &nc, part, s, red, &mval));
    double sa[2] = {0, 0};  // total parametric and original area
    PGCP_TRY(dsum2(m, Plain{a_new.p}, m, Plain{a_ref.p}, part, sa, s));
    PGCP_TRY(red.host(sa, 2, PGCP_RED_SUM));
    k_area_logratio<<<grid_for(m, 256), 256, 0, s>>>(m, a_new.p, a_ref.p, sa[0], sa[1], aabs.p);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY(summarize_dev(aabs.p, m, ar, &nf, part, s, red));
    for (int i = 0; i < 4; ++i) {
        summary[i] = ang[i];
        summary[4 + i] = ar[i];
    }
    summary[8] = (double)(3 * m - nc);
    summary[9] = (double)(m - nf);
    summary[12] = (double)nc;
    summary[13] = (double)nf;
    // histogram of |d| in 0.1-degree bins (metrics.py:140-149)
    double top = std::max(0.1, nc > 0 ? mval : 0.0);
    summary[10] = nc > 0 ? mval : 0.0;
    // np.arange(0.0, top + 0.1, 0.1): len = ceil((stop - start) / step), e_i = i * delta
    double stop = top + 0.1;
    int64_t len = (int64_t)std::ceil((stop - 0.0) / 0.1);
    int64_t nb = len - 1;
    summary[11] = (double)nb;
    if (hist && hist_cap >= nb && nb > 0 && nc > 0) {
        std::vector<double> edges(len);
        double delta = (0.0 + 0.1) - 0.0;
        edges[0] = 0.0;
        if (len > 1) edges[1] = 0.0 + 0.1;
        for (int64_t i = 2; i < len; ++i) edges[i] = 0.0 + (double)i * delta;
        DevBuf<double> de;
        DevBuf<unsigned long long> cnt;
        PGCP_TRY(de.alloc(len, s));
        PGCP_TRY(cnt.alloc(nb, s));
        PGCP_TRY(cnt.zero(s));
        PGCP_TRY_CUDA(cudaMemcpyAsync(de.p, edges.data(), len * sizeof(double), cudaMemcpyHostToDevice, s));
        if (nb <= HIST_SMEM_BINS)
            k_hist_bins_smem<<<(int)std::min<int64_t>(SEL_BLOCKS, (3 * m + 511) / 512), 512, 0, s>>>(
                absd.p, 3 * m, de.p, (int)nb, cnt.p);
        else
            k_hist_bins<<<grid_for(3 * m, 256), 256, 0, s>>>(absd.p, 3 * m, de.p, (int)nb, cnt.p);
        PGCP_LAUNCH_CHECK();
        PGCP_TRY(red.dev(cnt.p, nb, PGCP_RED_U64, PGCP_RED_SUM));
        PGCP_TRY(d2h_async(hist, cnt.p, nb * sizeof(uint64_t), s));
        PGCP_TRY(d2h_flush(s));
    }
    summary[14] = (double)red.bytes;
    return PGCP_OK;
}

}  // extern "C"
