// direct.cu -- K3d: batched multifrontal Cholesky of the per-subdomain
// systems (the DNCP flatten H = L_UU + 2i M_xy, complex Hermitian, and the
// Dirichlet system L_II, real symmetric), all subdomains of a solve at once.
//
// Replaces the two `spsolve` calls of the hot path (flatten.py:167,
// assemble.py:42) with what SuperLU does on the CPU -- a sparse direct
// factorization -- laid out for the GPU:
//
//   ordering   geometric nested dissection of every subdomain, level by level
//              over all subdomains: a region is split at the midpoint of the
//              longest axis of its bounding box; its separator is the set of
//              near-side vertices with an edge to the far side. Per-vertex
//              kernels with warp-aggregated atomics, one host sync per level.
//   symbolic   update sets U(N) = (adj(pivots) u U(children)) beyond N's
//              pivots, one CTA per front (shared-memory sort + unique),
//              level by level from the leaves.
//   numeric    one CTA per front, level by level from the leaves: assemble
//              the matrix entries of the pivots, extend-add the children's
//              update blocks, blocked partial Cholesky of the pivot columns
//              (warp-factored 16x16 diagonal blocks, per-row TRSM, 64x64
//              tiled updates staged in shared memory), then one tiled
//              Schur update of the U block that the parent reads in place.
//   solve      forward (leaves -> roots) and backward (roots -> leaves)
//              substitution, one CTA per front, deterministic extend-add of
//              the children's partial sums.
//
// Everything is fixed-order (no floating-point atomics): results are bitwise
// reproducible. The system is the Jacobi-scaled one pcg.cu builds (unit
// diagonal), so the PCG path's post-processing (true residual, scatter,
// flatten checks) applies unchanged.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <memory>
#include <mutex>
#include <cstdlib>
#include <vector>

#include "direct.cuh"

namespace pgcp {

namespace {

constexpr int DNT = 128;        // threads per CTA of the per-front kernels (4 CTAs per SM)
constexpr int NB = 16;          // diagonal block of the partial factorization
constexpr int TR = 32;          // update tiles: TR rows x TC columns, 4x4 outputs per thread
constexpr int TC = 64;
constexpr int KC = 16;          // k-chunk staged per update tile
constexpr int CAND_MAX = 8192;  // symbolic: candidates per front (shared memory)
constexpr unsigned FULL = 0xffffffffu;

// ---------------------------------------------------------------------------
// scalar helpers: T = double (real symmetric) or double2 (complex Hermitian)

__device__ __forceinline__ double re(double a) { return a; }
__device__ __forceinline__ double re(double2 a) { return a.x; }
template <class T> __device__ __forceinline__ T zero_t();
template <> __device__ __forceinline__ double zero_t<double>() { return 0.0; }
template <> __device__ __forceinline__ double2 zero_t<double2>() { return make_double2(0.0, 0.0); }
template <class T> __device__ __forceinline__ T from_c(double2 v);
template <> __device__ __forceinline__ double from_c<double>(double2 v) { return v.x; }
template <> __device__ __forceinline__ double2 from_c<double2>(double2 v) { return v; }
__device__ __forceinline__ double cj(double a) { return a; }
__device__ __forceinline__ double2 cj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double scale(double a, double s) { return a * s; }
__device__ __forceinline__ double2 scale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double add(double a, double b) { return a + b; }
__device__ __forceinline__ double2 add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double sub(double a, double b) { return a - b; }
__device__ __forceinline__ double2 sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// acc += a * conj(b)
__device__ __forceinline__ void fma_cj(double& acc, double a, double b) { acc = fma(a, b, acc); }
__device__ __forceinline__ void fma_cj(double2& acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, fma(a.y, b.y, acc.x));
    acc.y = fma(a.y, b.x, fma(-a.x, b.y, acc.y));
}
// complex vector entry times a matrix entry: v * a, and v * conj(a)
__device__ __forceinline__ double2 vmul(double a, double2 v) { return make_double2(a * v.x, a * v.y); }
__device__ __forceinline__ double2 vmul(double2 a, double2 v) {
    return make_double2(a.x * v.x - a.y * v.y, a.x * v.y + a.y * v.x);
}
__device__ __forceinline__ double2 vmul_cj(double a, double2 v) { return make_double2(a * v.x, a * v.y); }
__device__ __forceinline__ double2 vmul_cj(double2 a, double2 v) {
    return make_double2(a.x * v.x + a.y * v.y, a.x * v.y - a.y * v.x);
}

__device__ __forceinline__ int dbsearch(const int64_t* __restrict__ off, int n, int64_t e) {
    int lo = 0, hi = n - 1;  // largest j with off[j] <= e
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (off[mid] <= e) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ int lower_bound_i32(const int32_t* a, int n, int32_t x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint32_t ford(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float funord(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// warp-aggregated atomics keyed by a node id: every lane of the warp must
// call (active or not)
__device__ __forceinline__ void agg_min_max(uint32_t* bb, int key, bool active, uint32_t v, int which) {
    unsigned act = __ballot_sync(FULL, active);
    const int lane = threadIdx.x & 31;
    while (act) {
        const int leader = __ffs(act) - 1;
        const int k = __shfl_sync(FULL, key, leader);
        const bool mine = active && key == k;
        const unsigned m = __ballot_sync(FULL, mine);
        if (mine) {
            const uint32_t lo = __reduce_min_sync(m, v), hi = __reduce_max_sync(m, v);
            if (lane == leader) {
                atomicMin(bb + 6 * (int64_t)k + which, lo);
                atomicMax(bb + 6 * (int64_t)k + 3 + which, hi);
            }
        }
        act &= ~m;
    }
}
__device__ __forceinline__ void agg_count(int32_t* cnt, int key, bool active, int g) {
    unsigned act = __ballot_sync(FULL, active);
    const int lane = threadIdx.x & 31;
    while (act) {
        const int leader = __ffs(act) - 1;
        const int k = __shfl_sync(FULL, key, leader);
        const int gg = __shfl_sync(FULL, g, leader);
        const bool mine = active && key == k && g == gg;
        const unsigned m = __ballot_sync(FULL, mine);
        if (lane == leader) atomicAdd(cnt + 3 * (int64_t)k + gg, __popc(m));
        act &= ~m;
    }
}

// ---------------------------------------------------------------------------
// unknowns, coordinates, adjacency

__global__ void k_d_urow(int64_t NU, int32_t nslot, const int64_t* __restrict__ uoff,
                         const int64_t* __restrict__ sl_off, int32_t* __restrict__ urow,
                         int32_t* __restrict__ uslot) {
    GRID_STRIDE(u, NU) {
        const int j = dbsearch(uoff, nslot + 1, u);
        urow[u] = (int32_t)(32 * sl_off[j] + (u - uoff[j]));
        uslot[u] = j;
    }
}

__global__ void k_d_pos(int64_t NU, const int32_t* __restrict__ urow, const int32_t* __restrict__ uslot,
                        const int32_t* __restrict__ rowsrc, const int64_t* __restrict__ sv_off,
                        const int32_t* __restrict__ comps, const int64_t* __restrict__ vert_off,
                        const int32_t* __restrict__ vmap, const double* __restrict__ V, float4* __restrict__ pos) {
    GRID_STRIDE(u, NU) {
        const int j = uslot[u];
        const int e = rowsrc[urow[u]];
        const int64_t gid = vert_off[comps[j]] + (e - sv_off[j]);
        const int64_t pv = vmap[gid];
        pos[u] = make_float4((float)V[3 * pv], (float)V[3 * pv + 1], (float)V[3 * pv + 2], 0.f);
    }
}

struct AdjArgs {
    const int32_t* urow;
    const int32_t* uslot;
    const int64_t* uoff;
    const int64_t* sl_off;
    const int64_t* sl_ptr;
    const int32_t* col;
    const double* val;
    const uint32_t* sl_mask;
    const int2* cpl;
    const double2* cplc;
};

__device__ __forceinline__ int64_t sp_pos(int64_t e0, int k, int lane) {
    return e0 + ((int64_t)(k >> 1) << 6) + (lane << 1) + (k & 1);
}

// row u's off-diagonal entries: the ELL entries (column != own row) and the
// coupling partners not already among them; fill=false only counts
template <bool FILL>
__device__ __forceinline__ int adj_row(const AdjArgs& a, int64_t u, int32_t* oc, double2* ov) {
    const int r = a.urow[u];
    const int j = a.uslot[u];
    const int64_t rbase = 32 * a.sl_off[j];
    const int self = (int)(r - rbase);
    const int64_t s = r >> 5;
    const int lane = r & 31;
    const int64_t e0 = a.sl_ptr[s];
    const int w = (int)((a.sl_ptr[s + 1] - e0) >> 5);
    int2 cp = make_int2(-1, -1);
    double2 cc = make_double2(0.0, 0.0);
    const bool has_c = a.sl_mask && ((a.sl_mask[s] >> lane) & 1u);
    if (has_c) {
        cp = a.cpl[r];
        cc = a.cplc[r];
    }
    bool seen_n = false, seen_p = false;
    int k = 0;
    for (int q = 0; q < w; ++q) {
        const int64_t e = sp_pos(e0, q, lane);
        const int c = a.col[e];
        if (c == self) continue;
        if (FILL) {
            double im = 0.0;
            if (c == cp.x) im += cc.x;
            if (c == cp.y) im -= cc.y;
            oc[k] = (int32_t)(a.uoff[j] + c);
            ov[k] = make_double2(a.val[e], im);
        }
        seen_n |= c == cp.x;
        seen_p |= c == cp.y;
        ++k;
    }
    if (cp.x >= 0 && !seen_n) {
        if (FILL) {
            oc[k] = (int32_t)(a.uoff[j] + cp.x);
            ov[k] = make_double2(0.0, cp.x == cp.y ? cc.x - cc.y : cc.x);
        }
        ++k;
    }
    if (cp.y >= 0 && !seen_p && cp.y != cp.x) {
        if (FILL) {
            oc[k] = (int32_t)(a.uoff[j] + cp.y);
            ov[k] = make_double2(0.0, -cc.y);
        }
        ++k;
    }
    return k;
}

__global__ void k_d_adj_count(int64_t NU, AdjArgs a, int64_t* __restrict__ cnt) {
    GRID_STRIDE(u, NU) cnt[u] = adj_row<false>(a, u, nullptr, nullptr);
}
__global__ void k_d_adj_fill(int64_t NU, AdjArgs a, const int64_t* __restrict__ ptr, int32_t* __restrict__ oc,
                             double2* __restrict__ ov) {
    GRID_STRIDE(u, NU) adj_row<true>(a, u, oc + ptr[u], ov + ptr[u]);
}

// ---------------------------------------------------------------------------
// nested dissection

struct NodeArrays {
    int32_t* parent;
    int32_t* chA;
    int32_t* chB;
    int32_t* cnt;     // unknowns in the region when it was created
    int32_t* npiv;    // pivots (separator, or all of a leaf)
    int32_t* slot;
    int8_t* leaf;
    uint32_t* bbox;   // [6] ordered floats, min xyz then max xyz
    int32_t* gcnt;    // [3] near side / far side / separator
    float2* split;    // (axis, mid)
    int32_t* nchild;
};

__global__ void k_nd_roots(int32_t nslot, const int64_t* __restrict__ uoff, int leafmax, NodeArrays nd) {
    GRID_STRIDE(j, nslot) {
        const int32_t c = (int32_t)(uoff[j + 1] - uoff[j]);
        nd.parent[j] = -1;
        nd.chA[j] = nd.chB[j] = -1;
        nd.cnt[j] = c;
        nd.slot[j] = (int32_t)j;
        nd.leaf[j] = c <= leafmax;
        nd.npiv[j] = c <= leafmax ? c : 0;
    }
}

// Boundary-last ordering of the DNCP system: every slot's loop unknowns form
// its root front (eliminated last, complex), the interior gets the nested
// dissection below it. The interior block of the factor is then the factor
// of the Dirichlet system L_II (direct_solve_interior).
__global__ void k_nd_bl_count(int64_t NU, const int32_t* __restrict__ uslot, const int32_t* __restrict__ urow,
                              const uint8_t* __restrict__ onloop, int32_t* __restrict__ cnt2) {
    GRID_STRIDE(u, NU) atomicAdd(cnt2 + 2 * uslot[u] + (onloop[urow[u]] ? 0 : 1), 1);
}
__global__ void k_nd_bl_roots(int32_t nslot, const int32_t* __restrict__ cnt2, int leafmax, NodeArrays nd) {
    GRID_STRIDE(j, nslot) {
        const int32_t nb = cnt2[2 * j], ni = cnt2[2 * j + 1];
        const int64_t C = nslot + j;
        nd.parent[j] = -1;                 // the loop's front
        nd.chA[j] = (int32_t)C;
        nd.chB[j] = -1;
        nd.cnt[j] = nb;
        nd.npiv[j] = nb;
        nd.leaf[j] = 2;
        nd.slot[j] = (int32_t)j;
        nd.parent[C] = (int32_t)j;         // the interior's root region
        nd.chA[C] = nd.chB[C] = -1;
        nd.cnt[C] = ni;
        nd.slot[C] = (int32_t)j;
        nd.leaf[C] = ni <= leafmax;
        nd.npiv[C] = ni <= leafmax ? ni : 0;
    }
}
__global__ void k_nd_bl_init_u(int64_t NU, int32_t nslot, const int32_t* __restrict__ uslot,
                               const int32_t* __restrict__ urow, const uint8_t* __restrict__ onloop,
                               const int8_t* __restrict__ leaf, int32_t* __restrict__ reg,
                               int32_t* __restrict__ node_of) {
    GRID_STRIDE(u, NU) {
        const int j = uslot[u];
        if (onloop[urow[u]]) {
            node_of[u] = j;
            reg[u] = -1;
            continue;
        }
        const int C = nslot + j;
        if (leaf[C]) {
            node_of[u] = C;
            reg[u] = -1;
        } else {
            reg[u] = C;
            node_of[u] = -1;
        }
    }
}
__global__ void k_d_rowel(int64_t NU, const int32_t* __restrict__ urow, const int32_t* __restrict__ elim,
                          int32_t* __restrict__ rowel) {
    GRID_STRIDE(u, NU) rowel[urow[u]] = elim[u];
}

__global__ void k_nd_init_u(int64_t NU, const int32_t* __restrict__ uslot, const int8_t* __restrict__ leaf,
                            int32_t* __restrict__ reg, int32_t* __restrict__ node_of) {
    GRID_STRIDE(u, NU) {
        const int j = uslot[u];
        if (leaf[j]) {
            node_of[u] = j;
            reg[u] = -1;
        } else {
            reg[u] = j;
            node_of[u] = -1;
        }
    }
}

// region kernels read the level's node range [rng[0], rng[1]) from device
// memory (no host round trip per level) and stride over it
#define RANGE_LOOP(N, rng)                                                                  \
    for (int64_t N = (rng)[0] + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; N < (rng)[1]; \
         N += (int64_t)gridDim.x * blockDim.x)

__global__ void k_nd_reset(const int32_t* __restrict__ rng, NodeArrays nd) {
    RANGE_LOOP(N, rng) {
        for (int q = 0; q < 3; ++q) {
            nd.bbox[6 * N + q] = 0xffffffffu;
            nd.bbox[6 * N + 3 + q] = 0u;
            nd.gcnt[3 * N + q] = 0;
        }
    }
}

__global__ void k_nd_bbox(int64_t NU, const int32_t* __restrict__ reg, const float4* __restrict__ pos, NodeArrays nd) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < NU; base += stride) {
        const int64_t u = base + threadIdx.x;
        const int r = u < NU ? reg[u] : -1;
        const bool act = r >= 0;
        const float4 p = act ? pos[u] : make_float4(0.f, 0.f, 0.f, 0.f);
        agg_min_max(nd.bbox, r, act, ford(p.x), 0);
        agg_min_max(nd.bbox, r, act, ford(p.y), 1);
        agg_min_max(nd.bbox, r, act, ford(p.z), 2);
    }
}

__global__ void k_nd_split(const int32_t* __restrict__ rng, NodeArrays nd) {
    RANGE_LOOP(N, rng) {
        if (nd.leaf[N]) continue;
        float lo[3], hi[3];
        int ax = 0;
        float best = -1.f;
        for (int q = 0; q < 3; ++q) {
            lo[q] = funord(nd.bbox[6 * N + q]);
            hi[q] = funord(nd.bbox[6 * N + 3 + q]);
            if (hi[q] - lo[q] > best) {
                best = hi[q] - lo[q];
                ax = q;
            }
        }
        float mid = 0.5f * (lo[ax] + hi[ax]);
        if (!(mid > lo[ax])) mid = hi[ax];  // ties: the far side is the maximum
        if (!(best > 0.f)) {                 // all points coincide: a dense leaf
            nd.leaf[N] = 2;
            nd.npiv[N] = nd.cnt[N];
        }
        nd.split[N] = make_float2((float)ax, mid);
    }
}

__global__ void k_nd_side(int64_t NU, const int32_t* __restrict__ reg, const float4* __restrict__ pos, NodeArrays nd,
                          int8_t* __restrict__ side) {
    GRID_STRIDE(u, NU) {
        const int r = reg[u];
        if (r < 0) continue;
        const float2 sp = nd.split[r];
        const float4 p = pos[u];
        const float c = sp.x == 0.f ? p.x : (sp.x == 1.f ? p.y : p.z);
        side[u] = c >= sp.y ? 1 : 0;
    }
}

__global__ void k_nd_sep(int64_t NU, const int32_t* __restrict__ reg, const int8_t* __restrict__ side,
                         const int64_t* __restrict__ aptr, const int32_t* __restrict__ acol, NodeArrays nd,
                         int8_t* __restrict__ grp) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < NU; base += stride) {
        const int64_t u = base + threadIdx.x;
        const int r = u < NU ? reg[u] : -1;
        const bool act = r >= 0 && nd.leaf[r] == 0;
        int g = 0;
        if (act) {
            if (side[u]) {
                g = 1;
            } else {
                for (int64_t q = aptr[u]; q < aptr[u + 1]; ++q) {
                    const int w = acol[q];
                    if (reg[w] == r && side[w]) {
                        g = 2;
                        break;
                    }
                }
            }
            grp[u] = (int8_t)g;
        }
        agg_count(nd.gcnt, r, act, g);
    }
}

__global__ void k_nd_count_children(const int32_t* __restrict__ rng, NodeArrays nd) {
    RANGE_LOOP(N, rng) {
        const int64_t i = N - rng[0];
        int nc = 0;
        if (!nd.leaf[N]) {
            const int nA = nd.gcnt[3 * N], nB = nd.gcnt[3 * N + 1], nS = nd.gcnt[3 * N + 2];
            if (nB == 0 || nA + nS == 0) {  // no split: a dense leaf
                nd.leaf[N] = 2;
                nd.npiv[N] = nd.cnt[N];
            } else {
                nd.npiv[N] = nS;
                nc = (nA > 0) + 1;
            }
        }
        nd.nchild[i] = nc;
    }
}

// `cur` = this level's recorded range (the live range already points at the
// next level); children ids start at cur[1]
__global__ void k_nd_link(const int32_t* __restrict__ cur, const int32_t* __restrict__ scan, int leafmax,
                          NodeArrays nd) {
    const int32_t next = cur[1];
    RANGE_LOOP(N, cur) {
        const int64_t i = N - cur[0];
        if (nd.nchild[i] == 0) continue;
        const int nA = nd.gcnt[3 * N], nB = nd.gcnt[3 * N + 1];
        int id = next + scan[i];
        int c[2] = {-1, -1}, n[2] = {nA, nB};
        if (nA > 0) c[0] = id++;
        c[1] = id;
        nd.chA[N] = c[0];
        nd.chB[N] = c[1];
        for (int q = 0; q < 2; ++q) {
            if (c[q] < 0) continue;
            const int C = c[q];
            nd.parent[C] = (int32_t)N;
            nd.chA[C] = nd.chB[C] = -1;
            nd.cnt[C] = n[q];
            nd.slot[C] = nd.slot[N];
            nd.leaf[C] = n[q] <= leafmax;
            nd.npiv[C] = n[q] <= leafmax ? n[q] : 0;
        }
    }
}

// exclusive scan of the level's child counts (one CTA), the level recorded in
// hist[2 level..], the live range advanced to the children
__global__ void __launch_bounds__(1024) k_nd_scan(int32_t* __restrict__ rng, const int32_t* __restrict__ nchild,
                                                  int32_t* __restrict__ scan, int32_t* __restrict__ hist, int level,
                                                  int64_t ncap, int32_t* __restrict__ ovf) {
    __shared__ int32_t wsum[33];
    const int lb = rng[0], le = rng[1], n = le - lb;
    const int per = (n + 1023) / 1024;
    const int i0 = min(n, (int)threadIdx.x * per), i1 = min(n, i0 + per);
    int loc = 0;
    for (int i = i0; i < i1; ++i) loc += nchild[i];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int inc = loc;
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int q = 0; q < 32; ++q) {
            const int v = wsum[q];
            wsum[q] = acc;
            acc += v;
        }
        wsum[32] = acc;
    }
    __syncthreads();
    int off = wsum[w] + inc - loc;
    for (int i = i0; i < i1; ++i) {
        scan[i] = off;
        off += nchild[i];
    }
    if (threadIdx.x == 0) {
        const int total = wsum[32];
        hist[2 * level] = lb;
        hist[2 * level + 1] = le;
        if ((int64_t)le + total > ncap) {
            *ovf = 1;
            rng[0] = rng[1] = le;
        } else {
            rng[0] = le;
            rng[1] = le + total;
        }
    }
}

__global__ void k_nd_assign(int64_t NU, int32_t* __restrict__ reg, const int8_t* __restrict__ grp, NodeArrays nd,
                            int32_t* __restrict__ node_of) {
    GRID_STRIDE(u, NU) {
        const int r = reg[u];
        if (r < 0) continue;
        if (nd.leaf[r]) {  // dense leaf (no split possible)
            node_of[u] = r;
            reg[u] = -1;
            continue;
        }
        const int g = grp[u];
        if (g == 2) {
            node_of[u] = r;
            reg[u] = -1;
            continue;
        }
        const int C = g == 0 ? nd.chA[r] : nd.chB[r];
        if (nd.leaf[C]) {
            node_of[u] = C;
            reg[u] = -1;
        } else {
            reg[u] = C;
        }
    }
}

// postorder numbering: subtree sizes bottom-up, then starts top-down
__global__ void k_nd_subtree(int32_t lb, int32_t le, NodeArrays nd, int64_t* __restrict__ tsz) {
    GRID_STRIDE(i, (int64_t)(le - lb)) {
        const int64_t N = lb + i;
        int64_t t = nd.npiv[N];
        if (nd.chA[N] >= 0) t += tsz[nd.chA[N]];
        if (nd.chB[N] >= 0) t += tsz[nd.chB[N]];
        tsz[N] = t;
    }
}
__global__ void k_nd_start(int32_t lb, int32_t le, NodeArrays nd, const int64_t* __restrict__ tsz,
                           const int64_t* __restrict__ uoff, int64_t* __restrict__ start, int64_t* __restrict__ pfirst) {
    GRID_STRIDE(i, (int64_t)(le - lb)) {
        const int64_t N = lb + i;
        if (nd.parent[N] < 0) start[N] = uoff[nd.slot[N]];
        const int64_t s0 = start[N];
        int64_t off = s0;
        if (nd.chA[N] >= 0) {
            start[nd.chA[N]] = off;
            off += tsz[nd.chA[N]];
        }
        if (nd.chB[N] >= 0) start[nd.chB[N]] = off;
        pfirst[N] = s0 + tsz[N] - nd.npiv[N];
    }
}
__global__ void k_iota(int64_t n, int32_t* __restrict__ v) {
    GRID_STRIDE(i, n) v[i] = (int32_t)i;
}
__global__ void k_nd_elim(int64_t NU, const int32_t* __restrict__ skey, const int32_t* __restrict__ sval,
                          const int64_t* __restrict__ gstart, const int64_t* __restrict__ pfirst,
                          int32_t* __restrict__ elim, int32_t* __restrict__ perm) {
    GRID_STRIDE(i, NU) {
        const int N = skey[i];
        const int u = sval[i];
        const int64_t e = pfirst[N] + (i - gstart[N]);
        elim[u] = (int32_t)e;
        perm[e] = u;
    }
}
__global__ void k_nd_npiv64(int32_t n, const int32_t* __restrict__ a, int64_t* __restrict__ b) {
    GRID_STRIDE(i, (int64_t)n) b[i] = a[i];
}

// the adjacency in elimination order, entries above the row only (w > e):
// what assembly and the symbolic pass read, contiguous per front
__global__ void k_eadj_count(int64_t NU, const int32_t* __restrict__ perm, const int32_t* __restrict__ elim,
                             const int64_t* __restrict__ aptr, const int32_t* __restrict__ acol,
                             int64_t* __restrict__ cnt) {
    GRID_STRIDE(e, NU) {
        const int u = perm[e];
        int c = 0;
        for (int64_t q = aptr[u]; q < aptr[u + 1]; ++q) c += elim[acol[q]] > e;
        cnt[e] = c;
    }
}
__global__ void k_eadj_fill(int64_t NU, const int32_t* __restrict__ perm, const int32_t* __restrict__ elim,
                            const int64_t* __restrict__ aptr, const int32_t* __restrict__ acol,
                            const double2* __restrict__ aval, const int64_t* __restrict__ eptr,
                            int32_t* __restrict__ erow, int32_t* __restrict__ ecol, double2* __restrict__ eval) {
    GRID_STRIDE(e, NU) {
        const int u = perm[e];
        int64_t o = eptr[e];
        for (int64_t q = aptr[u]; q < aptr[u + 1]; ++q) {
            const int w = elim[acol[q]];
            if (w > e) {
                erow[o] = (int32_t)e;
                ecol[o] = w;
                eval[o] = aval[q];
                ++o;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// symbolic: update sets

struct SymArgs {
    NodeArrays nd;
    const int64_t* pfirst;
    const int32_t* perm;
    const int32_t* elim;
    const int64_t* eptr;     // adjacency in elimination order (entries above the row only)
    const int32_t* ecol;
    int32_t* ucnt;
    int64_t* ustart;
    int32_t* upool;
    unsigned long long* bump;
    int64_t ucap;
    int32_t* overflow;
};

__global__ void __launch_bounds__(DNT) k_sym(int32_t lb, SymArgs a) {
    __shared__ int32_t cand[CAND_MAX];
    __shared__ int32_t ncand;
    __shared__ int32_t wsum[DNT / 32 + 1];
    __shared__ unsigned long long base;
    const int N = lb + blockIdx.x;
    const int64_t pf = a.pfirst[N];
    const int s = a.nd.npiv[N];
    const int64_t pend = pf + s;
    if (threadIdx.x == 0) ncand = 0;
    __syncthreads();
    for (int64_t q = a.eptr[pf] + threadIdx.x; q < a.eptr[pend]; q += DNT) {
        const int e = a.ecol[q];
        if (e >= pend) {
            const int i = atomicAdd(&ncand, 1);
            if (i < CAND_MAX) cand[i] = e;
        }
    }
    const int ch[2] = {a.nd.chA[N], a.nd.chB[N]};
    for (int c = 0; c < 2; ++c) {
        if (ch[c] < 0) continue;
        const int n = a.ucnt[ch[c]];
        const int32_t* U = a.upool + a.ustart[ch[c]];
        for (int t = threadIdx.x; t < n; t += DNT) {
            const int e = U[t];
            if (e >= pend) {
                const int i = atomicAdd(&ncand, 1);
                if (i < CAND_MAX) cand[i] = e;
            }
        }
    }
    __syncthreads();
    const int n = ncand;
    if (n > CAND_MAX) {
        if (threadIdx.x == 0) {
            atomicExch(a.overflow, 1);
            a.ucnt[N] = 0;
            a.ustart[N] = 0;
        }
        return;
    }
    int p2 = 1;
    while (p2 < n) p2 <<= 1;
    for (int i = n + threadIdx.x; i < p2; i += DNT) cand[i] = INT_MAX;
    __syncthreads();
    // bitonic sort (ascending)
    for (int k = 2; k <= p2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < p2; i += DNT) {
                const int l = i ^ j;
                if (l > i) {
                    const int x = cand[i], y = cand[l];
                    const bool up = (i & k) == 0;
                    if ((x > y) == up) {
                        cand[i] = y;
                        cand[l] = x;
                    }
                }
            }
            __syncthreads();
        }
    }
    // unique: contiguous chunks per thread, block scan of the kept counts
    const int per = (n + DNT - 1) / DNT;
    const int i0 = min(n, (int)threadIdx.x * per), i1 = min(n, i0 + per);
    int keep = 0;
    for (int i = i0; i < i1; ++i) keep += (i == 0 || cand[i] != cand[i - 1]);
    // inclusive warp scan, then warp offsets
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int inc = keep;
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int q = 0; q < DNT / 32; ++q) {
            const int v = wsum[q];
            wsum[q] = acc;
            acc += v;
        }
        wsum[DNT / 32] = acc;
        const unsigned long long b = atomicAdd(a.bump, (unsigned long long)acc);
        base = b;
        if ((int64_t)(b + acc) > a.ucap) atomicExch(a.overflow, 1);
        a.ucnt[N] = acc;
        a.ustart[N] = (int64_t)b;
    }
    __syncthreads();
    const int total = wsum[DNT / 32];
    if ((int64_t)(base + total) > a.ucap) return;
    int o = wsum[w] + inc - keep;
    int32_t* out = a.upool + base;
    for (int i = i0; i < i1; ++i)
        if (i == 0 || cand[i] != cand[i - 1]) out[o++] = cand[i];
}

// front sizes; storage in doubles (complex: 2 per entry; real: padded to
// an even count so every complex front stays 16-byte aligned)
__global__ void k_front_sizes(int32_t n, const int32_t* __restrict__ npiv, const int32_t* __restrict__ ucnt,
                              const int8_t* __restrict__ ntype, int32_t* __restrict__ fsz, int64_t* __restrict__ f2,
                              int64_t* __restrict__ f1) {
    GRID_STRIDE(i, (int64_t)n) {
        const int64_t f = (int64_t)npiv[i] + ucnt[i];
        fsz[i] = (int32_t)f;
        const int64_t np = f * (f + 1) / 2;  // packed lower triangle
        f2[i] = ntype[i] ? 2 * np : ((np + 1) & ~1ll);
        f1[i] = f;
    }
}

// a front is complex when its subtree holds a row with DNCP coupling
// (imaginary entries); marks walk up from the row's node (idempotent stores)
__global__ void k_mark_cplx(int64_t NU, const int64_t* __restrict__ aptr, const double2* __restrict__ aval,
                            const int32_t* __restrict__ node_of, const int32_t* __restrict__ parent,
                            int8_t* __restrict__ ntype) {
    GRID_STRIDE(u, NU) {
        bool c = false;
        for (int64_t q = aptr[u]; q < aptr[u + 1]; ++q) c |= aval[q].y != 0.0;
        if (!c) continue;
        for (int N = node_of[u]; N >= 0; N = parent[N]) ntype[N] = 1;
    }
}

// ---------------------------------------------------------------------------
// numeric factorization

struct FacArgs {
    NodeArrays nd;
    const int64_t* pfirst;
    const int32_t* perm;
    const int32_t* elim;
    const int64_t* eptr;     // adjacency in elimination order: row e's entries w > e
    const int32_t* erow;
    const int32_t* ecol;
    const double2* eval;     // A(row, col)
    const int32_t* ucnt;
    const int64_t* ustart;
    const int32_t* upool;
    const int32_t* fsz;
    const int64_t* foff;     // front offsets in doubles (complex fronts: 16-byte aligned)
    void* fpool;
    const int8_t* ntype;     // 1: complex front (its subtree holds DNCP coupling entries)
    const int32_t* list;     // the fronts of one launch (one level, one type)
    int32_t* err;  // per slot: nonpositive pivot
};

template <class T>
__device__ __forceinline__ T* front_ptr(void* pool, int64_t off) {
    return reinterpret_cast<T*>(reinterpret_cast<double*>(pool) + off);
}
template <class T>
__device__ __forceinline__ const T* front_ptr(const void* pool, int64_t off) {
    return reinterpret_cast<const T*>(reinterpret_cast<const double*>(pool) + off);
}
// fronts live in global memory as packed lower triangles, column-major:
// column j holds rows j..f-1 and starts at j (2f - j - 1) / 2
__device__ __forceinline__ int64_t pk64(int i, int j, int f) { return (int64_t)j * (2 * f - j - 1) / 2 + i; }
__device__ __forceinline__ int64_t npk(int f) { return (int64_t)f * (f + 1) / 2; }
template <class T> __device__ __forceinline__ T narrow(double2 v);
template <> __device__ __forceinline__ double narrow<double>(double2 v) { return v.x; }
template <> __device__ __forceinline__ double2 narrow<double2>(double2 v) { return v; }

// position of elimination index x in front N's row list (pivots, then U)
__device__ __forceinline__ int front_pos(int64_t x, int64_t pf, int s, const int32_t* U, int nu) {
    if (x < pf + s) return (int)(x - pf);
    return s + lower_bound_i32(U, nu, (int32_t)x);
}

// matrix entries of pivots [kb, ke) of a front (lower part, column-major,
// leading dimension f): S[pos(w)][k] = A(w, u) = conj(A(u, w)), unit diagonal.
// One thread per stored entry: independent, coalesced loads.
template <class T, bool PACKED>
__device__ __forceinline__ void assemble_entries(T* S, int f, int64_t pf, int s, const int32_t* Us, int nu, int kb,
                                                 int ke, const FacArgs& a) {
    auto at = [&](int i, int j) -> int64_t { return PACKED ? pk64(i, j, f) : (int64_t)i + (int64_t)j * f; };
    for (int k = kb + threadIdx.x; k < ke; k += DNT) S[at(k, k)] = from_c<T>(make_double2(1.0, 0.0));
    const int64_t q1 = a.eptr[pf + ke];
    for (int64_t q = a.eptr[pf + kb] + threadIdx.x; q < q1; q += DNT) {
        const int k = (int)(a.erow[q] - pf);
        const int i = front_pos(a.ecol[q], pf, s, Us, nu);
        S[at(i, k)] = cj(from_c<T>(a.eval[q]));
    }
}

// One TR x TC tile (rows [ti, ti+TR) below rlim, columns [tj, tj+TC) below
// clim, lower part r >= c only): F[r][c] -= sum_{k in [kb, ke)} F[r][k]
// conj(F[c][k]), k staged in chunks of KC through shared memory (the next
// chunk's global loads issued before the current chunk's multiply-adds).
// Thread (ty, tx) owns rows ty + 8 i and columns tx + 16 j: for a fixed
// (i, j) a warp reads consecutive shared-memory entries (no bank conflicts).
template <class T>
__device__ __forceinline__ void tile_one(T* F, int f, int ti, int tj, int rlim, int clim, int kb, int ke, T* As,
                                         T* Bs) {
    const int t = threadIdx.x;
    const int ty = t >> 4, tx = t & 15;
    constexpr int QA = (TR * KC) / DNT, QB = (TC * KC) / DNT;
    T acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = zero_t<T>();
    T ra[QA], rb[QB];
    auto fetch = [&](int kc) {
#pragma unroll
        for (int q = 0; q < QA; ++q) {
            const int idx = t + q * DNT;
            const int r = idx % TR, k = kc + idx / TR;
            ra[q] = (k < ke && ti + r < rlim) ? F[pk64(ti + r, k, f)] : zero_t<T>();
        }
#pragma unroll
        for (int q = 0; q < QB; ++q) {
            const int idx = t + q * DNT;
            const int r = idx % TC, k = kc + idx / TC;
            rb[q] = (k < ke && tj + r < clim) ? F[pk64(tj + r, k, f)] : zero_t<T>();
        }
    };
    if (kb < ke) fetch(kb);
    for (int kc = kb; kc < ke; kc += KC) {
#pragma unroll
        for (int q = 0; q < QA; ++q) As[t + q * DNT] = ra[q];
#pragma unroll
        for (int q = 0; q < QB; ++q) Bs[t + q * DNT] = rb[q];
        __syncthreads();
        if (kc + KC < ke) fetch(kc + KC);
#pragma unroll 4
        for (int kk = 0; kk < KC; ++kk) {
            T av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[kk * TR + ty + 8 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Bs[kk * TC + tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) fma_cj(acc[i][j], av[i], bv[j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = ti + ty + 8 * i;
        if (r >= rlim) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = tj + tx + 16 * j;
            if (c >= clim || r < c) continue;
            T& dst = F[pk64(r, c, f)];
            dst = sub(dst, acc[i][j]);
        }
    }
}

// F[i][j] -= sum_{k in [kb, ke)} F[i][k] conj(F[j][k]) for j in [c0, c1),
// i in [j, f): every lower tile in turn (one CTA)
template <class T>
__device__ void tile_update(T* F, int f, int c0, int c1, int kb, int ke, T* As, T* Bs) {
    for (int tj = c0; tj < c1; tj += TC)
        for (int ti = tj; ti < f; ti += TR) tile_one<T>(F, f, ti, tj, f, c1, kb, ke, As, Bs);
    __syncthreads();
}

// lower tiles of an n x n block: column tile j (TC wide) has ceil((n - TC j) / TR) row tiles
__host__ __device__ inline int schur_tiles(int n) {
    int t = 0;
    for (int c = 0; c < n; c += TC) t += (n - c + TR - 1) / TR;
    return t;
}

__device__ __forceinline__ double shfl_t(double v, int src) { return __shfl_sync(FULL, v, src); }
__device__ __forceinline__ double2 shfl_t(double2 v, int src) {
    return make_double2(__shfl_sync(FULL, v.x, src), __shfl_sync(FULL, v.y, src));
}

// Cholesky of the nb x nb lower block Ld (leading dimension LDB <= 32) by
// one warp: lane i keeps row i in registers, column k's entries travel by
// shuffles; a nonpositive pivot sets *bad and continues with 1
template <class T, int LDB>
__device__ __forceinline__ void diag_factor(T* Ld, int nb, int* bad) {
    const int lane = threadIdx.x & 31;
    T r[LDB];
#pragma unroll
    for (int j = 0; j < LDB; ++j) r[j] = (lane < nb && j < nb) ? Ld[lane + j * LDB] : zero_t<T>();
#pragma unroll
    for (int k = 0; k < LDB; ++k) {
        if (k < nb) {
            double d = re(shfl_t(r[k], k));
            if (!(d > 0.0) || !isfinite(d)) {
                if (lane == 0) *bad = 1;
                d = 1.0;
            }
            const double inv = rsqrt(d);  // one reciprocal square root per pivot
            if (lane == k) r[k] = from_c<T>(make_double2(d * inv, 0.0));
            else if (lane > k) r[k] = scale(r[k], inv);
#pragma unroll
            for (int j = k + 1; j < LDB; ++j) {
                const T ljk = shfl_t(r[k], j);
                if (lane >= j && j < nb) fma_cj(r[j], scale(r[k], -1.0), ljk);
            }
        }
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < LDB; ++j)
        if (lane < nb && j <= lane) Ld[lane + j * LDB] = r[j];
    __syncwarp();
}

// the same by the whole CTA in shared memory (no register arrays: for
// kernels whose register budget is set by other work)
template <class T, int LDB, int NTH>
__device__ __forceinline__ void diag_factor_cta(T* Ld, int nb, int* bad) {
    __shared__ double sinv;
    for (int k = 0; k < nb; ++k) {
        if (threadIdx.x == 0) {
            double d = re(Ld[k + k * LDB]);
            if (!(d > 0.0) || !isfinite(d)) {
                *bad = 1;
                d = 1.0;
            }
            const double inv = rsqrt(d);
            Ld[k + k * LDB] = from_c<T>(make_double2(d * inv, 0.0));
            sinv = inv;
        }
        __syncthreads();
        for (int i = k + 1 + threadIdx.x; i < nb; i += NTH) Ld[i + k * LDB] = scale(Ld[i + k * LDB], sinv);
        __syncthreads();
        {   // trailing update: lane = row, the warps stride over the columns (no
            // index divisions, conflict-free rows, broadcast l_jk); each entry
            // takes the same one multiply-add per k as before
            static_assert(LDB <= 32, "one lane per row of the block");
            const int i = k + 1 + (int)(threadIdx.x & 31);
            if (i < nb) {
                const T lik = scale(Ld[i + k * LDB], -1.0);
                for (int j = k + 1 + (int)(threadIdx.x >> 5); j <= i; j += NTH / 32)
                    fma_cj(Ld[i + j * LDB], lik, Ld[j + k * LDB]);
            }
        }
        __syncthreads();
    }
}

constexpr int FAC_SCHUR_INLINE = 1;  // k_factor: Schur update of the U block in this CTA
constexpr int FAC_ASSEMBLE_ONLY = 2; // k_factor: assembly only (the level-synchronous panel follows)

// real fronts: 8 CTAs per SM (64 registers); complex: 4
template <class T>
__global__ void __launch_bounds__(DNT, sizeof(T) == 8 ? 8 : 4) k_factor(FacArgs a, int mode) {
    extern __shared__ __align__(16) unsigned char dsm[];
    T* As = reinterpret_cast<T*>(dsm);
    T* Bs = As + KC * TR;
    T* Ld = Bs + KC * TC;                                // NB x NB, column-major
    int32_t* Us = reinterpret_cast<int32_t*>(Ld + NB * NB);  // my U list, then a child's rel map
    __shared__ int bad;
    __shared__ double dinv[NB];
    const int N = a.list[blockIdx.x];
    const int s = a.nd.npiv[N];
    const int nu = a.ucnt[N];
    const int f = s + nu;
    const int64_t pf = a.pfirst[N];
    T* F = front_ptr<T>(a.fpool, a.foff[N]);
    int32_t* rel = Us + nu;
    if (threadIdx.x == 0) bad = 0;
    for (int i = threadIdx.x; i < nu; i += DNT) Us[i] = a.upool[a.ustart[N] + i];
    {   // zero the front (16-byte stores)
        const int64_t nd2 = npk(f) * (int64_t)(sizeof(T) / 8);
        double2* z2 = reinterpret_cast<double2*>(F);
        const bool al = (reinterpret_cast<uintptr_t>(F) & 15) == 0;
        if (al) {
            for (int64_t i = threadIdx.x; i < nd2 / 2; i += DNT) z2[i] = make_double2(0.0, 0.0);
            if ((nd2 & 1) && threadIdx.x == 0) reinterpret_cast<double*>(F)[nd2 - 1] = 0.0;
        } else {
            for (int64_t i = threadIdx.x; i < nd2; i += DNT) reinterpret_cast<double*>(F)[i] = 0.0;
        }
    }
    __syncthreads();
    assemble_entries<T, true>(F, f, pf, s, Us, nu, 0, s, a);
    __syncthreads();
    // extend-add the children's update blocks (fixed order: A, then B; every
    // entry of one child's block lands on a distinct position)
    const int ch[2] = {a.nd.chA[N], a.nd.chB[N]};
    for (int c = 0; c < 2; ++c) {
        const int C = ch[c];
        if (C < 0) continue;
        const int sc = a.nd.npiv[C], uc = a.ucnt[C], fc = sc + uc;
        const int32_t* UC = a.upool + a.ustart[C];
        for (int i = threadIdx.x; i < uc; i += DNT) rel[i] = front_pos(UC[i], pf, s, Us, nu);
        __syncthreads();
        const bool ccx = a.ntype[C] != 0;  // a real child may feed a complex front
        const double* __restrict__ FC = reinterpret_cast<const double*>(a.fpool) + a.foff[C];
        const int tot = uc * uc;
        for (int t0 = threadIdx.x; t0 < tot; t0 += 4 * DNT) {
            double2 v[4];
            int pos[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int t = t0 + q * DNT;
                const int bcol = t / max(uc, 1), i = t - bcol * uc;
                const bool ok = t < tot && i >= bcol;
                pos[q] = ok ? pk64(rel[i], rel[bcol], f) : -1;
                const int64_t e = pk64(sc + i, sc + bcol, fc);
                v[q] = !ok ? make_double2(0.0, 0.0)
                           : (ccx ? reinterpret_cast<const double2*>(FC)[e] : make_double2(FC[e], 0.0));
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (pos[q] >= 0) F[pos[q]] = add(F[pos[q]], narrow<T>(v[q]));
        }
        __syncthreads();
    }
    if (mode & FAC_ASSEMBLE_ONLY) return;
    // partial factorization of the pivot columns
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int k0 = 0; k0 < s; k0 += NB) {
        const int nb = min(NB, s - k0);
        // diagonal block: one warp, unblocked
        if (warp == 0) {
            for (int idx = lane; idx < NB * NB; idx += 32) {
                const int i = idx % NB, j = idx / NB;
                Ld[idx] = (i < nb && j < nb && i >= j) ? F[pk64(k0 + i, k0 + j, f)] : zero_t<T>();
            }
            __syncwarp();
            diag_factor<T, NB>(Ld, nb, &bad);
            for (int idx = lane; idx < NB * NB; idx += 32) {
                const int i = idx % NB, j = idx / NB;
                if (i < nb && j < nb && i >= j) F[pk64(k0 + i, k0 + j, f)] = Ld[idx];
            }
        }
        if (threadIdx.x < nb) dinv[threadIdx.x] = 1.0 / re(Ld[threadIdx.x + threadIdx.x * NB]);
        __syncthreads();
        // rows below the block: x L^H = row -> forward substitution per row
        for (int r = k0 + nb + threadIdx.x; r < f; r += DNT) {
            T x[NB];
#pragma unroll
            for (int k = 0; k < NB; ++k) x[k] = k < nb ? F[pk64(r, k0 + k, f)] : zero_t<T>();
#pragma unroll
            for (int k = 0; k < NB; ++k) {
                if (k < nb) {
                    T v = x[k];
#pragma unroll
                    for (int j = 0; j < NB; ++j)
                        if (j < k) fma_cj(v, scale(x[j], -1.0), Ld[k + j * NB]);
                    x[k] = scale(v, dinv[k]);
                }
            }
#pragma unroll
            for (int k = 0; k < NB; ++k)
                if (k < nb) F[pk64(r, k0 + k, f)] = x[k];
        }
        __syncthreads();
        // the remaining pivot columns
        if (k0 + nb < s) tile_update<T>(F, f, k0 + nb, s, k0, k0 + nb, As, Bs);
    }
    // Schur complement of the update block (read in place by the parent):
    // here, or by k_schur's tiles spread over CTAs
    if ((mode & FAC_SCHUR_INLINE) && nu > 0 && s > 0) tile_update<T>(F, f, s, f, 0, s, As, Bs);
    if (threadIdx.x == 0 && bad) atomicExch(a.err + a.nd.slot[N], 1);
}

// Level-synchronous blocked panel for the large fronts of a level: all
// fronts advance through their pivot columns in blocks of PB together.
// k_pdiag: the diagonal block (redundantly per CTA, written by row chunk 0)
// and the TRSM of DNT rows below it per CTA; k_pupd: the update of the
// remaining pivot columns, one CTA per TR x TC tile.
constexpr int PB = 32;
constexpr int FUSED_MAXS = 48;
constexpr size_t SM_FRONT_BYTES = 112 * 1024;  // k_factor_sm: two CTAs per SM
// k_factor_warp fronts split off a list of larger ones: up to 70 wide (real and complex)
constexpr size_t warp_split_bytes(size_t tsz) { return tsz == 8 ? 20 * 1024 : 40 * 1024; }
constexpr size_t WARP_FRONT_BYTES = 40 * 1024; // k_factor_warp: per warp (packed lower triangle)  // levels whose fronts all have <= this many pivots stay fused

// phase 0 (one CTA per front): factor the diagonal block in place;
// phase 1 (CTAs over row chunks): TRSM of the rows below it
template <class T>
__global__ void __launch_bounds__(DNT) k_pdiag(FacArgs a, int k0, int phase) {
    __shared__ __align__(16) T Ld[PB * PB];
    __shared__ double dinvp[PB];
    __shared__ int bad;
    const int N = a.list[blockIdx.x];
    const int s = a.nd.npiv[N];
    if (k0 >= s) return;
    const int f = s + a.ucnt[N];
    const int nb = min(PB, s - k0);
    const int r0 = k0 + nb + blockIdx.y * DNT;
    if (blockIdx.y > 0 && r0 >= f) return;
    T* F = front_ptr<T>(a.fpool, a.foff[N]);
    if (threadIdx.x == 0) bad = 0;
    for (int idx = threadIdx.x; idx < PB * PB; idx += DNT) {
        const int i = idx % PB, j = idx / PB;
        Ld[idx] = (i < nb && j < nb && i >= j) ? F[pk64(k0 + i, k0 + j, f)] : zero_t<T>();
    }
    if (phase == 0) {
        __syncthreads();
        // by the whole CTA in shared memory: the one-warp register form is a
        // fully unrolled 32 x 32 block (~10K straight-line instructions for
        // complex fronts, every one a cold instruction fetch): 54-105 us per
        // level in the launch list against ~15 us this way
        diag_factor_cta<T, PB, DNT>(Ld, nb, &bad);
        __syncthreads();
        for (int idx = threadIdx.x; idx < PB * PB; idx += DNT) {
            const int i = idx % PB, j = idx / PB;
            if (i < nb && j < nb && i >= j) F[pk64(k0 + i, k0 + j, f)] = Ld[idx];
        }
        if (threadIdx.x == 0 && bad) atomicExch(a.err + a.nd.slot[N], 1);
        return;
    }
    __syncthreads();
    if (threadIdx.x < nb) dinvp[threadIdx.x] = 1.0 / re(Ld[threadIdx.x + threadIdx.x * PB]);
    __syncthreads();
    // TRSM of my row in two halves of 16: a dependency chain per half, the
    // coupling between the halves as independent multiply-adds
    const int r = r0 + threadIdx.x;
    if (r < f) {
        T x[16], y[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) x[k] = k < nb ? F[pk64(r, k0 + k, f)] : zero_t<T>();
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            T v = x[k];
#pragma unroll
            for (int j = 0; j < k; ++j) fma_cj(v, scale(x[j], -1.0), Ld[k + j * PB]);
            x[k] = k < nb ? scale(v, dinvp[k]) : zero_t<T>();
        }
#pragma unroll
        for (int k = 0; k < 16; ++k)
            if (k < nb) F[pk64(r, k0 + k, f)] = x[k];
        if (nb > 16) {
#pragma unroll
            for (int k = 0; k < 16; ++k) y[k] = 16 + k < nb ? F[pk64(r, k0 + 16 + k, f)] : zero_t<T>();
#pragma unroll
            for (int j = 0; j < 16; ++j)
#pragma unroll
                for (int k = 0; k < 16; ++k) fma_cj(y[k], scale(x[j], -1.0), Ld[(16 + k) + j * PB]);
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                T v = y[k];
#pragma unroll
                for (int j = 0; j < k; ++j) fma_cj(v, scale(y[j], -1.0), Ld[(16 + k) + (16 + j) * PB]);
                y[k] = 16 + k < nb ? scale(v, dinvp[16 + k]) : zero_t<T>();
            }
#pragma unroll
            for (int k = 0; k < 16; ++k)
                if (16 + k < nb) F[pk64(r, k0 + 16 + k, f)] = y[k];
        }
    }
}

// Multi-CTA assembly of the large fronts of a level. k_asm_cols: CTA y owns
// columns [y cw, (y+1) cw): zeroes them and writes the matrix entries of the
// pivots among them. k_asm_child: one child's update block, CTA y adding
// columns [y cw, (y+1) cw) of it. Launched zero, child A, child B: every
// position's sum is formed in a fixed order.
template <class T>
__global__ void __launch_bounds__(DNT) k_asm_cols(FacArgs a, int cw) {
    extern __shared__ __align__(16) unsigned char dsm[];
    int32_t* Us = reinterpret_cast<int32_t*>(dsm);
    const int N = a.list[blockIdx.x];
    const int s = a.nd.npiv[N];
    const int nu = a.ucnt[N];
    const int f = s + nu;
    const int c0 = blockIdx.y * cw;
    if (c0 >= f) return;
    const int c1 = min(f, c0 + cw);
    const int64_t pf = a.pfirst[N];
    T* F = front_ptr<T>(a.fpool, a.foff[N]);
    const int kb = c0, ke = min(c1, s);
    if (ke > kb)
        for (int i = threadIdx.x; i < nu; i += DNT) Us[i] = a.upool[a.ustart[N] + i];
    for (int64_t i = pk64(c0, c0, f) + threadIdx.x; i < pk64(c1, c1, f); i += DNT) F[i] = zero_t<T>();
    __syncthreads();
    if (ke > kb) assemble_entries<T, true>(F, f, pf, s, Us, nu, kb, ke, a);
}

template <class T>
__global__ void __launch_bounds__(DNT) k_asm_child(FacArgs a, int which, int cw) {
    extern __shared__ __align__(16) unsigned char dsm[];
    int32_t* Us = reinterpret_cast<int32_t*>(dsm);
    const int N = a.list[blockIdx.x];
    const int C = which ? a.nd.chB[N] : a.nd.chA[N];
    if (C < 0) return;
    const int sc = a.nd.npiv[C], uc = a.ucnt[C], fc = sc + uc;
    const int b0 = blockIdx.y * cw;
    if (b0 >= uc) return;
    const int b1 = min(uc, b0 + cw);
    const int s = a.nd.npiv[N];
    const int nu = a.ucnt[N];
    const int f = s + nu;
    const int64_t pf = a.pfirst[N];
    int32_t* rel = Us + nu;
    for (int i = threadIdx.x; i < nu; i += DNT) Us[i] = a.upool[a.ustart[N] + i];
    __syncthreads();
    const int32_t* UC = a.upool + a.ustart[C];
    for (int i = b0 + threadIdx.x; i < uc; i += DNT) rel[i] = front_pos(UC[i], pf, s, Us, nu);
    __syncthreads();
    T* F = front_ptr<T>(a.fpool, a.foff[N]);
    const bool ccx = a.ntype[C] != 0;
    const double* FC = reinterpret_cast<const double*>(a.fpool) + a.foff[C];
    const int tot = (b1 - b0) * uc;
    constexpr int BAT = 4;
    for (int t0 = threadIdx.x; t0 < tot; t0 += DNT * BAT) {
        double2 v[BAT];
        int64_t pos[BAT];
#pragma unroll
        for (int q = 0; q < BAT; ++q) {
            const int t = t0 + DNT * q;
            const int b = b0 + t / uc, i = t % uc;
            const bool ok = t < tot && i >= b;
            pos[q] = ok ? pk64(rel[i], rel[b], f) : -1;
            const int64_t e = pk64(sc + i, sc + b, fc);
            v[q] = !ok ? make_double2(0.0, 0.0)
                       : (ccx ? reinterpret_cast<const double2*>(FC)[e] : make_double2(FC[e], 0.0));
        }
#pragma unroll
        for (int q = 0; q < BAT; ++q)
            if (pos[q] >= 0) F[pos[q]] = add(F[pos[q]], narrow<T>(v[q]));
    }
}

// tiles of the pivot-column update after block k0: columns [c0, s), rows [tj, f)
__host__ __device__ inline int pupd_tiles(int s, int f, int c0) {
    int t = 0;
    for (int tj = c0; tj < s; tj += TC) t += (f - tj + TR - 1) / TR;
    return t;
}

template <class T>
__global__ void __launch_bounds__(DNT, 4) k_pupd(FacArgs a, int k0) {
    __shared__ __align__(16) T As[KC * TR];
    __shared__ __align__(16) T Bs[KC * TC];  // then the next diagonal block (PB x PB <= KC x TC)
    __shared__ int bad;
    const int N = a.list[blockIdx.x];
    const int s = a.nd.npiv[N];
    const int nb = min(PB, s - k0);
    const int c0 = k0 + nb;
    if (k0 >= s || c0 >= s) return;
    const int f = s + a.ucnt[N];
    int p = blockIdx.y;
    int tj = c0;
    for (; tj < s; tj += TC) {
        const int nr = (f - tj + TR - 1) / TR;
        if (p < nr) break;
        p -= nr;
    }
    if (tj >= s) return;
    T* F = front_ptr<T>(a.fpool, a.foff[N]);
    tile_one<T>(F, f, tj + TR * p, tj, f, s, k0, k0 + nb, As, Bs);
    if (tj != c0 || p != 0) return;
    // this tile holds the next diagonal block: factor it now (the next
    // step's TRSM reads it; no other CTA of this launch touches it)
    __syncthreads();
    const int nb2 = min(PB, s - c0);
    T* Ld = Bs;
    if (threadIdx.x == 0) bad = 0;
    for (int idx = threadIdx.x; idx < PB * PB; idx += DNT) {
        const int i = idx % PB, j = idx / PB;
        Ld[idx] = (i < nb2 && j < nb2 && i >= j) ? F[pk64(c0 + i, c0 + j, f)] : zero_t<T>();
    }
    __syncthreads();
    diag_factor_cta<T, PB, DNT>(Ld, nb2, &bad);
    for (int idx = threadIdx.x; idx < PB * PB; idx += DNT) {
        const int i = idx % PB, j = idx / PB;
        if (i < nb2 && j < nb2 && i >= j) F[pk64(c0 + i, c0 + j, f)] = Ld[idx];
    }
    if (threadIdx.x == 0 && bad) atomicExch(a.err + a.nd.slot[N], 1);
}

// Small fronts, resident in shared memory for the whole factorization:
// zero, matrix entries, children's update blocks (fixed order), then per
// 16-column block: the diagonal block by one warp (registers + shuffles),
// the rows below by one thread each, and the trailing lower triangle
// (pivot columns and the update block alike) in 4x4 register tiles read
// straight from shared memory. One coalesced write-back at the end.
template <class T, int SBK>
__global__ void __launch_bounds__(DNT) k_factor_sm(FacArgs a) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ int bad;
    __shared__ double dsm_inv[SBK];
    const int N = a.list[blockIdx.x];
    const int s = a.nd.npiv[N];
    const int nu = a.ucnt[N];
    const int f = s + nu;
    const int64_t pf = a.pfirst[N];
    T* S = reinterpret_cast<T*>(dsm);
    int32_t* Us = reinterpret_cast<int32_t*>(S + (int64_t)f * f);
    int32_t* rel = Us + nu;
    if (threadIdx.x == 0) bad = 0;
    for (int i = threadIdx.x; i < f * f; i += DNT) S[i] = zero_t<T>();
    for (int i = threadIdx.x; i < nu; i += DNT) Us[i] = a.upool[a.ustart[N] + i];
    __syncthreads();
    assemble_entries<T, false>(S, f, pf, s, Us, nu, 0, s, a);
    __syncthreads();
    const int ch[2] = {a.nd.chA[N], a.nd.chB[N]};
    for (int c = 0; c < 2; ++c) {
        const int C = ch[c];
        if (C < 0) continue;
        const int sc = a.nd.npiv[C], uc = a.ucnt[C], fc = sc + uc;
        const int32_t* UC = a.upool + a.ustart[C];
        for (int i = threadIdx.x; i < uc; i += DNT) rel[i] = front_pos(UC[i], pf, s, Us, nu);
        __syncthreads();
        const bool ccx = a.ntype[C] != 0;
        const double* FC = reinterpret_cast<const double*>(a.fpool) + a.foff[C];
        const int tot = uc * uc;
        for (int t0 = threadIdx.x; t0 < tot; t0 += 4 * DNT) {
            double2 v[4];
            int pos[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int t = t0 + q * DNT;
                const int bcol = t / uc, i = t - bcol * uc;
                const bool ok = t < tot && i >= bcol;
                pos[q] = ok ? rel[i] + rel[bcol] * f : -1;
                const int64_t e = pk64(sc + i, sc + bcol, fc);
                v[q] = !ok ? make_double2(0.0, 0.0)
                           : (ccx ? reinterpret_cast<const double2*>(FC)[e] : make_double2(FC[e], 0.0));
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (pos[q] >= 0) S[pos[q]] = add(S[pos[q]], narrow<T>(v[q]));
        }
        __syncthreads();
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int k0 = 0; k0 < s; k0 += SBK) {
        const int nb = min(SBK, s - k0);
        if (warp == 0) {  // diagonal block: lane i keeps row i
            T r[SBK];
#pragma unroll
            for (int j = 0; j < SBK; ++j) r[j] = (lane < nb && j < nb) ? S[(k0 + lane) + (k0 + j) * f] : zero_t<T>();
#pragma unroll
            for (int k = 0; k < SBK; ++k) {
                if (k < nb) {
                    double d = re(shfl_t(r[k], k));
                    if (!(d > 0.0) || !isfinite(d)) {
                        if (lane == 0) bad = 1;
                        d = 1.0;
                    }
                    const double inv = rsqrt(d);
                    if (lane == k) r[k] = from_c<T>(make_double2(d * inv, 0.0));
                    else if (lane > k) r[k] = scale(r[k], inv);
#pragma unroll
                    for (int j = k + 1; j < SBK; ++j) {
                        const T ljk = shfl_t(r[k], j);
                        if (lane >= j && j < nb) fma_cj(r[j], scale(r[k], -1.0), ljk);
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < SBK; ++j)
                if (lane < nb && j <= lane) S[(k0 + lane) + (k0 + j) * f] = r[j];
        }
        if (threadIdx.x < nb) dsm_inv[threadIdx.x] = 1.0 / re(S[(k0 + threadIdx.x) + (k0 + threadIdx.x) * f]);
        __syncthreads();
        for (int rr = k0 + nb + threadIdx.x; rr < f; rr += DNT) {
            T x[SBK];
#pragma unroll
            for (int k = 0; k < SBK; ++k) x[k] = k < nb ? S[rr + (k0 + k) * f] : zero_t<T>();
#pragma unroll
            for (int k = 0; k < SBK; ++k) {
                if (k < nb) {
                    T v = x[k];
#pragma unroll
                    for (int j = 0; j < SBK; ++j)
                        if (j < k) fma_cj(v, scale(x[j], -1.0), S[(k0 + k) + (k0 + j) * f]);
                    x[k] = scale(v, dsm_inv[k]);
                }
            }
#pragma unroll
            for (int k = 0; k < SBK; ++k)
                if (k < nb) S[rr + (k0 + k) * f] = x[k];
        }
        __syncthreads();
        // trailing lower triangle, 4x4 tiles (tile row ti >= tile column tj)
        const int c0 = k0 + nb, m = f - c0;
        if (m > 0) {
            const int nt = (m + 3) >> 2;
            const int ntiles = nt * (nt + 1) / 2;
            for (int t = threadIdx.x; t < ntiles; t += DNT) {
                // t -> (ti, tj), ti >= tj, row-major over the lower tiles
                int ti = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
                while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
                while (ti * (ti + 1) / 2 > t) --ti;
                const int tj = t - ti * (ti + 1) / 2;
                const int rb = c0 + 4 * ti, cb = c0 + 4 * tj;
                T acc[4][4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = zero_t<T>();
                for (int k = 0; k < nb; ++k) {
                    const T* colk = S + (k0 + k) * f;
                    T av[4], bv[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) av[i] = rb + i < f ? colk[rb + i] : zero_t<T>();
#pragma unroll
                    for (int j = 0; j < 4; ++j) bv[j] = cb + j < f ? colk[cb + j] : zero_t<T>();
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) fma_cj(acc[i][j], av[i], bv[j]);
                }
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int r = rb + i, c = cb + j;
                        if (r < f && c < f && r >= c) S[r + c * f] = sub(S[r + c * f], acc[i][j]);
                    }
            }
        }
        __syncthreads();
    }
    T* F = front_ptr<T>(a.fpool, a.foff[N]);
    for (int j = 0; j < f; ++j) {  // square (shared) -> packed lower triangle (global)
        const int64_t b = pk64(0, j, f);
        for (int i = j + threadIdx.x; i < f; i += DNT) F[b + i] = S[i + j * f];
    }
    if (threadIdx.x == 0 && bad) atomicExch(a.err + a.nd.slot[N], 1);
}

// Warp-per-front factorization of the smallest fronts: each warp of the CTA
// owns one front, stored as a packed lower triangle (column-major) in its
// own slice of shared memory, and runs the whole partial factorization with
// __syncwarp only: diagonal blocks in registers (lane = row), TRSM with one
// lane per row, trailing updates in 4x4 register tiles. The result goes to
// the front's full-square storage (lower part) for the parent and the solves.
__device__ __forceinline__ int pk(int i, int j, int f) { return j * (2 * f - j - 1) / 2 + i; }

template <class T, int WB>
__global__ void __launch_bounds__(256) k_factor_warp(FacArgs a, const int32_t* __restrict__ gstart,
                                                     const int32_t* __restrict__ wsoff) {
    extern __shared__ __align__(16) unsigned char dsm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // a.list is the whole node list here; group blockIdx.x holds the list
    // positions [gstart[g], gstart[g + 1]), one per warp, each with its own
    // slice of the CTA's shared memory (sized by the front, not by the list)
    const int idx = gstart[blockIdx.x] + warp;
    if (idx >= gstart[blockIdx.x + 1]) return;
    const int N = a.list[idx];
    const int s = a.nd.npiv[N];
    const int nu = a.ucnt[N];
    const int f = s + nu;
    const int64_t pf = a.pfirst[N];
    unsigned char* base = dsm + wsoff[idx];
    T* S = reinterpret_cast<T*>(base);
    const int np = f * (f + 1) / 2;
    int32_t* Us = reinterpret_cast<int32_t*>(S + np);
    int32_t* rel = Us + nu;
    for (int i = lane; i < np; i += 32) S[i] = zero_t<T>();
    for (int i = lane; i < nu; i += 32) Us[i] = a.upool[a.ustart[N] + i];
    __syncwarp();
    for (int k = lane; k < s; k += 32) S[pk(k, k, f)] = from_c<T>(make_double2(1.0, 0.0));
    {
        const int64_t q1 = a.eptr[pf + s];
        for (int64_t q = a.eptr[pf] + lane; q < q1; q += 32) {
            const int k = (int)(a.erow[q] - pf);
            const int i = front_pos(a.ecol[q], pf, s, Us, nu);
            S[pk(i, k, f)] = cj(from_c<T>(a.eval[q]));
        }
    }
    __syncwarp();
    const int ch[2] = {a.nd.chA[N], a.nd.chB[N]};
    for (int c = 0; c < 2; ++c) {
        const int C = ch[c];
        if (C < 0) continue;
        const int sc = a.nd.npiv[C], uc = a.ucnt[C], fc = sc + uc;
        const int32_t* UC = a.upool + a.ustart[C];
        for (int i = lane; i < uc; i += 32) rel[i] = front_pos(UC[i], pf, s, Us, nu);
        __syncwarp();
        const bool ccx = a.ntype[C] != 0;
        const double* FC = reinterpret_cast<const double*>(a.fpool) + a.foff[C];
        const int tot = uc * uc;
        constexpr int BAT = 8;  // independent loads in flight per lane
        for (int t0 = lane; t0 < tot; t0 += 32 * BAT) {
            double2 v[BAT];
            int pos[BAT];
#pragma unroll
            for (int q = 0; q < BAT; ++q) {
                const int t = t0 + 32 * q;
                const int bcol = t / uc, i = t - bcol * uc;
                const bool ok = t < tot && i >= bcol;
                pos[q] = ok ? pk(rel[i], rel[bcol], f) : -1;
                const int64_t e = pk64(sc + i, sc + bcol, fc);
                v[q] = !ok ? make_double2(0.0, 0.0)
                           : (ccx ? reinterpret_cast<const double2*>(FC)[e] : make_double2(FC[e], 0.0));
            }
#pragma unroll
            for (int q = 0; q < BAT; ++q)
                if (pos[q] >= 0) S[pos[q]] = add(S[pos[q]], narrow<T>(v[q]));
        }
        __syncwarp();
    }
    int bad = 0;
    for (int k0 = 0; k0 < s; k0 += WB) {
        const int nb = min(WB, s - k0);
        {   // diagonal block: lane i keeps row i
            T r[WB];
#pragma unroll
            for (int j = 0; j < WB; ++j) r[j] = (lane < nb && j < nb && j <= lane) ? S[pk(k0 + lane, k0 + j, f)] : zero_t<T>();
#pragma unroll
            for (int k = 0; k < WB; ++k) {
                if (k < nb) {
                    double d = re(shfl_t(r[k], k));
                    if (!(d > 0.0) || !isfinite(d)) {
                        bad = 1;
                        d = 1.0;
                    }
                    const double inv = rsqrt(d);
                    if (lane == k) r[k] = from_c<T>(make_double2(d * inv, 0.0));
                    else if (lane > k) r[k] = scale(r[k], inv);
#pragma unroll
                    for (int j = k + 1; j < WB; ++j) {
                        const T ljk = shfl_t(r[k], j);
                        if (lane >= j && j < nb) fma_cj(r[j], scale(r[k], -1.0), ljk);
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < WB; ++j)
                if (lane < nb && j <= lane) S[pk(k0 + lane, k0 + j, f)] = r[j];
        }
        __syncwarp();
        double di[WB];
#pragma unroll
        for (int k = 0; k < WB; ++k) di[k] = k < nb ? 1.0 / re(S[pk(k0 + k, k0 + k, f)]) : 0.0;
        for (int rr = k0 + nb + lane; rr < f; rr += 32) {
            T x[WB];
#pragma unroll
            for (int k = 0; k < WB; ++k) x[k] = k < nb ? S[pk(rr, k0 + k, f)] : zero_t<T>();
#pragma unroll
            for (int k = 0; k < WB; ++k) {
                if (k < nb) {
                    T v = x[k];
#pragma unroll
                    for (int j = 0; j < WB; ++j)
                        if (j < k) fma_cj(v, scale(x[j], -1.0), S[pk(k0 + k, k0 + j, f)]);
                    x[k] = scale(v, di[k]);
                }
            }
#pragma unroll
            for (int k = 0; k < WB; ++k)
                if (k < nb) S[pk(rr, k0 + k, f)] = x[k];
        }
        __syncwarp();
        const int c0 = k0 + nb, m = f - c0;
        if (m > 0) {
            const int nt = (m + 3) >> 2;
            const int ntiles = nt * (nt + 1) / 2;
            for (int t = lane; t < ntiles; t += 32) {
                int ti = (int)((sqrtf(8.0f * (float)t + 1.0f) - 1.0f) * 0.5f);
                while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
                while (ti * (ti + 1) / 2 > t) --ti;
                const int tj = t - ti * (ti + 1) / 2;
                const int rb = c0 + 4 * ti, cb = c0 + 4 * tj;
                T acc[4][4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = zero_t<T>();
                for (int k = 0; k < nb; ++k) {
                    const T* colk = S + pk(0, k0 + k, f);
                    T av[4], bv[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) av[i] = rb + i < f ? colk[rb + i] : zero_t<T>();
#pragma unroll
                    for (int j = 0; j < 4; ++j) bv[j] = cb + j < f ? colk[cb + j] : zero_t<T>();
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) fma_cj(acc[i][j], av[i], bv[j]);
                }
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int r = rb + i, c = cb + j;
                        if (r < f && c < f && r >= c) {
                            T& d = S[pk(r, c, f)];
                            d = sub(d, acc[i][j]);
                        }
                    }
            }
        }
        __syncwarp();
    }
    T* F = front_ptr<T>(a.fpool, a.foff[N]);
    for (int t = lane; t < np; t += 32) F[t] = S[t];  // same packed layout
    bad = __any_sync(FULL, bad);
    if (lane == 0 && bad) atomicExch(a.err + a.nd.slot[N], 1);
}

// Schur update of the U block of every front of a level, one CTA per lower
// 64x64 tile (blockIdx.y = tile index within the front)
template <class T>
__global__ void __launch_bounds__(DNT, sizeof(T) == 8 ? 8 : 4) k_schur(FacArgs a) {
    __shared__ __align__(16) T As[KC * TR];
    __shared__ __align__(16) T Bs[KC * TC];
    const int N = a.list[blockIdx.x];
    const int s = a.nd.npiv[N];
    const int nu = a.ucnt[N];
    if (s == 0 || nu == 0) return;
    int p = blockIdx.y;
    int tj = 0;
    for (; tj < nu; tj += TC) {
        const int nr = (nu - tj + TR - 1) / TR;
        if (p < nr) break;
        p -= nr;
    }
    if (tj >= nu) return;
    const int f = s + nu;
    T* F = front_ptr<T>(a.fpool, a.foff[N]);
    tile_one<T>(F, f, s + tj + TR * p, s + tj, f, f, 0, s, As, Bs);
}

// ---------------------------------------------------------------------------
// solves

struct SolArgs {
    NodeArrays nd;
    const int64_t* pfirst;
    const int32_t* perm;
    const int32_t* urow;
    const int32_t* ucnt;
    const int64_t* ustart;
    const int32_t* upool;
    const int64_t* foff;
    const int64_t* woff;
    const void* fpool;
    const int32_t* list;  // the fronts of one launch (one level, one type)
    double2* W;   // per front partial sums (forward)
    double2* X;   // elimination order: y after the forward sweep, x after the backward one
    const double2* b;
};

constexpr int SB = 32;  // pivots per block of the blocked substitutions

// TMA bulk prefetch of a byte range into L2 (no registers, no completion to
// wait for): a front's pivot columns, issued as soon as the front is known,
// so the column loads that follow hit L2 instead of HBM
__device__ __forceinline__ void l2_prefetch(const void* p, int64_t bytes) {
    uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)15;
    int64_t n = (int64_t)((reinterpret_cast<uintptr_t>(p) + bytes - a0) & ~(uintptr_t)15);  // rounded down
    while (n > 0) {
        const uint32_t c = (uint32_t)min(n, (int64_t)(1 << 20));
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"(c) : "memory");
        a0 += c;
        n -= c;
    }
}
// the pivot columns of front N: s (2f - s + 1) / 2 entries from its start
__device__ __forceinline__ void prefetch_panel(const SolArgs& a, int N, bool cplx) {
    const int s = a.nd.npiv[N], f = s + a.ucnt[N];
    const int64_t n = (int64_t)s * (2 * f - s + 1) / 2;
    if (cplx) l2_prefetch(front_ptr<double2>(a.fpool, a.foff[N]), n * (int64_t)sizeof(double2));
    else l2_prefetch(front_ptr<double>(a.fpool, a.foff[N]), n * (int64_t)sizeof(double));
}
// right-hand side into elimination order: X[e] = b[row of e] (the forward
// step of a front then reads its pivots' entries contiguously)
__global__ void k_perm_rhs(int64_t NU, const int32_t* __restrict__ perm, const int32_t* __restrict__ urow,
                           const double2* __restrict__ b, double2* __restrict__ X) {
    GRID_STRIDE(e, NU) X[e] = b[urow[perm[e]]];
}


// Forward step of front N (CTA-wide): gather the pivots' right-hand side and
// the children's partial sums (fixed order; L2 loads: written by other CTAs
// of the same persistent launch), blocked substitution with L_PP (one warp
// per 32-pivot diagonal block, shuffles), GEMV for the rows below; W[N] and
// the pivots' y in X.
template <class T>
__device__ void fwd_front(const SolArgs& a, int N, unsigned char* dsm, T* Lb) {
    double2* w = reinterpret_cast<double2*>(dsm);
    __shared__ double dvi[SB];
    const int s = a.nd.npiv[N];
    const int nu = a.ucnt[N];
    const int f = s + nu;
    const int64_t pf = a.pfirst[N];
    int32_t* Us = reinterpret_cast<int32_t*>(w + f);
    for (int i = threadIdx.x; i < nu; i += DNT) Us[i] = a.upool[a.ustart[N] + i];
    for (int k = threadIdx.x; k < f; k += DNT)
        w[k] = k < s ? a.X[pf + k] : make_double2(0.0, 0.0);  // b in elimination order (k_perm_rhs)
    __syncthreads();
    const int ch[2] = {a.nd.chA[N], a.nd.chB[N]};
    for (int c = 0; c < 2; ++c) {
        const int C = ch[c];
        if (C < 0) continue;
        const int sc = a.nd.npiv[C], uc = a.ucnt[C];
        const int32_t* UC = a.upool + a.ustart[C];
        const double2* WC = a.W + a.woff[C] + sc;
        for (int i = threadIdx.x; i < uc; i += DNT) {
            const int p = front_pos(UC[i], pf, s, Us, nu);
            const double2 v = __ldcg(WC + i);
            w[p].x += v.x;
            w[p].y += v.y;
        }
        __syncthreads();
    }
    const T* F = front_ptr<T>(a.fpool, a.foff[N]);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ int64_t coff[SB];  // pk64(0, k0 + k, f): column starts of the block
    for (int k0 = 0; k0 < s; k0 += SB) {
        const int nb = min(SB, s - k0);
        if (threadIdx.x < SB) coff[threadIdx.x] = pk64(0, k0 + min((int)threadIdx.x, nb - 1), f);
        __syncthreads();
        for (int idx = threadIdx.x; idx < SB * SB; idx += DNT) {
            const int i = idx % SB, j = idx / SB;
            Lb[idx] = (i < nb && j < nb && i >= j) ? F[coff[j] + k0 + i] : zero_t<T>();
        }
        __syncthreads();
        if (threadIdx.x < nb) dvi[threadIdx.x] = 1.0 / re(Lb[threadIdx.x + threadIdx.x * SB]);
        __syncthreads();
        if (warp == 0) {  // lane i holds w[k0 + i]
            double2 wi = lane < nb ? w[k0 + lane] : make_double2(0.0, 0.0);
            for (int k = 0; k < nb; ++k) {
                const double2 wk = make_double2(__shfl_sync(FULL, wi.x, k), __shfl_sync(FULL, wi.y, k));
                const double2 yk = make_double2(wk.x * dvi[k], wk.y * dvi[k]);
                if (lane == k) {
                    wi = yk;
                } else if (lane > k && lane < nb) {
                    const double2 t = vmul(Lb[lane + k * SB], yk);
                    wi.x -= t.x;
                    wi.y -= t.y;
                }
            }
            if (lane < nb) w[k0 + lane] = wi;
        }
        __syncthreads();
        for (int i = k0 + nb + threadIdx.x; i < f; i += DNT) {
            double2 acc = w[i];
            for (int kc = 0; kc < nb; kc += 16) {  // 16 loads in flight, then the FMAs
                T l[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) l[k] = kc + k < nb ? F[coff[kc + k] + i] : zero_t<T>();
#pragma unroll
                for (int k = 0; k < 16; ++k)
                    if (kc + k < nb) {
                        const double2 t = vmul(l[k], w[k0 + kc + k]);
                        acc.x -= t.x;
                        acc.y -= t.y;
                    }
            }
            w[i] = acc;
        }
        __syncthreads();
    }
    double2* WN = a.W + a.woff[N];
    for (int i = threadIdx.x; i < f; i += DNT) {
        WN[i] = w[i];
        if (i < s) a.X[pf + i] = w[i];
    }
}

// Backward step of front N: t = y_P - L_UP^H x_U (one warp per pivot column;
// the ancestors' x through L2), then the blocked back substitution with L_PP^H.
template <class T>
__device__ void bwd_front(const SolArgs& a, int N, unsigned char* dsm, T* Lb) {
    double2* t = reinterpret_cast<double2*>(dsm);   // [s] right-hand sides, then x
    __shared__ double dvi[SB];
    const int s = a.nd.npiv[N];
    const int nu = a.ucnt[N];
    const int f = s + nu;
    if (s == 0) return;
    const int64_t pf = a.pfirst[N];
    double2* xu = t + s;                            // [nu] ancestors' x
    const int32_t* U = a.upool + a.ustart[N];
    for (int i = threadIdx.x; i < nu; i += DNT) xu[i] = __ldcg(a.X + U[i]);
    __syncthreads();
    const T* F = front_ptr<T>(a.fpool, a.foff[N]);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int k = warp; k < s; k += DNT / 32) {
        const T* colk = F + pk64(0, k, f) + s;  // column k, rows s..f-1
        double sx = 0.0, sy = 0.0;
#pragma unroll 4
        for (int q = lane; q < nu; q += 32) {
            const double2 v = vmul_cj(colk[q], xu[q]);
            sx += v.x;
            sy += v.y;
        }
        sx = warp_sum(sx);
        sy = warp_sum(sy);
        if (lane == 0) {
            const double2 y = a.X[pf + k];
            t[k] = make_double2(y.x - sx, y.y - sy);
        }
    }
    __syncthreads();
    for (int k1 = s; k1 > 0; k1 -= SB) {
        const int k0 = max(0, k1 - SB), nb = k1 - k0;
        for (int idx = threadIdx.x; idx < SB * SB; idx += DNT) {
            const int i = idx % SB, j = idx / SB;
            Lb[idx] = (i < nb && j < nb && i >= j) ? F[pk64(k0 + i, k0 + j, f)] : zero_t<T>();
        }
        __syncthreads();
        if (threadIdx.x < nb) dvi[threadIdx.x] = 1.0 / re(Lb[threadIdx.x + threadIdx.x * SB]);
        __syncthreads();
        if (warp == 0) {  // lane i holds t[k0 + i]
            double2 ti = lane < nb ? t[k0 + lane] : make_double2(0.0, 0.0);
            for (int k = nb - 1; k >= 0; --k) {
                const double2 tk = make_double2(__shfl_sync(FULL, ti.x, k), __shfl_sync(FULL, ti.y, k));
                const double2 xk = make_double2(tk.x * dvi[k], tk.y * dvi[k]);
                if (lane == k) {
                    ti = xk;
                } else if (lane < k) {  // t_i -= conj(L[k][i]) x_k
                    const double2 v = vmul_cj(Lb[k + lane * SB], xk);
                    ti.x -= v.x;
                    ti.y -= v.y;
                }
            }
            if (lane < nb) t[k0 + lane] = ti;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < k0; i += DNT) {
            double2 acc = t[i];
            const T* rowi = F + pk64(0, i, f) + k0;  // column i of L: entries L[k][i], k in the block
            for (int kc = 0; kc < nb; kc += 16) {  // 16 loads in flight, then the FMAs
                T l[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) l[k] = kc + k < nb ? rowi[kc + k] : zero_t<T>();
#pragma unroll
                for (int k = 0; k < 16; ++k)
                    if (kc + k < nb) {
                        const double2 v = vmul_cj(l[k], t[k0 + kc + k]);
                        acc.x -= v.x;
                        acc.y -= v.y;
                    }
            }
            t[i] = acc;
        }
        __syncthreads();
    }
    for (int k = threadIdx.x; k < s; k += DNT) a.X[pf + k] = t[k];
}

// per-level launches (PGCP_DIRECT_PERSIST=0)
template <class T>
__global__ void __launch_bounds__(DNT) k_fwd(SolArgs a) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ __align__(16) T Lb[SB * SB];
    fwd_front<T>(a, a.list[blockIdx.x], dsm, Lb);
}
template <class T>
__global__ void __launch_bounds__(DNT) k_bwd(SolArgs a) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ __align__(16) T Lb[SB * SB];
    bwd_front<T>(a, a.list[blockIdx.x], dsm, Lb);
}

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// spin until *flag != 0; gives up after 2 s (flags the solve instead of hanging)
__device__ __forceinline__ void wait_flag(const int* flag, int* err) {
    if (ld_acquire_gpu(flag)) return;
    const unsigned long long t0 = gtimer();
    while (!ld_acquire_gpu(flag)) {
        __nanosleep(64);
        if (gtimer() - t0 > 2000000000ull) {
            atomicExch(err, 1);
            return;
        }
    }
}

// One persistent launch per sweep. CTAs draw fronts from a ticket counter in
// `order` (leaves first for the forward sweep, read backwards for the
// backward one) and wait for the fronts they depend on (children / parent),
// whose tickets are smaller and so held by CTAs already running: no level
// barriers, no per-level launches, real and complex fronts in one launch.
// skip: fronts with id < skip are not solved (the loops' fronts in the
// interior-only solve: their x stays 0, set beforehand)
__global__ void __launch_bounds__(DNT, 6) k_solve_pers(SolArgs a, const int32_t* __restrict__ order, int nn,
                                                    int* __restrict__ done, int* ticket,
                                                    const int8_t* __restrict__ ntype, int backward, int skip,
                                                    unsigned long long* __restrict__ trace) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ __align__(16) double2 Lb[SB * SB];
    __shared__ int sq;
    unsigned long long tr0 = 0, tr1 = 0;
    for (;;) {
        if (threadIdx.x == 0) sq = atomicAdd(ticket, 1);
        __syncthreads();
        const int q = sq;
        __syncthreads();
        if (q >= nn) return;
        const int N = backward ? order[nn - 1 - q] : order[q];
        if (N < skip) {
            if (threadIdx.x == 0) st_release_gpu(done + N, 1);
            continue;
        }
        if (threadIdx.x == 0) {
            if (trace) tr0 = gtimer();
            if (backward) {
                const int P = a.nd.parent[N];
                if (P >= 0) wait_flag(done + P, ticket - 1);
            } else {
                const int A = a.nd.chA[N], B = a.nd.chB[N];
                if (A >= 0) wait_flag(done + A, ticket - 1);
                if (B >= 0) wait_flag(done + B, ticket - 1);
            }
            prefetch_panel(a, N, ntype[N] != 0);
            if (trace) tr1 = gtimer();
        }
        __syncthreads();
        if (backward) {
            if (ntype[N]) bwd_front<double2>(a, N, dsm, Lb);
            else bwd_front<double>(a, N, dsm, reinterpret_cast<double*>(Lb));
        } else {
            if (ntype[N]) fwd_front<double2>(a, N, dsm, Lb);
            else fwd_front<double>(a, N, dsm, reinterpret_cast<double*>(Lb));
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
            st_release_gpu(done + N, 1);
            if (trace) {
                trace[3 * N] = tr0;
                trace[3 * N + 1] = tr1;
                trace[3 * N + 2] = gtimer();
            }
        }
    }
}

// ---- warp-per-front substitutions for the small fronts (the deep levels:
// tens of thousands of fronts with f <= SW_F rows, s <= SW_S pivots). One
// warp owns a front: no CTA barriers, 4 warps of a CTA on 4 fronts, every
// resident warp of the GPU on its own front. L columns are read SWC at a
// time with every load of the chunk in flight before the chain consumes
// them (one memory round trip per chunk instead of one per pivot).
constexpr int SW_NS = 4;             // rows per lane (forward)
constexpr int SW_F = 32 * SW_NS;     // largest front on the warp path
constexpr int SW_NP = 2;             // pivot columns per lane (backward)
constexpr int SW_S = 32 * SW_NP;     // most pivots on the warp path
constexpr int SWC = 4;               // columns per chunk (forward chain)
constexpr int SWQ = 8;               // update rows per chunk (backward GEMV)
constexpr int SWK = 8;               // chain steps per chunk (backward)

// Forward step by one warp: lane l holds rows l, l+32, ... of w in registers;
// column k of L (rows k..f-1, contiguous in the packed front) is one
// coalesced load per slot; y_k is broadcast from the owner lane.
template <class T>
__device__ void fwd_front_w(const SolArgs& a, int N, double2* w, int32_t* Us, int lane) {
    const int s = a.nd.npiv[N];
    const int nu = a.ucnt[N];
    const int f = s + nu;
    const int64_t pf = a.pfirst[N];
    const int32_t* U = a.upool + a.ustart[N];
    for (int i = lane; i < nu; i += 32) Us[i] = U[i];
    for (int k = lane; k < f; k += 32) w[k] = k < s ? a.X[pf + k] : make_double2(0.0, 0.0);
    __syncwarp();
    {   // both children's partial sums: loads of both issued together, then
        // added in fixed order (A, then B) for bitwise-repeatable results
        const int A = a.nd.chA[N], B = a.nd.chB[N];
        const int ua = A >= 0 ? a.ucnt[A] : 0, ub = B >= 0 ? a.ucnt[B] : 0;
        const int32_t* UA = A >= 0 ? a.upool + a.ustart[A] : nullptr;
        const int32_t* UB = B >= 0 ? a.upool + a.ustart[B] : nullptr;
        const double2* WA = A >= 0 ? a.W + a.woff[A] + a.nd.npiv[A] : nullptr;
        const double2* WB = B >= 0 ? a.W + a.woff[B] + a.nd.npiv[B] : nullptr;
        const int um = max(ua, ub);
        for (int i0 = 0; i0 < um; i0 += 32) {
            const int i = i0 + lane;
            int pa = -1, pb = -1;
            double2 va = make_double2(0.0, 0.0), vb = va;
            if (i < ua) {
                pa = UA[i];
                va = __ldcg(WA + i);
            }
            if (i < ub) {
                pb = UB[i];
                vb = __ldcg(WB + i);
            }
            if (pa >= 0) {
                const int p = front_pos(pa, pf, s, Us, nu);
                w[p].x += va.x;
                w[p].y += va.y;
            }
            __syncwarp();
            if (pb >= 0) {
                const int p = front_pos(pb, pf, s, Us, nu);
                w[p].x += vb.x;
                w[p].y += vb.y;
            }
            __syncwarp();
        }
    }
    double2 r[SW_NS];
#pragma unroll
    for (int j = 0; j < SW_NS; ++j) {
        const int i = lane + 32 * j;
        r[j] = i < f ? w[i] : make_double2(0.0, 0.0);
    }
    const T* F = front_ptr<T>(a.fpool, a.foff[N]);
    int64_t col = 0;  // pk64(0, k, f): column k starts at col + k
    for (int k0 = 0; k0 < s; k0 += SWC) {
        T l[SWC][SW_NS];
        int64_t cc = col;
#pragma unroll
        for (int c = 0; c < SWC; ++c) {
            const int k = k0 + c;
#pragma unroll
            for (int j = 0; j < SW_NS; ++j) {
                const int i = lane + 32 * j;
                l[c][j] = (k < s && i >= k && i < f) ? F[cc + i] : zero_t<T>();
            }
            cc += f - k - 1;
        }
        col = cc;
#pragma unroll
        for (int c = 0; c < SWC; ++c) {
            const int k = k0 + c;
            if (k >= s) break;
            const int jk = k >> 5, lk = k & 31;
            double2 v = r[0];
            double d = re(l[c][0]);
#pragma unroll
            for (int j = 1; j < SW_NS; ++j)
                if (j == jk) {
                    v = r[j];
                    d = re(l[c][j]);
                }
            const double dv = 1.0 / d;
            double2 y = make_double2(v.x * dv, v.y * dv);
            y.x = __shfl_sync(FULL, y.x, lk);
            y.y = __shfl_sync(FULL, y.y, lk);
#pragma unroll
            for (int j = 0; j < SW_NS; ++j) {
                const int i = lane + 32 * j;
                if (i == k) {
                    r[j] = y;
                } else if (i > k && i < f) {
                    const double2 t = vmul(l[c][j], y);
                    r[j].x -= t.x;
                    r[j].y -= t.y;
                }
            }
        }
    }
    double2* WN = a.W + a.woff[N];
#pragma unroll
    for (int j = 0; j < SW_NS; ++j) {
        const int i = lane + 32 * j;
        if (i < f) {
            WN[i] = r[j];
            if (i < s) a.X[pf + i] = r[j];
        }
    }
}

// Backward step by one warp: lane l owns pivot columns l, l+32 (x_k and its
// running right-hand side). The update rows' contribution is a per-lane walk
// down the lane's own column (no reductions); the chain k = s-1..0 then
// broadcasts x_k and every lane i < k subtracts conj(L[k][i]) x_k.
template <class T>
__device__ void bwd_front_w(const SolArgs& a, int N, double2* xs, int lane) {
    const int s = a.nd.npiv[N];
    if (s == 0) return;
    const int nu = a.ucnt[N];
    const int f = s + nu;
    const int64_t pf = a.pfirst[N];
    const int32_t* U = a.upool + a.ustart[N];
    for (int i = lane; i < nu; i += 32) xs[i] = __ldcg(a.X + U[i]);
    __syncwarp();
    const T* F = front_ptr<T>(a.fpool, a.foff[N]);
    double2 acc[SW_NP];
    int64_t ck[SW_NP];
#pragma unroll
    for (int j = 0; j < SW_NP; ++j) {
        const int k = lane + 32 * j;
        ck[j] = pk64(0, min(k, max(s - 1, 0)), f);
        acc[j] = k < s ? a.X[pf + k] : make_double2(0.0, 0.0);
    }
    double dinv[SW_NP];
#pragma unroll
    for (int j = 0; j < SW_NP; ++j) {
        const int k = lane + 32 * j;
        dinv[j] = k < s ? 1.0 / re(F[ck[j] + k]) : 0.0;
    }
    for (int q0 = 0; q0 < nu; q0 += SWQ) {
        T l[SWQ][SW_NP];
#pragma unroll
        for (int q = 0; q < SWQ; ++q)
#pragma unroll
            for (int j = 0; j < SW_NP; ++j)
                l[q][j] = (q0 + q < nu && lane + 32 * j < s) ? F[ck[j] + s + q0 + q] : zero_t<T>();
#pragma unroll
        for (int q = 0; q < SWQ; ++q) {
            if (q0 + q >= nu) break;
            const double2 xq = xs[q0 + q];
#pragma unroll
            for (int j = 0; j < SW_NP; ++j) {
                const double2 t = vmul_cj(l[q][j], xq);
                acc[j].x -= t.x;
                acc[j].y -= t.y;
            }
        }
    }
    for (int k1 = s; k1 > 0; k1 -= SWK) {
        T l[SWK][SW_NP];  // l[c][j] = L[k1-1-c][lane + 32 j]
#pragma unroll
        for (int c = 0; c < SWK; ++c)
#pragma unroll
            for (int j = 0; j < SW_NP; ++j) {
                const int k = k1 - 1 - c, i = lane + 32 * j;
                l[c][j] = (k >= 0 && i < k) ? F[ck[j] + k] : zero_t<T>();
            }
#pragma unroll
        for (int c = 0; c < SWK; ++c) {
            const int k = k1 - 1 - c;
            if (k < 0) break;
            const int jk = k >> 5, lk = k & 31;
            double2 v = acc[0];
            double dv = dinv[0];
#pragma unroll
            for (int j = 1; j < SW_NP; ++j)
                if (j == jk) {
                    v = acc[j];
                    dv = dinv[j];
                }
            double2 x = make_double2(v.x * dv, v.y * dv);
            x.x = __shfl_sync(FULL, x.x, lk);
            x.y = __shfl_sync(FULL, x.y, lk);
#pragma unroll
            for (int j = 0; j < SW_NP; ++j) {
                const int i = lane + 32 * j;
                if (i == k) {
                    acc[j] = x;
                } else if (i < k) {
                    const double2 t = vmul_cj(l[c][j], x);
                    acc[j].x -= t.x;
                    acc[j].y -= t.y;
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < SW_NP; ++j) {
        const int k = lane + 32 * j;
        if (k < s) a.X[pf + k] = acc[j];
    }
}

// persistent warp-per-front sweep over order[0, nn) (forward) or its reverse
// (backward); the same ticket / done-flag protocol as k_solve_pers, per warp
template <bool backward, int MINB>
__global__ void __launch_bounds__(DNT, MINB) k_solve_warp(SolArgs a, const int32_t* __restrict__ order, int nn,
                                                    int* __restrict__ done, int* ticket,
                                                    const int8_t* __restrict__ ntype, int skip,
                                                    unsigned long long* __restrict__ trace) {
    __shared__ __align__(16) double2 wbuf[DNT / 32][SW_F];
    __shared__ int32_t ubuf[DNT / 32][SW_F];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (;;) {
        int q = 0;
        if (lane == 0) q = atomicAdd(ticket, 1);
        q = __shfl_sync(FULL, q, 0);
        if (q >= nn) return;
        const int N = backward ? order[nn - 1 - q] : order[q];
        if (N < skip) {
            if (lane == 0) st_release_gpu(done + N, 1);
            continue;
        }
        unsigned long long tr0 = 0, tr1 = 0;
        if (lane == 0) {
            if (trace) tr0 = gtimer();
            if (backward) {
                const int P = a.nd.parent[N];
                if (P >= 0) wait_flag(done + P, ticket - 1);
            } else {
                const int A = a.nd.chA[N], B = a.nd.chB[N];
                if (A >= 0) wait_flag(done + A, ticket - 1);
                if (B >= 0) wait_flag(done + B, ticket - 1);
            }
            prefetch_panel(a, N, ntype[N] != 0);
            if (trace) tr1 = gtimer();
        }
        __syncwarp();
        if (backward) {
            if (ntype[N]) bwd_front_w<double2>(a, N, wbuf[warp], lane);
            else bwd_front_w<double>(a, N, wbuf[warp], lane);
        } else {
            if (ntype[N]) fwd_front_w<double2>(a, N, wbuf[warp], ubuf[warp], lane);
            else fwd_front_w<double>(a, N, wbuf[warp], ubuf[warp], lane);
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) {
            st_release_gpu(done + N, 1);
            if (trace) {
                trace[3 * N] = tr0;
                trace[3 * N + 1] = tr1;
                trace[3 * N + 2] = gtimer();
            }
        }
    }
}

__global__ void k_d_scatter(int64_t NU, const int32_t* __restrict__ urow, const int32_t* __restrict__ elim,
                            const double2* __restrict__ X, double2* __restrict__ x) {
    GRID_STRIDE(u, NU) x[urow[u]] = X[elim[u]];
}

int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}

// k_factor_warp CTA: up to 8 warps share this much dynamic shared memory (real
// fronts: three CTAs per SM at 80 registers; complex: two at 125); tunable for sweeps
inline size_t warp_cta_bytes(size_t tsz) {
    const int kb = env_int(tsz == 8 ? "PGCP_DIRECT_WCTA_KB" : "PGCP_DIRECT_WCTA_KB_C", tsz == 8 ? 75 : 112);
    return (size_t)std::max(40, std::min(kb, 220)) * 1024;  // at least one WARP_FRONT_BYTES front
}
// warps (= fronts) per k_factor_warp CTA
inline int warp_cta_warps() { return std::max(1, std::min(8, env_int("PGCP_DIRECT_WCTA_W", 8))); }

// PGCP_DIRECT_TIMING=1: CUDA-event split of the phases (and the host time
// between the marks), printed to stderr
struct PhaseTimer {
    bool on = false;
    cudaStream_t s = nullptr;
    std::vector<std::pair<const char*, cudaEvent_t>> ev;
    std::vector<double> host;
    explicit PhaseTimer(cudaStream_t st) : on(getenv("PGCP_DIRECT_TIMING") != nullptr), s(st) { mark("start"); }
    void mark(const char* name) {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        ev.push_back({name, e});
        host.push_back(1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count());
    }
    ~PhaseTimer() {
        if (!on) return;
        cudaEventSynchronize(ev.back().second);
        fprintf(stderr, "[direct timing]");
        for (size_t i = 1; i < ev.size(); ++i) {
            float ms = 0;
            cudaEventElapsedTime(&ms, ev[i - 1].second, ev[i].second);
            fprintf(stderr, " %s %.3f", ev[i].first, ms);
        }
        fprintf(stderr, " (ms)\n[direct host]  ");
        for (size_t i = 1; i < ev.size(); ++i) fprintf(stderr, " %s %.3f", ev[i].first, host[i] - host[i - 1]);
        fprintf(stderr, " (ms)\n");
        for (auto& p : ev) cudaEventDestroy(p.second);
    }
};


}  // namespace

// ---------------------------------------------------------------------------
// Workspace cache for the large per-factorization buffers (front storage,
// update sets, forward partial sums: GBs at cfg 2). Stream-ordered pool
// allocations of that size sometimes make the pool map new memory (ms of
// host time); these blocks are instead kept per process, grow-only, and
// handed out again after an event on the releasing stream (the acquiring
// stream waits on it).
struct WsSlot {
    int dev = -1;
    void* p = nullptr;
    size_t bytes = 0;
    bool busy = false;
    cudaEvent_t ready = nullptr;
};
static std::mutex g_ws_mu;
static std::vector<WsSlot> g_ws;
static long long g_ws_grows = 0;  // slot (re)allocations since load
static double g_ws_grow_ms = 0;   // host time spent in them (cudaFree + cudaMalloc)

static int ws_acquire(size_t bytes, cudaStream_t s, int* slot_out, void** p_out) {
    int dev = 0;
    PGCP_TRY_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_ws_mu);
    int best = -1;
    for (int i = 0; i < (int)g_ws.size(); ++i) {
        const WsSlot& w = g_ws[i];
        if (w.dev != dev || w.busy || w.bytes < bytes) continue;
        if (best < 0 || w.bytes < g_ws[best].bytes) best = i;
    }
    if (best < 0) {  // grow: a new slot while the cache stays under half the device memory, else evict an idle one
        size_t cached = 0, free_b = 0, total_b = 0;
        for (const WsSlot& w : g_ws)
            if (w.dev == dev) cached += w.bytes;
        PGCP_TRY_CUDA(cudaMemGetInfo(&free_b, &total_b));
        const bool room = cached + bytes + bytes * 3 / 10 <= total_b / 2;
        for (int i = 0; i < (int)g_ws.size() && best < 0 && !room; ++i)
            if (g_ws[i].dev == dev && !g_ws[i].busy) best = i;
        if (best < 0) {
            g_ws.push_back(WsSlot());
            best = (int)g_ws.size() - 1;
            g_ws[best].dev = dev;
        }
        WsSlot& w = g_ws[best];
        const auto t_grow = std::chrono::steady_clock::now();
        if (w.p) {
            if (w.ready) PGCP_TRY_CUDA(cudaEventSynchronize(w.ready));
            PGCP_TRY_CUDA(cudaFree(w.p));
            w.p = nullptr;
            w.bytes = 0;
        }
        // 30 % headroom: the flatten's and the Dirichlet system's buffers are
        // close in size and are acquired concurrently in either order
        const size_t want = std::max<size_t>(bytes + bytes * 3 / 10, 1 << 20);
        PGCP_TRY_CUDA(cudaMalloc(&w.p, want));
        w.bytes = want;
        ++g_ws_grows;
        g_ws_grow_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_grow).count();
        if (getenv("PGCP_DIRECT_TIMING")) {
            size_t cached = 0;
            int nsl = 0;
            for (const WsSlot& q : g_ws)
                if (q.dev == dev) cached += q.bytes, ++nsl;
            fprintf(stderr, "[direct workspace] slot %d sized %.3f GB (%d slots, %.2f GB cached)\n", best, 1e-9 * want,
                    nsl, 1e-9 * cached);
        }
    }
    WsSlot& w = g_ws[best];
    if (w.ready) PGCP_TRY_CUDA(cudaStreamWaitEvent(s, w.ready, 0));
    w.busy = true;
    *slot_out = best;
    *p_out = w.p;
    return PGCP_OK;
}

static void ws_release(int slot, cudaStream_t s) {
    std::lock_guard<std::mutex> lock(g_ws_mu);
    WsSlot& w = g_ws[slot];
    if (!w.ready) cudaEventCreateWithFlags(&w.ready, cudaEventDisableTiming);
    cudaEventRecord(w.ready, s);
    w.busy = false;
}

template <class T>
struct WsBuf {
    T* p = nullptr;
    int slot = -1;
    cudaStream_t s = nullptr;
    WsBuf() = default;
    WsBuf(const WsBuf&) = delete;
    WsBuf& operator=(const WsBuf&) = delete;
    ~WsBuf() { release(); }
    int alloc(int64_t n, cudaStream_t st) {
        release();
        void* q = nullptr;
        PGCP_TRY(ws_acquire((size_t)std::max<int64_t>(n, 1) * sizeof(T), st, &slot, &q));
        p = static_cast<T*>(q);
        s = st;
        return PGCP_OK;
    }
    void release() {
        if (slot >= 0) ws_release(slot, s);
        slot = -1;
        p = nullptr;
    }
};

struct DirectFactor {
    bool cplx = false;
    int32_t nslot = 0;
    int64_t NU = 0, rows = 0;
    std::vector<int64_t> h_uoff;
    DevBuf<int64_t> uoff;
    DevBuf<int32_t> urow, uslot;
    DevBuf<int64_t> aptr;
    DevBuf<int32_t> acol;
    DevBuf<double2> aval;
    DevBuf<int32_t> elim, perm;
    DevBuf<int64_t> eptr;
    DevBuf<int32_t> erow, ecol;
    DevBuf<double2> eval;
    // tree
    int32_t nnodes = 0;
    std::vector<std::pair<int32_t, int32_t>> levels;  // node id ranges, level 0 = roots
    DevBuf<int32_t> parent, chA, chB, cnt, npiv, slot, nchild;
    DevBuf<int8_t> leaf;
    DevBuf<uint32_t> bbox;
    DevBuf<int32_t> gcnt;
    DevBuf<float2> split;
    DevBuf<int64_t> pfirst;
    DevBuf<int32_t> ucnt, fsz;
    WsBuf<int32_t> upool;
    DevBuf<int64_t> ustart, foff, woff;
    WsBuf<unsigned char> fpool;
    WsBuf<double2> W;
    DevBuf<double2> X;
    DevBuf<int32_t> err;
    DevBuf<int8_t> ntype;
    bool boundary_last = false;   // level 0 = the loops' fronts (the interior block factors L_II)
    DevBuf<int32_t> rowel;        // system row -> elimination index (-1: padding)
    DevBuf<int32_t> order;   // fronts deepest level first (the persistent solves' ticket order)
    DevBuf<int32_t> sync;    // [0] ticket counter, [1 + N] front N done
    // fronts per (level, type): nlist[lst_off[2 l + t], lst_off[2 l + t + 1])
    DevBuf<int32_t> nlist;
    std::vector<int64_t> lst_off;
    std::vector<int> lst_maxs;               // per (level, type): largest pivot count
    std::vector<int> lst_maxf;               // ... largest front
    std::vector<int32_t> h_nlist, h_npiv, h_fsz, h_order;  // host copies (uploads stay async)
    // k_factor_warp groups: every list is sorted by front size (largest
    // first); the fronts small enough for one warp (from lst_wfirst on) are
    // packed, in that order, into CTAs of up to 8 fronts whose packed
    // triangles fill the CTA's shared memory -- so a CTA of leaf-sized fronts
    // runs 8 warps where a CTA of the list's largest fronts runs 2
    std::vector<int64_t> lst_wfirst;         // per (level, type): first list position handled by k_factor_warp
    std::vector<int64_t> grp_off;            // per (level, type): its groups are [grp_off[q], grp_off[q + 1])
    std::vector<int32_t> h_gstart, h_wsoff;  // group -> first list position (+ end sentinel per list); position -> smem offset
    DevBuf<int32_t> gstart, wsoff;
    std::vector<int> lvl_maxf, lvl_maxu;
    int ncplx = 0;
    std::vector<int32_t> h_err;
    double fmas = 0, factor_ms = 0, solve_ms = 0, front_bytes = 0, numeric_ms = 0;
    int maxf = 0;

    NodeArrays na() {
        NodeArrays n;
        n.parent = parent.p;
        n.chA = chA.p;
        n.chB = chB.p;
        n.cnt = cnt.p;
        n.npiv = npiv.p;
        n.slot = slot.p;
        n.leaf = leaf.p;
        n.bbox = bbox.p;
        n.gcnt = gcnt.p;
        n.split = split.p;
        n.nchild = nchild.p;
        return n;
    }
};

void direct_free(DirectFactor* F) { delete F; }

void direct_stats(const DirectFactor* F, double* o) {
    for (int i = 0; i < 9; ++i) o[i] = 0;
    if (!F) return;
    o[0] = F->nnodes;
    o[1] = (double)F->levels.size();
    o[2] = F->maxf;
    o[3] = F->fmas;
    o[4] = F->factor_ms;
    o[5] = F->solve_ms;
    o[6] = F->front_bytes;
    o[7] = (double)F->NU;
    o[8] = F->numeric_ms;
}

const std::vector<int32_t>& direct_slot_status(const DirectFactor* F) { return F->h_err; }

namespace {

// Dynamic shared-memory limit of a kernel: raised once to the most the
// kernel can take and never lowered. Concurrent solves (the flatten worker
// and the Dirichlet preparation) launch the same kernels with different
// sizes; a per-launch attribute could be lowered by one thread between the
// other's set and launch.
std::mutex g_smem_mu;
std::vector<const void*> g_smem_done;  // kernels whose limit is raised (keyed by entry point)
template <class K>
int set_smem(K kern, size_t bytes) {
    std::lock_guard<std::mutex> lock(g_smem_mu);
    const void* key = reinterpret_cast<const void*>(kern);
    if (std::find(g_smem_done.begin(), g_smem_done.end(), key) == g_smem_done.end()) {
        cudaFuncAttributes fa;
        PGCP_TRY_CUDA(cudaFuncGetAttributes(&fa, kern));
        const int cap = 227 * 1024 - (int)fa.sharedSizeBytes;
        PGCP_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, cap));
        g_smem_done.push_back(key);
    }
    if (bytes + 0 > (size_t)(227 * 1024)) {
        set_error("direct solver: %zu bytes of shared memory requested", bytes);
        return DIRECT_FALLBACK;
    }
    return PGCP_OK;
}

template <class T>
int factor_level(DirectFactor* D, FacArgs fa, int l, int type, cudaStream_t s) {
    const int64_t o0 = D->lst_off[2 * l + type];
    if (D->lst_off[2 * l + type + 1] <= o0) return PGCP_OK;
    fa.list = D->nlist.p + o0;
    const size_t tsz = sizeof(T);
    const int maxu_child = (l + 1 < (int)D->levels.size()) ? D->lvl_maxu[l + 1] : 0;
    const size_t smem = (KC * (TR + TC) + NB * NB) * tsz + (size_t)(D->lvl_maxu[l] + maxu_child) * 4 + 16;
    if (smem > 227 * 1024) {
        set_error("direct solver: front update set too large (%d)", D->lvl_maxu[l]);
        return DIRECT_FALLBACK;
    }
    // the fronts small enough for one warp each (the tail of the size-sorted
    // list), grouped into CTAs by packed size (see DirectFactor::grp_off)
    if (D->grp_off[2 * l + type + 1] > D->grp_off[2 * l + type]) {
        const int64_t g0 = D->grp_off[2 * l + type], g1 = D->grp_off[2 * l + type + 1];
        const int ng = (int)(g1 - g0) - 1;  // the list's last entry is its end sentinel
        FacArgs fw = fa;
        fw.list = D->nlist.p;
        const size_t cta = warp_cta_bytes(tsz);
        const int wbk = env_int("PGCP_DIRECT_WB", 8);
        if (wbk == 4) {
            PGCP_TRY(set_smem(k_factor_warp<T, 4>, cta));
            k_factor_warp<T, 4><<<ng, 32 * warp_cta_warps(), cta, s>>>(fw, D->gstart.p + g0, D->wsoff.p);
        } else if (wbk == 8) {
            PGCP_TRY(set_smem(k_factor_warp<T, 8>, cta));
            k_factor_warp<T, 8><<<ng, 32 * warp_cta_warps(), cta, s>>>(fw, D->gstart.p + g0, D->wsoff.p);
        } else {
            PGCP_TRY(set_smem(k_factor_warp<T, 16>, cta));
            k_factor_warp<T, 16><<<ng, 32 * warp_cta_warps(), cta, s>>>(fw, D->gstart.p + g0, D->wsoff.p);
        }
        PGCP_LAUNCH_CHECK();
    }
    // the larger fronts of the list: [o0, lst_wfirst)
    const int64_t o1 = D->lst_wfirst[2 * l + type];
    if (o1 <= o0) return PGCP_OK;
    const int n = (int)(o1 - o0);
    int maxf_t = 0, maxs = 0;
    for (int64_t q = o0; q < o1; ++q) {
        maxf_t = std::max(maxf_t, D->h_fsz[D->h_nlist[q]]);
        maxs = std::max(maxs, D->h_npiv[D->h_nlist[q]]);
    }
    {   // fronts that fit in shared memory: the resident kernel
        const size_t sm = (size_t)maxf_t * maxf_t * tsz + (size_t)(D->lvl_maxu[l] + maxu_child) * 4 + 16;
        if (sm <= SM_FRONT_BYTES && !getenv("PGCP_DIRECT_NO_SMEM")) {
            if (env_int("PGCP_DIRECT_SB", 8) == 8) {
                PGCP_TRY(set_smem(k_factor_sm<T, 8>, sm));
                k_factor_sm<T, 8><<<n, DNT, sm, s>>>(fa);
            } else {
                PGCP_TRY(set_smem(k_factor_sm<T, 16>, sm));
                k_factor_sm<T, 16><<<n, DNT, sm, s>>>(fa);
            }
            PGCP_LAUNCH_CHECK();
            return PGCP_OK;
        }
    }
    PGCP_TRY(set_smem(k_factor<T>, smem));
    const int nt = schur_tiles(D->lvl_maxu[l]);
    static const int fused_maxs = env_int("PGCP_DIRECT_FUSED_MAXS", FUSED_MAXS);
    if (maxs <= fused_maxs) {
        const bool inl = nt <= 1;
        k_factor<T><<<n, DNT, smem, s>>>(fa, inl ? FAC_SCHUR_INLINE : 0);
        PGCP_LAUNCH_CHECK();
    } else {
        {
            constexpr int CW = 8;
            const int maxf = D->lvl_maxf[l];
            const size_t sm1 = (size_t)D->lvl_maxu[l] * 4 + 16;
            const size_t sm2 = (size_t)(D->lvl_maxu[l] + maxu_child) * 4 + 16;
            PGCP_TRY(set_smem(k_asm_cols<T>, sm1));
            PGCP_TRY(set_smem(k_asm_child<T>, sm2));
            k_asm_cols<T><<<dim3(n, (maxf + CW - 1) / CW), DNT, sm1, s>>>(fa, CW);
            PGCP_LAUNCH_CHECK();
            for (int w = 0; w < 2; ++w) {
                k_asm_child<T><<<dim3(n, (std::max(maxu_child, 1) + CW - 1) / CW), DNT, sm2, s>>>(fa, w, CW);
                PGCP_LAUNCH_CHECK();
            }
        }
        const size_t xs = 0;
        for (int k0 = 0; k0 < maxs; k0 += PB) {
            int chunks = 1, tiles = 0;
            for (int64_t q = o0; q < o1; ++q) {
                const int N = D->h_nlist[q];
                const int sp = D->h_npiv[N], f = D->h_fsz[N];
                if (k0 >= sp) continue;
                const int nb = std::min(PB, sp - k0);
                chunks = std::max(chunks, (f - k0 - nb + DNT - 1) / DNT);
                tiles = std::max(tiles, pupd_tiles(sp, f, k0 + nb));
            }
            if (k0 == 0) {  // later diagonal blocks are factored by the previous k_pupd
                k_pdiag<T><<<dim3(n, 1), DNT, xs, s>>>(fa, k0, 0);
                PGCP_LAUNCH_CHECK();
            }
            k_pdiag<T><<<dim3(n, chunks), DNT, xs, s>>>(fa, k0, 1);
            PGCP_LAUNCH_CHECK();
            if (tiles > 0) {
                k_pupd<T><<<dim3(n, tiles), DNT, 0, s>>>(fa, k0);
                PGCP_LAUNCH_CHECK();
            }
        }
    }
    if (nt > 1 || (maxs > FUSED_MAXS && nt > 0)) {
        k_schur<T><<<dim3(n, nt), DNT, 0, s>>>(fa);
        PGCP_LAUNCH_CHECK();
    }
    return PGCP_OK;
}

int factor_levels(DirectFactor* D, FacArgs& fa, cudaStream_t s, PhaseTimer& pt) {
    static const char* names[] = {"L0", "L1", "L2", "L3", "L4", "L5", "L6", "L7", "L8", "L9", "L10", "L11",
                                  "L12", "L13", "L14", "L15", "L16", "L17", "L18", "L19", "L20+"};
    // The real and the complex fronts of a level are independent lists. On
    // the upper levels each is a chain of ~10 small dependent launches that
    // leaves most SMs idle, so the complex list runs on a second stream of
    // the same priority, forked and joined per level with events
    // (PGCP_DIRECT_TWO_STREAMS=0: one stream).
    const bool two = env_int("PGCP_DIRECT_TWO_STREAMS", 1) != 0;
    cudaStream_t s2 = nullptr;
    cudaEvent_t ef = nullptr, ej = nullptr;
    if (two && D->ncplx > 0 && D->ncplx < D->nnodes) {
        int prio = 0;
        PGCP_TRY_CUDA(cudaStreamGetPriority(s, &prio));
        PGCP_TRY_CUDA(cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, prio));
        PGCP_TRY_CUDA(cudaEventCreateWithFlags(&ef, cudaEventDisableTiming));
        PGCP_TRY_CUDA(cudaEventCreateWithFlags(&ej, cudaEventDisableTiming));
    }
    int rc = PGCP_OK;
    for (int l = (int)D->levels.size() - 1; l >= 0 && rc == PGCP_OK; --l) {
        const bool both = s2 && D->lst_off[2 * l + 1] > D->lst_off[2 * l] && D->lst_off[2 * l + 2] > D->lst_off[2 * l + 1];
        if (both) {
            if (cudaEventRecord(ef, s) != cudaSuccess || cudaStreamWaitEvent(s2, ef, 0) != cudaSuccess) rc = PGCP_E_CUDA;
        }
        if (rc == PGCP_OK) rc = factor_level<double>(D, fa, l, 0, s);
        if (rc == PGCP_OK) rc = factor_level<double2>(D, fa, l, 1, both ? s2 : s);
        if (both) {  // joined even after an error: nothing may outlive the aux stream unordered
            if (cudaEventRecord(ej, s2) != cudaSuccess || cudaStreamWaitEvent(s, ej, 0) != cudaSuccess) {
                if (rc == PGCP_OK) rc = PGCP_E_CUDA;
            }
        }
        pt.mark(names[std::min(l, 20)]);
    }
    if (s2) {
        cudaEventDestroy(ef);
        cudaEventDestroy(ej);
        cudaStreamDestroy(s2);  // its work is ordered before s by the last join
    }
    if (rc == PGCP_E_CUDA && !cudaGetLastError()) set_error("direct solver: stream fork/join failed");
    return rc;
}

}  // namespace

int direct_factor(pgcp_batch* b, const DirectInput& in, DirectFactor** out, cudaStream_t s) {
    *out = nullptr;
    auto* D = new DirectFactor();
    std::unique_ptr<DirectFactor> guard(D);
    D->cplx = in.cplx;
    D->nslot = in.nslot;
    const int32_t nslot = in.nslot;
    D->h_uoff.assign(nslot + 1, 0);
    for (int j = 0; j < nslot; ++j) D->h_uoff[j + 1] = D->h_uoff[j] + in.h_nu[j];
    const int64_t NU = D->h_uoff[nslot];
    D->NU = NU;
    D->rows = 32 * in.h_sl_off[nslot];
    const int leafmax = std::max(4, env_int("PGCP_DIRECT_LEAF", 48));
    cudaEvent_t e0, e1;
    PGCP_TRY_CUDA(cudaEventCreate(&e0));
    PGCP_TRY_CUDA(cudaEventCreate(&e1));
    PGCP_TRY_CUDA(cudaEventRecord(e0, s));
    PhaseTimer pt(s);
    PGCP_TRY(D->err.alloc(std::max(nslot, 1), s));
    PGCP_TRY(D->err.zero(s));
    D->h_err.assign(nslot, 0);
    if (NU == 0) {
        *out = guard.release();
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        return PGCP_OK;
    }
    PGCP_TRY(D->uoff.alloc(nslot + 1, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(D->uoff.p, D->h_uoff.data(), (nslot + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    PGCP_TRY(D->urow.alloc(NU, s));
    PGCP_TRY(D->uslot.alloc(NU, s));
    k_d_urow<<<grid_for(NU, 256), 256, 0, s>>>(NU, nslot, D->uoff.p, in.sl_off, D->urow.p, D->uslot.p);
    PGCP_LAUNCH_CHECK();
    DevBuf<float4> pos;
    PGCP_TRY(pos.alloc(NU, s));
    k_d_pos<<<grid_for(NU, 256), 256, 0, s>>>(NU, D->urow.p, D->uslot.p, in.rowsrc, in.sv_off, in.comps,
                                            b->vert_off.p, b->vmap.p, b->V.p, pos.p);
    PGCP_LAUNCH_CHECK();
    // adjacency (the system's rows in unknown space)
    AdjArgs aa;
    aa.urow = D->urow.p;
    aa.uslot = D->uslot.p;
    aa.uoff = D->uoff.p;
    aa.sl_off = in.sl_off;
    aa.sl_ptr = in.sl_ptr;
    aa.col = in.col;
    aa.val = in.val;
    aa.sl_mask = in.cplx ? in.sl_mask : nullptr;
    aa.cpl = in.cpl;
    aa.cplc = in.cplc;
    {
        DevBuf<int64_t> cntb;
        PGCP_TRY(cntb.alloc(NU, s));
        k_d_adj_count<<<grid_for(NU, 256), 256, 0, s>>>(NU, aa, cntb.p);
        PGCP_LAUNCH_CHECK();
        PGCP_TRY(D->aptr.alloc(NU + 1, s));
        PGCP_TRY(exclusive_scan_i64(cntb.p, D->aptr.p, NU, s));
    }
    // upper bound of the stored entries (no host round trip): every ELL slot
    // (padding included) plus the two coupling partners of a row
    const int64_t annz = in.nnz_ell + 2 * NU;
    PGCP_TRY(D->acol.alloc(annz, s));
    PGCP_TRY(D->aval.alloc(annz, s));
    k_d_adj_fill<<<grid_for(NU, 256), 256, 0, s>>>(NU, aa, D->aptr.p, D->acol.p, D->aval.p);
    PGCP_LAUNCH_CHECK();
    pt.mark("adjacency");

    // ---- nested dissection, level by level
    const int64_t ncap = NU / 4 + 4 * (int64_t)nslot + 4096;
    PGCP_TRY(D->parent.alloc(ncap, s));
    PGCP_TRY(D->chA.alloc(ncap, s));
    PGCP_TRY(D->chB.alloc(ncap, s));
    PGCP_TRY(D->cnt.alloc(ncap, s));
    PGCP_TRY(D->npiv.alloc(ncap, s));
    PGCP_TRY(D->slot.alloc(ncap, s));
    PGCP_TRY(D->nchild.alloc(ncap, s));
    PGCP_TRY(D->leaf.alloc(ncap, s));
    PGCP_TRY(D->bbox.alloc(6 * ncap, s));
    PGCP_TRY(D->gcnt.alloc(3 * ncap, s));
    PGCP_TRY(D->split.alloc(ncap, s));
    NodeArrays nd = D->na();
    DevBuf<int32_t> reg, node_of;
    DevBuf<int8_t> side, grp;
    PGCP_TRY(reg.alloc(NU, s));
    PGCP_TRY(node_of.alloc(NU, s));
    PGCP_TRY(side.alloc(NU, s));
    PGCP_TRY(grp.alloc(NU, s));
    D->boundary_last = in.cplx && in.onloop != nullptr;
    if (D->boundary_last) {
        DevBuf<int32_t> cnt2;
        PGCP_TRY(cnt2.alloc(2 * (int64_t)nslot, s));
        PGCP_TRY(cnt2.zero(s));
        k_nd_bl_count<<<grid_for(NU, 256), 256, 0, s>>>(NU, D->uslot.p, D->urow.p, in.onloop, cnt2.p);
        PGCP_LAUNCH_CHECK();
        k_nd_bl_roots<<<grid_for(nslot, 128), 128, 0, s>>>(nslot, cnt2.p, leafmax, nd);
        PGCP_LAUNCH_CHECK();
        k_nd_bl_init_u<<<grid_for(NU, 256), 256, 0, s>>>(NU, nslot, D->uslot.p, D->urow.p, in.onloop, D->leaf.p,
                                                        reg.p, node_of.p);
        PGCP_LAUNCH_CHECK();
    } else {
        k_nd_roots<<<grid_for(nslot, 128), 128, 0, s>>>(nslot, D->uoff.p, leafmax, nd);
        PGCP_LAUNCH_CHECK();
        k_nd_init_u<<<grid_for(NU, 256), 256, 0, s>>>(NU, D->uslot.p, D->leaf.p, reg.p, node_of.p);
        PGCP_LAUNCH_CHECK();
    }
    DevBuf<int32_t> scan, ndst;  // ndst: [0..1] live level range, [2] overflow, [4..] per-level ranges
    PGCP_TRY(scan.alloc(ncap + 1, s));
    constexpr int MAXL = 96;
    PGCP_TRY(ndst.alloc(4 + 2 * MAXL, s));
    PGCP_TRY(ndst.zero(s));
    const int level0 = D->boundary_last ? 1 : 0;  // boundary-last: level 0 = the loops' fronts
    {
        const int32_t r0[6] = {D->boundary_last ? nslot : 0, D->boundary_last ? 2 * nslot : nslot, 0, 0, 0, nslot};
        PGCP_TRY_CUDA(cudaMemcpyAsync(ndst.p, r0, sizeof(r0), cudaMemcpyHostToDevice, s));  // [4..5] = level 0
    }
    int32_t* rng = ndst.p;
    int32_t* hist = ndst.p + 4;
    D->levels.clear();
    const int ugrid = grid_for(NU, 256);
    const int rgrid = 4 * 148;
    int nlev = 0;
    const bool nd_detail = env_int("PGCP_DIRECT_TIMING", 0) >= 2;
    for (int level = level0;; ++level) {
        if (level >= MAXL) {
            set_error("direct solver: nested dissection did not terminate");
            return DIRECT_FALLBACK;
        }
        k_nd_reset<<<rgrid, 256, 0, s>>>(rng, nd);
        PGCP_LAUNCH_CHECK();
        k_nd_bbox<<<ugrid, 256, 0, s>>>(NU, reg.p, pos.p, nd);
        PGCP_LAUNCH_CHECK();
        k_nd_split<<<rgrid, 256, 0, s>>>(rng, nd);
        PGCP_LAUNCH_CHECK();
        k_nd_side<<<ugrid, 256, 0, s>>>(NU, reg.p, pos.p, nd, side.p);
        PGCP_LAUNCH_CHECK();
        k_nd_sep<<<ugrid, 256, 0, s>>>(NU, reg.p, side.p, D->aptr.p, D->acol.p, nd, grp.p);
        PGCP_LAUNCH_CHECK();
        k_nd_count_children<<<rgrid, 256, 0, s>>>(rng, nd);
        PGCP_LAUNCH_CHECK();
        k_nd_scan<<<1, 1024, 0, s>>>(rng, D->nchild.p, scan.p, hist, level, ncap, ndst.p + 2);
        PGCP_LAUNCH_CHECK();
        k_nd_link<<<rgrid, 256, 0, s>>>(hist + 2 * level, scan.p, leafmax, nd);
        PGCP_LAUNCH_CHECK();
        k_nd_assign<<<ugrid, 256, 0, s>>>(NU, reg.p, grp.p, nd, node_of.p);
        PGCP_LAUNCH_CHECK();
        if (nd_detail) pt.mark("ndlvl");
        // termination: checked on the host every other level past the 9th
        if (level >= 8 && (level & 1)) {
            int32_t h[4];
            PGCP_TRY(d2h_async(h, ndst.p, sizeof(h), s));
            PGCP_TRY(d2h_flush(s));
            if (h[2]) {
                set_error("direct solver: nested dissection node capacity exceeded");
                return DIRECT_FALLBACK;
            }
            if (h[0] >= h[1]) {
                nlev = level + 1;
                break;
            }
        }
    }
    std::vector<int32_t> hh(2 * nlev);
    PGCP_TRY(d2h_async(hh.data(), hist, hh.size() * sizeof(int32_t), s));
    PGCP_TRY(d2h_flush(s));
    int32_t le = nslot;
    for (int l = 0; l < nlev; ++l) {
        if (hh[2 * l + 1] <= hh[2 * l]) break;  // trailing empty levels
        D->levels.push_back({hh[2 * l], hh[2 * l + 1]});
        le = hh[2 * l + 1];
    }
    D->nnodes = le;
    const int32_t nn = D->nnodes;
    pt.mark("nd");
    // ---- postorder: elimination indices
    DevBuf<int64_t> tsz, start, npiv64, gstart;
    PGCP_TRY(tsz.alloc(nn, s));
    PGCP_TRY(start.alloc(nn, s));
    PGCP_TRY(D->pfirst.alloc(nn, s));
    for (int l = (int)D->levels.size() - 1; l >= 0; --l) {
        const int a0 = D->levels[l].first, a1 = D->levels[l].second;
        k_nd_subtree<<<grid_for(a1 - a0, 256), 256, 0, s>>>(a0, a1, nd, tsz.p);
        PGCP_LAUNCH_CHECK();
    }
    for (size_t l = 0; l < D->levels.size(); ++l) {
        const int a0 = D->levels[l].first, a1 = D->levels[l].second;
        k_nd_start<<<grid_for(a1 - a0, 256), 256, 0, s>>>(a0, a1, nd, tsz.p, D->uoff.p, start.p, D->pfirst.p);
        PGCP_LAUNCH_CHECK();
    }
    PGCP_TRY(npiv64.alloc(nn, s));
    PGCP_TRY(gstart.alloc(nn + 1, s));
    k_nd_npiv64<<<grid_for(nn, 256), 256, 0, s>>>(nn, D->npiv.p, npiv64.p);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY(exclusive_scan_i64(npiv64.p, gstart.p, nn, s));
    {
        DevBuf<int32_t> kin, vin, kout, vout;
        PGCP_TRY(vin.alloc(NU, s));
        PGCP_TRY(kout.alloc(NU, s));
        PGCP_TRY(vout.alloc(NU, s));
        k_iota<<<grid_for(NU, 256), 256, 0, s>>>(NU, vin.p);
        PGCP_LAUNCH_CHECK();
        int bits = 1;
        while ((1ll << bits) < nn) ++bits;
        size_t need = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, need, node_of.p, kout.p, vin.p, vout.p, (int)NU, 0, bits, s);
        DevBuf<unsigned char> tmp;
        PGCP_TRY(tmp.alloc((int64_t)need, s));
        PGCP_TRY_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, need, node_of.p, kout.p, vin.p, vout.p, (int)NU, 0, bits, s));
        PGCP_TRY(D->elim.alloc(NU, s));
        PGCP_TRY(D->perm.alloc(NU, s));
        k_nd_elim<<<grid_for(NU, 256), 256, 0, s>>>(NU, kout.p, vout.p, gstart.p, D->pfirst.p, D->elim.p, D->perm.p);
        PGCP_LAUNCH_CHECK();
        PGCP_TRY(D->rowel.alloc(D->rows, s));
        PGCP_TRY(D->rowel.fill_bytes(0xff, s));
        k_d_rowel<<<grid_for(NU, 256), 256, 0, s>>>(NU, D->urow.p, D->elim.p, D->rowel.p);
        PGCP_LAUNCH_CHECK();
    }
    pt.mark("postorder");
    // ---- adjacency in elimination order
    {
        DevBuf<int64_t> ecnt;
        PGCP_TRY(ecnt.alloc(NU, s));
        k_eadj_count<<<grid_for(NU, 256), 256, 0, s>>>(NU, D->perm.p, D->elim.p, D->aptr.p, D->acol.p, ecnt.p);
        PGCP_LAUNCH_CHECK();
        PGCP_TRY(D->eptr.alloc(NU + 1, s));
        PGCP_TRY(exclusive_scan_i64(ecnt.p, D->eptr.p, NU, s));
        const int64_t ne = annz;  // upper bound (each stored entry once per direction)
        PGCP_TRY(D->erow.alloc(ne, s));
        PGCP_TRY(D->ecol.alloc(ne, s));
        PGCP_TRY(D->eval.alloc(ne, s));
        k_eadj_fill<<<grid_for(NU, 256), 256, 0, s>>>(NU, D->perm.p, D->elim.p, D->aptr.p, D->acol.p, D->aval.p,
                                                    D->eptr.p, D->erow.p, D->ecol.p, D->eval.p);
        PGCP_LAUNCH_CHECK();
    }
    // ---- symbolic: update sets, leaves first
    PGCP_TRY(D->ucnt.alloc(nn, s));
    PGCP_TRY(D->ustart.alloc(nn, s));
    const int64_t ucap = 24 * NU + 65536;
    PGCP_TRY(D->upool.alloc(ucap, s));
    DevBuf<unsigned long long> bump;
    DevBuf<int32_t> ovf;
    PGCP_TRY(bump.alloc(1, s));
    PGCP_TRY(bump.zero(s));
    PGCP_TRY(ovf.alloc(1, s));
    PGCP_TRY(ovf.zero(s));
    SymArgs sa;
    sa.nd = nd;
    sa.pfirst = D->pfirst.p;
    sa.perm = D->perm.p;
    sa.elim = D->elim.p;
    sa.eptr = D->eptr.p;
    sa.ecol = D->ecol.p;
    sa.ucnt = D->ucnt.p;
    sa.ustart = D->ustart.p;
    sa.upool = D->upool.p;
    sa.bump = bump.p;
    sa.ucap = ucap;
    sa.overflow = ovf.p;
    for (int l = (int)D->levels.size() - 1; l >= 0; --l) {
        const int a0 = D->levels[l].first, a1 = D->levels[l].second;
        k_sym<<<a1 - a0, DNT, 0, s>>>(a0, sa);
        PGCP_LAUNCH_CHECK();
    }
    pt.mark("symbolic");  // the overflow flag is read with the layout below
    // ---- front types: complex where the subtree holds coupling entries
    PGCP_TRY(D->ntype.alloc(nn, s));
    PGCP_TRY(D->ntype.zero(s));
    if (D->cplx) {
        k_mark_cplx<<<grid_for(NU, 256), 256, 0, s>>>(NU, D->aptr.p, D->aval.p, node_of.p, D->parent.p, D->ntype.p);
        PGCP_LAUNCH_CHECK();
    }
    // ---- front layout
    PGCP_TRY(D->fsz.alloc(nn, s));
    PGCP_TRY(D->foff.alloc(nn + 1, s));
    PGCP_TRY(D->woff.alloc(nn + 1, s));
    {
        DevBuf<int64_t> f2, f1;
        PGCP_TRY(f2.alloc(nn, s));
        PGCP_TRY(f1.alloc(nn, s));
        k_front_sizes<<<grid_for(nn, 256), 256, 0, s>>>(nn, D->npiv.p, D->ucnt.p, D->ntype.p, D->fsz.p, f2.p, f1.p);
        PGCP_LAUNCH_CHECK();
        PGCP_TRY(exclusive_scan_i64(f2.p, D->foff.p, nn, s));
        PGCP_TRY(exclusive_scan_i64(f1.p, D->woff.p, nn, s));
    }
    std::vector<int32_t> hf(nn), hp(nn);
    std::vector<int8_t> ht(nn);
    int64_t ftot = 0, wtot = 0;
    PGCP_TRY(d2h_async(ht.data(), D->ntype.p, nn * sizeof(int8_t), s));
    PGCP_TRY(d2h_async(hf.data(), D->fsz.p, nn * sizeof(int32_t), s));
    PGCP_TRY(d2h_async(hp.data(), D->npiv.p, nn * sizeof(int32_t), s));
    PGCP_TRY(d2h_async(&ftot, D->foff.p + nn, sizeof(int64_t), s));
    PGCP_TRY(d2h_async(&wtot, D->woff.p + nn, sizeof(int64_t), s));
    int32_t hov = 0;
    PGCP_TRY(d2h_async(&hov, ovf.p, sizeof(int32_t), s));
    PGCP_TRY(d2h_flush(s));
    if (hov) {  // some update set was cut short: nothing after it is valid
        set_error("direct solver: symbolic capacity exceeded");
        return DIRECT_FALLBACK;
    }
    D->lvl_maxf.assign(D->levels.size(), 0);
    D->lvl_maxu.assign(D->levels.size(), 0);
    D->fmas = 0;
    D->maxf = 0;
    D->ncplx = 0;
    std::vector<int32_t> hl;
    hl.reserve(nn);
    D->lst_off.assign(2 * D->levels.size() + 1, 0);
    for (size_t l = 0; l < D->levels.size(); ++l) {
        for (int t = 0; t < 2; ++t) {
            D->lst_off[2 * l + t] = (int64_t)hl.size();
            for (int N = D->levels[l].first; N < D->levels[l].second; ++N)
                if (ht[N] == t) hl.push_back(N);
        }
        for (int N = D->levels[l].first; N < D->levels[l].second; ++N) {
            const double f = hf[N], sp = hp[N], u = f - sp;
            D->lvl_maxf[l] = std::max(D->lvl_maxf[l], hf[N]);
            D->lvl_maxu[l] = std::max(D->lvl_maxu[l], hf[N] - hp[N]);
            D->maxf = std::max(D->maxf, hf[N]);
            D->fmas += (ht[N] ? 4.0 : 1.0) * (sp * sp * sp / 6.0 + u * sp * sp / 2.0 + u * u * sp / 2.0);
            D->ncplx += ht[N] != 0;
        }
    }
    D->lst_off[2 * D->levels.size()] = (int64_t)hl.size();
    // every list largest front first (ties by node id: deterministic), then
    // the warp-sized tail of each list packed into k_factor_warp's groups
    {
        const size_t nq = 2 * D->levels.size();
        D->lst_wfirst.assign(nq, 0);
        D->grp_off.assign(nq + 1, 0);
        D->h_gstart.clear();
        D->h_wsoff.assign(std::max<size_t>(hl.size(), 1), 0);
        const bool no_warp = getenv("PGCP_DIRECT_NO_WARP") != nullptr;
        for (size_t q = 0; q < nq; ++q) {
            const int64_t o0 = D->lst_off[q], o1 = D->lst_off[q + 1];
            {   // stable counting sort by front size, descending (the list is in node order)
                int fmax = 0;
                for (int64_t i = o0; i < o1; ++i) fmax = std::max(fmax, hf[hl[i]]);
                std::vector<int32_t> start(fmax + 2, 0), tmp(hl.begin() + o0, hl.begin() + o1);
                for (int32_t N : tmp) ++start[fmax - hf[N] + 1];
                for (int k = 0; k <= fmax; ++k) start[k + 1] += start[k];
                for (int32_t N : tmp) hl[o0 + start[fmax - hf[N]]++] = N;
            }
            const size_t l = q / 2, tsz = (q & 1) ? 16 : 8;
            const int maxu_child = l + 1 < D->levels.size() ? D->lvl_maxu[l + 1] : 0;
            // bytes of front N in k_factor_warp: packed triangle, its update
            // rows and the relative indices of a child's update rows
            auto wbytes = [&](int32_t N) {
                const size_t f = (size_t)hf[N], nu = (size_t)(hf[N] - hp[N]);
                return (f * (f + 1) / 2 * tsz + (nu + (size_t)maxu_child) * 4 + 16 + 15) & ~(size_t)15;
            };
            // A list whose largest front fits a warp goes to k_factor_warp whole.
            // Otherwise the fronts up to warp_split_bytes (f <= 70:
            // measured 3x faster per front there than a CTA each, while
            // a lone warp on an 80-100 wide front is slower than a CTA) split
            // off, if they are most of the list; the few larger ones take a CTA
            // each. PGCP_DIRECT_WSPLIT=0: no split (a mixed list takes CTAs).
            const bool wsplit = env_int("PGCP_DIRECT_WSPLIT", 1) != 0;
            int64_t w0 = o0;
            if (no_warp) {
                w0 = o1;
            } else if (o1 > o0 && wbytes(hl[o0]) > WARP_FRONT_BYTES) {
                while (w0 < o1 && wbytes(hl[w0]) > warp_split_bytes(tsz)) ++w0;
                if (!wsplit || 2 * (o1 - w0) < (o1 - o0)) w0 = o1;
            }
            D->lst_wfirst[q] = w0;
            D->grp_off[q] = (int64_t)D->h_gstart.size();
            if (w0 < o1) {
                const size_t cap = warp_cta_bytes(tsz);
                const int maxw = warp_cta_warps();
                size_t used = cap + 1;  // forces a new group at the first front
                int cnt = 0;
                for (int64_t i = w0; i < o1; ++i) {
                    const size_t wb = wbytes(hl[i]);
                    if (cnt == maxw || used + wb > cap) {
                        D->h_gstart.push_back((int32_t)i);
                        used = 0;
                        cnt = 0;
                    }
                    D->h_wsoff[i] = (int32_t)used;
                    used += wb;
                    ++cnt;
                }
                D->h_gstart.push_back((int32_t)o1);  // end sentinel of this list's groups
            }
        }
        D->grp_off[nq] = (int64_t)D->h_gstart.size();
        PGCP_TRY(D->gstart.alloc(std::max<int64_t>((int64_t)D->h_gstart.size(), 1), s));
        PGCP_TRY(D->wsoff.alloc((int64_t)D->h_wsoff.size(), s));
        if (!D->h_gstart.empty())
            PGCP_TRY_CUDA(cudaMemcpyAsync(D->gstart.p, D->h_gstart.data(), D->h_gstart.size() * sizeof(int32_t),
                                          cudaMemcpyHostToDevice, s));
        PGCP_TRY_CUDA(cudaMemcpyAsync(D->wsoff.p, D->h_wsoff.data(), D->h_wsoff.size() * sizeof(int32_t),
                                      cudaMemcpyHostToDevice, s));
    }
    D->lst_maxs.assign(2 * D->levels.size(), 0);
    D->lst_maxf.assign(2 * D->levels.size(), 0);
    for (size_t q = 0; q < 2 * D->levels.size(); ++q)
        for (int64_t i = D->lst_off[q]; i < D->lst_off[q + 1]; ++i) {
            D->lst_maxs[q] = std::max(D->lst_maxs[q], hp[hl[i]]);
            D->lst_maxf[q] = std::max(D->lst_maxf[q], hf[hl[i]]);
        }
    D->h_nlist = hl;
    D->h_npiv = hp;
    D->h_fsz = hf;
    PGCP_TRY(D->nlist.alloc(nn, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(D->nlist.p, hl.data(), nn * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    {   // deepest level first: every front after its children (host copy kept: async upload)
        std::vector<int32_t>& ord = D->h_order;
        ord.clear();
        ord.reserve(nn);
        for (int l = (int)D->levels.size() - 1; l >= 0; --l)
            for (int N = D->levels[l].first; N < D->levels[l].second; ++N) ord.push_back(N);
        PGCP_TRY(D->order.alloc(nn, s));
        PGCP_TRY_CUDA(cudaMemcpyAsync(D->order.p, ord.data(), nn * sizeof(int32_t), cudaMemcpyHostToDevice, s));
        PGCP_TRY(D->sync.alloc(nn + 2, s));
        PGCP_TRY(D->sync.zero(s));
    }
    if (pt.on) {
        for (size_t l = 0; l < D->levels.size(); ++l) {
            double lf = 0;
            int maxp = 0;
            for (int N = D->levels[l].first; N < D->levels[l].second; ++N) {
                const double f = hf[N], sp = hp[N], u = f - sp;
                lf += (ht[N] ? 4.0 : 1.0) * (sp * sp * sp / 6.0 + u * sp * sp / 2.0 + u * u * sp / 2.0);
                maxp = std::max(maxp, hp[N]);
            }
            fprintf(stderr, "[direct levels] L%zu nodes %d max front %d max pivots %d max update %d FMAs %.3g\n", l,
                    D->levels[l].second - D->levels[l].first, D->lvl_maxf[l], maxp, D->lvl_maxu[l], lf);
            if (env_int("PGCP_DIRECT_TIMING", 0) >= 2) {  // front-size distribution (count and FMA shares)
                std::vector<std::pair<int, double>> fs;
                for (int N = D->levels[l].first; N < D->levels[l].second; ++N) {
                    const double f = hf[N], sp = hp[N], u = f - sp;
                    fs.push_back({hf[N], (ht[N] ? 4.0 : 1.0) * (sp * sp * sp / 6.0 + u * sp * sp / 2.0 + u * u * sp / 2.0)});
                }
                std::sort(fs.begin(), fs.end());
                const size_t n = fs.size();
                double acc = 0;
                fprintf(stderr, "[direct levels]    front size quantiles 10/50/90%%: %d %d %d; FMA share of fronts <=",
                        fs[n / 10].first, fs[n / 2].first, fs[(9 * n) / 10].first);
                size_t i = 0;
                for (int cut : {40, 48, 56, 64, 72, 80}) {
                    while (i < n && fs[i].first <= cut) acc += fs[i++].second;
                    fprintf(stderr, " %d: %.2f (%zu)", cut, lf > 0 ? acc / lf : 0.0, i);
                }
                fprintf(stderr, "\n");
            }
        }
    }
    D->front_bytes = 8.0 * (double)ftot;
    auto ta = std::chrono::steady_clock::now();
    PGCP_TRY(D->fpool.alloc(8 * ftot, s));  // every front zeroes itself
    PGCP_TRY(D->W.alloc(wtot, s));
    PGCP_TRY(D->X.alloc(NU, s));
    if (pt.on)
        fprintf(stderr, "[direct timing] front storage %.3f GB, allocation %.3f ms (host)\n", 8e-9 * (double)ftot,
                1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - ta).count());
    pt.mark("layout");
    // ---- numeric
    FacArgs fa;
    fa.nd = nd;
    fa.pfirst = D->pfirst.p;
    fa.perm = D->perm.p;
    fa.elim = D->elim.p;
    fa.eptr = D->eptr.p;
    fa.erow = D->erow.p;
    fa.ecol = D->ecol.p;
    fa.eval = D->eval.p;
    fa.ucnt = D->ucnt.p;
    fa.ustart = D->ustart.p;
    fa.upool = D->upool.p;
    fa.fsz = D->fsz.p;
    fa.foff = D->foff.p;
    fa.fpool = D->fpool.p;
    fa.ntype = D->ntype.p;
    fa.list = nullptr;
    fa.err = D->err.p;
    cudaEvent_t n0, n1;
    PGCP_TRY_CUDA(cudaEventCreate(&n0));
    PGCP_TRY_CUDA(cudaEventCreate(&n1));
    PGCP_TRY_CUDA(cudaEventRecord(n0, s));
    PGCP_TRY(factor_levels(D, fa, s, pt));
    PGCP_TRY_CUDA(cudaEventRecord(n1, s));
    PGCP_TRY_CUDA(cudaEventRecord(e1, s));
    PGCP_TRY(d2h_async(D->h_err.data(), D->err.p, nslot * sizeof(int32_t), s));
    PGCP_TRY(d2h_flush(s));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    D->factor_ms = ms;
    cudaEventElapsedTime(&ms, n0, n1);
    D->numeric_ms = ms;
    cudaEventDestroy(n0);
    cudaEventDestroy(n1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *out = guard.release();
    return PGCP_OK;
}

// The forward and backward sweeps as persistent launches: the deep levels
// whose fronts fit a warp (f <= SW_F, s <= SW_S: closed under descent, as
// every level below qualifies too) warp-per-front (k_solve_warp), the rest
// CTA-per-front (k_solve_pers). Both share the done flags; the ticket
// counter restarts per launch. zero_roots: x of the roots (< skip) := 0
// before the backward sweep (the interior-only solve).
int solve_trace_report(DirectFactor* D, const unsigned long long* tr, int bwd, int grid, int per_sm, size_t smem,
                       cudaStream_t s);
__global__ void k_zero_roots(int32_t nroot, const int64_t* __restrict__ pfirst, const int32_t* __restrict__ npiv,
                             double2* __restrict__ X) {
    const int j = blockIdx.x;
    if (j >= nroot) return;
    for (int k = threadIdx.x; k < npiv[j]; k += blockDim.x) X[pfirst[j] + k] = make_double2(0.0, 0.0);
}
int solve_sweeps(DirectFactor* D, const SolArgs& a, int skip, bool zero_roots, cudaStream_t s, PhaseTimer* pt) {
    const int L = (int)D->levels.size();
    const int nn = D->nnodes;
    int lcut = L;
    if (env_int("PGCP_DIRECT_SOLVE_WARP", 1))
        for (int l = L - 1; l >= 0; --l) {
            const int ms = std::max(D->lst_maxs[2 * l], D->lst_maxs[2 * l + 1]);
            if (D->lvl_maxf[l] > SW_F || ms > SW_S) break;
            lcut = l;
        }
    int nsmall = 0;
    for (int l = lcut; l < L; ++l) nsmall += D->levels[l].second - D->levels[l].first;
    const int nbig = nn - nsmall;
    int maxf = 0, maxu = 0;
    for (int l = 0; l < lcut; ++l) {
        maxf = std::max(maxf, D->lvl_maxf[l]);
        maxu = std::max(maxu, D->lvl_maxu[l]);
    }
    const size_t smem = (size_t)maxf * sizeof(double2) + (size_t)maxu * 4 + 16;
    int dev = 0, sms = 148, per_sm = 1, per_sm_w = 1;
    PGCP_TRY_CUDA(cudaGetDevice(&dev));
    PGCP_TRY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (nbig > 0) {
        PGCP_TRY(set_smem(k_solve_pers, smem));
        PGCP_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_solve_pers, DNT, smem));
    }
    int per_sm_wb = 1;
    using WarpSweep = void (*)(SolArgs, const int32_t*, int, int*, int*, const int8_t*, int, unsigned long long*);
    WarpSweep kw[2] = {k_solve_warp<false, 4>, k_solve_warp<true, 4>};
    switch (env_int("PGCP_DIRECT_SOLVE_MINB", 4)) {  // register cap (resident CTAs per SM) of the warp sweeps
        case 6: kw[0] = k_solve_warp<false, 6>; kw[1] = k_solve_warp<true, 6>; break;
        case 8: kw[0] = k_solve_warp<false, 8>; kw[1] = k_solve_warp<true, 8>; break;
        default: break;
    }
    PGCP_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_w, kw[0], DNT, 0));
    PGCP_TRY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_wb, kw[1], DNT, 0));
    const int grid = std::max(1, std::min(per_sm * sms, nbig));
    const int grid_wf = std::max(1, std::min(per_sm_w * sms, (nsmall + DNT / 32 - 1) / (DNT / 32)));
    const int grid_wb = std::max(1, std::min(per_sm_wb * sms, (nsmall + DNT / 32 - 1) / (DNT / 32)));
    const bool trace_on = getenv("PGCP_DIRECT_SOLVE_TRACE") != nullptr;
    DevBuf<unsigned long long> tr;
    if (trace_on) PGCP_TRY(tr.alloc(3 * (int64_t)nn, s));
    int* ticket = D->sync.p + 1;
    int* done = D->sync.p + 2;
    k_perm_rhs<<<grid_for(D->NU, 256), 256, 0, s>>>(D->NU, D->perm.p, D->urow.p, a.b, D->X.p);
    PGCP_LAUNCH_CHECK();
    for (int bwd = 0; bwd < 2; ++bwd) {
        if (bwd && zero_roots) {
            k_zero_roots<<<D->nslot, 128, 0, s>>>(D->nslot, D->pfirst.p, D->npiv.p, D->X.p);
            PGCP_LAUNCH_CHECK();
        }
        PGCP_TRY_CUDA(cudaMemsetAsync(ticket, 0, (size_t)(nn + 1) * sizeof(int), s));
        for (int part = 0; part < 2; ++part) {
            const bool warp_part = (part == 0) != (bwd != 0);  // forward: small first; backward: big first
            if (warp_part ? nsmall == 0 : nbig == 0) continue;
            if (part == 1) PGCP_TRY_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int), s));
            if (warp_part)
                kw[bwd]<<<bwd ? grid_wb : grid_wf, DNT, 0, s>>>(a, D->order.p, nsmall, done, ticket, D->ntype.p, skip,
                                                              trace_on ? tr.p : nullptr);
            else
                k_solve_pers<<<grid, DNT, smem, s>>>(a, D->order.p + nsmall, nbig, done, ticket, D->ntype.p, bwd, skip,
                                                     trace_on ? tr.p : nullptr);
            PGCP_LAUNCH_CHECK();
        }
        if (pt) pt->mark(bwd ? "backward" : "forward");
        if (trace_on) {
            fprintf(stderr, "[solve trace] warp path: levels >= %d (%d fronts, grid %d, %d/SM)\n", lcut, nsmall,
                    bwd ? grid_wb : grid_wf, bwd ? per_sm_wb : per_sm_w);
            PGCP_TRY(solve_trace_report(D, tr.p, bwd, grid, per_sm, smem, s));
        }
    }
    return PGCP_OK;
}

// PGCP_DIRECT_SOLVE_TRACE=1: per-level timeline of one persistent sweep from
// the per-front globaltimer stamps (ticket drawn, dependencies met, done)
int solve_trace_report(DirectFactor* D, const unsigned long long* tr, int bwd, int grid, int per_sm,
                              size_t smem, cudaStream_t s) {
    const int nn = D->nnodes;
    std::vector<unsigned long long> h(3 * (size_t)nn);
    PGCP_TRY_CUDA(cudaMemcpyAsync(h.data(), tr, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaStreamSynchronize(s));
    unsigned long long t0 = ~0ull, tend = 0;
    for (int N = 0; N < nn; ++N) {
        t0 = std::min(t0, h[3 * N]);
        tend = std::max(tend, h[3 * N + 2]);
    }
    fprintf(stderr, "[solve trace] %s grid %d (%d/SM, smem %zu B) span %.1f us\n", bwd ? "backward" : "forward", grid,
            per_sm, smem, 1e-3 * (double)(tend - t0));
    for (size_t l = 0; l < D->levels.size(); ++l) {
        const int b = D->levels[l].first, e = D->levels[l].second;
        double wsum = 0, wmax = 0, ksum = 0, kmax = 0;
        unsigned long long lo = ~0ull, hi = 0, wl = ~0ull;
        for (int N = b; N < e; ++N) {
            const double w = 1e-3 * (double)(h[3 * N + 1] - h[3 * N]), k = 1e-3 * (double)(h[3 * N + 2] - h[3 * N + 1]);
            wsum += w;
            ksum += k;
            wmax = std::max(wmax, w);
            kmax = std::max(kmax, k);
            lo = std::min(lo, h[3 * N]);
            wl = std::min(wl, h[3 * N + 1]);
            hi = std::max(hi, h[3 * N + 2]);
        }
        const int n = e - b;
        fprintf(stderr,
                "[solve trace]   L%zu fronts %d  first ticket %.1f  first start %.1f  last done %.1f us  "
                "work mean %.2f max %.2f  wait mean %.2f max %.2f us\n",
                l, n, 1e-3 * (double)(lo - t0), 1e-3 * (double)(wl - t0), 1e-3 * (double)(hi - t0), ksum / n, kmax,
                wsum / n, wmax);
    }
    return PGCP_OK;
}

int direct_solve(DirectFactor* D, const double2* b_rows, double2* x_rows, cudaStream_t s) {
    PGCP_TRY_CUDA(cudaMemsetAsync(x_rows, 0, (size_t)D->rows * sizeof(double2), s));
    if (D->NU == 0) return PGCP_OK;
    cudaEvent_t e0, e1;
    PGCP_TRY_CUDA(cudaEventCreate(&e0));
    PGCP_TRY_CUDA(cudaEventCreate(&e1));
    PGCP_TRY_CUDA(cudaEventRecord(e0, s));
    PhaseTimer pt(s);
    SolArgs a;
    a.nd = D->na();
    a.pfirst = D->pfirst.p;
    a.perm = D->perm.p;
    a.urow = D->urow.p;
    a.ucnt = D->ucnt.p;
    a.ustart = D->ustart.p;
    a.upool = D->upool.p;
    a.foff = D->foff.p;
    a.woff = D->woff.p;
    a.fpool = D->fpool.p;
    a.list = nullptr;
    a.W = D->W.p;
    a.X = D->X.p;
    a.b = b_rows;
    const int L = (int)D->levels.size();
    auto launch = [&](bool fwd, int l, int t) -> int {
        const int64_t o0 = D->lst_off[2 * l + t], o1 = D->lst_off[2 * l + t + 1];
        if (o1 <= o0) return PGCP_OK;
        SolArgs aa = a;
        aa.list = D->nlist.p + o0;
        const int n = (int)(o1 - o0);
        const int maxu_child = (l + 1 < L) ? D->lvl_maxu[l + 1] : 0;
        const size_t smem = fwd ? (size_t)D->lvl_maxf[l] * sizeof(double2) + (size_t)(D->lvl_maxu[l] + maxu_child) * 4 + 16
                                : (size_t)D->lvl_maxf[l] * sizeof(double2) + 16;
        if (fwd && t) {
            PGCP_TRY(set_smem(k_fwd<double2>, smem));
            k_fwd<double2><<<n, DNT, smem, s>>>(aa);
        } else if (fwd) {
            PGCP_TRY(set_smem(k_fwd<double>, smem));
            k_fwd<double><<<n, DNT, smem, s>>>(aa);
        } else if (t) {
            PGCP_TRY(set_smem(k_bwd<double2>, smem));
            k_bwd<double2><<<n, DNT, smem, s>>>(aa);
        } else {
            PGCP_TRY(set_smem(k_bwd<double>, smem));
            k_bwd<double><<<n, DNT, smem, s>>>(aa);
        }
        PGCP_LAUNCH_CHECK();
        return PGCP_OK;
    };
    const char* ep = getenv("PGCP_DIRECT_PERSIST");
    if (!(ep && atoi(ep) == 0)) {  // persistent, dependency-driven launches
        PGCP_TRY(solve_sweeps(D, a, 0, false, s, &pt));
    } else {
        k_perm_rhs<<<grid_for(D->NU, 256), 256, 0, s>>>(D->NU, D->perm.p, D->urow.p, a.b, D->X.p);
        PGCP_LAUNCH_CHECK();
        for (int l = L - 1; l >= 0; --l) {
            PGCP_TRY(launch(true, l, 0));
            PGCP_TRY(launch(true, l, 1));
        }
        pt.mark("forward");
        for (int l = 0; l < L; ++l) {
            PGCP_TRY(launch(false, l, 0));
            PGCP_TRY(launch(false, l, 1));
        }
        pt.mark("backward");
    }
    k_d_scatter<<<grid_for(D->NU, 256), 256, 0, s>>>(D->NU, D->urow.p, D->elim.p, D->X.p, x_rows);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY_CUDA(cudaEventRecord(e1, s));
    PGCP_TRY_CUDA(cudaEventSynchronize(e1));
    {
        int timeout_flag = 0;
        PGCP_TRY_CUDA(cudaMemcpy(&timeout_flag, D->sync.p, sizeof(int), cudaMemcpyDeviceToHost));
        if (timeout_flag) {
            set_error("direct solver: substitution dependency wait timed out");
            return PGCP_E_CUDA;
        }
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    D->solve_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return PGCP_OK;
}

namespace {
__global__ void k_h2f_rhs(int64_t rows_h, const int32_t* __restrict__ h2f, const double2* __restrict__ bh,
                          double2* __restrict__ bf) {
    GRID_STRIDE(r, rows_h) {
        const int f = h2f[r];
        if (f >= 0) bf[f] = bh[r];
    }
}
__global__ void k_f2h_x(int64_t rows_h, const int32_t* __restrict__ h2f, const int32_t* __restrict__ rowel,
                        const double2* __restrict__ X, double2* __restrict__ xh) {
    GRID_STRIDE(r, rows_h) {
        const int f = h2f[r];
        const int e = f >= 0 ? rowel[f] : -1;
        xh[r] = e >= 0 ? X[e] : make_double2(0.0, 0.0);
    }
}
}  // namespace

bool direct_is_boundary_last(const DirectFactor* F) { return F && F->boundary_last; }

// The Dirichlet solve L_II x = b with the interior block of a boundary-last
// DNCP factor (the interior rows of the scaled DNCP system are the scaled
// Dirichlet system's): forward and backward sweeps over every front but the
// loops', whose x is held at 0. h2f maps the Dirichlet system's rows to the
// DNCP system's rows (-1: padding).
int direct_solve_interior(DirectFactor* D, const int32_t* h2f, int64_t rows_h, const double2* b_h, double2* x_h,
                          cudaStream_t s) {
    if (!D->boundary_last) {
        set_error("direct solver: interior solve needs a boundary-last factor");
        return PGCP_E_INVALID;
    }
    cudaEvent_t e0, e1;
    PGCP_TRY_CUDA(cudaEventCreate(&e0));
    PGCP_TRY_CUDA(cudaEventCreate(&e1));
    PGCP_TRY_CUDA(cudaEventRecord(e0, s));
    DevBuf<double2> bf;
    PGCP_TRY(bf.alloc(D->rows, s));
    PGCP_TRY(bf.zero(s));
    k_h2f_rhs<<<grid_for(rows_h, 256), 256, 0, s>>>(rows_h, h2f, b_h, bf.p);
    PGCP_LAUNCH_CHECK();
    SolArgs a;
    a.nd = D->na();
    a.pfirst = D->pfirst.p;
    a.perm = D->perm.p;
    a.urow = D->urow.p;
    a.ucnt = D->ucnt.p;
    a.ustart = D->ustart.p;
    a.upool = D->upool.p;
    a.foff = D->foff.p;
    a.woff = D->woff.p;
    a.fpool = D->fpool.p;
    a.list = nullptr;
    a.W = D->W.p;
    a.X = D->X.p;
    a.b = bf.p;
    PGCP_TRY(solve_sweeps(D, a, D->nslot, true, s, nullptr));
    k_f2h_x<<<grid_for(rows_h, 256), 256, 0, s>>>(rows_h, h2f, D->rowel.p, D->X.p, x_h);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY_CUDA(cudaEventRecord(e1, s));
    PGCP_TRY_CUDA(cudaEventSynchronize(e1));
    int timeout_flag = 0;
    PGCP_TRY(d2h_async(&timeout_flag, D->sync.p, sizeof(int), s));
    PGCP_TRY(d2h_flush(s));
    if (timeout_flag) {
        set_error("direct solver: substitution dependency wait timed out");
        return PGCP_E_CUDA;
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    D->solve_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return PGCP_OK;
}

}  // namespace pgcp

// diagnostics: the direct solver's workspace cache on the current device
// (out[0] slots, out[1] cached bytes, out[2] slot (re)allocations since the
// library was loaded, out[3] host ms spent in them)
extern "C" PGCP_API int pgcp_workspace_stats(double* out, int nout) {
    if (!out || nout < 4) {
        pgcp::set_error("pgcp_workspace_stats: invalid arguments");
        return PGCP_E_INVALID;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(pgcp::g_ws_mu);
    double slots = 0, bytes = 0;
    for (const pgcp::WsSlot& w : pgcp::g_ws)
        if (w.dev == dev) slots += 1, bytes += (double)w.bytes;
    out[0] = slots;
    out[1] = bytes;
    out[2] = (double)pgcp::g_ws_grows;
    out[3] = pgcp::g_ws_grow_ms;
    return PGCP_OK;
}
