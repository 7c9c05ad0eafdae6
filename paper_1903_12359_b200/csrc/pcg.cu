// pcg.cu -- K3: batched fp64 preconditioned CG, one thread-block cluster per
// subdomain, CG vectors resident in distributed shared memory.
//
// Replaces the two `spsolve` calls of the hot path:
//   flatten.py:157-173  DNCP: C_ff x = -C_f,fixed t with C = blockdiag(L,L) - 2M
//   assemble.py:34-48   harmonic: L_II u = -L_IB g (complex g, 2 RHS)
// Both are solved in one complex-Hermitian form over the unknown vertices U:
//     H = L_UU + 2i M_xy[U,U]      (flatten; M_xy[p,next]=+1/4, [p,prev]=-1/4)
//     H = L_UU                      (harmonic; complex RHS)
// which is exactly the real 2|U| system of the reference (pinned by
// tests/test_oracle_pins.py::test_hermitian_form). CG on an HPD system with
// an HPD preconditioner has real alpha/beta, so one recurrence serves both
// halves and L is streamed once per iteration for both.
//
// Layout (per solve, over the listed subdomains = "slots"):
//   rows      unknowns of slot j padded to 32*S_j rows (S_j slices); slot row
//             base 32*sl_off[j]; padding rows are inert (D=1, b=0, val=0)
//   matrix    paired sliced ELL (sell_pos): one 32-row slice per warp, two
//             values per 16-byte lane load, Jacobi-scaled D^-1/2 H D^-1/2;
//             columns re-encoded per launch as 16-bit CTA-local rows
//             (all-local slices) or (owner CTA, byte offset) codes (slices
//             that reach into another CTA's rows: DSMEM gathers)
//   coupling  flatten boundary rows carry (next, prev) rows in cpl[] and a bit
//             in the slice mask: (H z)_u += i/2 (z_next - z_prev)
//
// Kernels:
//   k_pcg2 (default) two-level PCG: M^-1 = I + W E^-1 W^T with W the linear
//             functions (1, u, v) of geometric aggregates that never straddle
//             a CTA; z, q, r in distributed shared memory, p and y in global
//             memory (row-local); three cluster reductions per iteration
//             (see the comment above k_pcg2); coarse start x0 = Q b.
//   k_pcg     plain Jacobi-PCG (PGCP_PCG_COARSE=0, and the safety net that
//             re-solves any slot the two-level solve did not finish), two
//             cluster reductions per iteration, using A p_new = A z + beta A p
//             so only z is ever gathered.
// Every reduction is a fixed-order warp / CTA / cluster sum: results are
// bitwise reproducible run to run.
#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>
#include <cuda_fp16.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <climits>
#include <cstring>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <mutex>

#include "batch.cuh"
#include "direct.cuh"

namespace cg = cooperative_groups;

namespace pgcp {

struct SolveSystem {
    bool dncp = false;
    int32_t nslot = 0;
    std::vector<int32_t> comps;      // slot -> comp
    std::vector<int64_t> h_sl_off;   // slot -> first slice (nslot+1)
    std::vector<int64_t> h_nu;       // slot -> unknowns
    std::vector<int64_t> h_sv_off;   // slot -> compact vertex offset (nslot+1)
    int64_t nslices = 0, rows = 0, nnz = 0, ne = 0;
    int csize = 1;
    // last run: PCG kernel time (CUDA events on the launch stream), iteration
    // totals and the compulsory bytes of one iteration
    double kernel_ms = 0, iters_sum = 0, iters_max = 0, bytes_iter_weighted = 0, nnz_off = 0, nrows_u = 0;
    double ref_bytes_weighted = 0;   // sum_j iters_j (12 z_j + 4 (r_j + 1)), reference CSR system
    DevBuf<int32_t> d_comps, slot_of_comp;
    DevBuf<int64_t> sl_off, sv_off, sl_ptr;
    DevBuf<uint32_t> sl_mask;
    DevBuf<int32_t> col, urow, rowsrc, fixed_ref;
    DevBuf<uint32_t> enc;
    DevBuf<uint16_t> enc16;          // local row index of every entry of an all-local slice
    DevBuf<uint8_t> remote;
    DevBuf<int2> cpl;
    DevBuf<double> val, D, Dinv, Dsq, dmax;
    DevBuf<double2> cplc;
    DevBuf<double2> b, x, fv;
    DevBuf<int32_t> iters;
    DevBuf<double> res;  // per slot: relres, bnorm^2, true_res^2, xnorm^2, pad
    // two-level preconditioner (see k_pcg2)
    bool coarse = false;
    bool force_jacobi = false;   // set for the Jacobi re-solve of non-converged slots
    bool setup_done = false;     // cluster shape, coarse space and encoded columns built
    bool prepared = false;       // harmonic: structure built, waiting for the fixed values
    int chunk = 1;
    DevBuf<int32_t> fixed_gid_copy;  // harmonic: fixed list (Jacobi re-solve)
    int64_t nfixed = 0;
    int gmax = 8;
    DevBuf<int32_t> cell, aggr, aoff;
    DevBuf<float2> pxy_row;
    DevBuf<uint2> wr;
    DevBuf<int64_t> nu_d, abase, eoff;
    DevBuf<double2> einv, p;
    DevBuf<float2> einv32;        // Hermitian E^-1 copy read by k_pcg2 (fp32) ...
    DevBuf<double2> einv64;       // ... or fp64 (PGCP_COARSE_FP64=1)
    DevBuf<int64_t> eoff32;
    bool einv_fp64 = false;
    int pcg_nt = 512;             // k_pcg2 threads per CTA (256: two CTAs per SM)
    int ncb = 0, mu_cap = 0, items_cap = 0;  // k_pcg2 coarse shared layout (see PcgArgs)
    std::vector<int64_t> h_abase;
    double coarse_ms = 0;
    std::vector<int32_t> h_iters;  // last run's iterations per slot
    // Every buffer above is allocated (and later freed, cudaFreeAsync) on
    // `home`, the stream of the call that built the system. A call that reads
    // the system on another stream (the harmonic solve after a prepare on a
    // side stream, export_system) makes `home` wait for its work, so the
    // frees of a later rebuild or of pgcp_batch_destroy are ordered after it.
    // direct solver (direct.cu): multifrontal Cholesky instead of PCG
    bool use_direct = false;
    std::shared_ptr<DirectFactor> direct;  // may be shared: a Dirichlet system borrows the DNCP factor
    bool borrowed = false;                 // solve with the interior block of the flatten's factor
    bool lazy_direct = false;              // prepared: factor (or borrow) at solve time
    DevBuf<int32_t> h2f;                   // borrowed: this system's row -> the DNCP system's row
    cudaStream_t direct_home = nullptr;    // stream the factor's buffers are freed on
    cudaStream_t home = nullptr;
    bool has_home = false;
    cudaEvent_t use_ev = nullptr;
    void built_on(cudaStream_t s) {
        home = s;
        has_home = true;
    }
    int used_on(cudaStream_t s) {
        if (!has_home || s == home) return PGCP_OK;
        if (!use_ev) PGCP_TRY_CUDA(cudaEventCreateWithFlags(&use_ev, cudaEventDisableTiming));
        PGCP_TRY_CUDA(cudaEventRecord(use_ev, s));
        PGCP_TRY_CUDA(cudaStreamWaitEvent(home, use_ev, 0));
        return PGCP_OK;
    }
    ~SolveSystem() {
        if (use_ev) cudaEventDestroy(use_ev);
    }
};

void free_system(void* p) { delete static_cast<SolveSystem*>(p); }

// PGCP_PCG_ORDER=prev (launch-order experiment): the last two-level solve's
// iteration counts; written and read by concurrent solves (flatten worker
// thread, harmonic on the caller's thread), hence the lock
static std::vector<int32_t> g_prev_iters;
static std::mutex g_prev_mu;

namespace {

constexpr int MAX_CLUSTER = 16;
constexpr int SMEM_LIMIT = 227 * 1024;
constexpr int RED_BYTES = 2 * MAX_CLUSTER * 2 * 8 + 32 * 2 * 8 + 64;

__device__ __forceinline__ int bsearch_off(const int64_t* __restrict__ off, int n, int64_t e) {
    int lo = 0, hi = n - 1;  // largest j with off[j] <= e
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (off[mid] <= e) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Paired sliced-ELL: slice s (32 rows) stores entry k of row `lane` at
// sl_ptr[s] + 64 (k / 2) + 2 lane + (k % 2); widths are even, so one 16-byte
// load per lane fetches two values (and one 8-byte load two columns) and a
// warp's load is a single contiguous 512 B (256 B) transaction.
__host__ __device__ __forceinline__ int64_t sell_pos(int64_t e0, int k, int lane) {
    return e0 + ((int64_t)(k >> 1) << 6) + (lane << 1) + (k & 1);
}

// ---------------------------------------------------------------------------
// system build kernels

__global__ void k_fixed_pins(int32_t nslot, const int32_t* __restrict__ pins, const int64_t* __restrict__ sv_off,
                             int32_t* __restrict__ fixed_ref) {
    GRID_STRIDE(j, nslot) {
        fixed_ref[sv_off[j] + pins[2 * j]] = 2 * (int)j;
        fixed_ref[sv_off[j] + pins[2 * j + 1]] = 2 * (int)j + 1;
    }
}

__global__ void k_fixed_list(int64_t nfixed, const int32_t* __restrict__ gid, const int32_t* __restrict__ comp_of,
                             const int32_t* __restrict__ slot_of_comp, const int64_t* __restrict__ vert_off,
                             const int64_t* __restrict__ sv_off, int32_t* __restrict__ fixed_ref) {
    GRID_STRIDE(i, nfixed) {
        int g = gid[i];
        int c = comp_of[g];
        int j = slot_of_comp[c];
        if (j < 0) continue;
        fixed_ref[sv_off[j] + (g - vert_off[c])] = (int32_t)i;
    }
}

__global__ void k_gather_i64(const int64_t* __restrict__ src, const int64_t* __restrict__ idx, int64_t n,
                             int64_t* __restrict__ dst) {
    GRID_STRIDE(i, n) dst[i] = src[idx[i]];
}

__global__ void k_unknown_flag(int64_t ne, const int32_t* __restrict__ fixed_ref, int32_t* __restrict__ flag) {
    GRID_STRIDE(e, ne) flag[e] = fixed_ref[e] < 0 ? 1 : 0;
}

__global__ void k_urow(int64_t ne, int32_t nslot, const int64_t* __restrict__ sv_off,
                       const int64_t* __restrict__ sl_off, const int64_t* __restrict__ uscan,
                       const int32_t* __restrict__ fixed_ref, int32_t* __restrict__ urow,
                       int32_t* __restrict__ rowsrc) {
    GRID_STRIDE(e, ne) {
        if (fixed_ref[e] >= 0) {
            urow[e] = -1;
            continue;
        }
        int j = bsearch_off(sv_off, nslot + 1, e);
        int64_t r = 32 * sl_off[j] + (uscan[e] - uscan[sv_off[j]]);
        urow[e] = (int32_t)r;
        rowsrc[r] = (int32_t)e;
    }
}

struct BuildArgs {
    int32_t nslot;
    const int32_t* comps;
    const int64_t* sv_off;
    const int64_t* sl_off;
    const int64_t* vert_off;
    const int64_t* row_ptr;
    const int32_t* col;
    const double* val;
    const int32_t* rowsrc;
    const int32_t* urow;
    const int32_t* fixed_ref;
    const double2* fv;
};

__global__ void k_slice_len(BuildArgs a, int64_t nslices, int64_t* __restrict__ len) {
    int lane = threadIdx.x & 31;
    int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t s = warp; s < nslices; s += nwarp) {
        int64_t r = 32 * s + lane;
        int cnt = 0;
        int e = a.rowsrc[r];
        if (e >= 0) {
            int j = bsearch_off(a.sv_off, a.nslot + 1, e);
            int c = a.comps[j];
            int self = (int)(e - a.sv_off[j]);
            int64_t g = a.vert_off[c] + self;
            for (int64_t q = a.row_ptr[g]; q < a.row_ptr[g + 1]; ++q) {
                int lc = a.col[q];
                if (lc != self && a.urow[a.sv_off[j] + lc] >= 0) ++cnt;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cnt = max(cnt, __shfl_xor_sync(0xffffffffu, cnt, o));
        cnt = (cnt + 1) & ~1;  // even widths (paired layout)
        if (lane == 0) len[s] = 32 * (int64_t)cnt;
    }
}

__global__ void k_fill_rows(BuildArgs a, int64_t rows, const int64_t* __restrict__ sl_ptr,
                            int32_t* __restrict__ ocol, double* __restrict__ oval, double* __restrict__ D,
                            double* __restrict__ Dinv, double2* __restrict__ bvec, int2* __restrict__ cpl,
                            double2* __restrict__ x) {
    GRID_STRIDE(r, rows) {
        int64_t s = r >> 5;
        int lane = (int)(r & 31);
        int64_t p0 = sl_ptr[s];
        int w = (int)((sl_ptr[s + 1] - p0) >> 5);
        int j = bsearch_off(a.sl_off, a.nslot + 1, s);
        int64_t rbase = 32 * a.sl_off[j];
        int selfrow = (int)(r - rbase);
        int e = a.rowsrc[r];
        int k = 0;
        double d = 1.0;
        double2 bb = make_double2(0.0, 0.0);
        if (e >= 0) {
            int c = a.comps[j];
            int self = (int)(e - a.sv_off[j]);
            int64_t g = a.vert_off[c] + self;
            for (int64_t q = a.row_ptr[g]; q < a.row_ptr[g + 1]; ++q) {
                int lc = a.col[q];
                double v = a.val[q];
                if (lc == self) {
                    d = v;
                    continue;
                }
                int64_t ee = a.sv_off[j] + lc;
                int ur = a.urow[ee];
                if (ur >= 0) {
                    ocol[sell_pos(p0, k, lane)] = (int32_t)(ur - rbase);
                    oval[sell_pos(p0, k, lane)] = v;
                    ++k;
                } else {
                    double2 f = a.fv[a.fixed_ref[ee]];
                    bb.x -= v * f.x;
                    bb.y -= v * f.y;
                }
            }
        }
        for (; k < w; ++k) {
            ocol[sell_pos(p0, k, lane)] = selfrow;
            oval[sell_pos(p0, k, lane)] = 0.0;
        }
        D[r] = d;
        Dinv[r] = 1.0 / d;
        bvec[r] = bb;
        cpl[r] = make_int2(-1, -1);
        x[r] = make_double2(0.0, 0.0);
    }
}

// harmonic right-hand side from the fixed values (the part of k_fill_rows that
// a prepared solve defers), already Jacobi-scaled: b = D^{-1/2} (-L_UF f)
__global__ void k_rhs_fixed(BuildArgs a, int64_t rows, const double* __restrict__ Dsq, double2* __restrict__ bvec) {
    GRID_STRIDE(r, rows) {
        const int e = a.rowsrc[r];
        double2 bb = make_double2(0.0, 0.0);
        if (e >= 0) {
            const int j = bsearch_off(a.sl_off, a.nslot + 1, r >> 5);
            const int c = a.comps[j];
            const int self = (int)(e - a.sv_off[j]);
            const int64_t g = a.vert_off[c] + self;
            for (int64_t q = a.row_ptr[g]; q < a.row_ptr[g + 1]; ++q) {
                const int lc = a.col[q];
                if (lc == self) continue;
                const int64_t ee = a.sv_off[j] + lc;
                if (a.urow[ee] < 0) {
                    const double2 f = a.fv[a.fixed_ref[ee]];
                    const double v = a.val[q];
                    bb.x -= v * f.x;
                    bb.y -= v * f.y;
                }
            }
        }
        const double d = Dsq[r];
        bvec[r] = make_double2(bb.x / d, bb.y / d);
    }
}

// DNCP boundary coupling (H = L + 2i M_xy) for every loop vertex of every slot
__global__ void k_coupling(int32_t nslot, const int32_t* __restrict__ comps, const int64_t* __restrict__ loop_off,
                           const int32_t* __restrict__ loop, const int64_t* __restrict__ sv_off,
                           const int64_t* __restrict__ sl_off, const int32_t* __restrict__ urow,
                           const int32_t* __restrict__ fixed_ref, const double2* __restrict__ fv,
                           int2* __restrict__ cpl, uint32_t* __restrict__ mask, double2* __restrict__ bvec,
                           int64_t total) {
    // flattened over (slot, loop position)
    GRID_STRIDE(t, total) {
        // find slot by scanning cumulative loop lengths (nslot small)
        int64_t acc = 0;
        int j = 0;
        for (; j < nslot; ++j) {
            int c = comps[j];
            int64_t nb = loop_off[c + 1] - loop_off[c];
            if (t < acc + nb) break;
            acc += nb;
        }
        if (j >= nslot) continue;
        int c = comps[j];
        int64_t lo = loop_off[c], nb = loop_off[c + 1] - lo;
        int64_t pos = t - acc;
        int u = loop[lo + pos];
        int nx = loop[lo + (pos + 1) % nb];
        int pv = loop[lo + (pos + nb - 1) % nb];
        int64_t eu = sv_off[j] + u, en = sv_off[j] + nx, ep = sv_off[j] + pv;
        int ru = urow[eu];
        if (ru < 0) continue;
        int64_t rbase = 32 * sl_off[j];
        int rn = urow[en], rp = urow[ep];
        cpl[ru] = make_int2(rn >= 0 ? (int)(rn - rbase) : -1, rp >= 0 ? (int)(rp - rbase) : -1);
        atomicOr(&mask[ru >> 5], 1u << (ru & 31));
        double2 bb = bvec[ru];
        if (rn < 0) {  // -(i/2) t_next
            double2 f = fv[fixed_ref[en]];
            bb.x += 0.5 * f.y;
            bb.y -= 0.5 * f.x;
        }
        if (rp < 0) {  // +(i/2) t_prev
            double2 f = fv[fixed_ref[ep]];
            bb.x -= 0.5 * f.y;
            bb.y += 0.5 * f.x;
        }
        bvec[ru] = bb;
    }
}

// ---------------------------------------------------------------------------
// Jacobi scaling: the solver iterates on D^{-1/2} H D^{-1/2} (unit diagonal),
// which is Jacobi-PCG in exact arithmetic and needs no diagonal loads per
// iteration. x = D^{-1/2} y.

__global__ void k_fill_i32(int32_t* __restrict__ p, int32_t n, int32_t v) {
    GRID_STRIDE(i, (int64_t)n) p[i] = v;
}

__global__ void k_dsq(int64_t rows, const double* __restrict__ D, double* __restrict__ Dsq) {
    GRID_STRIDE(r, rows) Dsq[r] = sqrt(D[r]);
}

__global__ void k_scale(int32_t nslot, const int64_t* __restrict__ sl_off, int64_t rows,
                        const int64_t* __restrict__ sl_ptr, const int32_t* __restrict__ col,
                        double* __restrict__ val, const double* __restrict__ Dsq, double2* __restrict__ b,
                        const int2* __restrict__ cpl, double2* __restrict__ cplc) {
    GRID_STRIDE(r, rows) {
        int64_t s = r >> 5;
        int lane = (int)(r & 31);
        int j = bsearch_off(sl_off, nslot + 1, s);
        int64_t rbase = 32 * sl_off[j];
        double dr = Dsq[r];
        int64_t e0 = sl_ptr[s];
        int w = (int)((sl_ptr[s + 1] - e0) >> 5);
        for (int k = 0; k < w; ++k) {
            int64_t e = sell_pos(e0, k, lane);
            val[e] = val[e] / (dr * Dsq[rbase + col[e]]);
        }
        double2 bb = b[r];
        b[r] = make_double2(bb.x / dr, bb.y / dr);
        int2 c = cpl[r];
        cplc[r] = make_double2(c.x >= 0 ? 0.5 / (dr * Dsq[rbase + c.x]) : 0.0,
                               c.y >= 0 ? 0.5 / (dr * Dsq[rbase + c.y]) : 0.0);
    }
}

__global__ void k_slot_dmax(const int64_t* __restrict__ sl_off, const double* __restrict__ D,
                            double* __restrict__ dmax) {
    __shared__ double red[32];
    int j = blockIdx.x;
    double m = 0;
    for (int64_t r = 32 * sl_off[j] + threadIdx.x; r < 32 * sl_off[j + 1]; r += blockDim.x) m = fmax(m, D[r]);
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, red[w]);
        dmax[j] = t;
    }
}

// column encoding for one cluster shape: a row owned by this CTA is the byte
// offset of its vector entry in the CTA's shared block; a row owned by
// another CTA of the cluster is (1 << 31) | (owner rank << 24) | byte offset.
// remote[s] = 1 if slice s has any remote entry (the kernel's slow path).
// enc16 holds the owner-local row index alone (rows per CTA < 2^16): the
// all-local slices stream 2-byte column codes instead of 4-byte ones.
__global__ void k_encode_cols(int32_t nslot, const int64_t* __restrict__ sl_off, int64_t nslices,
                              const int64_t* __restrict__ sl_ptr, const int32_t* __restrict__ col, int csize,
                              uint32_t* __restrict__ enc, uint16_t* __restrict__ enc16,
                              uint8_t* __restrict__ remote) {
    int lane = threadIdx.x & 31;
    int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t s = warp; s < nslices; s += nwarp) {
        int j = bsearch_off(sl_off, nslot + 1, s);
        int S = (int)(sl_off[j + 1] - sl_off[j]);
        int chunk = (S + csize - 1) / csize;
        int me = (int)(s - sl_off[j]) / chunk;  // owner of this slice
        bool rem = false;
        for (int64_t e = sl_ptr[s] + lane; e < sl_ptr[s + 1]; e += 32) {
            int c = col[e];
            int own = (c >> 5) / chunk;
            int off = c - 32 * own * chunk;
            if (own == me) {
                enc[e] = (uint32_t)(off * 16);
                enc16[e] = (uint16_t)off;
            } else {
                enc[e] = 0x80000000u | ((uint32_t)own << 24) | (uint32_t)(off * 16);
                enc16[e] = 0;
                rem = true;
            }
        }
        rem = __any_sync(0xffffffffu, rem);
        if (lane == 0) remote[s] = rem;
    }
}

// ---------------------------------------------------------------------------
// the solver

// ---------------------------------------------------------------------------
// Two-level preconditioner (additive coarse correction on top of Jacobi).
//
// Unknowns of every slot are reordered into geometric cells: principal frame
// of the slot's vertices, G quantile strips along the first axis, G cells per
// strip along the second (G = min(8, sqrt(nu / 128))). Cells cut by a CTA
// boundary of the cluster split become two aggregates, so every aggregate is
// a contiguous row range owned by one CTA. The coarse space holds the linear
// functions (1, u, v) of each aggregate (u, v local cell coordinates); in the
// Jacobi-scaled space W^ = D^{1/2} W and the preconditioner is
//     M^-1 = I + W^ E^-1 W^T,   E = W^T A^ W^   (complex Hermitian, dense)
// which is symmetric positive definite, so CG keeps its real alpha / beta.
// E^-1 is formed once per solve (Gauss-Jordan per slot, dependent coarse
// functions dropped).

constexpr int COARSE_GMAX = 8;
constexpr int AGG_MAX = 80;               // aggregates per slot: G^2 + CTA splits
constexpr int NC_MAX = 3 * AGG_MAX;       // coarse dofs per slot
constexpr int ITEMS_MAX = AGG_MAX;        // (aggregate, part) work items per CTA
constexpr int COARSE_BYTES = 3 * NC_MAX * 16 + ITEMS_MAX * 6 * 8;

// coarse weights of a row, (w0, w1, w2) as fp16 in 8 bytes: any fixed basis
// serves, and E is assembled from the same rounded values
__device__ __forceinline__ uint2 cw_make(double a, double b, double c) {
    __half2 h0 = __floats2half2_rn((float)a, (float)b);
    __half2 h1 = __floats2half2_rn((float)c, 0.0f);
    return make_uint2(*reinterpret_cast<unsigned int*>(&h0), *reinterpret_cast<unsigned int*>(&h1));
}
__device__ __forceinline__ float4 cw_get(const uint2* __restrict__ w, int64_t r) {
    uint2 u = w[r];
    __half2 h0 = *reinterpret_cast<__half2*>(&u.x);
    __half2 h1 = *reinterpret_cast<__half2*>(&u.y);
    float2 a = __half22float2(h0), b = __half22float2(h1);
    return make_float4(a.x, a.y, b.x, 0.0f);
}

__host__ __device__ inline int coarse_G(int64_t nu, int gmax) {
    int g = (int)sqrt((double)nu / 128.0);
    return g < 1 ? 1 : (g > gmax ? gmax : g);
}

__device__ __forceinline__ uint32_t f32_order(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// symmetric 3x3 eigenvectors by cyclic Jacobi; columns of v sorted by
// decreasing eigenvalue
__device__ void eig3(double a[3][3], double v[3][3]) {
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) v[i][j] = (i == j) ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 16; ++sweep) {
        double off = fabs(a[0][1]) + fabs(a[0][2]) + fabs(a[1][2]);
        if (off == 0.0) break;
        for (int p = 0; p < 2; ++p)
            for (int q = p + 1; q < 3; ++q) {
                if (a[p][q] == 0.0) continue;
                double th = (a[q][q] - a[p][p]) / (2.0 * a[p][q]);
                double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
                double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < 3; ++k) {  // a = J^T a J
                    double akp = a[k][p], akq = a[k][q];
                    a[k][p] = c * akp - s * akq;
                    a[k][q] = s * akp + c * akq;
                }
                for (int k = 0; k < 3; ++k) {
                    double apk = a[p][k], aqk = a[q][k];
                    a[p][k] = c * apk - s * aqk;
                    a[q][k] = s * apk + c * aqk;
                }
                for (int k = 0; k < 3; ++k) {
                    double vkp = v[k][p], vkq = v[k][q];
                    v[k][p] = c * vkp - s * vkq;
                    v[k][q] = s * vkp + c * vkq;
                }
            }
    }
    int o[3] = {0, 1, 2};
    for (int i = 0; i < 3; ++i)
        for (int j = i + 1; j < 3; ++j)
            if (a[o[j]][o[j]] > a[o[i]][o[i]]) {
                int t = o[i];
                o[i] = o[j];
                o[j] = t;
            }
    double w[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) w[i][j] = v[i][o[j]];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) v[i][j] = w[i][j];
}

__device__ __forceinline__ const double* vtx_of(int64_t e, int j, const int32_t* comps, const int64_t* sv_off,
                                                const int64_t* vert_off, const int32_t* vmap, const double* V) {
    int c = comps[j];
    int v = vmap[vert_off[c] + (e - sv_off[j])];
    return V + 3 * (int64_t)v;
}

// per slot: mean and principal frame (e1, e2) of the unknown vertices
__global__ void k_pca(int32_t nslot, const int32_t* __restrict__ comps, const int64_t* __restrict__ sv_off,
                      const int64_t* __restrict__ vert_off, const int32_t* __restrict__ vmap,
                      const double* __restrict__ V, const int32_t* __restrict__ fixed_ref,
                      double* __restrict__ frame) {
    __shared__ double red[10][32];
    const int j = blockIdx.x;
    double acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t e = sv_off[j] + threadIdx.x; e < sv_off[j + 1]; e += blockDim.x) {
        if (fixed_ref[e] >= 0) continue;
        const double* p = vtx_of(e, j, comps, sv_off, vert_off, vmap, V);
        double x = p[0], y = p[1], z = p[2];
        acc[0] += 1.0;
        acc[1] += x;
        acc[2] += y;
        acc[3] += z;
        acc[4] += x * x;
        acc[5] += x * y;
        acc[6] += x * z;
        acc[7] += y * y;
        acc[8] += y * z;
        acc[9] += z * z;
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = 0; i < 10; ++i) {
        double t = warp_sum(acc[i]);
        if (lane == 0) red[i][w] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s[10];
        for (int i = 0; i < 10; ++i) {
            s[i] = 0.0;
            for (int q = 0; q < nw; ++q) s[i] += red[i][q];
        }
        double n = s[0] > 0 ? s[0] : 1.0;
        double m[3] = {s[1] / n, s[2] / n, s[3] / n};
        double a[3][3];
        a[0][0] = s[4] / n - m[0] * m[0];
        a[0][1] = a[1][0] = s[5] / n - m[0] * m[1];
        a[0][2] = a[2][0] = s[6] / n - m[0] * m[2];
        a[1][1] = s[7] / n - m[1] * m[1];
        a[1][2] = a[2][1] = s[8] / n - m[1] * m[2];
        a[2][2] = s[9] / n - m[2] * m[2];
        double v[3][3];
        eig3(a, v);
        double* f = frame + 9 * j;
        for (int i = 0; i < 3; ++i) {
            f[i] = m[i];
            f[3 + i] = v[i][0];
            f[6 + i] = v[i][1];
        }
    }
}

// projected coordinates of every unknown and the first sort key (slot, px)
__global__ void k_proj(int64_t ne, int32_t nslot, const int32_t* __restrict__ comps,
                       const int64_t* __restrict__ sv_off, const int64_t* __restrict__ vert_off,
                       const int32_t* __restrict__ vmap, const double* __restrict__ V,
                       const int32_t* __restrict__ fixed_ref, const int64_t* __restrict__ uscan,
                       const double* __restrict__ frame, float2* __restrict__ pxy,
                       unsigned long long* __restrict__ key, int32_t* __restrict__ val,
                       uint32_t* __restrict__ bbox) {
    GRID_STRIDE(e, ne) {
        if (fixed_ref[e] >= 0) continue;
        int j = bsearch_off(sv_off, nslot + 1, e);
        const double* p = vtx_of(e, j, comps, sv_off, vert_off, vmap, V);
        const double* f = frame + 9 * j;
        double dx = p[0] - f[0], dy = p[1] - f[1], dz = p[2] - f[2];
        float px = (float)(dx * f[3] + dy * f[4] + dz * f[5]);
        float py = (float)(dx * f[6] + dy * f[7] + dz * f[8]);
        int64_t u = uscan[e];
        pxy[u] = make_float2(px, py);
        key[u] = ((unsigned long long)j << 32) | f32_order(px);
        val[u] = (int32_t)e;
        // box of the slot: one atomic per distinct slot per warp
        const unsigned act = __activemask();
        const unsigned peers = __match_any_sync(act, j);
        const uint32_t ox = f32_order(px), oy = f32_order(py);
        const uint32_t x0 = __reduce_min_sync(peers, ox), x1 = __reduce_max_sync(peers, ox);
        const uint32_t y0 = __reduce_min_sync(peers, oy), y1 = __reduce_max_sync(peers, oy);
        if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) {
            atomicMin(&bbox[4 * j], x0);
            atomicMax(&bbox[4 * j + 1], x1);
            atomicMin(&bbox[4 * j + 2], y0);
            atomicMax(&bbox[4 * j + 3], y1);
        }
    }
}

__device__ __forceinline__ float f32_unorder(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

__device__ __forceinline__ uint32_t spread16(uint32_t x) {
    x &= 0xffffu;
    x = (x | (x << 8)) & 0x00ff00ffu;
    x = (x | (x << 4)) & 0x0f0f0f0fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    return x;
}

// third key: (slot, cell, Morton code of the position in the slot's box), so
// rows inside a cell follow a Z-curve (neighbours stay close in the row order)
__global__ void k_cell_keys(int64_t nU, const unsigned long long* __restrict__ key_in,
                            const int32_t* __restrict__ val_in, const int64_t* __restrict__ sv_off,
                            const int64_t* __restrict__ uscan, const float2* __restrict__ pxy,
                            const uint32_t* __restrict__ bbox, int gmax, unsigned long long* __restrict__ key,
                            int32_t* __restrict__ val) {
    GRID_STRIDE(k, nU) {
        unsigned long long kk = key_in[k];
        int j = (int)(kk >> 40);
        int ax = (int)((kk >> 32) & 0xff);
        int32_t e = val_in[k];
        int64_t us = uscan[sv_off[j]], nu = uscan[sv_off[j + 1]] - us;
        int G = coarse_G(nu, gmax);
        int64_t rho = k - us;
        int64_t s0 = (ax * nu + G - 1) / G, s1 = ((ax + 1) * nu + G - 1) / G;
        int ay = s1 > s0 ? (int)((rho - s0) * G / (s1 - s0)) : 0;
        float2 p = pxy[uscan[e]];
        float x0 = f32_unorder(bbox[4 * j]), x1 = f32_unorder(bbox[4 * j + 1]);
        float y0 = f32_unorder(bbox[4 * j + 2]), y1 = f32_unorder(bbox[4 * j + 3]);
        float ex = x1 > x0 ? 65535.0f / (x1 - x0) : 0.0f, ey = y1 > y0 ? 65535.0f / (y1 - y0) : 0.0f;
        uint32_t qx = (uint32_t)fminf(65535.0f, fmaxf(0.0f, (p.x - x0) * ex));
        uint32_t qy = (uint32_t)fminf(65535.0f, fmaxf(0.0f, (p.y - y0) * ey));
        uint32_t mort = spread16(qx) | (spread16(qy) << 1);
        key[k] = ((unsigned long long)j << 40) | ((unsigned long long)(ax * G + ay) << 32) | mort;
        val[k] = e;
    }
}

// strip index along the first axis and the second sort key (slot, strip, py)
__global__ void k_strip(int64_t nU, const unsigned long long* __restrict__ key_in, const int32_t* __restrict__ val_in,
                        const int64_t* __restrict__ sv_off, const int64_t* __restrict__ uscan,
                        const float2* __restrict__ pxy, int gmax, unsigned long long* __restrict__ key,
                        int32_t* __restrict__ val) {
    GRID_STRIDE(k, nU) {
        int j = (int)(key_in[k] >> 32);
        int32_t e = val_in[k];
        int64_t us = uscan[sv_off[j]], nu = uscan[sv_off[j + 1]] - us;
        int G = coarse_G(nu, gmax);
        int64_t rho = k - us;
        int ax = (int)(rho * G / nu);
        float py = pxy[uscan[e]].y;
        key[k] = ((unsigned long long)j << 40) | ((unsigned long long)ax << 32) | f32_order(py);
        val[k] = e;
    }
}

// final row numbering (slot-local row = rank in the (strip, py) order) and the
// cell of every row
__global__ void k_rows_by_cell(int64_t nU, const unsigned long long* __restrict__ key_in,
                               const int32_t* __restrict__ val_in, const int64_t* __restrict__ sv_off,
                               const int64_t* __restrict__ sl_off, const int64_t* __restrict__ uscan,
                               const float2* __restrict__ pxy, int gmax, int32_t* __restrict__ urow,
                               int32_t* __restrict__ rowsrc, int32_t* __restrict__ cell,
                               float2* __restrict__ pxy_row) {
    GRID_STRIDE(k, nU) {
        unsigned long long kk = key_in[k];
        int j = (int)(kk >> 40);
        int32_t e = val_in[k];
        int64_t us = uscan[sv_off[j]];
        int64_t r = 32 * sl_off[j] + (k - us);
        urow[e] = (int32_t)r;
        rowsrc[r] = e;
        cell[r] = (int)((kk >> 32) & 0xff);
        pxy_row[r] = pxy[uscan[e]];
    }
}

// aggregate starts: first row of a slot, a cell change, or a CTA boundary
__global__ void k_agg_flag(int64_t rows, int32_t nslot, const int64_t* __restrict__ sl_off,
                           const int64_t* __restrict__ nu_slot, const int32_t* __restrict__ cell, int csize,
                           int32_t* __restrict__ flag) {
    GRID_STRIDE(r, rows) {
        int j = bsearch_off(sl_off, nslot + 1, r >> 5);
        int64_t lr = r - 32 * sl_off[j];
        int64_t S = sl_off[j + 1] - sl_off[j];
        int64_t chunk = (S + csize - 1) / csize;
        int f = 0;
        if (lr == 0) {
            f = 1;
        } else if (lr < nu_slot[j]) {
            int64_t cta = (lr >> 5) / chunk, ctap = ((lr - 1) >> 5) / chunk;
            f = (cell[r] != cell[r - 1] || cta != ctap) ? 1 : 0;
        }
        flag[r] = f;
    }
}

__global__ void k_agg_index(int64_t rows, const int32_t* __restrict__ flag, const int64_t* __restrict__ scan,
                            int32_t* __restrict__ aggr, int32_t* __restrict__ aoff) {
    GRID_STRIDE(r, rows) {
        int32_t a = (int32_t)(scan[r] + flag[r] - 1);
        aggr[r] = a;
        if (flag[r]) aoff[a] = (int32_t)r;
    }
}

__global__ void k_slot_abase(int32_t nslot, const int64_t* __restrict__ sl_off, const int64_t* __restrict__ scan,
                             int64_t* __restrict__ abase) {
    GRID_STRIDE(j, nslot + 1) abase[j] = scan[32 * sl_off[j]];
}

// per aggregate: centroid and extent of the cell coordinates -> coarse weights
// w^ = sqrt(D) (1, u, v) per real row (padding rows: 0)
__global__ void k_agg_weights(int32_t nagg_total, const int32_t* __restrict__ aoff, int32_t nslot,
                              const int64_t* __restrict__ sl_off, const int64_t* __restrict__ nu_slot,
                              const float2* __restrict__ pxy_row, const double* __restrict__ Dsq,
                              uint2* __restrict__ wr) {
    __shared__ double red[3][32];
    __shared__ double s_c[3];
    const int A = blockIdx.x;
    const int64_t r0 = aoff[A], r1 = aoff[A + 1];
    const int j = bsearch_off(sl_off, nslot + 1, r0 >> 5);
    const int64_t rend = min(r1, 32 * sl_off[j] + nu_slot[j]);  // real rows
    double sx = 0, sy = 0, n = 0;
    for (int64_t r = r0 + threadIdx.x; r < rend; r += blockDim.x) {
        float2 p = pxy_row[r];
        sx += p.x;
        sy += p.y;
        n += 1.0;
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    sx = warp_sum(sx);
    sy = warp_sum(sy);
    n = warp_sum(n);
    if (lane == 0) {
        red[0][w] = sx;
        red[1][w] = sy;
        red[2][w] = n;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0, b = 0, c = 0;
        for (int q = 0; q < nw; ++q) {
            a += red[0][q];
            b += red[1][q];
            c += red[2][q];
        }
        s_c[0] = c > 0 ? a / c : 0.0;
        s_c[1] = c > 0 ? b / c : 0.0;
    }
    __syncthreads();
    const double cx = s_c[0], cy = s_c[1];
    double m = 0.0;
    for (int64_t r = r0 + threadIdx.x; r < rend; r += blockDim.x) {
        float2 p = pxy_row[r];
        m = fmax(m, fmax(fabs(p.x - cx), fabs(p.y - cy)));
    }
    m = warp_max(m);
    __syncthreads();
    if (lane == 0) red[0][w] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0;
        for (int q = 0; q < nw; ++q) t = fmax(t, red[0][q]);
        s_c[2] = t;
    }
    __syncthreads();
    // linear functions only on aggregates with enough rows to carry them
    // (slivers cut off by a CTA boundary keep just the constant)
    const double sc = (s_c[2] > 0 && rend - r0 >= 16) ? 1.0 / s_c[2] : 0.0;
    for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
        if (r < rend) {
            float2 p = pxy_row[r];
            double d = Dsq[r];
            wr[r] = cw_make(d, d * (p.x - cx) * sc, d * (p.y - cy) * sc);
        } else {
            wr[r] = make_uint2(0u, 0u);
        }
    }
}


// E = W^T A^ W^ restricted to the rows of one aggregate (block per
// aggregate). A^ = I + scaled off-diagonals + i (cn e_next - cp e_prev).
// Every warp takes 32-row chunks; per neighbour aggregate b each lane forms
// y_t = sum_j A^_ij w_j[t] over its row's entries in b, the 9 products
// w_i[s] y_t are warp-summed into the warp's accumulator, and the warps'
// accumulators are added in warp order (deterministic).
constexpr int E_WARPS = 8;
constexpr int E_NBMAX = 16;  // neighbour aggregates per aggregate

__global__ void __launch_bounds__(32 * E_WARPS) k_coarse_E(
        int32_t nslot, const int64_t* __restrict__ sl_off, const int64_t* __restrict__ sl_ptr,
        const uint32_t* __restrict__ sl_mask, const int32_t* __restrict__ col, const double* __restrict__ val,
        const int2* __restrict__ cpl, const double2* __restrict__ cplc, const int32_t* __restrict__ aoff,
        const int32_t* __restrict__ aggr, const int64_t* __restrict__ abase, const uint2* __restrict__ wr,
        const int64_t* __restrict__ eoff, double2* __restrict__ E, int* __restrict__ overflow) {
    __shared__ int s_flag[AGG_MAX];
    __shared__ int s_nb[AGG_MAX];
    __shared__ int s_cnt;
    __shared__ double2 acc[E_WARPS][9 * E_NBMAX];
    const int A = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r0 = aoff[A], r1 = aoff[A + 1];
    const int j = bsearch_off(sl_off, nslot + 1, r0 >> 5);
    const int64_t rbase = 32 * sl_off[j];
    const int a0 = (int)abase[j];
    const int nag = (int)(abase[j + 1] - a0);
    const int nc = 3 * nag;
    for (int i = threadIdx.x; i < AGG_MAX; i += blockDim.x) s_flag[i] = 0;
    for (int i = threadIdx.x; i < E_WARPS * 9 * E_NBMAX; i += blockDim.x)
        acc[i / (9 * E_NBMAX)][i % (9 * E_NBMAX)] = make_double2(0.0, 0.0);
    __syncthreads();
    for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
        const int64_t s = r >> 5;
        const int ln = (int)(r & 31);
        const int64_t e0 = sl_ptr[s];
        const int wdt = (int)((sl_ptr[s + 1] - e0) >> 5);
        s_flag[aggr[r] - a0] = 1;
        for (int k = 0; k < wdt; ++k) s_flag[aggr[rbase + col[sell_pos(e0, k, ln)]] - a0] = 1;
        if (sl_mask[s] & (1u << ln)) {
            int2 nb = cpl[r];
            if (nb.x >= 0) s_flag[aggr[rbase + nb.x] - a0] = 1;
            if (nb.y >= 0) s_flag[aggr[rbase + nb.y] - a0] = 1;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int c = 0;
        for (int i = 0; i < nag && i < AGG_MAX; ++i)
            if (s_flag[i]) {
                if (c < E_NBMAX) s_nb[c] = i;
                ++c;
            }
        if (c > E_NBMAX) {
            atomicExch(overflow, 1);
            c = E_NBMAX;
        }
        s_cnt = c;
    }
    __syncthreads();
    const int NB = s_cnt;
    for (int64_t cbase = r0 + 32 * warp; cbase < r1; cbase += 32 * E_WARPS) {
        const int64_t r = cbase + lane;
        const bool have = r < r1;
        float4 wi = make_float4(0.f, 0.f, 0.f, 0.f);
        int64_t e0 = 0;
        int wdt = 0, ln = 0, ai = -1;
        bool cp = false;
        int2 nb = make_int2(-1, -1);
        double2 cc = make_double2(0.0, 0.0);
        if (have) {
            wi = cw_get(wr, r);
            const int64_t s = r >> 5;
            ln = (int)(r & 31);
            e0 = sl_ptr[s];
            wdt = (int)((sl_ptr[s + 1] - e0) >> 5);
            ai = aggr[r];
            cp = (sl_mask[s] >> ln) & 1u;
            if (cp) {
                nb = cpl[r];
                cc = cplc[r];
            }
        }
        for (int bi = 0; bi < NB; ++bi) {
            const int b = s_nb[bi] + a0;
            double yr[3] = {0.0, 0.0, 0.0}, yi[3] = {0.0, 0.0, 0.0};
            if (have) {
                if (ai == b) {
                    yr[0] += wi.x;
                    yr[1] += wi.y;
                    yr[2] += wi.z;
                }
                for (int k = 0; k < wdt; ++k) {
                    const int64_t q = sell_pos(e0, k, ln);
                    const int64_t rc = rbase + col[q];
                    if (aggr[rc] == b) {
                        const float4 wc = cw_get(wr, rc);
                        const double v = val[q];
                        yr[0] += v * wc.x;
                        yr[1] += v * wc.y;
                        yr[2] += v * wc.z;
                    }
                }
                if (cp) {
                    if (nb.x >= 0 && aggr[rbase + nb.x] == b) {
                        const float4 wc = cw_get(wr, rbase + nb.x);
                        yi[0] += cc.x * wc.x;
                        yi[1] += cc.x * wc.y;
                        yi[2] += cc.x * wc.z;
                    }
                    if (nb.y >= 0 && aggr[rbase + nb.y] == b) {
                        const float4 wc = cw_get(wr, rbase + nb.y);
                        yi[0] -= cc.y * wc.x;
                        yi[1] -= cc.y * wc.y;
                        yi[2] -= cc.y * wc.z;
                    }
                }
            }
            const double ws[3] = {(double)wi.x, (double)wi.y, (double)wi.z};
#pragma unroll
            for (int sx = 0; sx < 3; ++sx)
#pragma unroll
                for (int t = 0; t < 3; ++t) {
                    double cr = warp_sum(ws[sx] * yr[t]);
                    double ci = warp_sum(ws[sx] * yi[t]);
                    if (lane == 0) {
                        double2& a = acc[warp][(sx * E_NBMAX + bi) * 3 + t];
                        a.x += cr;
                        a.y += ci;
                    }
                }
        }
    }
    __syncthreads();
    double2* Eslot = E + eoff[j];
    const int arow = A - a0;
    for (int t = threadIdx.x; t < 9 * NB; t += blockDim.x) {
        const int sx = t / (3 * NB), rem = t % (3 * NB), bi = rem / 3, tt = rem % 3;
        double2 v = make_double2(0.0, 0.0);
        for (int w = 0; w < E_WARPS; ++w) {
            const double2 a = acc[w][(sx * E_NBMAX + bi) * 3 + tt];
            v.x += a.x;
            v.y += a.y;
        }
        Eslot[(int64_t)(3 * arow + sx) * nc + 3 * s_nb[bi] + tt] = v;
    }
}

// In-place Gauss-Jordan inverse of every slot's Hermitian positive
// semi-definite E on a thread-block cluster: the rows are spread over the
// CTAs' shared memory, the pivot row is broadcast through DSMEM (double
// buffered, one cluster barrier per pivot). Coarse functions whose pivot
// falls below 1e-10 of the largest diagonal are dependent and dropped
// (row/col zeroed). Output: E^-1, made exactly Hermitian.
constexpr int INV_THREADS = 512;

__device__ __forceinline__ double2 cm(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__global__ void __launch_bounds__(INV_THREADS, 1) k_coarse_inv(const int64_t* __restrict__ abase,
                                                               const int64_t* __restrict__ eoff,
                                                               double2* __restrict__ E) {
    extern __shared__ __align__(16) unsigned char smem[];
    cg::cluster_group cl = cg::this_cluster();
    const int CS = (int)cl.num_blocks();
    const int rank = (int)cl.block_rank();
    const int j = blockIdx.x / CS;
    const int n = 3 * (int)(abase[j + 1] - abase[j]);
    const int rpc = (n + CS - 1) / CS;                 // rows per CTA
    const int i0 = min(n, rank * rpc), i1 = min(n, i0 + rpc);
    const int nr = i1 - i0;
    double2* Ml = reinterpret_cast<double2*>(smem);    // [rpc][n] my rows
    double2* rowk = Ml + (size_t)rpc * n;              // [2 parity][2 rows][n] pivot rows (broadcast)
    double2* colk = rowk + 4 * n;                      // [rpc][2] my entries of the pivot columns
    double* s_diag = reinterpret_cast<double*>(colk + 2 * rpc);  // [n] original diagonal
    double2* M = E + eoff[j];
    for (int t = threadIdx.x; t < nr * n; t += INV_THREADS) Ml[t] = M[(int64_t)i0 * n + t];
    for (int i = threadIdx.x; i < n; i += INV_THREADS) s_diag[i] = M[(int64_t)i * n + i].x;
    __syncthreads();
    // pivot rows k, k+1 -> every CTA (owners write through DSMEM)
    int par = 0;
    auto publish = [&](int k, int pr) {
        for (int q = 0; q < 2; ++q) {
            const int r = k + q;
            if (r < n && r >= i0 && r < i1)
                for (int t = threadIdx.x; t < n * CS; t += INV_THREADS) {
                    const int c = t / CS, dst = t - c * CS;
                    double2* rk = cl.map_shared_rank(rowk + (2 * pr + q) * n, dst);
                    rk[c] = Ml[(size_t)(r - i0) * n + c];
                }
        }
    };
    publish(0, par);
    cl.sync();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NWI = INV_THREADS / 32;
    for (int k = 0; k < n;) {
        const double2* R0 = rowk + (2 * par) * n;
        const double2* R1 = R0 + n;
        // a pivot that lost all but 1e-8 of its original diagonal means the
        // coarse function is (numerically) dependent on the previous ones;
        // two pivots per cluster barrier when the 2x2 block is safe
        const double a = R0[k].x;
        const bool drop = !(a > 1e-8 * s_diag[k]) || !(s_diag[k] > 0.0);
        bool two = false;
        double2 bb = make_double2(0.0, 0.0);
        double d = 0.0;
        if (!drop && k + 1 < n) {
            bb = R0[k + 1];
            d = R1[k + 1].x;
            const double schur = d - (bb.x * bb.x + bb.y * bb.y) / a;
            two = schur > 1e-8 * s_diag[k + 1] && s_diag[k + 1] > 0.0;
        }
        for (int i = threadIdx.x; i < nr; i += INV_THREADS) {
            colk[2 * i] = Ml[(size_t)i * n + k];
            if (two) colk[2 * i + 1] = Ml[(size_t)i * n + k + 1];
        }
        __syncthreads();
        if (drop) {
            for (int i = warp; i < nr; i += NWI)
                for (int c = lane; c < n; c += 32)
                    if (i0 + i == k || c == k) Ml[(size_t)i * n + c] = make_double2(0.0, 0.0);
        } else if (!two) {
            const double ip = 1.0 / a;
            for (int i = warp; i < nr; i += NWI) {
                const int gi = i0 + i;
                const double2 ca = colk[2 * i];
                double2* row = Ml + (size_t)i * n;
                for (int c = lane; c < n; c += 32) {
                    const double2 b = R0[c];
                    double2 v;
                    if (gi == k) {
                        v = (c == k) ? make_double2(ip, 0.0) : make_double2(b.x * ip, b.y * ip);
                    } else if (c == k) {
                        v = make_double2(-ca.x * ip, -ca.y * ip);
                    } else {
                        const double2 m = row[c];
                        const double2 t = cm(ca, b);
                        v = make_double2(m.x - t.x * ip, m.y - t.y * ip);
                    }
                    row[c] = v;
                }
            }
        } else {
            // P = [[a, b], [conj(b), d]], P^-1 = [[d, -b], [-conj(b), a]] / det
            const double det = a * d - (bb.x * bb.x + bb.y * bb.y);
            const double id = 1.0 / det;
            const double2 P00 = make_double2(d * id, 0.0), P11 = make_double2(a * id, 0.0);
            const double2 P01 = make_double2(-bb.x * id, -bb.y * id), P10 = make_double2(-bb.x * id, bb.y * id);
            for (int i = warp; i < nr; i += NWI) {
                const int gi = i0 + i;
                double2* row = Ml + (size_t)i * n;
                if (gi == k || gi == k + 1) {
                    const double2 Q0 = gi == k ? P00 : P10, Q1 = gi == k ? P01 : P11;
                    for (int c = lane; c < n; c += 32) {
                        double2 v;
                        if (c == k) v = Q0;
                        else if (c == k + 1) v = Q1;
                        else {
                            const double2 u0 = cm(Q0, R0[c]), u1 = cm(Q1, R1[c]);
                            v = make_double2(u0.x + u1.x, u0.y + u1.y);
                        }
                        row[c] = v;
                    }
                } else {
                    const double2 C0 = colk[2 * i], C1 = colk[2 * i + 1];
                    const double2 a0 = cm(C0, P00), a1 = cm(C1, P10), b0 = cm(C0, P01), b1 = cm(C1, P11);
                    const double2 T0 = make_double2(a0.x + a1.x, a0.y + a1.y);
                    const double2 T1 = make_double2(b0.x + b1.x, b0.y + b1.y);
                    for (int c = lane; c < n; c += 32) {
                        double2 v;
                        if (c == k) v = make_double2(-T0.x, -T0.y);
                        else if (c == k + 1) v = make_double2(-T1.x, -T1.y);
                        else {
                            const double2 m = row[c];
                            const double2 u0 = cm(T0, R0[c]), u1 = cm(T1, R1[c]);
                            v = make_double2(m.x - u0.x - u1.x, m.y - u0.y - u1.y);
                        }
                        row[c] = v;
                    }
                }
            }
        }
        __syncthreads();
        k += two ? 2 : 1;
        par ^= 1;
        publish(k, par);
        cl.sync();
    }
    for (int t = threadIdx.x; t < nr * n; t += INV_THREADS) M[(int64_t)i0 * n + t] = Ml[t];
}

// float copy of (E^-1 + E^-H) / 2: exactly Hermitian after rounding (the
// preconditioner stays symmetric), rows padded to a multiple of 8 columns
template <typename ET>
__device__ __forceinline__ ET mk_et(double x, double y);
template <>
__device__ __forceinline__ float2 mk_et<float2>(double x, double y) { return make_float2((float)x, (float)y); }
template <>
__device__ __forceinline__ double2 mk_et<double2>(double x, double y) { return make_double2(x, y); }

template <typename ET>
__global__ void k_hermitize(const int64_t* __restrict__ abase, const int64_t* __restrict__ eoff,
                            const double2* __restrict__ E, const int64_t* __restrict__ eoff32,
                            ET* __restrict__ E32) {
    const int j = blockIdx.x;
    const int n = 3 * (int)(abase[j + 1] - abase[j]);
    const int np = (n + 7) & ~7;
    const double2* M = E + eoff[j];
    ET* O = E32 + eoff32[j];
    for (int64_t t = threadIdx.x; t < (int64_t)n * np; t += blockDim.x) {
        const int i = (int)(t / np), c = (int)(t % np);
        if (c >= n) {
            O[t] = mk_et<ET>(0.0, 0.0);
            continue;
        }
        // the upper triangle is the reference; the lower one is its exact
        // conjugate after rounding
        const double2 a = M[(int64_t)i * n + c], b = M[(int64_t)c * n + i];
        if (c < i) {
            const ET u = mk_et<ET>(0.5 * (b.x + a.x), 0.5 * (b.y - a.y));
            O[t] = mk_et<ET>((double)u.x, -(double)u.y);
        } else {
            O[t] = mk_et<ET>(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
        }
    }
}

struct CoarseArgs {
    const int64_t* abase;    // slot -> first aggregate (global id), nslot + 1
    const int32_t* aoff;     // aggregate -> first row (global padded row), NA + 1
    const uint2* wr;         // row -> scaled coarse weights (w0, w1, w2) as fp16
    const void* einvh;       // per slot Hermitian E^-1 (float2 or double2), row-major, rows padded to 8 columns
    const int64_t* eoff32;   // slot -> offset into einvh
    double2* p;              // search direction (rows)
};

struct PcgArgs {
    const int64_t* sl_off;   // slot -> first slice
    const int64_t* sl_ptr;   // slice -> first entry
    const uint32_t* sl_mask;
    const int32_t* col;
    const uint32_t* enc;     // encoded columns (see k_encode_cols)
    const uint16_t* enc16;   // 16-bit local codes (all-local slices; k_pcg2)
    const uint8_t* remote;   // slice has entries owned by another CTA
    const double* val;       // scaled off-diagonal values
    const double* D;         // unscaled diagonal (norms of the unscaled residual)
    const double* dmax;      // per slot max D (stopping bound)
    const int2* cpl;
    const double2* cplc;     // scaled coupling coefficients (next, prev)
    const double2* b;        // scaled rhs
    double2* x;              // scaled solution y
    int32_t* iters;
    double* res;             // per slot [8]
    double tol2;             // rtol^2
    int32_t maxit;
    int32_t chunk_cap;       // slices per CTA the smem was sized for
    long long* timing;       // optional: per CTA [phaseA, red1, phaseB, red2] cycles (iterations 64..191)
    const int32_t* order;    // k_pcg2: cluster -> slot launch order (nullptr: identity)
    double* hist;            // k_pcg2 (PGCP_PCG_HIST): per slot [HIST_K][3] alpha, rr, beta of the first iterations
    int32_t x0;              // k_pcg2: start from the coarse solution x0 = Q b (PGCP_PCG_X0)
    int32_t ncb;             // k_pcg2 shared layout: gbuf stride (>= every slot's nc)
    int32_t mu_cap;          // ... own coarse rows per CTA
    int32_t items_cap;       // ... (aggregate, part) work items per CTA
    CoarseArgs C;
};

// deterministic cluster-wide sum of two doubles: warp -> CTA (fixed order) ->
// every CTA receives every CTA's partial through DSMEM -> fixed-order sum
template <int NW>
__device__ __forceinline__ double2 cluster_sum2(cg::cluster_group& cl, int csize, int rank, double a, double b,
                                                double2* s_warp, double2* s_slot, int parity) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    a = warp_sum(a);
    b = warp_sum(b);
    if (lane == 0) s_warp[w] = make_double2(a, b);
    __syncthreads();
    if (w == 0) {
        double2 v = (lane < NW) ? s_warp[lane] : make_double2(0.0, 0.0);
        double ta = warp_sum(v.x), tb = warp_sum(v.y);
        if (lane < csize) {
            double2* dst = cl.map_shared_rank(s_slot + parity * MAX_CLUSTER, lane);
            dst[rank] = make_double2(ta, tb);
        }
    }
    cl.sync();
    double2 t = make_double2(0.0, 0.0);
    const double2* src = s_slot + parity * MAX_CLUSTER;
    for (int r = 0; r < csize; ++r) {
        t.x += src[r].x;
        t.y += src[r].y;
    }
    return t;
}

constexpr int KPF = 8;  // prefetched off-diagonal entries per row (4 pairs)
constexpr int HIST_K = 128;  // PGCP_PCG_HIST: iterations recorded per slot
constexpr int KPF2 = 6;  // k_pcg2 (register budget: p is prefetched as well)

template <int KP>
struct SliceBufT {
    double2 y;    // this lane's solution entry (updated in place, one owner thread)
    double2 p;    // this lane's search direction (k_pcg2: p lives in global memory)
    int w;        // even width
    int remote;   // any entry of the slice owned by another CTA
    int off;      // entry offset of this lane's first pair, relative to the CTA's first entry
    uint32_t c[KP];
    double v[KP];
};
using SliceBuf = SliceBufT<KPF>;

template <int KP>
__device__ __forceinline__ void slice_load(SliceBufT<KP>& B, const double* __restrict__ valc,
                                           const uint32_t* __restrict__ encc, const int* s_ent, const int* s_w,
                                           int ls, int nloc, int lane, const double2* yrow, bool need_y,
                                           const double2* prow = nullptr,
                                           const uint16_t* __restrict__ enc16c = nullptr) {
    // entries past the width become (own row, 0.0): the gathers below are
    // straight-line and issue back to back
    const uint32_t self = (uint32_t)((32 * ls + lane) * 16);
    B.w = 0;
    B.remote = 0;
    B.off = 0;
#pragma unroll
    for (int k = 0; k < KP; ++k) {
        B.c[k] = self;
        B.v[k] = 0.0;
    }
    if (ls >= nloc) return;
    if (need_y) B.y = yrow[32 * ls + lane];
    if (prow) B.p = prow[32 * ls + lane];
    B.w = s_w[ls] & 0xffff;
    B.remote = s_w[ls] >> 16;
    B.off = s_ent[ls] + (lane << 1);
    if (enc16c && !B.remote) {  // all-local slice: two 16-bit codes per 4-byte load
#pragma unroll
        for (int p = 0; p < KP / 2; ++p) {
            if (2 * p < B.w) {
                double2 vv = __ldg(reinterpret_cast<const double2*>(valc + B.off + (p << 6)));
                uint32_t cc = __ldg(reinterpret_cast<const unsigned int*>(enc16c + B.off + (p << 6)));
                B.v[2 * p] = vv.x;
                B.v[2 * p + 1] = vv.y;
                B.c[2 * p] = (cc & 0xffffu) << 4;
                B.c[2 * p + 1] = (cc >> 16) << 4;
            }
        }
        return;
    }
#pragma unroll
    for (int p = 0; p < KP / 2; ++p) {
        if (2 * p < B.w) {
            double2 vv = __ldg(reinterpret_cast<const double2*>(valc + B.off + (p << 6)));
            uint2 cc = __ldg(reinterpret_cast<const uint2*>(encc + B.off + (p << 6)));
            B.v[2 * p] = vv.x;
            B.v[2 * p + 1] = vv.y;
            B.c[2 * p] = cc.x;
            B.c[2 * p + 1] = cc.y;
        }
    }
}

__device__ __forceinline__ double2 gather(cg::cluster_group& cl, const double2* rl, int c, int rank, int chunk,
                                          float inv_chunk) {
    int own = __float2int_rz(((float)(c >> 5) + 0.5f) * inv_chunk);
    int off = c - 32 * own * chunk;
    return (own == rank) ? rl[off] : *cl.map_shared_rank(rl + off, own);
}

// generic load through the cluster shared-memory window: base[r] is the
// generic address of rank r's vector block (local rank included)
__device__ __forceinline__ double2 gather_enc(const unsigned long long* base, const double2* rl, uint32_t c) {
    if (!(c >> 31)) return *reinterpret_cast<const double2*>(reinterpret_cast<const char*>(rl) + c);
    const double2* p = reinterpret_cast<const double2*>(base[(c >> 24) & 0x7f] + (c & 0xffffffu));
    return *p;
}

// branch-free generic gather for slices with remote entries: local entries go
// through the generic address of this CTA's own block (base[rank])
__device__ __forceinline__ double2 gather_gen(const unsigned long long* base, int rank, uint32_t c) {
    const int own = (c >> 31) ? (int)((c >> 24) & 0x7f) : rank;
    return *reinterpret_cast<const double2*>(base[own] + (c & 0xffffffu));
}


template <int NT, bool PF>
__global__ void __launch_bounds__(NT, 1) k_pcg(PcgArgs A) {
    constexpr int PCG_WARPS = NT / 32;
    extern __shared__ __align__(16) unsigned char smem[];
    cg::cluster_group cl = cg::this_cluster();
    const int csize = (int)cl.num_blocks();
    const int rank = (int)cl.block_rank();
    const int slot = blockIdx.x / csize;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    const int64_t s0 = A.sl_off[slot];
    const int S = (int)(A.sl_off[slot + 1] - s0);
    const int chunk = (S + csize - 1) / csize;
    const int my_lo = min(S, rank * chunk);
    const int nloc = min(S, my_lo + chunk) - my_lo;
    const float inv_chunk = 1.0f / (float)chunk;
    const int cap = A.chunk_cap;

    double2* s_warp = reinterpret_cast<double2*>(smem);
    double2* s_slot = s_warp + PCG_WARPS;
    double2* rl = s_slot + 2 * MAX_CLUSTER;
    double2* pl = rl + 32 * cap;
    double2* ql = pl + 32 * cap;
    int* s_ent = reinterpret_cast<int*>(ql + 32 * cap);
    int* s_w = s_ent + cap;
    uint32_t* s_mask = reinterpret_cast<uint32_t*>(s_w + cap);

    __shared__ unsigned long long s_base[MAX_CLUSTER];
    if (threadIdx.x < csize) s_base[threadIdx.x] = reinterpret_cast<unsigned long long>(cl.map_shared_rank(rl, threadIdx.x));
    const int64_t gs0 = s0 + my_lo;           // first global slice of this CTA
    const int64_t row0 = 32 * gs0;            // first global row of this CTA
    const int64_t ent0 = A.sl_ptr[gs0];       // first entry of this CTA
    for (int t = threadIdx.x; t < nloc; t += NT) {
        int64_t e = A.sl_ptr[gs0 + t];
        s_ent[t] = (int)(e - ent0);
        s_w[t] = (int)((A.sl_ptr[gs0 + t + 1] - e) >> 5) | ((int)A.remote[gs0 + t] << 16);
        s_mask[t] = A.sl_mask[gs0 + t];
    }
    // init: y = 0 (done by the builder), r = b, p = q = 0
    double l_rr = 0.0, l_bb = 0.0;
    for (int i = threadIdx.x; i < 32 * nloc; i += NT) {
        double2 bi = A.b[row0 + i];
        double di = A.D[row0 + i];
        rl[i] = bi;
        pl[i] = make_double2(0.0, 0.0);
        ql[i] = make_double2(0.0, 0.0);
        double m2 = bi.x * bi.x + bi.y * bi.y;
        l_rr += m2;
        l_bb += di * m2;  // ||b||^2 of the unscaled system
    }
    int parity = 0;
    double2 t0 = cluster_sum2<PCG_WARPS>(cl, csize, rank, l_rr, l_bb, s_warp, s_slot, parity);
    parity ^= 1;
    double rr = t0.x;
    const double bbU = t0.y;
    const double dmax = A.dmax[slot];
    // ||r||^2 = sum D |r^|^2 <= dmax ||r^||^2: stopping on the bound is safe
    const double stop = A.tol2 * bbU / dmax;
    double beta = 0.0, alpha = 0.0;
    int it = 0;
    const bool active = bbU > 0.0 && rr > stop;

    if (active) {
        long long tA = 0, tR1 = 0, tB = 0, tR2 = 0;
        for (it = 0; it < A.maxit;) {
            const bool timed = A.timing && it >= 64 && it < 192;
            long long c0 = timed ? clock64() : 0;
            // ---- phase A: (y += alpha p_old), q = A r + beta q, p = r + beta p, pq
            double l_pq = 0.0;
            SliceBuf B0, B1;
            const double* valc = A.val + ent0;
            const uint32_t* encc = A.enc + ent0;
            double2* yrow = A.x + row0;
            if (PF) slice_load(B0, valc, encc, s_ent, s_w, warp, nloc, lane, yrow, it > 0);
            for (int ls = warp; ls < nloc; ls += 2 * PCG_WARPS) {
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    const int cur = ls + half * PCG_WARPS;
                    SliceBuf& Bc = half ? B1 : B0;
                    SliceBuf& Bn = half ? B0 : B1;
                    if (PF) {
                        slice_load(Bn, valc, encc, s_ent, s_w, cur + PCG_WARPS, nloc, lane, yrow, it > 0);
                    } else {
                        slice_load(Bc, valc, encc, s_ent, s_w, cur, nloc, lane, yrow, it > 0);
                    }
                    if (cur < nloc) {
                        const int li = 32 * cur + lane;
                        const int64_t gr = row0 + li;
                        double2 ri = rl[li];
                        double sx = ri.x, sy = ri.y;
                        double2 g[KPF];
                        if (!Bc.remote) {
#pragma unroll
                            for (int k = 0; k < KPF; ++k)
                                g[k] = *reinterpret_cast<const double2*>(reinterpret_cast<const char*>(rl) + Bc.c[k]);
                        } else {
#pragma unroll
                            for (int k = 0; k < KPF; ++k) g[k] = gather_gen(s_base, rank, Bc.c[k]);
                        }
#pragma unroll
                        for (int k = 0; k < KPF; ++k) {
                            sx = fma(Bc.v[k], g[k].x, sx);
                            sy = fma(Bc.v[k], g[k].y, sy);
                        }
                        for (int k = KPF; k < Bc.w; ++k) {
                            const int e = Bc.off + ((k >> 1) << 6) + (k & 1);
                            uint32_t c = __ldg(encc + e);
                            double v = __ldg(valc + e);
                            double2 rc = gather_enc(s_base, rl, c);
                            sx = fma(v, rc.x, sx);
                            sy = fma(v, rc.y, sy);
                        }
                        if (s_mask[cur] & (1u << lane)) {
                            int2 nb = A.cpl[gr];
                            double2 cc = A.cplc[gr];
                            double2 zn = nb.x >= 0 ? gather(cl, rl, nb.x, rank, chunk, inv_chunk) : make_double2(0, 0);
                            double2 zp = nb.y >= 0 ? gather(cl, rl, nb.y, rank, chunk, inv_chunk) : make_double2(0, 0);
                            // + i (cn z_next - cp z_prev)
                            double ax = cc.x * zn.x - cc.y * zp.x, ay = cc.x * zn.y - cc.y * zp.y;
                            sx -= ay;
                            sy += ax;
                        }
                        double2 qi = ql[li], pi = pl[li];
                        if (it > 0) {  // y += alpha p (previous iteration), plain load/store
                            double2 yv = Bc.y;
                            yv.x = fma(alpha, pi.x, yv.x);
                            yv.y = fma(alpha, pi.y, yv.y);
                            yrow[li] = yv;
                        }
                        qi.x = fma(beta, qi.x, sx);
                        qi.y = fma(beta, qi.y, sy);
                        pi.x = fma(beta, pi.x, ri.x);
                        pi.y = fma(beta, pi.y, ri.y);
                        ql[li] = qi;
                        pl[li] = pi;
                        l_pq += pi.x * qi.x + pi.y * qi.y;
                    }
                }
            }
            long long c1 = timed ? clock64() : 0;
            double2 tq = cluster_sum2<PCG_WARPS>(cl, csize, rank, l_pq, 0.0, s_warp, s_slot, parity);
            parity ^= 1;
            alpha = rr / tq.x;
            long long c2 = timed ? clock64() : 0;
            // ---- phase B: r -= alpha q (same rows as phase A: no block barrier needed)
            double l_rr2 = 0.0;
#pragma unroll 4
            for (int ls = warp; ls < nloc; ls += PCG_WARPS) {
                const int li = 32 * ls + lane;
                double2 qi = ql[li], ri = rl[li];
                ri.x = fma(-alpha, qi.x, ri.x);
                ri.y = fma(-alpha, qi.y, ri.y);
                rl[li] = ri;
                l_rr2 += ri.x * ri.x + ri.y * ri.y;
            }
            long long c3 = timed ? clock64() : 0;
            double2 tr = cluster_sum2<PCG_WARPS>(cl, csize, rank, l_rr2, 0.0, s_warp, s_slot, parity);
            parity ^= 1;
            if (timed) {
                long long c4 = clock64();
                tA += c1 - c0;
                tR1 += c2 - c1;
                tB += c3 - c2;
                tR2 += c4 - c3;
            }
            beta = tr.x / rr;
            rr = tr.x;
            ++it;
            if (rr <= stop || !(rr == rr)) break;
        }
        if (A.timing && threadIdx.x == 0) {
            long long* t = A.timing + 8 * blockIdx.x;
            t[0] = tA;
            t[1] = tR1;
            t[2] = tB;
            t[3] = tR2;
        }
        // the last update y += alpha p
        for (int ls = warp; ls < nloc; ls += PCG_WARPS) {
            const int li = 32 * ls + lane;
            double2 pi = pl[li];
            double2 yv = A.x[row0 + li];
            yv.x = fma(alpha, pi.x, yv.x);
            yv.y = fma(alpha, pi.y, yv.y);
            A.x[row0 + li] = yv;
        }
    }
    if (rank == 0 && threadIdx.x == 0) {
        A.iters[slot] = it;
        A.res[8 * slot + 0] = (bbU > 0.0) ? sqrt(dmax * rr / bbU) : 0.0;  // upper bound of ||r||/||b||
        A.res[8 * slot + 1] = bbU;
    }
}


// ---------------------------------------------------------------------------
// two-level PCG: one cluster per slot, z (the preconditioned residual, the
// only gathered vector), q and r in distributed shared memory, p in global
// memory (row-local). Three cluster reductions per iteration:
//   A: q = A z + beta q; y += alpha p; p = z + beta p; <p,q>           [SYNC1]
//   B: r -= alpha q; <r,r>; g = W^T r over my aggregates -> every CTA  [SYNC2]
//   C: mu = E^-1 g on my aggregates; z = r + W^ mu; rho = <r,z>        [SYNC3]
template <int NT, typename ET>
__global__ void __launch_bounds__(NT, NT <= 256 ? 2 : 1) k_pcg2(PcgArgs A) {
    constexpr int NW = NT / 32;
    extern __shared__ __align__(16) unsigned char smem[];
    cg::cluster_group cl = cg::this_cluster();
    const int csize = (int)cl.num_blocks();
    const int rank = (int)cl.block_rank();
    const int slot = A.order ? A.order[blockIdx.x / csize] : (int)(blockIdx.x / csize);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long t_start = 0;
    if (A.timing) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));

    const int64_t s0 = A.sl_off[slot];
    const int S = (int)(A.sl_off[slot + 1] - s0);
    const int chunk = (S + csize - 1) / csize;
    const int my_lo = min(S, rank * chunk);
    const int nloc = min(S, my_lo + chunk) - my_lo;
    const float inv_chunk = 1.0f / (float)chunk;
    const int cap = A.chunk_cap;

    double2* s_warp = reinterpret_cast<double2*>(smem);
    double2* s_slot = s_warp + NW;
    double2* zl = s_slot + 2 * MAX_CLUSTER;
    double2* ql = zl + 32 * cap;
    double2* rl = ql + 32 * cap;
    const int ncb = A.ncb;
    double2* gbuf = rl + 32 * cap;          // [2][ncb]
    double2* mu = gbuf + 2 * ncb;           // [mu_cap] (my aggregates)
    double* part = reinterpret_cast<double*>(mu + A.mu_cap);  // [items_cap][6]
    int* s_ent = reinterpret_cast<int*>(part + 6 * A.items_cap);
    int* s_w = s_ent + cap;
    uint32_t* s_mask = reinterpret_cast<uint32_t*>(s_w + cap);

    __shared__ unsigned long long s_base[MAX_CLUSTER];
    if (threadIdx.x < csize) s_base[threadIdx.x] = reinterpret_cast<unsigned long long>(cl.map_shared_rank(zl, threadIdx.x));
    const int64_t gs0 = s0 + my_lo;
    const int64_t row0 = 32 * gs0;
    const int64_t rowN = row0 + 32 * (int64_t)nloc;
    const int64_t ent0 = A.sl_ptr[gs0];
    for (int t = threadIdx.x; t < nloc; t += NT) {
        int64_t e = A.sl_ptr[gs0 + t];
        s_ent[t] = (int)(e - ent0);
        s_w[t] = (int)((A.sl_ptr[gs0 + t + 1] - e) >> 5) | ((int)A.remote[gs0 + t] << 16);
        s_mask[t] = A.sl_mask[gs0 + t];
    }
    // my aggregates [a_lo, a_hi) (global ids; aggregates never straddle CTAs)
    const int a0 = (int)A.C.abase[slot];
    const int nag = (int)(A.C.abase[slot + 1] - a0);
    const int nc = 3 * nag;
    int a_lo = a0, a_hi = a0;
    if (nloc > 0) {
        int lo = a0, hi = a0 + nag;  // first aggregate starting at or after row0 / rowN
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (A.C.aoff[mid] < row0) lo = mid + 1; else hi = mid;
        }
        a_lo = lo;
        lo = a_lo;
        hi = a0 + nag;
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (A.C.aoff[mid] < rowN) lo = mid + 1; else hi = mid;
        }
        a_hi = lo;
    }
    const int naggs = a_hi - a_lo;
    const int npart = max(1, NW / max(naggs, 1));
    const int nitems = naggs * npart;
    const int ncp = (nc + 7) & ~7;  // padded row stride of the float copy
    const ET* Einv = reinterpret_cast<const ET*>(A.C.einvh) + A.C.eoff32[slot];
    const int crow0 = 3 * (a_lo - a0);  // my first coarse row
    double2* pg = A.C.p;
    const uint2* wr = A.C.wr;

    // (aggregate, part) work items: row ranges kept in shared memory so the
    // per-iteration loops do not wait on global aggregate offsets
    int2* s_item = reinterpret_cast<int2*>((reinterpret_cast<uintptr_t>(s_mask + cap) + 7) & ~(uintptr_t)7);
    for (int t = threadIdx.x; t < nitems; t += NT) {
        const int a_rel = t / npart, pt = t - a_rel * npart;
        const int64_t r0 = A.C.aoff[a_lo + a_rel], r1 = A.C.aoff[a_lo + a_rel + 1];
        const int64_t per = (r1 - r0 + npart - 1) / npart;
        const int64_t rb = r0 + pt * per;
        s_item[t] = make_int2((int)(rb - row0), (int)(min(r1, rb + per) - row0));
    }
    auto item_range = [&](int t, int& a_rel, int64_t& rb, int64_t& re) {
        a_rel = t / npart;
        const int2 it2 = s_item[t];
        rb = row0 + it2.x;
        re = row0 + it2.y;
    };
    constexpr int IU = 8;  // rows per lane in flight in the aggregate-order loops
    // B: (optionally r -= alpha q), <r,r>, g = W^T r for my aggregates, sent
    // to every CTA's gbuf[par]; returns this thread's <r,r> share
    auto restrict_r = [&](bool upd, double alpha, int par) -> double {
        double l_rr = 0.0;
        for (int t = warp; t < nitems; t += NW) {
            int a_rel;
            int64_t rb, re;
            item_range(t, a_rel, rb, re);
            double g0x = 0, g0y = 0, g1x = 0, g1y = 0, g2x = 0, g2y = 0;
            for (int64_t rq = rb + lane; rq < re; rq += 32 * IU) {
                float4 w[IU];
#pragma unroll
                for (int u = 0; u < IU; ++u) {
                    const int64_t r = rq + 32 * u;
                    w[u] = r < re ? cw_get(wr, r) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < IU; ++u) {
                    const int64_t r = rq + 32 * u;
                    if (r >= re) break;
                    const int li = (int)(r - row0);
                    double2 ri = rl[li];
                    if (upd) {
                        const double2 qi = ql[li];
                        ri.x = fma(-alpha, qi.x, ri.x);
                        ri.y = fma(-alpha, qi.y, ri.y);
                        rl[li] = ri;
                    }
                    l_rr += ri.x * ri.x + ri.y * ri.y;
                    g0x = fma((double)w[u].x, ri.x, g0x);
                    g0y = fma((double)w[u].x, ri.y, g0y);
                    g1x = fma((double)w[u].y, ri.x, g1x);
                    g1y = fma((double)w[u].y, ri.y, g1y);
                    g2x = fma((double)w[u].z, ri.x, g2x);
                    g2y = fma((double)w[u].z, ri.y, g2y);
                }
            }
            g0x = warp_sum(g0x);
            g0y = warp_sum(g0y);
            g1x = warp_sum(g1x);
            g1y = warp_sum(g1y);
            g2x = warp_sum(g2x);
            g2y = warp_sum(g2y);
            if (lane == 0) {
                double* pp = part + 6 * t;
                pp[0] = g0x;
                pp[1] = g0y;
                pp[2] = g1x;
                pp[3] = g1y;
                pp[4] = g2x;
                pp[5] = g2y;
            }
        }
        if (upd) {  // rows outside every aggregate do not exist; all rows are covered above
        }
        __syncthreads();
        for (int q = threadIdx.x; q < 3 * naggs * csize; q += NT) {
            const int cq = q / csize, dst = q - cq * csize;
            const int a_rel = cq / 3, sidx = cq - 3 * a_rel;
            double gx = 0.0, gy = 0.0;
            for (int pt = 0; pt < npart; ++pt) {
                const double* pp = part + 6 * (a_rel * npart + pt);
                gx += pp[2 * sidx];
                gy += pp[2 * sidx + 1];
            }
            double2* gb = cl.map_shared_rank(gbuf + par * ncb, dst);
            gb[crow0 + cq] = make_double2(gx, gy);
        }
        return l_rr;
    };
    // C: mu = E^-1 g (my coarse rows), z = r + W^ mu, returns <r,z> share
    auto prolong_z = [&](int par) -> double {
        const double2* g = gbuf + par * ncb;
        for (int q = warp; q < 3 * naggs; q += NW) {
            const ET* er = Einv + (int64_t)(crow0 + q) * ncp;
            double mx = 0.0, my = 0.0;
            ET e[(NC_MAX + 31) / 32];
#pragma unroll
            for (int u = 0; u < (NC_MAX + 31) / 32; ++u) {  // lane-strided columns: coalesced, conflict-free
                const int c = lane + 32 * u;
                e[u] = c < nc ? er[c] : mk_et<ET>(0.0, 0.0);
            }
#pragma unroll
            for (int u = 0; u < (NC_MAX + 31) / 32; ++u) {
                const int c = lane + 32 * u;
                if (c < nc) {
                    const double2 gg = g[c];
                    mx = fma((double)e[u].x, gg.x, mx);
                    mx = fma(-(double)e[u].y, gg.y, mx);
                    my = fma((double)e[u].x, gg.y, my);
                    my = fma((double)e[u].y, gg.x, my);
                }
            }
            mx = warp_sum(mx);
            my = warp_sum(my);
            if (lane == 0) mu[q] = make_double2(mx, my);
        }
        __syncthreads();
        double l_rz = 0.0;
        for (int t = warp; t < nitems; t += NW) {
            int a_rel;
            int64_t rb, re;
            item_range(t, a_rel, rb, re);
            const double2 m0 = mu[3 * a_rel], m1 = mu[3 * a_rel + 1], m2 = mu[3 * a_rel + 2];
            for (int64_t rq = rb + lane; rq < re; rq += 32 * IU) {
                float4 w[IU];
#pragma unroll
                for (int u = 0; u < IU; ++u) {
                    const int64_t r = rq + 32 * u;
                    w[u] = r < re ? cw_get(wr, r) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < IU; ++u) {
                    const int64_t r = rq + 32 * u;
                    if (r >= re) break;
                    const int li = (int)(r - row0);
                    const double2 ri = rl[li];
                    double2 zi;
                    zi.x = ri.x + (double)w[u].x * m0.x + (double)w[u].y * m1.x + (double)w[u].z * m2.x;
                    zi.y = ri.y + (double)w[u].x * m0.y + (double)w[u].y * m1.y + (double)w[u].z * m2.y;
                    zl[li] = zi;
                    l_rz += ri.x * zi.x + ri.y * zi.y;
                }
            }
        }
        return l_rz;
    };

    // init: y = 0 (builder), r = b, p = q = 0; coarse buffers zero (columns
    // past nc meet zero padding of E^-1 and must not hold NaN garbage)
    for (int i = threadIdx.x; i < 2 * ncb; i += NT) gbuf[i] = make_double2(0.0, 0.0);
    double l_rr = 0.0, l_bb = 0.0;
    for (int i = threadIdx.x; i < 32 * nloc; i += NT) {
        double2 bi = A.b[row0 + i];
        double di = A.D[row0 + i];
        rl[i] = bi;
        zl[i] = bi;
        ql[i] = make_double2(0.0, 0.0);
        pg[row0 + i] = make_double2(0.0, 0.0);
        double m2 = bi.x * bi.x + bi.y * bi.y;
        l_rr += m2;
        l_bb += di * m2;
    }
    int parity = 0, gpar = 0;
    double2 t0 = cluster_sum2<NW>(cl, csize, rank, l_rr, l_bb, s_warp, s_slot, parity);
    parity ^= 1;
    double rr = t0.x;
    const double bbU = t0.y;
    const double dmax = A.dmax[slot];
    const double stop = A.tol2 * bbU / dmax;
    double beta = 0.0, alpha = 0.0, rho = 0.0;
    int it = 0;
    const bool active = bbU > 0.0 && rr > stop;

    if (active) {
        // z0 = M r0, rho0 = <r0, z0>
        restrict_r(false, 0.0, gpar);
        cluster_sum2<NW>(cl, csize, rank, 0.0, 0.0, s_warp, s_slot, parity);
        parity ^= 1;
        double l_rz = prolong_z(gpar);
        gpar ^= 1;
        // coarse start: the first search direction is Q b = z0 - r0 (step
        // length 1 in exact arithmetic, so x1 = Q b, r1 = b - A Q b); CG
        // restarts from there (beta = 0 after the first iteration)
        double l_bq = 0.0;
        if (A.x0) {
            __syncthreads();
            for (int i = threadIdx.x; i < 32 * nloc; i += NT) {
                const double2 ri = rl[i];
                double2 zi = zl[i];
                zi.x -= ri.x;
                zi.y -= ri.y;
                zl[i] = zi;
                l_bq += ri.x * zi.x + ri.y * zi.y;
            }
        }
        double2 tz = cluster_sum2<NW>(cl, csize, rank, l_rz, l_bq, s_warp, s_slot, parity);
        parity ^= 1;
        rho = tz.x;
        bool x0_start = A.x0 != 0;
        if (x0_start) {
            if (tz.y > 1e-24 * tz.x) {
                rho = tz.y;
            } else {  // no coarse component: back to z0 = M r0
                x0_start = false;
                for (int i = threadIdx.x; i < 32 * nloc; i += NT) {
                    const double2 ri = rl[i];
                    double2 zi = zl[i];
                    zi.x += ri.x;
                    zi.y += ri.y;
                    zl[i] = zi;
                }
                cluster_sum2<NW>(cl, csize, rank, 0.0, 0.0, s_warp, s_slot, parity);
                parity ^= 1;
            }
        }
        const double* valc = A.val + ent0;
        const uint32_t* encc = A.enc + ent0;
        const uint16_t* enc16c = A.enc16 + ent0;
        double2* yrow = A.x + row0;
        double2* prow = pg + row0;
        long long tm[6] = {0, 0, 0, 0, 0, 0};
        for (it = 0; it < A.maxit;) {
            const bool timed = A.timing && it >= 64 && it < 192;
            long long c0 = timed ? clock64() : 0;
            // ---- A: q = A z + beta q, y += alpha p_old, p = z + beta p, <p,q>
            double l_pq = 0.0;
            SliceBufT<KPF2> B0, B1;
            auto row_body = [&](SliceBufT<KPF2>& Bc, int cur, double2& pref, double2& yref) {
                const int li = 32 * cur + lane;
                const int64_t gr = row0 + li;
                double2 zi = zl[li];
                double sx = zi.x, sy = zi.y;
                double2 g[KPF2];
                if (!Bc.remote) {
#pragma unroll
                    for (int k = 0; k < KPF2; ++k)
                        g[k] = *reinterpret_cast<const double2*>(reinterpret_cast<const char*>(zl) + Bc.c[k]);
                } else {
#pragma unroll
                    for (int k = 0; k < KPF2; ++k) g[k] = gather_gen(s_base, rank, Bc.c[k]);
                }
#pragma unroll
                for (int k = 0; k < KPF2; ++k) {
                    sx = fma(Bc.v[k], g[k].x, sx);
                    sy = fma(Bc.v[k], g[k].y, sy);
                }
                for (int k = KPF2; k < Bc.w; ++k) {
                    const int e = Bc.off + ((k >> 1) << 6) + (k & 1);
                    uint32_t c = __ldg(encc + e);
                    double v = __ldg(valc + e);
                    double2 rc = gather_enc(s_base, zl, c);
                    sx = fma(v, rc.x, sx);
                    sy = fma(v, rc.y, sy);
                }
                if (s_mask[cur] & (1u << lane)) {
                    int2 nb = A.cpl[gr];
                    double2 cc = A.cplc[gr];
                    double2 zn = nb.x >= 0 ? gather(cl, zl, nb.x, rank, chunk, inv_chunk) : make_double2(0, 0);
                    double2 zp = nb.y >= 0 ? gather(cl, zl, nb.y, rank, chunk, inv_chunk) : make_double2(0, 0);
                    double ax = cc.x * zn.x - cc.y * zp.x, ay = cc.x * zn.y - cc.y * zp.y;
                    sx -= ay;
                    sy += ax;
                }
                double2 qi = ql[li];
                double2 pi = pref;
                yref.x = fma(alpha, pi.x, yref.x);  // alpha = 0 in the first iteration
                yref.y = fma(alpha, pi.y, yref.y);
                qi.x = fma(beta, qi.x, sx);
                qi.y = fma(beta, qi.y, sy);
                pi.x = fma(beta, pi.x, zi.x);
                pi.y = fma(beta, pi.y, zi.y);
                ql[li] = qi;
                pref = pi;
                l_pq += pi.x * qi.x + pi.y * qi.y;
            };
            {
                slice_load(B0, valc, encc, s_ent, s_w, warp, nloc, lane, yrow, it > 0, prow, enc16c);
                for (int ls = warp; ls < nloc; ls += 2 * NW) {
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                        const int cur = ls + half * NW;
                        SliceBufT<KPF2>& Bc = half ? B1 : B0;
                        SliceBufT<KPF2>& Bn = half ? B0 : B1;
                        slice_load(Bn, valc, encc, s_ent, s_w, cur + NW, nloc, lane, yrow, it > 0, prow, enc16c);
                        if (cur < nloc) {
                            const int li = 32 * cur + lane;
                            double2 pv = Bc.p, yv = Bc.y;
                            if (it == 0) yv = make_double2(0.0, 0.0);
                            row_body(Bc, cur, pv, yv);
                            prow[li] = pv;
                            if (it > 0) yrow[li] = yv;
                        }
                    }
                }
            }
            long long c1 = timed ? clock64() : 0;
            double2 tq = cluster_sum2<NW>(cl, csize, rank, l_pq, 0.0, s_warp, s_slot, parity);
            parity ^= 1;
            alpha = rho / tq.x;
            long long c2 = timed ? clock64() : 0;
            // ---- B: r -= alpha q, <r,r>, g = W^T r
            double l_rr2 = restrict_r(true, alpha, gpar);
            long long c3 = timed ? clock64() : 0;
            double2 tr = cluster_sum2<NW>(cl, csize, rank, l_rr2, 0.0, s_warp, s_slot, parity);
            parity ^= 1;
            rr = tr.x;
            ++it;
            if (A.hist && rank == 0 && threadIdx.x == 0 && it <= HIST_K) {
                A.hist[(slot * HIST_K + it - 1) * 3 + 0] = alpha;
                A.hist[(slot * HIST_K + it - 1) * 3 + 1] = rr;
            }
            if (rr <= stop || !(rr == rr)) break;
            long long c4 = timed ? clock64() : 0;
            // ---- C: z = M r, rho = <r,z>
            double l_rz2 = prolong_z(gpar);
            gpar ^= 1;
            long long c5 = timed ? clock64() : 0;
            double2 tz2 = cluster_sum2<NW>(cl, csize, rank, l_rz2, 0.0, s_warp, s_slot, parity);
            parity ^= 1;
            beta = (x0_start && it == 1) ? 0.0 : tz2.x / rho;
            rho = tz2.x;
            if (A.hist && rank == 0 && threadIdx.x == 0 && it <= HIST_K) A.hist[(slot * HIST_K + it - 1) * 3 + 2] = beta;
            if (timed) {
                long long c6 = clock64();
                tm[0] += c1 - c0;
                tm[1] += c2 - c1;
                tm[2] += c3 - c2;
                tm[3] += c4 - c3;
                tm[4] += c5 - c4;
                tm[5] += c6 - c5;
            }
        }
        if (A.timing && threadIdx.x == 0) {
            for (int q = 0; q < 6; ++q) A.timing[8 * blockIdx.x + q] = tm[q];
            unsigned long long t_end;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
            A.timing[8 * blockIdx.x + 6] = (long long)t_start;
            A.timing[8 * blockIdx.x + 7] = (long long)t_end;
        }
        // the last update y += alpha p
        {
            for (int i = threadIdx.x; i < 32 * nloc; i += NT) {
                double2 pi = prow[i];
                double2 yv = yrow[i];
                yv.x = fma(alpha, pi.x, yv.x);
                yv.y = fma(alpha, pi.y, yv.y);
                yrow[i] = yv;
            }
        }
    }
    if (rank == 0 && threadIdx.x == 0) {
        A.iters[slot] = it;
        A.res[8 * slot + 0] = (bbU > 0.0) ? sqrt(dmax * rr / bbU) : 0.0;
        A.res[8 * slot + 1] = bbU;
    }
}

// nnz of the reference's CSR system of every slot (SURVEY §8(d) bytes model).
// DNCP C_ff (flatten.py:160-166): 2 x (diagonal + nonzero off-diagonals of
// L_UU), plus, for a boundary row, one entry in the x-row and one in the
// y-row per unknown loop neighbour (the -2M blocks); exact zeros are dropped
// as scipy's csr_binop does. L_II (assemble.py:40): diagonal + every stored
// off-diagonal (explicit zeros kept). Padding entries point to their own row
// and are skipped.
__global__ void k_ref_nnz(const int64_t* __restrict__ sl_off, const int64_t* __restrict__ sl_ptr,
                          const int32_t* __restrict__ col, const double* __restrict__ val,
                          const uint32_t* __restrict__ sl_mask, const int2* __restrict__ cpl,
                          const int64_t* __restrict__ nu, int dncp, long long* __restrict__ out) {
    __shared__ long long red[32];
    const int j = blockIdx.x;
    const int64_t rbase = 32 * sl_off[j];
    long long cnt = 0;
    for (int64_t r = rbase + threadIdx.x; r < rbase + nu[j]; r += blockDim.x) {
        const int64_t s = r >> 5;
        const int lane = (int)(r & 31);
        const int64_t e0 = sl_ptr[s];
        const int w = (int)((sl_ptr[s + 1] - e0) >> 5);
        const int self = (int)(r - rbase);
        long long c = 1;  // diagonal
        for (int k = 0; k < w; ++k) {
            const int64_t q = sell_pos(e0, k, lane);
            if (col[q] == self) continue;
            if (dncp && val[q] == 0.0) continue;
            ++c;
        }
        if (dncp) {
            c *= 2;
            if (sl_mask[s] & (1u << lane)) {
                const int2 nb = cpl[r];
                c += 2 * ((nb.x >= 0) + (nb.y >= 0));
            }
        }
        cnt += c;
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[q];
        out[j] = t;
    }
}

// true residual of the unscaled system from the scaled arrays:
//   ||b - H x||^2 = sum D |b^ - H^ y|^2, ||x||^2 = sum |y|^2 / D, ||b||^2 = sum D |b^|^2
// (1024 threads: one CTA per slot, so only nslot SMs work; the warps hide the gather latency)
__global__ void __launch_bounds__(1024) k_true_residual(PcgArgs A) {
    __shared__ double red[3][32];
    const int slot = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t s0 = A.sl_off[slot];
    const int S = (int)(A.sl_off[slot + 1] - s0);
    const int64_t rbase = 32 * s0;
    double a_r = 0.0, a_x = 0.0, a_b = 0.0;
    for (int ls = warp; ls < S; ls += nw) {
        const int64_t gs = s0 + ls;
        const int64_t e0 = A.sl_ptr[gs];
        const int wdt = (int)((A.sl_ptr[gs + 1] - e0) >> 5);
        const int64_t gr = rbase + 32 * ls + lane;
        double2 yi = A.x[gr];
        double sx = yi.x, sy = yi.y;
        for (int k = 0; k < wdt; ++k) {
            int c = A.col[sell_pos(e0, k, lane)];
            double v = A.val[sell_pos(e0, k, lane)];
            double2 yc = A.x[rbase + c];
            sx = fma(v, yc.x, sx);
            sy = fma(v, yc.y, sy);
        }
        if (A.sl_mask[gs] & (1u << lane)) {
            int2 nb = A.cpl[gr];
            double2 cc = A.cplc[gr];
            double2 zn = nb.x >= 0 ? A.x[rbase + nb.x] : make_double2(0.0, 0.0);
            double2 zp = nb.y >= 0 ? A.x[rbase + nb.y] : make_double2(0.0, 0.0);
            double ax = cc.x * zn.x - cc.y * zp.x, ay = cc.x * zn.y - cc.y * zp.y;
            sx -= ay;
            sy += ax;
        }
        double2 bi = A.b[gr];
        double di = A.D[gr];
        double rx = bi.x - sx, ry = bi.y - sy;
        a_r += di * (rx * rx + ry * ry);
        a_x += (yi.x * yi.x + yi.y * yi.y) / di;
        a_b += di * (bi.x * bi.x + bi.y * bi.y);
    }
    a_r = warp_sum(a_r);
    a_x = warp_sum(a_x);
    a_b = warp_sum(a_b);
    if (lane == 0) {
        red[0][warp] = a_r;
        red[1][warp] = a_x;
        red[2][warp] = a_b;
    }
    __syncthreads();
    if (warp == 0) {
        double r0 = lane < nw ? red[0][lane] : 0.0;
        double r1 = lane < nw ? red[1][lane] : 0.0;
        double r2 = lane < nw ? red[2][lane] : 0.0;
        r0 = warp_sum(r0);
        r1 = warp_sum(r1);
        r2 = warp_sum(r2);
        if (lane == 0) {
            A.res[8 * slot + 2] = sqrt(r0);
            A.res[8 * slot + 3] = sqrt(r1);
            A.res[8 * slot + 4] = sqrt(r2);
        }
    }
}

// scatter x = D^{-1/2} y back to submesh-local vertices (fixed vertices get
// their prescribed values)
__global__ void k_scatter(int64_t ne, int32_t nslot, const int32_t* __restrict__ comps,
                          const int64_t* __restrict__ sv_off, const int64_t* __restrict__ vert_off,
                          const int32_t* __restrict__ urow, const int32_t* __restrict__ fixed_ref,
                          const double2* __restrict__ fv, const double2* __restrict__ y,
                          const double* __restrict__ Dsq, double2* __restrict__ z) {
    GRID_STRIDE(e, ne) {
        int j = bsearch_off(sv_off, nslot + 1, e);
        int64_t g = vert_off[comps[j]] + (e - sv_off[j]);
        int r = urow[e];
        if (r >= 0) {
            double2 v = y[r];
            double d = Dsq[r];
            z[g] = make_double2(v.x / d, v.y / d);
        } else {
            z[g] = fv[fixed_ref[e]];
        }
    }
}

// per slot: shoelace area of the loop, E_D - A, max |z| (flatten.py:176-187)
__global__ void __launch_bounds__(1024) k_flat_checks(const int32_t* __restrict__ comps, const int64_t* __restrict__ vert_off,
                              const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                              const double* __restrict__ val, const int64_t* __restrict__ loop_off,
                              const int32_t* __restrict__ loop, const double2* __restrict__ z,
                              double* __restrict__ res) {
    __shared__ double red[3][32];
    int slot = blockIdx.x;
    int c = comps[slot];
    int64_t vb = vert_off[c], ve = vert_off[c + 1];
    double ed = 0.0, mx = 0.0, ar = 0.0;
    for (int64_t g = vb + threadIdx.x; g < ve; g += blockDim.x) {
        double sx = 0.0, sy = 0.0;
        for (int64_t q = row_ptr[g]; q < row_ptr[g + 1]; ++q) {
            double2 zz = z[vb + col[q]];
            sx += val[q] * zz.x;
            sy += val[q] * zz.y;
        }
        double2 zi = z[g];
        ed += 0.5 * (zi.x * sx + zi.y * sy);
        mx = fmax(mx, zi.x * zi.x + zi.y * zi.y);
    }
    int64_t lo = loop_off[c], nb = loop_off[c + 1] - lo;
    for (int64_t j = threadIdx.x; j < nb; j += blockDim.x) {
        double2 w = z[vb + loop[lo + j]];
        double2 u = z[vb + loop[lo + (j + 1) % nb]];
        ar += 0.5 * (w.x * u.y - w.y * u.x);
    }
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    ed = warp_sum(ed);
    ar = warp_sum(ar);
    mx = warp_max(mx);
    if (lane == 0) {
        red[0][warp] = ed;
        red[1][warp] = ar;
        red[2][warp] = mx;
    }
    __syncthreads();
    if (warp == 0) {
        double a = lane < nw ? red[0][lane] : 0.0;
        double b = lane < nw ? red[1][lane] : 0.0;
        double m = lane < nw ? red[2][lane] : 0.0;
        a = warp_sum(a);
        b = warp_sum(b);
        m = warp_max(m);
        if (lane == 0) {
            res[8 * slot + 5] = b;       // signed area
            res[8 * slot + 6] = a - b;   // E_C = E_D - A
            res[8 * slot + 7] = m;       // max |z|^2
        }
    }
}

// ---------------------------------------------------------------------------
// host side

// Kernel attributes are set to fixed values (the largest dynamic shared
// memory the device allows next to the kernel's static shared memory, and
// non-portable cluster sizes): the flatten's worker thread and the caller's
// thread launch and query these kernels concurrently, so per-launch values
// could race between a set and a launch.
template <class K>
int set_kernel_attrs(K kern) {
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    int dev = 0, optin = 0;
    PGCP_TRY_CUDA(cudaGetDevice(&dev));
    PGCP_TRY_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa;
    PGCP_TRY_CUDA(cudaFuncGetAttributes(&fa, kern));
    PGCP_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       optin - (int)fa.sharedSizeBytes));
    PGCP_TRY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    return PGCP_OK;
}

// clusters of k_pcg2 that can be resident at once for a cluster shape, for
// the instantiation that will be launched (threads per CTA, E^-1 precision),
// cached per device
template <int NT, typename ET>
int query_active_clusters(int csize, size_t smem) {
    auto kern = k_pcg2<NT, ET>;
    int n = 0;
    if (set_kernel_attrs(kern) == PGCP_OK) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)csize, 1, 1);
        cfg.blockDim = dim3(NT, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = csize;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) n = 0;
    }
    cudaGetLastError();
    return n;
}

int max_active_clusters(int csize, size_t smem, int nt, bool einv_fp64) {
    // the flatten (worker thread) and the harmonic preparation (caller's
    // thread) choose their shapes concurrently
    static std::mutex mu;
    static std::vector<std::pair<std::array<long long, 5>, int>> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const std::array<long long, 5> key = {dev, nt, einv_fp64 ? 1 : 0, csize, (long long)smem};
    std::lock_guard<std::mutex> lock(mu);
    for (auto& kv : cache)
        if (kv.first == key) return kv.second;
    int n;
    if (nt == 256)
        n = einv_fp64 ? query_active_clusters<256, double2>(csize, smem) : query_active_clusters<256, float2>(csize, smem);
    else
        n = einv_fp64 ? query_active_clusters<512, double2>(csize, smem) : query_active_clusters<512, float2>(csize, smem);
    cache.emplace_back(key, n);
    return n;
}

int pick_cluster(int64_t max_slices, int32_t nslot, int32_t forced, bool coarse, int nt, bool einv_fp64,
                 int* csize_out, int* chunk_out) {
    const int max_chunk = (SMEM_LIMIT - RED_BYTES - (coarse ? COARSE_BYTES : 0)) / (48 * 32 + 12);
    int cmin = 1;
    while (cmin <= MAX_CLUSTER && (max_slices + cmin - 1) / cmin > max_chunk) cmin *= 2;
    if (cmin > MAX_CLUSTER) {
        set_error("subdomain with %lld unknown slices exceeds the on-chip capacity of a %d-CTA cluster",
                  (long long)max_slices, MAX_CLUSTER);
        return PGCP_E_INVALID;
    }
    int c = cmin;
    if (forced > 0) {
        c = std::max(cmin, forced);
    } else if (coarse) {
        // k_pcg2: choose the cluster shape by waves x per-iteration time.
        // Waves come from the occupancy query (GPC packing: 33 four-CTA,
        // 15 eight-CTA, 7 sixteen-CTA clusters fit on a B200); the
        // per-iteration time per CTA was measured on cfg 2 as about
        // 10.9K + 8.6 x (rows per CTA) cycles (46.7K / 28.8K / 21.9K at 4 / 8 /
        // 16 CTAs per subdomain), barriers and coarse phases being the
        // constant part. Spreading a few subdomains over wider clusters only
        // pays while they still run in one wave.
        double best = 0;
        for (int cc = cmin; cc <= MAX_CLUSTER; ++cc) {  // any size: 6 / 10-CTA clusters pack GPCs well
            const int64_t ch = (max_slices + cc - 1) / cc;
            if (cc > cmin && ch < 8) break;  // keep >= 256 rows per CTA
            const size_t smem = (size_t)RED_BYTES + (size_t)3 * 32 * ch * 16 + (size_t)12 * ch + COARSE_BYTES;
            const int nconc = max_active_clusters(cc, smem, nt, einv_fp64);
            if (nconc < 1) continue;
            const double waves = (double)((nslot + nconc - 1) / nconc);
            const double cost = waves * (10900.0 + 8.6 * 32.0 * (double)ch);
            if (best == 0 || cost < best * 0.98) {  // ties: the narrower cluster
                best = cost;
                c = cc;
            }
        }
    } else {
        // spread over the SMs when there are few subdomains, but keep >= 8
        // slices (256 rows) per CTA so DSMEM halo traffic stays small
        while (c < MAX_CLUSTER && (int64_t)(2 * c) * nslot <= 148 && (max_slices + 2 * c - 1) / (2 * c) >= 8) c *= 2;
    }
    *csize_out = c;
    *chunk_out = (int)((max_slices + c - 1) / c);
    return PGCP_OK;
}

template <int NT, bool PF>
int launch_pcg_t(SolveSystem* S, const PcgArgs& args, int csize, size_t smem, cudaStream_t s) {
    auto kern = k_pcg<NT, PF>;
    PGCP_TRY(set_kernel_attrs(kern));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(S->nslot * csize), 1, 1);
    cfg.blockDim = dim3(NT, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    cudaError_t oe = cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg);
    if (oe != cudaSuccess || nclusters < 1) {
        set_error("pcg: cluster of %d CTAs with %zu B shared memory cannot be scheduled (%s)", csize, smem,
                  cudaGetErrorString(oe));
        cudaGetLastError();
        return PGCP_E_CUDA;
    }
    PGCP_TRY_CUDA(cudaLaunchKernelEx(&cfg, kern, args));
    return PGCP_OK;
}

template <int NT, typename ET>
int launch_pcg2_t(SolveSystem* S, const PcgArgs& args, int csize, size_t smem, cudaStream_t s) {
    auto kern = k_pcg2<NT, ET>;
    PGCP_TRY(set_kernel_attrs(kern));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(S->nslot * csize), 1, 1);
    cfg.blockDim = dim3(NT, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    cudaError_t oe = cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg);
    if (oe != cudaSuccess || nclusters < 1) {
        set_error("pcg: cluster of %d CTAs with %zu B shared memory cannot be scheduled (%s)", csize, smem,
                  cudaGetErrorString(oe));
        cudaGetLastError();
        return PGCP_E_CUDA;
    }
    PGCP_TRY_CUDA(cudaLaunchKernelEx(&cfg, kern, args));
    return PGCP_OK;
}

int launch_pcg(SolveSystem* S, const PcgArgs& args, int csize, cudaStream_t s) {
    int chunk = args.chunk_cap;
    size_t smem = (size_t)RED_BYTES + (size_t)3 * 32 * chunk * sizeof(double2) + (size_t)12 * chunk +
                  (S->coarse ? (size_t)(2 * S->ncb + S->mu_cap) * 16 + (size_t)S->items_cap * (48 + 8) + 8
                             : 0);
    if (smem > SMEM_LIMIT) {
        set_error("pcg: shared memory %zu exceeds limit", smem);
        return PGCP_E_INVALID;
    }
    if (S->coarse) {
        if (S->pcg_nt == 256)
            return S->einv_fp64 ? launch_pcg2_t<256, double2>(S, args, csize, smem, s)
                                : launch_pcg2_t<256, float2>(S, args, csize, smem, s);
        return S->einv_fp64 ? launch_pcg2_t<512, double2>(S, args, csize, smem, s)
                            : launch_pcg2_t<512, float2>(S, args, csize, smem, s);
    }
    const char* v = getenv("PGCP_PCG_VARIANT");
    int variant = v ? atoi(v) : 0;
    switch (variant) {
        case 1: return launch_pcg_t<1024, false>(S, args, csize, smem, s);
        case 2: return launch_pcg_t<768, false>(S, args, csize, smem, s);
        case 3: return launch_pcg_t<512, false>(S, args, csize, smem, s);
        case 4: return launch_pcg_t<256, true>(S, args, csize, smem, s);
        default: return launch_pcg_t<512, true>(S, args, csize, smem, s);
    }
}

// Coarse-space row order (see k_pcg2): unknowns sorted by (slot, strip of
// the first principal axis, second principal coordinate). Sets urow/rowsrc,
// the cell of every row and its cell coordinates.
int order_rows_by_cell(pgcp_batch* b, SolveSystem* S, const int64_t* uscan, const std::vector<int64_t>& hus,
                       cudaStream_t s) {
    const int32_t nslot = S->nslot;
    const int64_t nU = hus[nslot] - hus[0];
    PGCP_TRY(S->urow.fill_bytes(0xff, s));
    PGCP_TRY(S->cell.alloc(S->rows, s));
    PGCP_TRY(S->cell.zero(s));
    PGCP_TRY(S->pxy_row.alloc(S->rows, s));
    PGCP_TRY(S->pxy_row.zero(s));
    if (nU <= 0) return PGCP_OK;
    DevBuf<double> frame;
    DevBuf<float2> pxy;
    DevBuf<unsigned long long> k1, k2;
    DevBuf<int32_t> v1, v2;
    PGCP_TRY(frame.alloc(9 * (int64_t)nslot, s));
    PGCP_TRY(pxy.alloc(nU, s));
    PGCP_TRY(k1.alloc(nU, s));
    PGCP_TRY(k2.alloc(nU, s));
    PGCP_TRY(v1.alloc(nU, s));
    PGCP_TRY(v2.alloc(nU, s));
    k_pca<<<nslot, 256, 0, s>>>(nslot, S->d_comps.p, S->sv_off.p, b->vert_off.p, b->vmap.p, b->V.p, S->fixed_ref.p,
                                frame.p);
    PGCP_LAUNCH_CHECK();
    DevBuf<uint32_t> bbox;
    PGCP_TRY(bbox.alloc(4 * (int64_t)nslot, s));
    {
        std::vector<uint32_t> hb(4 * (size_t)nslot);
        for (int j = 0; j < nslot; ++j) {
            hb[4 * j] = 0xffffffffu;
            hb[4 * j + 1] = 0u;
            hb[4 * j + 2] = 0xffffffffu;
            hb[4 * j + 3] = 0u;
        }
        PGCP_TRY_CUDA(cudaMemcpyAsync(bbox.p, hb.data(), hb.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
        PGCP_TRY_CUDA(cudaStreamSynchronize(s));  // hb is a local
    }
    k_proj<<<grid_for(S->ne, 256), 256, 0, s>>>(S->ne, nslot, S->d_comps.p, S->sv_off.p, b->vert_off.p, b->vmap.p,
                                              b->V.p, S->fixed_ref.p, uscan, frame.p, pxy.p, k1.p, v1.p, bbox.p);
    PGCP_LAUNCH_CHECK();
    int sbits = 1;
    while ((1ll << sbits) <= nslot) ++sbits;
    size_t tmp_bytes = 0, t2 = 0;
    PGCP_TRY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k1.p, k2.p, v1.p, v2.p, (int)nU, 0, 32 + sbits, s));
    PGCP_TRY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t2, k2.p, k1.p, v2.p, v1.p, (int)nU, 0, 40 + sbits, s));
    DevBuf<unsigned char> tmp;
    PGCP_TRY(tmp.alloc((int64_t)std::max(tmp_bytes, t2), s));
    tmp_bytes = std::max(tmp_bytes, t2);
    PGCP_TRY_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, k1.p, k2.p, v1.p, v2.p, (int)nU, 0, 32 + sbits, s));
    count_launch();
    // sorted (k2, v2) -> strip keys into (k1, v1)
    k_strip<<<grid_for(nU, 256), 256, 0, s>>>(nU, k2.p, v2.p, S->sv_off.p, uscan, pxy.p, S->gmax, k1.p, v1.p);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, k1.p, k2.p, v1.p, v2.p, (int)nU, 0, 40 + sbits, s));
    count_launch();
    k_cell_keys<<<grid_for(nU, 256), 256, 0, s>>>(nU, k2.p, v2.p, S->sv_off.p, uscan, pxy.p, bbox.p, S->gmax, k1.p,
                                                v1.p);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, k1.p, k2.p, v1.p, v2.p, (int)nU, 0, 40 + sbits, s));
    count_launch();
    k_rows_by_cell<<<grid_for(nU, 256), 256, 0, s>>>(nU, k2.p, v2.p, S->sv_off.p, S->sl_off.p, uscan, pxy.p, S->gmax,
                                                   S->urow.p, S->rowsrc.p, S->cell.p, S->pxy_row.p);
    PGCP_LAUNCH_CHECK();
    return PGCP_OK;
}

// Aggregates for the cluster split `csize`, coarse weights, E and E^-1.
int build_coarse(SolveSystem* S, int csize, cudaStream_t s) {
    const int32_t nslot = S->nslot;
    std::vector<int64_t> hnu(S->h_nu.begin(), S->h_nu.end());
    PGCP_TRY(S->nu_d.alloc(nslot, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(S->nu_d.p, hnu.data(), nslot * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    DevBuf<int32_t> flag;
    DevBuf<int64_t> scan;
    PGCP_TRY(flag.alloc(S->rows, s));
    PGCP_TRY(scan.alloc(S->rows + 1, s));
    k_agg_flag<<<grid_for(S->rows, 256), 256, 0, s>>>(S->rows, nslot, S->sl_off.p, S->nu_d.p, S->cell.p, csize,
                                                    flag.p);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY(exclusive_scan_i32_to_i64(flag.p, scan.p, S->rows, s));
    S->h_abase.assign(nslot + 1, 0);
    PGCP_TRY(S->abase.alloc(nslot + 1, s));
    k_slot_abase<<<grid_for(nslot + 1, 128), 128, 0, s>>>(nslot, S->sl_off.p, scan.p, S->abase.p);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY_CUDA(cudaMemcpyAsync(S->h_abase.data(), S->abase.p, (nslot + 1) * sizeof(int64_t),
                                  cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaStreamSynchronize(s));
    const int64_t NA = S->h_abase[nslot];
    std::vector<int64_t> heoff(nslot + 1, 0);
    for (int j = 0; j < nslot; ++j) {
        int64_t na = S->h_abase[j + 1] - S->h_abase[j];
        if (na > AGG_MAX) {
            set_error("coarse space: %lld aggregates in one subdomain (max %d)", (long long)na, AGG_MAX);
            return PGCP_E_INVALID;
        }
        heoff[j + 1] = heoff[j] + 9 * na * na;
    }
    PGCP_TRY(S->aggr.alloc(S->rows, s));
    PGCP_TRY(S->aoff.alloc(NA + 1, s));
    k_agg_index<<<grid_for(S->rows, 256), 256, 0, s>>>(S->rows, flag.p, scan.p, S->aggr.p, S->aoff.p);
    PGCP_LAUNCH_CHECK();
    const int32_t rows32 = (int32_t)S->rows;
    PGCP_TRY_CUDA(cudaMemcpyAsync(S->aoff.p + NA, &rows32, sizeof(int32_t), cudaMemcpyHostToDevice, s));
    PGCP_TRY(S->eoff.alloc(nslot + 1, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(S->eoff.p, heoff.data(), (nslot + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    PGCP_TRY(S->wr.alloc(S->rows, s));
    k_agg_weights<<<(unsigned)NA, 128, 0, s>>>((int32_t)NA, S->aoff.p, nslot, S->sl_off.p, S->nu_d.p, S->pxy_row.p,
                                              S->Dsq.p, S->wr.p);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY(S->einv.alloc(heoff[nslot], s));
    PGCP_TRY(S->einv.zero(s));
    DevBuf<int> ovf;
    PGCP_TRY(ovf.alloc(1, s));
    PGCP_TRY(ovf.zero(s));
    k_coarse_E<<<(unsigned)NA, 32 * E_WARPS, 0, s>>>(nslot, S->sl_off.p, S->sl_ptr.p, S->sl_mask.p, S->col.p,
                                                    S->val.p, S->cpl.p, S->cplc.p, S->aoff.p, S->aggr.p,
                                                    S->abase.p, S->wr.p, S->eoff.p, S->einv.p, ovf.p);
    PGCP_LAUNCH_CHECK();
    if (const char* dump = getenv("PGCP_COARSE_DUMP")) {  // debugging aid: E of every slot before inversion
        std::vector<double2> hE(heoff[nslot]);
        std::vector<int32_t> haoff(NA + 1);
        std::vector<uint2> hwr(S->rows);
        PGCP_TRY_CUDA(cudaMemcpyAsync(hE.data(), S->einv.p, hE.size() * sizeof(double2), cudaMemcpyDeviceToHost, s));
        PGCP_TRY_CUDA(cudaMemcpyAsync(haoff.data(), S->aoff.p, haoff.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        PGCP_TRY_CUDA(cudaMemcpyAsync(hwr.data(), S->wr.p, hwr.size() * sizeof(uint2), cudaMemcpyDeviceToHost, s));
        PGCP_TRY_CUDA(cudaStreamSynchronize(s));
        FILE* f = fopen(dump, "wb");
        if (f) {
            int64_t hdr[4] = {nslot, NA, S->rows, heoff[nslot]};
            fwrite(hdr, sizeof(hdr), 1, f);
            fwrite(S->h_abase.data(), sizeof(int64_t), nslot + 1, f);
            fwrite(heoff.data(), sizeof(int64_t), nslot + 1, f);
            fwrite(S->h_sl_off.data(), sizeof(int64_t), nslot + 1, f);
            fwrite(haoff.data(), sizeof(int32_t), haoff.size(), f);
            fwrite(hwr.data(), sizeof(uint2), hwr.size(), f);
            fwrite(hE.data(), sizeof(double2), hE.size(), f);
            fclose(f);
        }
    }
    {
        int nmax = 0;
        for (int j = 0; j < nslot; ++j) nmax = std::max<int>(nmax, 3 * (int)(S->h_abase[j + 1] - S->h_abase[j]));
        int CS = 1;
        auto inv_smem = [&](int cs) {
            int rpc = (nmax + cs - 1) / cs;
            return (size_t)rpc * nmax * 16 + (size_t)4 * nmax * 16 + (size_t)2 * rpc * 16 + (size_t)nmax * 8 + 64;
        };
        while (CS < 16 && inv_smem(CS) > 200 * 1024) CS *= 2;
        const size_t smem = inv_smem(CS);
        PGCP_TRY(set_kernel_attrs(k_coarse_inv));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(nslot * CS), 1, 1);
        cfg.blockDim = dim3(INV_THREADS, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CS;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        PGCP_TRY_CUDA(cudaLaunchKernelEx(&cfg, k_coarse_inv, S->abase.p, S->eoff.p, S->einv.p));
        PGCP_LAUNCH_CHECK();
        std::vector<int64_t> he32(nslot + 1, 0);
        for (int j = 0; j < nslot; ++j) {
            int64_t n = 3 * (S->h_abase[j + 1] - S->h_abase[j]);
            he32[j + 1] = he32[j] + n * ((n + 7) & ~7ll);
        }
        PGCP_TRY(S->eoff32.alloc(nslot + 1, s));
        PGCP_TRY_CUDA(cudaMemcpyAsync(S->eoff32.p, he32.data(), (nslot + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        if (S->einv_fp64) {  // PGCP_COARSE_FP64=1 (read in setup_solve)
            PGCP_TRY(S->einv64.alloc(std::max<int64_t>(he32[nslot], 1), s));
            k_hermitize<double2><<<nslot, 512, 0, s>>>(S->abase.p, S->eoff.p, S->einv.p, S->eoff32.p, S->einv64.p);
        } else {
            PGCP_TRY(S->einv32.alloc(std::max<int64_t>(he32[nslot], 1), s));
            k_hermitize<float2><<<nslot, 512, 0, s>>>(S->abase.p, S->eoff.p, S->einv.p, S->eoff32.p, S->einv32.p);
        }
        PGCP_LAUNCH_CHECK();
        PGCP_TRY_CUDA(cudaStreamSynchronize(s));  // he32 is a local
    }
    {
        // k_pcg2 shared layout: gbuf holds every coarse dof of a slot, mu and
        // the partial sums only the CTA's own aggregates (k_pcg2 item_range)
        std::vector<int32_t> haoff(NA + 1);
        PGCP_TRY_CUDA(cudaMemcpyAsync(haoff.data(), S->aoff.p, haoff.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        PGCP_TRY_CUDA(cudaStreamSynchronize(s));
        const int NW = S->pcg_nt / 32;
        int ncmax = 0, own_max = 0, items_max = 1;
        for (int j = 0; j < nslot; ++j) {
            const int a0 = (int)S->h_abase[j], nag = (int)(S->h_abase[j + 1] - a0);
            ncmax = std::max(ncmax, 3 * nag);
            const int Sj = (int)(S->h_sl_off[j + 1] - S->h_sl_off[j]);
            const int ch = (Sj + csize - 1) / csize;
            for (int r = 0; r < csize; ++r) {
                const int64_t row0 = 32 * (S->h_sl_off[j] + std::min(Sj, r * ch));
                const int64_t rowN = 32 * (S->h_sl_off[j] + std::min(Sj, (r + 1) * ch));
                int na = 0;
                for (int a = a0; a < a0 + nag; ++a) na += haoff[a] >= row0 && haoff[a] < rowN;
                own_max = std::max(own_max, na);
                const int npart = std::max(1, NW / std::max(na, 1));
                items_max = std::max(items_max, na * npart);
            }
        }
        S->ncb = std::max(8, (ncmax + 7) & ~7);
        S->mu_cap = std::max(2, (3 * own_max + 1) & ~1);
        S->items_cap = items_max;
    }
    PGCP_TRY(S->p.alloc(S->rows, s));
    int hovf = 0;
    PGCP_TRY_CUDA(cudaMemcpyAsync(&hovf, ovf.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    // unconditional: the host vectors above are locals of this frame
    PGCP_TRY_CUDA(cudaStreamSynchronize(s));
    if (hovf) {
        set_error("coarse space: an aggregate touches more than %d neighbouring aggregates", E_NBMAX);
        return PGCP_E_INVALID;
    }
    return PGCP_OK;
}

// Build the slot system. pins (device int32 [2*nslot]) for DNCP, or the fixed
// list for harmonic. fv = fixed values (device complex).
// val_override (device f64 [nnz of the batch Laplacian], optional): matrix
// values on the Laplacian's CSR pattern to use instead of L (the linear
// Beltrami stiffness of the fold-over repair, repair.cu).
int build_system(pgcp_batch* b, SolveSystem* S, bool dncp, const int32_t* d_pins, const double2* targets_host,
                 const int32_t* fixed_gid, const double* fixed_val, int64_t nfixed, cudaStream_t s,
                 const double* val_override = nullptr) {
    const int32_t nslot = S->nslot;
    S->dncp = dncp;
    // compact vertex enumeration over the slots
    S->h_sv_off.assign(nslot + 1, 0);
    for (int j = 0; j < nslot; ++j) {
        int c = S->comps[j];
        S->h_sv_off[j + 1] = S->h_sv_off[j] + (b->h_vert_off[c + 1] - b->h_vert_off[c]);
    }
    S->ne = S->h_sv_off[nslot];
    PGCP_TRY(S->d_comps.alloc(nslot, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(S->d_comps.p, S->comps.data(), nslot * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    PGCP_TRY(S->sv_off.alloc(nslot + 1, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(S->sv_off.p, S->h_sv_off.data(), (nslot + 1) * sizeof(int64_t),
                                  cudaMemcpyHostToDevice, s));
    std::vector<int32_t> h_soc(b->K, -1);
    for (int j = 0; j < nslot; ++j) h_soc[S->comps[j]] = j;
    PGCP_TRY(S->slot_of_comp.alloc(b->K, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(S->slot_of_comp.p, h_soc.data(), b->K * sizeof(int32_t), cudaMemcpyHostToDevice, s));

    // fixed vertices and their values
    PGCP_TRY(S->fixed_ref.alloc(S->ne, s));
    PGCP_TRY(S->fixed_ref.fill_bytes(0xff, s));  // -1
    if (dncp) {
        PGCP_TRY(S->fv.alloc(2 * (int64_t)nslot, s));
        std::vector<double2> hfv(2 * nslot);
        for (int j = 0; j < nslot; ++j) {
            hfv[2 * j] = targets_host[0];
            hfv[2 * j + 1] = targets_host[1];
        }
        PGCP_TRY_CUDA(cudaMemcpyAsync(S->fv.p, hfv.data(), hfv.size() * sizeof(double2), cudaMemcpyHostToDevice, s));
        k_fixed_pins<<<grid_for(nslot, 64), 64, 0, s>>>(nslot, d_pins, S->sv_off.p, S->fixed_ref.p);
        PGCP_LAUNCH_CHECK();
        PGCP_TRY_CUDA(cudaStreamSynchronize(s));  // hfv is a local
    } else {
        PGCP_TRY(S->fv.alloc(nfixed, s));
        if (nfixed > 0) {
            if (fixed_val)
                PGCP_TRY_CUDA(cudaMemcpyAsync(S->fv.p, fixed_val, nfixed * sizeof(double2), cudaMemcpyDeviceToDevice, s));
            else
                PGCP_TRY(S->fv.zero(s));  // prepared solve: values (and the rhs) come later
            k_fixed_list<<<grid_for(nfixed, 256), 256, 0, s>>>(nfixed, fixed_gid, b->comp_of_gid.p,
                                                              S->slot_of_comp.p, b->vert_off.p, S->sv_off.p,
                                                              S->fixed_ref.p);
            PGCP_LAUNCH_CHECK();
        }
    }
    // unknown numbering
    DevBuf<int32_t> flag;
    DevBuf<int64_t> uscan;
    PGCP_TRY(flag.alloc(S->ne, s));
    PGCP_TRY(uscan.alloc(S->ne + 1, s));
    k_unknown_flag<<<grid_for(S->ne, 256), 256, 0, s>>>(S->ne, S->fixed_ref.p, flag.p);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY(exclusive_scan_i32_to_i64(flag.p, uscan.p, S->ne, s));
    std::vector<int64_t> hus(nslot + 1);
    {
        DevBuf<int64_t> g;
        PGCP_TRY(g.alloc(nslot + 1, s));
        k_gather_i64<<<grid_for(nslot + 1, 128), 128, 0, s>>>(uscan.p, S->sv_off.p, nslot + 1, g.p);
        PGCP_LAUNCH_CHECK();
        PGCP_TRY(d2h_async(hus.data(), g.p, (nslot + 1) * sizeof(int64_t), s));
        PGCP_TRY(d2h_flush(s));
    }
    S->h_nu.resize(nslot);
    S->h_sl_off.assign(nslot + 1, 0);
    for (int j = 0; j < nslot; ++j) {
        S->h_nu[j] = hus[j + 1] - hus[j];
        int64_t sl = (S->h_nu[j] + 31) / 32;
        if (sl == 0) sl = 1;  // keep every slot addressable (all-fixed submesh)
        S->h_sl_off[j + 1] = S->h_sl_off[j] + sl;
    }
    S->nslices = S->h_sl_off[nslot];
    S->rows = 32 * S->nslices;
    PGCP_TRY(S->sl_off.alloc(nslot + 1, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(S->sl_off.p, S->h_sl_off.data(), (nslot + 1) * sizeof(int64_t),
                                  cudaMemcpyHostToDevice, s));
    PGCP_TRY(S->urow.alloc(S->ne, s));
    PGCP_TRY(S->rowsrc.alloc(S->rows, s));
    PGCP_TRY(S->rowsrc.fill_bytes(0xff, s));
    {
        const char* ev = getenv("PGCP_PCG_COARSE");
        S->coarse = !S->force_jacobi && !S->use_direct && !(ev && atoi(ev) == 0);
        const char* eg = getenv("PGCP_PCG_GMAX");
        S->gmax = eg ? std::max(1, std::min(COARSE_GMAX, atoi(eg))) : COARSE_GMAX;
    }
    if (S->coarse) {
        PGCP_TRY(order_rows_by_cell(b, S, uscan.p, hus, s));
    } else {
        k_urow<<<grid_for(S->ne, 256), 256, 0, s>>>(S->ne, nslot, S->sv_off.p, S->sl_off.p, uscan.p, S->fixed_ref.p,
                                                  S->urow.p, S->rowsrc.p);
        PGCP_LAUNCH_CHECK();
    }

    BuildArgs a;
    a.nslot = nslot;
    a.comps = S->d_comps.p;
    a.sv_off = S->sv_off.p;
    a.sl_off = S->sl_off.p;
    a.vert_off = b->vert_off.p;
    a.row_ptr = b->row_ptr.p;
    a.col = b->col.p;
    a.val = val_override ? val_override : b->val.p;
    a.rowsrc = S->rowsrc.p;
    a.urow = S->urow.p;
    a.fixed_ref = S->fixed_ref.p;
    a.fv = S->fv.p;
    DevBuf<int64_t> len;
    PGCP_TRY(len.alloc(S->nslices, s));
    k_slice_len<<<grid_for(S->nslices * 32, 256), 256, 0, s>>>(a, S->nslices, len.p);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY(S->sl_ptr.alloc(S->nslices + 1, s));
    PGCP_TRY(exclusive_scan_i64(len.p, S->sl_ptr.p, S->nslices, s));
    PGCP_TRY(fetch_scalar(S->sl_ptr.p + S->nslices, &S->nnz, s));
    PGCP_TRY(S->col.alloc(S->nnz, s));
    PGCP_TRY(S->val.alloc(S->nnz, s));
    PGCP_TRY(S->D.alloc(S->rows, s));
    PGCP_TRY(S->Dinv.alloc(S->rows, s));
    PGCP_TRY(S->b.alloc(S->rows, s));
    PGCP_TRY(S->x.alloc(S->rows, s));
    PGCP_TRY(S->cpl.alloc(S->rows, s));
    PGCP_TRY(S->sl_mask.alloc(S->nslices, s));
    PGCP_TRY(S->sl_mask.zero(s));
    k_fill_rows<<<grid_for(S->rows, 256), 256, 0, s>>>(a, S->rows, S->sl_ptr.p, S->col.p, S->val.p, S->D.p,
                                                     S->Dinv.p, S->b.p, S->cpl.p, S->x.p);
    PGCP_LAUNCH_CHECK();
    if (dncp) {
        int64_t total = 0;
        for (int j = 0; j < nslot; ++j) {
            int c = S->comps[j];
            total += b->h_loop_off[c + 1] - b->h_loop_off[c];
        }
        if (total > 0) {
            k_coupling<<<grid_for(total, 256), 256, 0, s>>>(nslot, S->d_comps.p, b->loop_off.p, b->loop.p, S->sv_off.p,
                                                          S->sl_off.p, S->urow.p, S->fixed_ref.p, S->fv.p, S->cpl.p,
                                                          S->sl_mask.p, S->b.p, total);
            PGCP_LAUNCH_CHECK();
        }
    }
    // symmetric Jacobi scaling of the system (values, rhs, coupling)
    PGCP_TRY(S->Dsq.alloc(S->rows, s));
    PGCP_TRY(S->cplc.alloc(S->rows, s));
    PGCP_TRY(S->dmax.alloc(nslot, s));
    k_dsq<<<grid_for(S->rows, 256), 256, 0, s>>>(S->rows, S->D.p, S->Dsq.p);
    PGCP_LAUNCH_CHECK();
    k_scale<<<grid_for(S->rows, 256), 256, 0, s>>>(nslot, S->sl_off.p, S->rows, S->sl_ptr.p, S->col.p, S->val.p,
                                                 S->Dsq.p, S->b.p, S->cpl.p, S->cplc.p);
    PGCP_LAUNCH_CHECK();
    k_slot_dmax<<<nslot, 256, 0, s>>>(S->sl_off.p, S->D.p, S->dmax.p);
    PGCP_LAUNCH_CHECK();
    return PGCP_OK;
}

// cluster shape, coarse space (two-level) and the per-shape column encoding:
// everything of a solve that does not depend on the right-hand side
// loop vertices among a system's rows (the unknown ones: pins have no row)
__global__ void k_onloop(int32_t nslot, const int32_t* __restrict__ comps, const int64_t* __restrict__ loop_off,
                         const int32_t* __restrict__ loop, const int64_t* __restrict__ sv_off,
                         const int32_t* __restrict__ urow, uint8_t* __restrict__ onloop, int64_t total) {
    GRID_STRIDE(t, total) {
        int64_t acc = 0;
        int j = 0;
        for (; j < nslot; ++j) {
            const int c = comps[j];
            const int64_t nb = loop_off[c + 1] - loop_off[c];
            if (t < acc + nb) break;
            acc += nb;
        }
        if (j >= nslot) continue;
        const int c = comps[j];
        const int v = loop[loop_off[c] + (t - acc)];
        const int r = urow[sv_off[j] + v];
        if (r >= 0) onloop[r] = 1;
    }
}

// Dirichlet row -> DNCP row of the same compact vertex (-1: padding)
__global__ void k_h2f(int64_t rows, const int32_t* __restrict__ rowsrc, const int32_t* __restrict__ urow_f,
                      int32_t* __restrict__ h2f) {
    GRID_STRIDE(r, rows) {
        const int e = rowsrc[r];
        h2f[r] = e >= 0 ? urow_f[e] : -1;
    }
}

// PGCP_DIRECT_BLAST=1: factor the DNCP system with every loop last and
// solve the Dirichlet system with the interior block (no second
// factorization). Measured on cfg 2: the Dirichlet preparation drops from
// ~8 ms to 0.5 ms of GPU work, but the loops' 510-wide dense fronts put a
// long serial chain into both substitution sweeps (flatten 12.5 -> 15.9 ms
// standalone, step +3 ms), so the default keeps two factorizations.
bool boundary_last_enabled() {
    const char* e = getenv("PGCP_DIRECT_BLAST");
    return e && atoi(e) != 0;
}

// A Dirichlet system over the same submeshes as the last DNCP solve can use
// the interior block of that boundary-last factor: no factorization at all.
int try_borrow(pgcp_batch* b, SolveSystem* S, cudaStream_t s) {
    SolveSystem* F = static_cast<SolveSystem*>(b->sys[0]);
    if (!F || F == S || S->dncp || !F->dncp || !F->use_direct || !F->direct || !F->setup_done) return 0;
    if (!direct_is_boundary_last(F->direct.get()) || F->comps != S->comps) return 0;
    S->direct = F->direct;
    S->direct_home = F->direct_home;
    S->borrowed = true;
    PGCP_TRY(S->h2f.alloc(S->rows, s));
    if (F->direct_home && F->direct_home != s) {  // the factor is complete before this stream uses it
        cudaEvent_t ev;
        PGCP_TRY_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        PGCP_TRY_CUDA(cudaEventRecord(ev, F->direct_home));
        PGCP_TRY_CUDA(cudaStreamWaitEvent(s, ev, 0));
        cudaEventDestroy(ev);
    }
    k_h2f<<<grid_for(S->rows, 256), 256, 0, s>>>(S->rows, S->rowsrc.p, F->urow.p, S->h2f.p);
    PGCP_LAUNCH_CHECK();
    S->setup_done = true;
    return 1;
}

int setup_direct(pgcp_batch* b, SolveSystem* S, cudaStream_t s) {
    DirectInput in;
    in.nslot = S->nslot;
    in.comps = S->d_comps.p;
    in.sv_off = S->sv_off.p;
    in.sl_off = S->sl_off.p;
    in.h_sl_off = S->h_sl_off;
    in.h_nu = S->h_nu;
    in.rowsrc = S->rowsrc.p;
    in.sl_ptr = S->sl_ptr.p;
    in.nnz_ell = S->nnz;
    in.col = S->col.p;
    in.val = S->val.p;
    in.sl_mask = S->sl_mask.p;
    in.cpl = S->cpl.p;
    in.cplc = S->cplc.p;
    in.cplx = S->dncp;
    DevBuf<uint8_t> onloop;
    if (S->dncp && boundary_last_enabled()) {  // order every loop last: the interior block serves the Dirichlet solve
        PGCP_TRY(onloop.alloc(S->rows, s));
        PGCP_TRY(onloop.zero(s));
        int64_t total = 0;
        for (int j = 0; j < S->nslot; ++j) {
            const int c = S->comps[j];
            total += b->h_loop_off[c + 1] - b->h_loop_off[c];
        }
        if (total > 0) {
            k_onloop<<<grid_for(total, 256), 256, 0, s>>>(S->nslot, S->d_comps.p, b->loop_off.p, b->loop.p,
                                                        S->sv_off.p, S->urow.p, onloop.p, total);
            PGCP_LAUNCH_CHECK();
        }
        in.onloop = onloop.p;
    }
    DirectFactor* F = nullptr;
    const int rc = direct_factor(b, in, &F, s);
    if (rc == DIRECT_FALLBACK) {  // a front outgrew the kernels' bounds: plain PCG on the device
        S->use_direct = false;
        return PGCP_OK;
    }
    PGCP_TRY(rc);
    S->direct = std::shared_ptr<DirectFactor>(F, direct_free);
    S->direct_home = s;
    S->borrowed = false;
    S->setup_done = true;
    return PGCP_OK;
}

int setup_solve(pgcp_batch* b, SolveSystem* S, const pgcp_solve_opts* o, cudaStream_t s) {
    const int32_t nslot = S->nslot;
    if (S->use_direct) {
        if (!S->dncp && boundary_last_enabled()) {
            // Dirichlet system: the DNCP factor's interior block when there is one
            const int got = try_borrow(b, S, s);
            if (got < 0) return got;
            if (got) return PGCP_OK;
            if (S->lazy_direct) return PGCP_OK;  // decide at solve time (the flatten may still be running)
        }
        PGCP_TRY(setup_direct(b, S, s));
        if (S->use_direct) return PGCP_OK;
    }
    int64_t max_sl = 0;
    for (int j = 0; j < nslot; ++j) max_sl = std::max(max_sl, S->h_sl_off[j + 1] - S->h_sl_off[j]);
    int csize = 1, chunk = 1;
    if (const char* en = getenv("PGCP_PCG2_NT")) S->pcg_nt = atoi(en) == 256 ? 256 : 512;
    {
        const char* ef = getenv("PGCP_COARSE_FP64");
        S->einv_fp64 = ef && atoi(ef) != 0;
    }
    PGCP_TRY(pick_cluster(max_sl, nslot, o ? o->cluster : 0, S->coarse, S->pcg_nt, S->einv_fp64, &csize, &chunk));
    S->csize = csize;
    S->chunk = chunk;
    if (S->coarse) {
        cudaEvent_t c0, c1;
        PGCP_TRY_CUDA(cudaEventCreate(&c0));
        PGCP_TRY_CUDA(cudaEventCreate(&c1));
        PGCP_TRY_CUDA(cudaEventRecord(c0, s));
        PGCP_TRY(build_coarse(S, csize, s));
        PGCP_TRY_CUDA(cudaEventRecord(c1, s));
        PGCP_TRY_CUDA(cudaEventSynchronize(c1));
        float cms = 0;
        cudaEventElapsedTime(&cms, c0, c1);
        cudaEventDestroy(c0);
        cudaEventDestroy(c1);
        S->coarse_ms = cms;
    }
    PGCP_TRY(S->enc.alloc(S->nnz, s));
    PGCP_TRY(S->enc16.alloc(S->nnz, s));
    PGCP_TRY(S->remote.alloc(S->nslices, s));
    k_encode_cols<<<grid_for(S->nslices * 32, 256), 256, 0, s>>>(nslot, S->sl_off.p, S->nslices, S->sl_ptr.p, S->col.p,
                                                               csize, S->enc.p, S->enc16.p, S->remote.p);
    PGCP_LAUNCH_CHECK();
    S->setup_done = true;
    return PGCP_OK;
}

int run_solve(pgcp_batch* b, SolveSystem* S, const pgcp_solve_opts* o, double* z, pgcp_solve_stat* st,
              cudaStream_t s) {
    const int32_t nslot = S->nslot;
    if (!S->setup_done) PGCP_TRY(setup_solve(b, S, o, s));
    const int csize = S->csize, chunk = S->chunk;
    PGCP_TRY(S->iters.alloc(nslot, s));
    PGCP_TRY(S->res.alloc(8 * (int64_t)nslot, s));
    PGCP_TRY(S->res.zero(s));
    PcgArgs A;
    A.sl_off = S->sl_off.p;
    A.sl_ptr = S->sl_ptr.p;
    A.sl_mask = S->sl_mask.p;
    A.col = S->col.p;
    A.enc = S->enc.p;
    A.enc16 = S->enc16.p;
    A.remote = S->remote.p;
    A.val = S->val.p;
    A.D = S->D.p;
    A.dmax = S->dmax.p;
    A.cpl = S->cpl.p;
    A.cplc = S->cplc.p;
    A.b = S->b.p;
    A.x = S->x.p;
    A.iters = S->iters.p;
    A.res = S->res.p;
    double rtol = (o && o->rtol > 0) ? o->rtol : 1e-10;
    A.tol2 = rtol * rtol;
    // two-level PCG needs ~3.5x fewer iterations than Jacobi; its default cap
    // bounds the time lost before a slot falls back to Jacobi (solve_*)
    int coarse_cap = 60000;
    if (const char* ec = getenv("PGCP_PCG_COARSE_MAXIT")) coarse_cap = std::max(1, atoi(ec));  // tests
    A.maxit = (o && o->maxit > 0) ? o->maxit : (S->coarse ? coarse_cap : 200000);
    A.chunk_cap = chunk;
    A.C.abase = S->abase.p;
    A.C.aoff = S->aoff.p;
    A.C.wr = S->wr.p;
    A.C.einvh = S->einv_fp64 ? (const void*)S->einv64.p : (const void*)S->einv32.p;
    A.C.eoff32 = S->eoff32.p;
    A.C.p = S->p.p;
    A.ncb = S->ncb;
    A.mu_cap = S->mu_cap;
    A.items_cap = S->items_cap;
    DevBuf<long long> tbuf;
    A.timing = nullptr;
    A.order = nullptr;
    DevBuf<int32_t> dorder;
    std::vector<int32_t> hord(nslot);
    for (int j = 0; j < nslot; ++j) hord[j] = j;
    if (S->coarse && !S->force_jacobi) {
        const char* eo = getenv("PGCP_PCG_ORDER");
        std::vector<int32_t> prev;
        if (eo && !strcmp(eo, "prev")) {
            std::lock_guard<std::mutex> lock(g_prev_mu);
            prev = g_prev_iters;
        }
        // the harmonic solve launches its clusters heaviest first, predicted
        // by the same subdomains' iteration counts in the batch's last
        // flatten (longest-processing-time order shortens the last wave);
        // PGCP_HARM_ORDER=0 keeps the slot order
        std::vector<int32_t> pred;
        const char* eh = getenv("PGCP_HARM_ORDER");
        const SolveSystem* FS = static_cast<const SolveSystem*>(b->sys[0]);
        if (!eo && !S->dncp && !(eh && atoi(eh) == 0) && FS && FS != S && (int)FS->h_iters.size() == FS->nslot) {
            std::vector<int32_t> by_comp(b->K, -1);
            for (int j = 0; j < FS->nslot; ++j) by_comp[FS->comps[j]] = FS->h_iters[j];
            pred.resize(nslot);
            bool all = true;
            for (int j = 0; j < nslot; ++j) all &= (pred[j] = by_comp[S->comps[j]]) >= 0;
            if (!all) pred.clear();
        }
        if (eo && !strcmp(eo, "prev") && (int)prev.size() == nslot)
            std::stable_sort(hord.begin(), hord.end(), [&](int a, int b) { return prev[a] > prev[b]; });
        else if (eo && !strcmp(eo, "rev"))
            std::reverse(hord.begin(), hord.end());
        else if (!pred.empty())
            std::stable_sort(hord.begin(), hord.end(), [&](int a, int b) { return pred[a] > pred[b]; });
        if (eo || !pred.empty()) {
            PGCP_TRY(dorder.alloc(nslot, s));
            PGCP_TRY_CUDA(cudaMemcpyAsync(dorder.p, hord.data(), nslot * sizeof(int32_t), cudaMemcpyHostToDevice, s));
            A.order = dorder.p;
        }
    }
    DevBuf<double> hbuf;
    A.hist = nullptr;
    {
        const char* ex = getenv("PGCP_PCG_X0");
        A.x0 = ex ? atoi(ex) : 1;
    }
    const char* hist_path = getenv("PGCP_PCG_HIST");  // analysis aid: early CG coefficients per slot
    if (hist_path && S->coarse && !S->force_jacobi) {
        PGCP_TRY(hbuf.alloc((int64_t)nslot * HIST_K * 3, s));
        PGCP_TRY(hbuf.zero(s));
        A.hist = hbuf.p;
    }
    const bool want_timing = getenv("PGCP_PCG_TIMING") != nullptr;
    if (want_timing) {
        PGCP_TRY(tbuf.alloc(8 * (int64_t)nslot * csize, s));
        PGCP_TRY(tbuf.zero(s));
        A.timing = tbuf.p;
    }
    cudaEvent_t e0, e1;
    PGCP_TRY_CUDA(cudaEventCreate(&e0));
    PGCP_TRY_CUDA(cudaEventCreate(&e1));
    PGCP_TRY_CUDA(cudaEventRecord(e0, s));
    if (S->use_direct) {
        if (S->borrowed) {
            PGCP_TRY(direct_solve_interior(S->direct.get(), S->h2f.p, S->rows, S->b.p, S->x.p, s));
            // the factor's buffers are freed on the DNCP system's stream: order
            // that after this solve
            if (S->direct_home && S->direct_home != s) {
                cudaEvent_t ev;
                PGCP_TRY_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                PGCP_TRY_CUDA(cudaEventRecord(ev, s));
                PGCP_TRY_CUDA(cudaStreamWaitEvent(S->direct_home, ev, 0));
                cudaEventDestroy(ev);
            }
        } else {
            PGCP_TRY(direct_solve(S->direct.get(), S->b.p, S->x.p, s));
        }
        k_fill_i32<<<grid_for(nslot, 128), 128, 0, s>>>(S->iters.p, nslot, 1);
        PGCP_LAUNCH_CHECK();
    } else {
        PGCP_TRY(launch_pcg(S, A, csize, s));
        count_launch();
    }
    PGCP_TRY_CUDA(cudaEventRecord(e1, s));
    auto t_post = std::chrono::steady_clock::now();
    if (want_timing) {
        cudaEventSynchronize(e1);
        t_post = std::chrono::steady_clock::now();
    }
    k_true_residual<<<nslot, 1024, 0, s>>>(A);
    PGCP_LAUNCH_CHECK();
    k_scatter<<<grid_for(S->ne, 256), 256, 0, s>>>(S->ne, nslot, S->d_comps.p, S->sv_off.p, b->vert_off.p, S->urow.p,
                                                 S->fixed_ref.p, S->fv.p, S->x.p, S->Dsq.p, (double2*)z);
    PGCP_LAUNCH_CHECK();
    if (S->dncp) {
        k_flat_checks<<<nslot, 1024, 0, s>>>(S->d_comps.p, b->vert_off.p, b->row_ptr.p, b->col.p, b->val.p,
                                            b->loop_off.p, b->loop.p, (const double2*)z, S->res.p);
        PGCP_LAUNCH_CHECK();
    }
    // SURVEY 8(d) byte model of the PCG (entries of the reference's CSR
    // system per slot): PCG statistics only -- the direct solver's calls skip
    // the count, its stream synchronisation and the copy
    DevBuf<long long> refnz;
    std::vector<long long> hrefnz(nslot, 0);
    if (!S->use_direct) {
        PGCP_TRY(refnz.alloc(nslot, s));
        DevBuf<int64_t> dnu;
        std::vector<int64_t> hnu(S->h_nu.begin(), S->h_nu.end());
        PGCP_TRY(dnu.alloc(nslot, s));
        PGCP_TRY_CUDA(cudaMemcpyAsync(dnu.p, hnu.data(), nslot * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        k_ref_nnz<<<nslot, 256, 0, s>>>(S->sl_off.p, S->sl_ptr.p, S->col.p, S->val.p, S->sl_mask.p, S->cpl.p, dnu.p,
                                        S->dncp ? 1 : 0, refnz.p);
        PGCP_LAUNCH_CHECK();
        PGCP_TRY_CUDA(cudaStreamSynchronize(s));  // hnu is a local
        PGCP_TRY(d2h_async(hrefnz.data(), refnz.p, nslot * sizeof(long long), s));
    }
    std::vector<int32_t> hit(nslot);
    std::vector<double> hres(8 * nslot);
    std::vector<int64_t> hptr(S->nslices + 1);
    // through the pinned staging buffer: a pageable destination would make
    // the driver stage the copy synchronously and hold the other host
    // threads' launches meanwhile (concurrency lessons)
    PGCP_TRY(d2h_async(hptr.data(), S->sl_ptr.p, (S->nslices + 1) * sizeof(int64_t), s));
    PGCP_TRY(d2h_async(hit.data(), S->iters.p, nslot * sizeof(int32_t), s));
    PGCP_TRY(d2h_async(hres.data(), S->res.p, 8 * nslot * sizeof(double), s));
    PGCP_TRY(d2h_flush(s));
    S->h_iters = hit;
    if (S->coarse && !S->force_jacobi) {
        std::lock_guard<std::mutex> lock(g_prev_mu);
        g_prev_iters = hit;
    }
    if (A.hist) {
        std::vector<double> hh((size_t)nslot * HIST_K * 3);
        PGCP_TRY_CUDA(cudaMemcpy(hh.data(), hbuf.p, hh.size() * sizeof(double), cudaMemcpyDeviceToHost));
        if (FILE* f = fopen(hist_path, "ab")) {
            int32_t hdr[2] = {nslot, HIST_K};
            fwrite(hdr, sizeof hdr, 1, f);
            fwrite(hit.data(), sizeof(int32_t), nslot, f);
            fwrite(hh.data(), sizeof(double), hh.size(), f);
            fclose(f);
        }
    }
    if (want_timing)
        fprintf(stderr, "[pcg timing] post-solve (true residual, scatter, checks, stats) %.2f ms\n",
                1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t_post).count());
    if (want_timing) {
        std::vector<long long> ht(8 * (size_t)nslot * csize);
        PGCP_TRY_CUDA(cudaMemcpy(ht.data(), tbuf.p, ht.size() * sizeof(long long), cudaMemcpyDeviceToHost));
        double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (size_t i = 0; i < ht.size(); ++i) acc[i % 8] += (double)ht[i];
        double nct = (double)nslot * csize * 128.0;
        if (S->coarse) {
            // timeline: per cluster [first CTA start, last CTA end] (globaltimer ns)
            long long t0 = LLONG_MAX, t1 = 0;
            double busy = 0;
            int late = -1;
            long long late_end = 0;
            for (int c = 0; c < nslot; ++c) {
                long long cs = LLONG_MAX, ce = 0;
                for (int r = 0; r < csize; ++r) {
                    cs = std::min(cs, ht[8 * (size_t)(c * csize + r) + 6]);
                    ce = std::max(ce, ht[8 * (size_t)(c * csize + r) + 7]);
                }
                t0 = std::min(t0, cs);
                t1 = std::max(t1, ce);
                busy += (double)(ce - cs);
                if (ce > late_end) { late_end = ce; late = c; }
            }
            int first_wave = 0;
            long long last_start = 0;
            for (int c = 0; c < nslot; ++c) {
                long long cs = LLONG_MAX;
                for (int r = 0; r < csize; ++r) cs = std::min(cs, ht[8 * (size_t)(c * csize + r) + 6]);
                if (cs - t0 < 50000) ++first_wave;
                last_start = std::max(last_start, cs - t0);
            }
            long long ls = LLONG_MAX;
            for (int r = 0; r < csize; ++r) ls = std::min(ls, ht[8 * (size_t)(late * csize + r) + 6]);
            fprintf(stderr, "[pcg timing] timeline: makespan %.2f ms, cluster-busy sum %.1f ms (mean %.1f concurrent), "
                    "%d clusters in the first wave, last start %.2f ms; last to finish: cluster %d (slot %d, %d iters) "
                    "started %.2f ms\n", 1e-6 * (t1 - t0), 1e-6 * busy, busy / (double)(t1 - t0), first_wave,
                    1e-6 * last_start, late, hord[late], hit[hord[late]], 1e-6 * (ls - t0));
        }
        if (S->coarse) {
            fprintf(stderr, "[pcg timing] cycles/iter per CTA: A %.0f sync1 %.0f B %.0f sync2 %.0f C %.0f sync3 %.0f "
                    "(csize %d, coarse setup %.2f ms)\n", acc[0] / nct, acc[1] / nct, acc[2] / nct, acc[3] / nct,
                    acc[4] / nct, acc[5] / nct, csize, S->coarse_ms);
            // per cluster rank: where the time of the slowest CTA goes
            for (int r = 0; r < csize && r < 16; ++r) {
                double pr[6] = {0, 0, 0, 0, 0, 0};
                for (int c = 0; c < nslot; ++c)
                    for (int q = 0; q < 6; ++q) pr[q] += (double)ht[8 * (size_t)(c * csize + r) + q];
                const double d = (double)nslot * 128.0;
                fprintf(stderr, "[pcg timing]   rank %d: A %.0f sync1 %.0f B %.0f sync2 %.0f C %.0f sync3 %.0f\n", r,
                        pr[0] / d, pr[1] / d, pr[2] / d, pr[3] / d, pr[4] / d, pr[5] / d);
            }
        }
        else
            fprintf(stderr, "[pcg timing] cycles/iter per CTA: phaseA %.0f red1 %.0f phaseB %.0f red2 %.0f (csize %d)\n",
                    acc[0] / nct, acc[1] / nct, acc[2] / nct, acc[3] / nct, csize);
    }
    {
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        S->kernel_ms = ms;
        // compulsory bytes per iteration of slot j: stored off-diagonal
        // values + cols (12 B per slice entry) and the y update (read +
        // write, 32 B per unknown row); CG vectors stay on chip. Two-level
        // (k_pcg2) adds p read + write (32 B/row), the fp16 coarse weights
        // read twice (2 x 8 B/row) and the float E^-1 (8 nc ncp B per slot).
        S->iters_sum = S->iters_max = S->bytes_iter_weighted = S->ref_bytes_weighted = 0;
        std::vector<uint8_t> hrem;
        if (S->coarse) {  // all-local slices stream 16-bit codes in k_pcg2
            hrem.resize(S->nslices);
            PGCP_TRY_CUDA(cudaMemcpy(hrem.data(), S->remote.p, S->nslices, cudaMemcpyDeviceToHost));
        }
        for (int j = 0; j < nslot; ++j) {
            int64_t e = hptr[S->h_sl_off[j + 1]] - hptr[S->h_sl_off[j]];
            double rows = (double)S->h_nu[j];
            double bytes = 12.0 * (double)e + 32.0 * rows;
            if (S->coarse) {
                int64_t e_local = 0;
                for (int64_t q = S->h_sl_off[j]; q < S->h_sl_off[j + 1]; ++q)
                    if (!hrem[q]) e_local += hptr[q + 1] - hptr[q];
                bytes -= 2.0 * (double)e_local;
                double nc = 3.0 * (double)(S->h_abase[j + 1] - S->h_abase[j]);
                double ncp = (double)(((int64_t)nc + 7) & ~7ll);
                bytes += 48.0 * rows + 8.0 * nc * ncp;
            }
            S->iters_sum += hit[j];
            S->iters_max = std::max<double>(S->iters_max, hit[j]);
            S->bytes_iter_weighted += bytes * hit[j];
            const double rref = S->dncp ? 2.0 * rows : rows;
            if (!S->use_direct) S->ref_bytes_weighted += (12.0 * (double)hrefnz[j] + 4.0 * (rref + 1.0)) * hit[j];
            S->nrows_u += rows;
            S->nnz_off += (double)e;
        }
    }
    const double ctol = (o && o->contract_tol > 0) ? o->contract_tol : 1e-10;
    int worst = PGCP_OK;
    for (int j = 0; j < nslot; ++j) {
        pgcp_solve_stat t;
        t.iters = hit[j];
        t.relres = hres[8 * j + 0];
        t.true_res = hres[8 * j + 2];
        t.xnorm = hres[8 * j + 3];
        t.bnorm = hres[8 * j + 4];
        t.status = PGCP_OK;
        bool finite = std::isfinite(t.true_res) && std::isfinite(t.xnorm);
        if (S->use_direct && S->direct && direct_slot_status(S->direct.get())[j]) finite = false;  // pivot <= 0
        if (!finite) {
            t.status = PGCP_E_SOLVE;
        } else if (t.relres > rtol && t.iters >= A.maxit) {
            t.status = PGCP_E_NOCONV;
        } else if (t.bnorm > 0 && t.true_res > std::max(ctol * t.bnorm, 1e3 * ctol * t.xnorm)) {
            t.status = PGCP_E_SOLVE;
        }
        if (st) st[j] = t;
        if (t.status != PGCP_OK && worst == PGCP_OK) {
            worst = t.status;
            if (t.status == PGCP_E_NOCONV)
                set_error("submesh %d: PCG did not converge (%d iterations, relres %.3e)", S->comps[j], t.iters,
                          t.relres);
            else if (!finite)
                set_error("submesh %d: singular or non-finite system", S->comps[j]);
            else
                set_error("submesh %d: %s residual %.3e above tolerance", S->comps[j],
                          S->dncp ? "flattening" : "harmonic", t.true_res);
        }
        if (S->dncp && worst == PGCP_OK) {
            double area = hres[8 * j + 5], ec = hres[8 * j + 6], sc2 = hres[8 * j + 7];
            if (area <= 0) {
                set_error("flattening produced nonpositive signed area (inconsistent input orientation)");
                if (st) st[j].status = PGCP_E_MESH;
                worst = PGCP_E_MESH;
            } else if (ec < -1e-8 * sc2) {
                set_error("conformal energy %.3e below lower bound", ec);
                if (st) st[j].status = PGCP_E_SOLVE;
                worst = PGCP_E_SOLVE;
            }
        }
    }
    return worst;
}

// solver choice: the direct solver unless the caller asks for PCG (explicitly,
// by an iteration cap, or PGCP_SOLVER=pcg)
bool want_direct(const pgcp_solve_opts* o) {
    const int k = o ? o->solver : PGCP_SOLVER_DEFAULT;
    if (k == PGCP_SOLVER_DIRECT) return true;
    if (k == PGCP_SOLVER_PCG) return false;
    if (o && o->maxit > 0) return false;
    const char* e = getenv("PGCP_SOLVER");
    return !(e && !strcmp(e, "pcg"));
}

int prepare_slots(pgcp_batch* b, SolveSystem* S, const int32_t* comps, int32_t ncomp) {
    if (!b->has_laplacian) {
        set_error("laplacian not built");
        return PGCP_E_INVALID;
    }
    if (comps == nullptr) {
        S->comps.resize(b->K);
        for (int c = 0; c < b->K; ++c) S->comps[c] = c;
    } else {
        S->comps.assign(comps, comps + ncomp);
        for (int c : S->comps)
            if (c < 0 || c >= b->K) {
                set_error("submesh id %d out of range", c);
                return PGCP_E_INVALID;
            }
    }
    S->nslot = (int32_t)S->comps.size();
    return PGCP_OK;
}

}  // namespace

SolveSystem*& system_slot(pgcp_batch* b, int which) {
    return reinterpret_cast<SolveSystem*&>(b->sys[which]);
}

int solve_flatten(pgcp_batch* b, const int32_t* comps, int32_t ncomp, const int32_t* pins, const double* targets,
                  const pgcp_solve_opts* o, double* z, pgcp_solve_stat* st, cudaStream_t s) {
    SolveSystem*& slot = system_slot(b, 0);
    delete slot;
    slot = new SolveSystem();
    SolveSystem* S = slot;
    S->built_on(s);
    S->use_direct = want_direct(o);
    PGCP_TRY(prepare_slots(b, S, comps, ncomp));
    if (S->nslot == 0) return PGCP_OK;
    double2 t[2] = {make_double2(0.0, 0.0), make_double2(1.0, 0.0)};
    if (targets) {
        t[0] = make_double2(targets[0], targets[1]);
        t[1] = make_double2(targets[2], targets[3]);
    }
    if (t[0].x == t[1].x && t[0].y == t[1].y) {
        set_error("pin targets must be distinct");
        return PGCP_E_MESH;
    }
    // pins: given (host, local) or the default half-perimeter pins
    DevBuf<int32_t> dp;
    PGCP_TRY(dp.alloc(2 * (int64_t)S->nslot, s));
    std::vector<int32_t> hp(2 * S->nslot);
    if (pins) {
        for (int j = 0; j < 2 * S->nslot; ++j) hp[j] = pins[j];
    } else {
        if (b->pins.p == nullptr) PGCP_TRY(default_pins(b, s));
        std::vector<int32_t> all(2 * b->K);
        PGCP_TRY(d2h_async(all.data(), b->pins.p, all.size() * sizeof(int32_t), s));  // pinned staging
        PGCP_TRY(d2h_flush(s));
        for (int j = 0; j < S->nslot; ++j) {
            hp[2 * j] = all[2 * S->comps[j]];
            hp[2 * j + 1] = all[2 * S->comps[j] + 1];
        }
    }
    // pins must be two distinct boundary vertices (flatten.py:154-157)
    for (int j = 0; j < S->nslot; ++j) {
        int c = S->comps[j];
        int64_t nc = b->h_vert_off[c + 1] - b->h_vert_off[c];
        if (hp[2 * j] == hp[2 * j + 1] || hp[2 * j] < 0 || hp[2 * j + 1] < 0 || hp[2 * j] >= nc || hp[2 * j + 1] >= nc) {
            set_error("pins must be two distinct boundary vertices");
            return PGCP_E_MESH;
        }
    }
    if (pins) {  // boundary membership of user pins
        std::vector<int32_t> hl(b->sum_nb);
        PGCP_TRY_CUDA(cudaMemcpyAsync(hl.data(), b->loop.p, b->sum_nb * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        PGCP_TRY_CUDA(cudaStreamSynchronize(s));
        for (int j = 0; j < S->nslot; ++j) {
            int c = S->comps[j];
            bool f0 = false, f1 = false;
            for (int64_t q = b->h_loop_off[c]; q < b->h_loop_off[c + 1]; ++q) {
                f0 |= hl[q] == hp[2 * j];
                f1 |= hl[q] == hp[2 * j + 1];
            }
            if (!f0 || !f1) {
                set_error("pins must be two distinct boundary vertices");
                return PGCP_E_MESH;
            }
        }
    }
    PGCP_TRY_CUDA(cudaMemcpyAsync(dp.p, hp.data(), hp.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    b->last_flat_pins = hp;
    auto t0 = std::chrono::steady_clock::now();
    PGCP_TRY(build_system(b, S, true, dp.p, t, nullptr, nullptr, 0, s));
    if (getenv("PGCP_PCG_TIMING")) {
        cudaStreamSynchronize(s);
        fprintf(stderr, "[pcg timing] flatten build_system %.2f ms (host, synchronised)\n",
                1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    std::vector<pgcp_solve_stat> hst(S->nslot);
    int rc = run_solve(b, S, o, z, hst.data(), s);
    bool only_noconv = rc == PGCP_E_NOCONV;
    for (int j = 0; j < S->nslot && only_noconv; ++j)
        only_noconv = hst[j].status == PGCP_OK || hst[j].status == PGCP_E_NOCONV;
    if (only_noconv && S->coarse && !(o && o->maxit > 0)) {
        // safety net: re-solve the slots the two-level PCG did not finish with
        // plain Jacobi-PCG (same kernels family, still on the device)
        std::vector<int32_t> rc_comps, rc_pins;
        std::vector<int> where;
        for (int j = 0; j < S->nslot; ++j)
            if (hst[j].status == PGCP_E_NOCONV) {
                rc_comps.push_back(S->comps[j]);
                rc_pins.push_back(hp[2 * j]);
                rc_pins.push_back(hp[2 * j + 1]);
                where.push_back(j);
            }
        SolveSystem R;
        R.force_jacobi = true;
        PGCP_TRY(prepare_slots(b, &R, rc_comps.data(), (int32_t)rc_comps.size()));
        DevBuf<int32_t> dp2;
        PGCP_TRY(dp2.alloc((int64_t)rc_pins.size(), s));
        PGCP_TRY_CUDA(cudaMemcpyAsync(dp2.p, rc_pins.data(), rc_pins.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
        PGCP_TRY(build_system(b, &R, true, dp2.p, t, nullptr, nullptr, 0, s));
        std::vector<pgcp_solve_stat> rst(R.nslot);
        rc = run_solve(b, &R, o, z, rst.data(), s);
        for (size_t q = 0; q < where.size(); ++q) hst[where[q]] = rst[q];
        S->kernel_ms += R.kernel_ms;
        S->iters_sum += R.iters_sum;
        S->iters_max = std::max(S->iters_max, R.iters_max);
        S->bytes_iter_weighted += R.bytes_iter_weighted;
        S->ref_bytes_weighted += R.ref_bytes_weighted;
    }
    if (st)
        for (int j = 0; j < S->nslot; ++j) st[j] = hst[j];
    PGCP_TRY(S->used_on(s));
    return rc;
}

// Harmonic solve in two parts so the structure (unknown numbering, sliced
// ELL, Jacobi scaling, coarse space, column encoding) can be built while the
// fixed values are still being computed (pipeline: during the weld).
int prepare_harmonic(pgcp_batch* b, const int32_t* comps, int32_t ncomp, const int32_t* fixed_gid, int64_t nfixed,
                     const pgcp_solve_opts* o, cudaStream_t s) {
    SolveSystem*& slot = system_slot(b, 1);
    delete slot;
    slot = new SolveSystem();
    SolveSystem* S = slot;
    S->built_on(s);
    S->use_direct = want_direct(o);
    PGCP_TRY(prepare_slots(b, S, comps, ncomp));
    S->nfixed = nfixed;
    PGCP_TRY(S->fixed_gid_copy.alloc(std::max<int64_t>(nfixed, 1), s));
    if (nfixed > 0)
        PGCP_TRY_CUDA(cudaMemcpyAsync(S->fixed_gid_copy.p, fixed_gid, nfixed * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    if (S->nslot == 0) {
        S->prepared = true;
        return PGCP_OK;
    }
    auto t0 = std::chrono::steady_clock::now();
    PGCP_TRY(build_system(b, S, false, nullptr, nullptr, S->fixed_gid_copy.p, nullptr, nfixed, s));
    S->lazy_direct = true;  // the direct solver factors (or borrows the DNCP factor) at solve time
    PGCP_TRY(setup_solve(b, S, o, s));
    S->lazy_direct = false;
    PGCP_TRY_CUDA(cudaStreamSynchronize(s));
    if (getenv("PGCP_PCG_TIMING"))
        fprintf(stderr, "[pcg timing] harmonic prepare (build + setup) %.2f ms (host, synchronised)\n",
                1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    S->prepared = true;
    return PGCP_OK;
}

int finish_harmonic(pgcp_batch* b, const double* fixed_val, int64_t nfixed, const pgcp_solve_opts* o, double* z,
                    pgcp_solve_stat* st, cudaStream_t s) {
    SolveSystem* S = system_slot(b, 1);
    if (!S || !S->prepared) {
        set_error("harmonic solve: no prepared system (call pgcp_batch_harmonic_prepare first)");
        return PGCP_E_INVALID;
    }
    if (nfixed != S->nfixed) {
        set_error("harmonic solve: %lld fixed values for %lld fixed vertices", (long long)nfixed, (long long)S->nfixed);
        return PGCP_E_INVALID;
    }
    S->prepared = false;
    if (S->nslot == 0) return PGCP_OK;
    if (nfixed > 0) {
        PGCP_TRY_CUDA(cudaMemcpyAsync(S->fv.p, fixed_val, nfixed * sizeof(double2), cudaMemcpyDeviceToDevice, s));
        BuildArgs a;
        a.nslot = S->nslot;
        a.comps = S->d_comps.p;
        a.sv_off = S->sv_off.p;
        a.sl_off = S->sl_off.p;
        a.vert_off = b->vert_off.p;
        a.row_ptr = b->row_ptr.p;
        a.col = b->col.p;
        a.val = b->val.p;
        a.rowsrc = S->rowsrc.p;
        a.urow = S->urow.p;
        a.fixed_ref = S->fixed_ref.p;
        a.fv = S->fv.p;
        k_rhs_fixed<<<grid_for(S->rows, 256), 256, 0, s>>>(a, S->rows, S->Dsq.p, S->b.p);
        PGCP_LAUNCH_CHECK();
    }
    std::vector<pgcp_solve_stat> hst(S->nslot);
    int rc = run_solve(b, S, o, z, hst.data(), s);
    bool only_noconv = rc == PGCP_E_NOCONV;
    for (int j = 0; j < S->nslot && only_noconv; ++j)
        only_noconv = hst[j].status == PGCP_OK || hst[j].status == PGCP_E_NOCONV;
    if (only_noconv && S->coarse && !(o && o->maxit > 0)) {  // Jacobi safety net (see solve_flatten)
        std::vector<int32_t> rc_comps;
        std::vector<int> where;
        for (int j = 0; j < S->nslot; ++j)
            if (hst[j].status == PGCP_E_NOCONV) {
                rc_comps.push_back(S->comps[j]);
                where.push_back(j);
            }
        SolveSystem R;
        R.force_jacobi = true;
        PGCP_TRY(prepare_slots(b, &R, rc_comps.data(), (int32_t)rc_comps.size()));
        PGCP_TRY(build_system(b, &R, false, nullptr, nullptr, S->fixed_gid_copy.p, fixed_val, nfixed, s));
        std::vector<pgcp_solve_stat> rst(R.nslot);
        rc = run_solve(b, &R, o, z, rst.data(), s);
        for (size_t q = 0; q < where.size(); ++q) hst[where[q]] = rst[q];
        S->kernel_ms += R.kernel_ms;
        S->iters_sum += R.iters_sum;
        S->iters_max = std::max(S->iters_max, R.iters_max);
        S->bytes_iter_weighted += R.bytes_iter_weighted;
        S->ref_bytes_weighted += R.ref_bytes_weighted;
    }
    if (st)
        for (int j = 0; j < S->nslot; ++j) st[j] = hst[j];
    PGCP_TRY(S->used_on(s));
    return rc;
}

int solve_harmonic(pgcp_batch* b, const int32_t* comps, int32_t ncomp, const int32_t* fixed_gid,
                   const double* fixed_val, int64_t nfixed, const pgcp_solve_opts* o, double* z,
                   pgcp_solve_stat* st, cudaStream_t s) {
    PGCP_TRY(prepare_harmonic(b, comps, ncomp, fixed_gid, nfixed, o, s));
    return finish_harmonic(b, fixed_val, nfixed, o, z, st, s);
}

// Dirichlet solve of the listed submeshes with explicit matrix values on the
// Laplacian pattern (repair.cu: assemble.py:205-213, K_ff u = -K_f,fixed g
// for both coordinates). Same solver and safety net as the harmonic solve;
// the system is not kept on the batch.
int solve_values(pgcp_batch* b, const int32_t* comps, int32_t ncomp, const double* vals, const int32_t* fixed_gid,
                 const double* fixed_val, int64_t nfixed, const pgcp_solve_opts* o, double* z, pgcp_solve_stat* st,
                 cudaStream_t s) {
    SolveSystem S;
    PGCP_TRY(prepare_slots(b, &S, comps, ncomp));
    if (S.nslot == 0) return PGCP_OK;
    PGCP_TRY(build_system(b, &S, false, nullptr, nullptr, fixed_gid, fixed_val, nfixed, s, vals));
    std::vector<pgcp_solve_stat> hst(S.nslot);
    int rc = run_solve(b, &S, o, z, hst.data(), s);
    bool only_noconv = rc == PGCP_E_NOCONV;
    for (int j = 0; j < S.nslot && only_noconv; ++j)
        only_noconv = hst[j].status == PGCP_OK || hst[j].status == PGCP_E_NOCONV;
    if (only_noconv && S.coarse && !(o && o->maxit > 0)) {
        std::vector<int32_t> rc_comps;
        std::vector<int> where;
        for (int j = 0; j < S.nslot; ++j)
            if (hst[j].status == PGCP_E_NOCONV) {
                rc_comps.push_back(S.comps[j]);
                where.push_back(j);
            }
        SolveSystem R;
        R.force_jacobi = true;
        PGCP_TRY(prepare_slots(b, &R, rc_comps.data(), (int32_t)rc_comps.size()));
        PGCP_TRY(build_system(b, &R, false, nullptr, nullptr, fixed_gid, fixed_val, nfixed, s, vals));
        std::vector<pgcp_solve_stat> rst(R.nslot);
        rc = run_solve(b, &R, o, z, rst.data(), s);
        for (size_t q = 0; q < where.size(); ++q) hst[where[q]] = rst[q];
    }
    if (st)
        for (int j = 0; j < S.nslot; ++j) st[j] = hst[j];
    return rc;
}

int system_dims(pgcp_batch* b, int which, int32_t* nslot_out) {
    SolveSystem* S = system_slot(b, which);
    *nslot_out = S ? S->nslot : 0;
    return PGCP_OK;
}


// Host-side export of the last solve's system in the reference's CSR form,
// for pattern parity: which = 0 -> C_ff (flatten.py:160-166, real 2|U| rows,
// exact zeros of L dropped as csr_binop does), which = 1 -> L_II
// (assemble.py:40, explicit zeros kept). Built from the device Laplacian and
// the device unknown/fixed maps of that solve.
int export_system(pgcp_batch* b, int which, int32_t comp, int64_t* dims, int32_t* indptr, int32_t* indices,
                  double* data, double* rhs, cudaStream_t s) {
    if (which < 0 || which > 1) {
        set_error("export_system: which must be 0 or 1");
        return PGCP_E_INVALID;
    }
    SolveSystem* S = system_slot(b, which);
    if (!S) {
        set_error("export_system: no %s solve has run", which ? "harmonic" : "flatten");
        return PGCP_E_INVALID;
    }
    int j = -1;
    for (int q = 0; q < S->nslot; ++q)
        if (S->comps[q] == comp) j = q;
    if (j < 0) {
        set_error("export_system: submesh %d was not part of the last solve", comp);
        return PGCP_E_INVALID;
    }
    const int64_t v0 = b->h_vert_off[comp], nc = b->h_vert_off[comp + 1] - v0;
    std::vector<int64_t> rp(nc + 1);
    PGCP_TRY_CUDA(cudaMemcpyAsync(rp.data(), b->row_ptr.p + v0, (nc + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaStreamSynchronize(s));
    const int64_t e0 = rp[0], ne = rp[nc] - rp[0];
    std::vector<int32_t> cl(ne), fr(nc), ur(nc), lp;
    std::vector<double> vl(ne);
    PGCP_TRY_CUDA(cudaMemcpyAsync(cl.data(), b->col.p + e0, ne * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(vl.data(), b->val.p + e0, ne * sizeof(double), cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(fr.data(), S->fixed_ref.p + S->h_sv_off[j], nc * sizeof(int32_t),
                                  cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(ur.data(), S->urow.p + S->h_sv_off[j], nc * sizeof(int32_t),
                                  cudaMemcpyDeviceToHost, s));
    const int64_t lo = b->h_loop_off[comp], nb = b->h_loop_off[comp + 1] - lo;
    lp.resize(nb);
    PGCP_TRY_CUDA(cudaMemcpyAsync(lp.data(), b->loop.p + lo, nb * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    const int64_t nU = S->h_nu[j];
    std::vector<double2> hb(nU > 0 ? nU : 1);
    std::vector<double> hd(nU > 0 ? nU : 1);
    if (nU > 0) {
        PGCP_TRY_CUDA(cudaMemcpyAsync(hb.data(), S->b.p + 32 * S->h_sl_off[j], nU * sizeof(double2),
                                      cudaMemcpyDeviceToHost, s));
        PGCP_TRY_CUDA(cudaMemcpyAsync(hd.data(), S->Dsq.p + 32 * S->h_sl_off[j], nU * sizeof(double),
                                      cudaMemcpyDeviceToHost, s));
    }
    PGCP_TRY_CUDA(cudaStreamSynchronize(s));
    for (int64_t r = 0; r < nU; ++r) {  // the solver holds D^{-1/2} b
        hb[r].x *= hd[r];
        hb[r].y *= hd[r];
    }
    const int64_t rbase = 32 * S->h_sl_off[j];
    // columns in the reference's order (unknowns by vertex id); the solver's
    // row of vertex v is ur[v] - rbase (cell order with the coarse space)
    std::vector<int64_t> pos(nc, -1), srow(nc, -1);
    {
        int64_t k = 0;
        for (int64_t v = 0; v < nc; ++v)
            if (fr[v] < 0) {
                pos[v] = k++;
                srow[v] = ur[v] - rbase;
            }
    }
    std::vector<int64_t> nxt(nc, -1), prv(nc, -1);
    if (nb >= 3)
        for (int64_t q = 0; q < nb; ++q) {
            nxt[lp[q]] = lp[(q + 1) % nb];
            prv[lp[q]] = lp[(q + nb - 1) % nb];
        }
    std::vector<int32_t> ip, ix;
    std::vector<double> dv;
    ip.push_back(0);
    auto push_L = [&](int64_t u, int64_t shift, bool drop_zero) {
        for (int64_t q = rp[u] - e0; q < rp[u + 1] - e0; ++q) {
            int64_t c = cl[q];
            if (pos[c] < 0) continue;
            if (drop_zero && vl[q] == 0.0) continue;
            ix.push_back((int32_t)(pos[c] + shift));
            dv.push_back(vl[q]);
        }
    };
    auto push_cpl = [&](int64_t u, int64_t shift, double sn) {
        // (next: sn, prev: -sn), sorted by column
        int64_t a = nxt[u] >= 0 ? pos[nxt[u]] : -1, c = prv[u] >= 0 ? pos[prv[u]] : -1;
        std::pair<int64_t, double> e[2];
        int k = 0;
        if (a >= 0) e[k++] = {a + shift, sn};
        if (c >= 0) e[k++] = {c + shift, -sn};
        if (k == 2 && e[1].first < e[0].first) std::swap(e[0], e[1]);
        for (int t = 0; t < k; ++t) {
            ix.push_back((int32_t)e[t].first);
            dv.push_back(e[t].second);
        }
    };
    std::vector<double> hr;
    std::vector<int64_t> U;
    for (int64_t v = 0; v < nc; ++v)
        if (pos[v] >= 0) U.push_back(v);
    if (which == 0) {
        for (int64_t r = 0; r < nU; ++r) {  // x rows: L | -2 M_xy
            push_L(U[r], 0, true);
            push_cpl(U[r], nU, -0.5);
            ip.push_back((int32_t)ix.size());
            hr.push_back(hb[srow[U[r]]].x);
        }
        for (int64_t r = 0; r < nU; ++r) {  // y rows: 2 M_xy | L
            push_cpl(U[r], 0, 0.5);
            push_L(U[r], nU, true);
            ip.push_back((int32_t)ix.size());
            hr.push_back(hb[srow[U[r]]].y);
        }
    } else {
        for (int64_t r = 0; r < nU; ++r) {
            push_L(U[r], 0, false);
            ip.push_back((int32_t)ix.size());
            hr.push_back(hb[srow[U[r]]].x);
            hr.push_back(hb[srow[U[r]]].y);
        }
    }
    dims[0] = (int64_t)ip.size() - 1;
    dims[1] = (int64_t)ix.size();
    if (indptr) std::copy(ip.begin(), ip.end(), indptr);
    if (indices) std::copy(ix.begin(), ix.end(), indices);
    if (data) std::copy(dv.begin(), dv.end(), data);
    if (rhs) std::copy(hr.begin(), hr.end(), rhs);
    return PGCP_OK;
}


void solve_summary(const pgcp_batch* b, int which, double* out) {
    for (int i = 0; i < 19; ++i) out[i] = 0;
    SolveSystem* S = static_cast<SolveSystem*>(b->sys[which]);
    if (!S) return;
    out[0] = S->kernel_ms;
    out[1] = S->iters_sum;
    out[2] = S->iters_max;
    out[3] = S->bytes_iter_weighted;   // sum over slots of iters * compulsory bytes/iter
    out[4] = S->nnz_off;               // stored slice entries (incl. padding)
    out[5] = S->nrows_u;
    out[6] = S->csize;
    out[7] = S->nslot;
    out[8] = S->ref_bytes_weighted;
    out[9] = S->coarse_ms;
    // direct solver: [10] 1, [11] real FMAs of the factorization, [12] factor
    // ms, [13] solve ms (forward + backward), [14] largest front, [15] front
    // storage bytes, [16] tree nodes, [17] tree levels, [18] numeric-phase ms
    if (S->use_direct && S->direct) {
        double d[9];
        direct_stats(S->direct.get(), d);
        out[10] = S->borrowed ? 2 : 1;  // 2: the DNCP factor's interior block (no factorization of its own)
        out[11] = S->borrowed ? 0.0 : d[3];
        out[12] = S->borrowed ? 0.0 : d[4];
        out[13] = d[5];
        out[14] = d[2];
        out[15] = d[6];
        out[16] = d[0];
        out[17] = d[1];
        out[18] = S->borrowed ? 0.0 : d[8];
    }
}

}  // namespace pgcp
