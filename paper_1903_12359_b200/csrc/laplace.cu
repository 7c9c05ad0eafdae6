// laplace.cu -- K1 cotangent weights and K2 canonical CSR cotangent Laplacian.
//
// K1 replaces flatten.py:39-57 (per face, per corner i with opposite edge
// (j,k): cot = (u1.u2)/|u1 x u2|, u1 = v_j - v_i, u2 = v_k - v_i). The
// arithmetic is written with explicit round-to-nearest intrinsics (no FMA
// contraction) in numpy's evaluation order -- cross = np.cross, norm =
// sqrt((cx^2 + cy^2) + cz^2), dot = (x + z) + y (einsum's SIMD pairing,
// verified bit-exact on the build host) -- so the weights, and therefore the
// exact-zero pattern of C = blockdiag(L,L) - 2M, match the reference.
//
// K2 replaces `csr_matrix((vals,(rows,cols)))` of flatten.py:61: one thread
// per submesh-local vertex gathers (neighbour, weight) pairs from the faces of
// its submesh around it, sorts them by column (the segment sort), and merges
// duplicates; off-diagonals are sums of <= 2 terms (order-free in IEEE), so
// they are bit-identical to scipy's; the diagonal is summed in the COO order
// of the reference's triplets.
#include "batch.cuh"

namespace pgcp {
namespace {

constexpr double COT_CLAMP = 1e8;  // flatten.py:21

__global__ void k_cot(const double* __restrict__ V, const int32_t* __restrict__ F, int64_t m,
                      double* __restrict__ w3, DevErr* err, unsigned long long* nclamp) {
    GRID_STRIDE(f, m) {
        int vid[3] = {F[3 * f], F[3 * f + 1], F[3 * f + 2]};
        double p[3][3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            p[c][0] = V[3 * vid[c]];
            p[c][1] = V[3 * vid[c] + 1];
            p[c][2] = V[3 * vid[c] + 2];
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int j = (c + 1) % 3, k = (c + 2) % 3;
            double ax = __dsub_rn(p[j][0], p[c][0]), ay = __dsub_rn(p[j][1], p[c][1]), az = __dsub_rn(p[j][2], p[c][2]);
            double bx = __dsub_rn(p[k][0], p[c][0]), by = __dsub_rn(p[k][1], p[c][1]), bz = __dsub_rn(p[k][2], p[c][2]);
            double cx = __dsub_rn(__dmul_rn(ay, bz), __dmul_rn(az, by));
            double cy = __dsub_rn(__dmul_rn(az, bx), __dmul_rn(ax, bz));
            double cz = __dsub_rn(__dmul_rn(ax, by), __dmul_rn(ay, bx));
            double nrm = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(cx, cx), __dmul_rn(cy, cy)), __dmul_rn(cz, cz)));
            double dot = __dadd_rn(__dadd_rn(__dmul_rn(ax, bx), __dmul_rn(az, bz)), __dmul_rn(ay, by));
            if (nrm == 0.0) {
                dev_fail(err, 1, f);
                w3[3 * f + c] = 0.0;
                continue;
            }
            double ct = __ddiv_rn(dot, nrm);
            if (fabs(ct) > COT_CLAMP) {
                atomicAdd(nclamp, 1ull);
                ct = fmin(fmax(ct, -COT_CLAMP), COT_CLAMP);
            }
            w3[3 * f + c] = __dmul_rn(0.5, ct);
        }
    }
}

constexpr int MAXF = 64;  // incident faces of one vertex inside one submesh

struct RowEntry {
    int32_t col;  // parent id while gathering
    double w;
};

// Gather the row of local vertex g. Returns the number of off-diagonal pairs
// (before merging) in e[], the diagonal in *diag; -1 on valence overflow.
__device__ int gather_row(const int32_t* __restrict__ F, const int64_t* __restrict__ inc_off,
                          const int32_t* __restrict__ inc, const int32_t* __restrict__ face_comp,
                          const double* __restrict__ w3, int v, int comp, RowEntry* e, double* diag) {
    int ne = 0;
    for (int64_t q = inc_off[v]; q < inc_off[v + 1]; ++q) {
        int f = inc[q];
        if (face_comp[f] != comp) continue;
        if (ne + 2 > 2 * MAXF) return -1;
        int cv = (F[3 * f] == v) ? 0 : ((F[3 * f + 1] == v) ? 1 : 2);
        int a = F[3 * f + (cv + 1) % 3];
        int b = F[3 * f + (cv + 2) % 3];
        e[ne].col = a;
        e[ne].w = w3[3 * f + (cv + 2) % 3];
        ++ne;
        e[ne].col = b;
        e[ne].w = w3[3 * f + (cv + 1) % 3];
        ++ne;
    }
    // diagonal in the reference COO order: corner-major, then the (j,j) block
    // (v = F[c+1]) before the (k,k) block (v = F[c+2]), faces ascending
    double d = 0.0;
    bool first = true;
    for (int c = 0; c < 3; ++c) {
        for (int blk = 0; blk < 2; ++blk) {
            int want = (c + 1 + blk) % 3;  // position of v in the face
            for (int64_t q = inc_off[v]; q < inc_off[v + 1]; ++q) {
                int f = inc[q];
                if (face_comp[f] != comp) continue;
                if (F[3 * f + want] != v) continue;
                double w = w3[3 * f + c];
                d = first ? w : __dadd_rn(d, w);
                first = false;
            }
        }
    }
    *diag = d;
    // insertion sort by column (stable: keeps face order of equal columns)
    for (int i = 1; i < ne; ++i) {
        RowEntry x = e[i];
        int j = i - 1;
        while (j >= 0 && e[j].col > x.col) {
            e[j + 1] = e[j];
            --j;
        }
        e[j + 1] = x;
    }
    return ne;
}

__global__ void k_row_count(int64_t sum_n, const int32_t* __restrict__ vmap, const int32_t* __restrict__ comp_of,
                            const int32_t* __restrict__ F, const int64_t* __restrict__ inc_off,
                            const int32_t* __restrict__ inc, const int32_t* __restrict__ face_comp,
                            const double* __restrict__ w3, int32_t* __restrict__ cnt, DevErr* err) {
    RowEntry e[2 * MAXF];
    GRID_STRIDE(g, sum_n) {
        double diag;
        int ne = gather_row(F, inc_off, inc, face_comp, w3, vmap[g], comp_of[g], e, &diag);
        if (ne < 0) {
            dev_fail(err, 2, g);
            cnt[g] = 1;
            continue;
        }
        int u = 0;
        for (int i = 0; i < ne; ++i)
            if (i == 0 || e[i].col != e[i - 1].col) ++u;
        cnt[g] = 1 + u;
    }
}

__device__ __forceinline__ int lv_find2(const int64_t* __restrict__ lv_off, const int32_t* __restrict__ lv_comp,
                                        const int32_t* __restrict__ lv_gid, int v, int c) {
    for (int64_t e = lv_off[v]; e < lv_off[v + 1]; ++e)
        if (lv_comp[e] == c) return lv_gid[e];
    return -1;
}

__global__ void k_row_fill(int64_t sum_n, const int32_t* __restrict__ vmap, const int32_t* __restrict__ comp_of,
                           const int32_t* __restrict__ F, const int64_t* __restrict__ inc_off,
                           const int32_t* __restrict__ inc, const int32_t* __restrict__ face_comp,
                           const double* __restrict__ w3, const int64_t* __restrict__ lv_off,
                           const int32_t* __restrict__ lv_comp, const int32_t* __restrict__ lv_gid,
                           const int64_t* __restrict__ vert_off, const int64_t* __restrict__ row_ptr,
                           int32_t* __restrict__ col, double* __restrict__ val) {
    RowEntry e[2 * MAXF];
    GRID_STRIDE(g, sum_n) {
        int v = vmap[g], c = comp_of[g];
        double diag;
        int ne = gather_row(F, inc_off, inc, face_comp, w3, v, c, e, &diag);
        if (ne < 0) continue;
        int64_t base = vert_off[c];
        int64_t o = row_ptr[g];
        int self = (int)(g - base);
        bool diag_done = false;
        int i = 0;
        while (i < ne) {
            int pc = e[i].col;
            double s = -e[i].w;
            int j = i + 1;
            if (j < ne && e[j].col == pc) {
                s = -e[i].w + (-e[j].w);  // scipy: (-w_a) + (-w_b), commutative
                ++j;
            }
            while (j < ne && e[j].col == pc) {  // non-manifold fan: keep summing
                s += -e[j].w;
                ++j;
            }
            int lc = lv_find2(lv_off, lv_comp, lv_gid, pc, c) - (int)base;
            if (!diag_done && lc > self) {
                col[o] = self;
                val[o] = diag;
                ++o;
                diag_done = true;
            }
            col[o] = lc;
            val[o] = s;
            ++o;
            i = j;
        }
        if (!diag_done) {
            col[o] = self;
            val[o] = diag;
        }
    }
}

// default pins (flatten.py:113-122): one warp per loop. The lanes compute 32
// segment lengths at a time; lane 0 adds them in loop order, so the running
// sums (cumsum) and the argmin (first minimum) are the reference's exactly.
__global__ void k_default_pins(int32_t K, const int64_t* __restrict__ loop_off, const int32_t* __restrict__ loop,
                               const int64_t* __restrict__ vert_off, const int32_t* __restrict__ vmap,
                               const double* __restrict__ V, int32_t* __restrict__ pins) {
    const int lane = threadIdx.x & 31;
    const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (c >= K) return;
    const int64_t lo = loop_off[c], nb = loop_off[c + 1] - lo;
    const int64_t vb = vert_off[c];
    if (nb <= 0) {
        if (lane == 0) pins[2 * c] = pins[2 * c + 1] = -1;
        return;
    }
    auto seg = [&](int64_t j) {
        int a = vmap[vb + loop[lo + j]];
        int b = vmap[vb + loop[lo + (j + 1) % nb]];
        double dx = __dsub_rn(V[3 * b], V[3 * a]);
        double dy = __dsub_rn(V[3 * b + 1], V[3 * a + 1]);
        double dz = __dsub_rn(V[3 * b + 2], V[3 * a + 2]);
        return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
    };
    double total = 0.0;
    for (int64_t j0 = 0; j0 < nb; j0 += 32) {
        double sl = j0 + lane < nb ? seg(j0 + lane) : 0.0;
        const int cnt = (int)min((int64_t)32, nb - j0);
        for (int t = 0; t < cnt; ++t) {
            double v = __shfl_sync(0xffffffffu, sl, t);
            total = __dadd_rn(total, v);
        }
    }
    const double half = total / 2.0;
    double cum = 0.0, best = fabs(0.0 - half);
    int64_t bj = 0;
    // cum after segment j-1 is compared at position j (j = 1..nb-1)
    for (int64_t j0 = 0; j0 < nb - 1; j0 += 32) {
        double sl = j0 + lane < nb - 1 ? seg(j0 + lane) : 0.0;
        const int cnt = (int)min((int64_t)32, nb - 1 - j0);
        for (int t = 0; t < cnt; ++t) {
            double v = __shfl_sync(0xffffffffu, sl, t);
            cum = __dadd_rn(cum, v);
            double d = fabs(__dsub_rn(cum, half));
            if (d < best) {
                best = d;
                bj = j0 + t + 1;
            }
        }
    }
    if (lane == 0) {
        if (bj == 0) bj = nb / 2;
        pins[2 * c] = loop[lo];
        pins[2 * c + 1] = loop[lo + bj];
    }
}

// per submesh E_D - A of a complex embedding (flatten.py:89-110); one block
// per submesh, fixed-order reduction
__global__ void __launch_bounds__(1024) k_energy(const int64_t* __restrict__ vert_off, const int64_t* __restrict__ row_ptr,
                         const int32_t* __restrict__ col, const double* __restrict__ val,
                         const int64_t* __restrict__ loop_off, const int32_t* __restrict__ loop,
                         const double2* __restrict__ z, double* __restrict__ energy) {
    __shared__ double red[32];
    int c = blockIdx.x;
    int64_t vb = vert_off[c], ve = vert_off[c + 1];
    double acc = 0.0;
    for (int64_t g = vb + threadIdx.x; g < ve; g += blockDim.x) {
        double sx = 0.0, sy = 0.0;
        for (int64_t q = row_ptr[g]; q < row_ptr[g + 1]; ++q) {
            double2 zz = z[vb + col[q]];
            sx += val[q] * zz.x;
            sy += val[q] * zz.y;
        }
        double2 zi = z[g];
        acc += 0.5 * (zi.x * sx + zi.y * sy);
    }
    int64_t lo = loop_off[c], nb = loop_off[c + 1] - lo;
    for (int64_t j = threadIdx.x; j < nb; j += blockDim.x) {
        double2 w = z[vb + loop[lo + j]];
        double2 u = z[vb + loop[lo + (j + 1) % nb]];
        acc -= 0.5 * (w.x * u.y - w.y * u.x);
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
        t = warp_sum(t);
        if (threadIdx.x == 0) energy[c] = t;
    }
}

}  // namespace

int build_laplacian(pgcp_batch* b, int64_t* clamped, cudaStream_t s) {
    const int BT = 256;
    DevBuf<DevErr> err;
    PGCP_TRY(err.alloc(1, s));
    DevErr init{0, 0, ~0ull, 0};
    PGCP_TRY_CUDA(cudaMemcpyAsync(err.p, &init, sizeof(DevErr), cudaMemcpyHostToDevice, s));
    DevBuf<unsigned long long> ncl;
    PGCP_TRY(ncl.alloc(1, s));
    PGCP_TRY(ncl.zero(s));
    PGCP_TRY(b->w3.alloc(3 * b->m, s));
    k_cot<<<grid_for(b->m, BT), BT, 0, s>>>(b->V.p, b->F.p, b->m, b->w3.p, err.p, ncl.p);
    PGCP_LAUNCH_CHECK();
    DevErr herr;
    unsigned long long hcl = 0;
    PGCP_TRY_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(DevErr), cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(&hcl, ncl.p, sizeof(hcl), cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaStreamSynchronize(s));
    if (herr.code) {
        set_error("zero-area face %llu in cotangent weights", herr.index);
        return PGCP_E_MESH;
    }
    if (clamped) *clamped = (int64_t)hcl;

    const int64_t N = b->sum_n;
    DevBuf<int32_t> cnt;
    PGCP_TRY(cnt.alloc(N, s));
    k_row_count<<<grid_for(N, 128), 128, 0, s>>>(N, b->vmap.p, b->comp_of_gid.p, b->F.p, b->inc_off.p, b->inc.p,
                                                 b->face_comp.p, b->w3.p, cnt.p, err.p);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY(b->row_ptr.alloc(N + 1, s));
    PGCP_TRY(exclusive_scan_i32_to_i64(cnt.p, b->row_ptr.p, N, s));
    PGCP_TRY(fetch_scalar(b->row_ptr.p + N, &b->nnz, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(&herr, err.p, sizeof(DevErr), cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaStreamSynchronize(s));
    if (herr.code) {
        set_error("local vertex %llu has more than %d incident faces", herr.index, MAXF);
        return PGCP_E_MESH;
    }
    PGCP_TRY(b->col.alloc(b->nnz, s));
    PGCP_TRY(b->val.alloc(b->nnz, s));
    k_row_fill<<<grid_for(N, 128), 128, 0, s>>>(N, b->vmap.p, b->comp_of_gid.p, b->F.p, b->inc_off.p, b->inc.p,
                                                b->face_comp.p, b->w3.p, b->lv_off.p, b->lv_comp.p, b->lv_gid.p,
                                                b->vert_off.p, b->row_ptr.p, b->col.p, b->val.p);
    PGCP_LAUNCH_CHECK();
    b->has_laplacian = true;
    return PGCP_OK;
}

int default_pins(pgcp_batch* b, cudaStream_t s) {
    PGCP_TRY(b->pins.alloc(2 * (int64_t)b->K, s));
    k_default_pins<<<(unsigned)((b->K + 3) / 4), 128, 0, s>>>(b->K, b->loop_off.p, b->loop.p, b->vert_off.p, b->vmap.p,
                                                    b->V.p, b->pins.p);
    PGCP_LAUNCH_CHECK();
    return PGCP_OK;
}

int conformal_energy(pgcp_batch* b, const double* z, double* energy, cudaStream_t s) {
    if (!b->has_laplacian) PGCP_TRY(build_laplacian(b, nullptr, s));
    DevBuf<double> e;
    PGCP_TRY(e.alloc(b->K, s));
    k_energy<<<b->K, 1024, 0, s>>>(b->vert_off.p, b->row_ptr.p, b->col.p, b->val.p, b->loop_off.p, b->loop.p,
                                  (const double2*)z, e.p);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY_CUDA(cudaMemcpyAsync(energy, e.p, b->K * sizeof(double), cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaStreamSynchronize(s));
    return PGCP_OK;
}

}  // namespace pgcp
