// repair.cu -- quasi-conformal fold-over repair on the device
// (assemble.py:53-217; called per submesh by pipeline.py:88-102 when the
// harmonic map flipped faces).
//
// Per repair iteration of every still-folded submesh (assemble.py:192-216):
//   mu_inv  Beltrami coefficient of the map embedding -> isometric face
//           layout, per face (beltrami_per_face, assemble.py:74-92);
//   mu      |mu_inv| capped at `cap`, non-finite -> 0 (assemble.py:193-200);
//   K       linear-element stiffness of the divergence-form operator with
//           Beltrami coefficient mu on the current embedding, absolute face
//           areas (lbs_stiffness, assemble.py:124-164) -- it lives on the
//           Laplacian's CSR pattern (same face-adjacency), one thread per
//           row gathers its incident faces in incidence order (deterministic);
//   solve   K_ff u = -K_f,fixed g for both coordinates at once (complex RHS,
//           real symmetric K) with the batched cluster PCG of pcg.cu;
//   flips   signed area <= 0 per face (assemble.py:95-102), counted per
//           submesh; a submesh stops at the first iteration with none.
// All submeshes that still fold are repaired in one batched solve per
// iteration.
#include <cmath>
#include <vector>

#include "batch.cuh"

namespace pgcp {
namespace {

__device__ __forceinline__ double2 C(double x, double y) { return make_double2(x, y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return C(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cconj(double2 a) { return C(a.x, -a.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return C(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
// numpy's complex division (Smith's method with a reciprocal)
__device__ double2 cdiv(double2 a, double2 b) {
    double abr = fabs(b.x), abi = fabs(b.y);
    if (abr >= abi) {
        if (abr == 0.0 && abi == 0.0) return C(a.x / abr, a.y / abi);
        double rat = b.y / b.x;
        double scl = 1.0 / (b.x + b.y * rat);
        return C((a.x + a.y * rat) * scl, (a.y - a.x * rat) * scl);
    }
    double rat = b.x / b.y;
    double scl = 1.0 / (b.y + b.x * rat);
    return C((a.x * rat + a.y) * scl, (a.y * rat - a.x) * scl);
}

// face_layout (assemble.py:53-67) of one face: corner 0 at the origin, corner
// 1 on the positive real axis; norm = sqrt((x^2+y^2)+z^2), dot = (x+z)+y
// (numpy's orders, as in laplace.cu)
__device__ void layout_of(const double* __restrict__ V, const int32_t* __restrict__ F, int64_t f, double2 t[3]) {
    const int a = F[3 * f], b = F[3 * f + 1], c = F[3 * f + 2];
    const double ex = __dsub_rn(V[3 * b], V[3 * a]), ey = __dsub_rn(V[3 * b + 1], V[3 * a + 1]),
                 ez = __dsub_rn(V[3 * b + 2], V[3 * a + 2]);
    const double gx = __dsub_rn(V[3 * c], V[3 * a]), gy = __dsub_rn(V[3 * c + 1], V[3 * a + 1]),
                 gz = __dsub_rn(V[3 * c + 2], V[3 * a + 2]);
    const double x1 = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey)), __dmul_rn(ez, ez)));
    const double dot = __dadd_rn(__dadd_rn(__dmul_rn(gx, ex), __dmul_rn(gz, ez)), __dmul_rn(gy, ey));
    const double cx = __dsub_rn(__dmul_rn(ey, gz), __dmul_rn(ez, gy));
    const double cy = __dsub_rn(__dmul_rn(ez, gx), __dmul_rn(ex, gz));
    const double cz = __dsub_rn(__dmul_rn(ex, gy), __dmul_rn(ey, gx));
    const double cn = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(cx, cx), __dmul_rn(cy, cy)), __dmul_rn(cz, cz)));
    t[0] = C(0.0, 0.0);
    t[1] = C(x1, 0.0);
    t[2] = C(__ddiv_rn(dot, x1), __ddiv_rn(cn, x1));
}

// beltrami_per_face (assemble.py:74-92) of source corners s -> target t.
// Returns false for a degenerate source triangle (det == 0).
__device__ bool beltrami(const double2 s[3], const double2 t[3], double2* mu) {
    const double2 d1 = csub(s[1], s[0]), d2 = csub(s[2], s[0]);
    const double2 e1 = csub(t[1], t[0]), e2 = csub(t[2], t[0]);
    const double2 det = csub(cmul(d1, cconj(d2)), cmul(cconj(d1), d2));
    if (det.x == 0.0 && det.y == 0.0) return false;
    const double2 fz = cdiv(csub(cmul(e1, cconj(d2)), cmul(cconj(d1), e2)), det);
    const double2 fzb = cdiv(csub(cmul(d1, e2), cmul(e1, d2)), det);
    *mu = (fz.x == 0.0 && fz.y == 0.0) ? C(INFINITY, 0.0) : cdiv(fzb, fz);
    return true;
}

// the capped coefficient fed to the linear Beltrami solve (assemble.py:193-200)
__device__ double2 cap_mu(double2 mi, double cap) {
    const double mag = hypot(mi.x, mi.y);
    const bool fin = isfinite(mi.x) && isfinite(mi.y);
    if (!isfinite(mag) || !fin) return C(0.0, 0.0);  // bad & non-finite: cap / inf = 0
    if (mag > cap) {
        const double sc = cap / (mag > 0.0 ? mag : INFINITY);
        return C(mi.x * sc, mi.y * sc);
    }
    return mi;
}

__device__ __forceinline__ int lv_find(const int64_t* __restrict__ lv_off, const int32_t* __restrict__ lv_comp,
                                       const int32_t* __restrict__ lv_gid, int v, int c) {
    for (int64_t e = lv_off[v]; e < lv_off[v + 1]; ++e)
        if (lv_comp[e] == c) return lv_gid[e];
    return -1;
}

struct RepairArgs {
    const double* V;
    const int32_t* F;
    const double2* layout;  // per parent face, 3 corners (nullptr: from V)
    const int64_t* inc_off;
    const int32_t* inc;
    const int32_t* face_comp;
    const int32_t* vmap;
    const int32_t* comp_of;
    const int64_t* lv_off;
    const int32_t* lv_comp;
    const int32_t* lv_gid;
    const int64_t* vert_off;
    const int64_t* row_ptr;
    const int32_t* col;
    const uint8_t* active;  // per submesh
    const double2* z;
    double cap;
    const double2* mu;      // per parent face: given coefficient (lbs_stiffness), or nullptr
};

// lbs_stiffness (assemble.py:124-164): the 3x3 element matrix row of corner i
__device__ bool face_row(const RepairArgs& A, int64_t f, int c, int i, int gids[3], double q[3]) {
    double2 s[3], t[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        gids[k] = lv_find(A.lv_off, A.lv_comp, A.lv_gid, A.F[3 * f + k], c);
        s[k] = A.z[gids[k]];
    }
    double2 mu;
    if (A.mu) {
        mu = A.mu[f];
    } else {
        if (A.layout) {
#pragma unroll
            for (int k = 0; k < 3; ++k) t[k] = A.layout[3 * f + k];
        } else {
            layout_of(A.V, A.F, f, t);
        }
        double2 mi;
        if (!beltrami(s, t, &mi)) return false;
        mu = cap_mu(mi, A.cap);
    }
    const double rho = mu.x, tau = mu.y;
    const double den = fmax(1.0 - rho * rho - tau * tau, 1e-12);
    const double a1 = ((rho - 1.0) * (rho - 1.0) + tau * tau) / den;
    const double a2 = -2.0 * tau / den;
    const double a3 = ((1.0 + rho) * (1.0 + rho) + tau * tau) / den;
    const double2 u = csub(s[1], s[0]), w = csub(s[2], s[0]);
    const double area = 0.5 * (u.x * w.y - u.y * w.x);
    const double absarea = fmax(fabs(area), 1e-300);
    double gx[3], gy[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double2 e = csub(s[(k + 2) % 3], s[(k + 1) % 3]);
        gx[k] = -e.y / (2.0 * area);
        gy[k] = e.x / (2.0 * area);
    }
#pragma unroll
    for (int j = 0; j < 3; ++j)
        q[j] = (a1 * gx[i] * gx[j] + a2 * (gx[i] * gy[j] + gy[i] * gx[j]) + a3 * gy[i] * gy[j]) * absarea;
    return true;
}

// one thread per local vertex of an active submesh: zero its CSR row, then
// add the element rows of its incident faces (incidence order)
__global__ void k_lbs_rows(RepairArgs A, int64_t sum_n, double* __restrict__ kval, DevErr* err) {
    GRID_STRIDE(g, sum_n) {
        const int c = A.comp_of[g];
        if (!A.active[c]) continue;
        const int v = A.vmap[g];
        const int64_t base = A.vert_off[c];
        const int64_t r0 = A.row_ptr[g], r1 = A.row_ptr[g + 1];
        for (int64_t q = r0; q < r1; ++q) kval[q] = 0.0;
        for (int64_t e = A.inc_off[v]; e < A.inc_off[v + 1]; ++e) {
            const int f = A.inc[e];
            if (A.face_comp[f] != c) continue;
            const int i = A.F[3 * f] == v ? 0 : (A.F[3 * f + 1] == v ? 1 : 2);
            int gids[3];
            double qv[3];
            if (!face_row(A, f, c, i, gids, qv)) {
                dev_fail(err, 1, f);
                continue;
            }
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const int lc = (int)(gids[j] - base);
                for (int64_t q = r0; q < r1; ++q)
                    if (A.col[q] == lc) {
                        kval[q] += qv[j];
                        break;
                    }
            }
        }
    }
}

// signed_areas(z, faces) <= 0 per face of an active submesh (assemble.py:95-102)
__global__ void k_flip_count(RepairArgs A, int64_t m, int32_t* __restrict__ cnt, uint8_t* __restrict__ flipped) {
    GRID_STRIDE(f, m) {
        const int c = A.face_comp[f];
        bool fl = false;
        if (A.active[c]) {
            double2 s[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) s[k] = A.z[lv_find(A.lv_off, A.lv_comp, A.lv_gid, A.F[3 * f + k], c)];
            const double2 u = csub(s[1], s[0]), w = csub(s[2], s[0]);
            fl = 0.5 * (u.x * w.y - u.y * w.x) <= 0.0;
            if (fl) atomicAdd(&cnt[c], 1);
        }
        if (flipped) flipped[f] = fl;
    }
}

__global__ void k_gather(const double2* __restrict__ z, const int32_t* __restrict__ gid, int64_t n,
                         double2* __restrict__ out) {
    GRID_STRIDE(i, n) out[i] = z[gid[i]];
}

__global__ void k_face_layout(const double* __restrict__ V, const int32_t* __restrict__ F, int64_t m,
                              double2* __restrict__ out) {
    GRID_STRIDE(f, m) {
        double2 t[3];
        layout_of(V, F, f, t);
        out[3 * f] = t[0];
        out[3 * f + 1] = t[1];
        out[3 * f + 2] = t[2];
    }
}

__global__ void k_beltrami(const double2* __restrict__ src, const int32_t* __restrict__ sf,
                           const double2* __restrict__ tgt, const int32_t* __restrict__ tf, int64_t m,
                           double2* __restrict__ mu, DevErr* err) {
    GRID_STRIDE(f, m) {
        double2 s[3], t[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            s[k] = sf ? src[sf[3 * f + k]] : src[3 * f + k];
            t[k] = tf ? tgt[tf[3 * f + k]] : tgt[3 * f + k];
        }
        double2 r;
        if (!beltrami(s, t, &r)) {
            dev_fail(err, 1, f);
            r = C(NAN, NAN);
        }
        mu[f] = r;
    }
}

int fetch_err(DevBuf<DevErr>& e, DevErr* h, cudaStream_t s) {
    PGCP_TRY_CUDA(cudaMemcpyAsync(h, e.p, sizeof(DevErr), cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaStreamSynchronize(s));
    return PGCP_OK;
}

int init_err(DevBuf<DevErr>& e, cudaStream_t s) {
    PGCP_TRY(e.alloc(1, s));
    DevErr h;
    h.code = 0;
    h.pad = 0;
    h.index = ~0ull;
    h.aux = 0;
    PGCP_TRY_CUDA(cudaMemcpyAsync(e.p, &h, sizeof(DevErr), cudaMemcpyHostToDevice, s));
    return PGCP_OK;
}

}  // namespace

int face_layout(const double* V, const int32_t* F, int64_t m, double* out, cudaStream_t s) {
    if (m <= 0) return PGCP_OK;
    k_face_layout<<<grid_for(m, 256), 256, 0, s>>>(V, F, m, reinterpret_cast<double2*>(out));
    PGCP_LAUNCH_CHECK();
    return PGCP_OK;
}

int beltrami_per_face(const double* src, const int32_t* sf, const double* tgt, const int32_t* tf, int64_t m,
                      double* mu, int64_t* first_degenerate, cudaStream_t s) {
    if (first_degenerate) *first_degenerate = -1;
    if (m <= 0) return PGCP_OK;
    DevBuf<DevErr> err;
    PGCP_TRY(init_err(err, s));
    k_beltrami<<<grid_for(m, 256), 256, 0, s>>>(reinterpret_cast<const double2*>(src), sf,
                                                reinterpret_cast<const double2*>(tgt), tf, m,
                                                reinterpret_cast<double2*>(mu), err.p);
    PGCP_LAUNCH_CHECK();
    DevErr h;
    PGCP_TRY(fetch_err(err, &h, s));
    if (h.code) {
        if (first_degenerate) *first_degenerate = (int64_t)h.index;
        set_error("degenerate source triangle %lld in Beltrami computation", (long long)h.index);
        return PGCP_E_SOLVE;
    }
    return PGCP_OK;
}

int qc_repair(pgcp_batch* b, const int32_t* comps, int32_t ncomp, const double* layout, const int32_t* fixed_gid,
              int64_t nfixed, int32_t max_iter, double cap, const pgcp_solve_opts* o, double* z, int32_t* info,
              uint8_t* flipped, cudaStream_t s) {
    if (!b->has_laplacian) PGCP_TRY(build_laplacian(b, nullptr, s));
    std::vector<int32_t> list;
    if (comps) {
        list.assign(comps, comps + ncomp);
    } else {
        for (int c = 0; c < b->K; ++c) list.push_back(c);
    }
    for (int c : list)
        if (c < 0 || c >= b->K) {
            set_error("submesh id %d out of range", c);
            return PGCP_E_INVALID;
        }
    const int n = (int)list.size();
    std::vector<uint8_t> act(b->K, 0);
    for (int c : list) act[c] = 1;
    DevBuf<uint8_t> d_act;
    DevBuf<int32_t> cnt;
    PGCP_TRY(d_act.alloc(b->K, s));
    PGCP_TRY(cnt.alloc(b->K, s));
    RepairArgs A;
    A.V = b->V.p;
    A.F = b->F.p;
    A.layout = reinterpret_cast<const double2*>(layout);
    A.inc_off = b->inc_off.p;
    A.inc = b->inc.p;
    A.face_comp = b->face_comp.p;
    A.vmap = b->vmap.p;
    A.comp_of = b->comp_of_gid.p;
    A.lv_off = b->lv_off.p;
    A.lv_comp = b->lv_comp.p;
    A.lv_gid = b->lv_gid.p;
    A.vert_off = b->vert_off.p;
    A.row_ptr = b->row_ptr.p;
    A.col = b->col.p;
    A.active = d_act.p;
    A.z = reinterpret_cast<const double2*>(z);
    A.cap = cap;
    A.mu = nullptr;
    std::vector<int32_t> hc(b->K);
    // flips of the active submeshes (and, on the last count, the face flags)
    auto count = [&](bool last) -> int {
        PGCP_TRY_CUDA(cudaMemcpyAsync(d_act.p, act.data(), act.size(), cudaMemcpyHostToDevice, s));
        PGCP_TRY(cnt.zero(s));
        k_flip_count<<<grid_for(b->m, 256), 256, 0, s>>>(A, b->m, cnt.p, last ? flipped : nullptr);
        PGCP_LAUNCH_CHECK();
        PGCP_TRY_CUDA(cudaMemcpyAsync(hc.data(), cnt.p, hc.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        PGCP_TRY_CUDA(cudaStreamSynchronize(s));
        return PGCP_OK;
    };
    PGCP_TRY(count(false));
    std::vector<int32_t> before(b->K, 0), iters(b->K, 0), after(b->K, 0);
    for (int c : list) {
        before[c] = after[c] = hc[c];
        act[c] = hc[c] > 0;
    }
    // the held values are the embedding's own (assemble.py:182)
    DevBuf<double2> fv;
    PGCP_TRY(fv.alloc(std::max<int64_t>(nfixed, 1), s));
    if (nfixed > 0) {
        k_gather<<<grid_for(nfixed, 256), 256, 0, s>>>(A.z, fixed_gid, nfixed, fv.p);
        PGCP_LAUNCH_CHECK();
    }
    DevBuf<double> kval;
    PGCP_TRY(kval.alloc(b->nnz, s));
    DevBuf<DevErr> err;
    for (int it = 1; it <= max_iter; ++it) {
        std::vector<int32_t> cur;
        for (int c : list)
            if (act[c]) cur.push_back(c);
        if (cur.empty()) break;
        PGCP_TRY_CUDA(cudaMemcpyAsync(d_act.p, act.data(), act.size(), cudaMemcpyHostToDevice, s));
        PGCP_TRY(init_err(err, s));
        k_lbs_rows<<<grid_for(b->sum_n, 128), 128, 0, s>>>(A, b->sum_n, kval.p, err.p);
        PGCP_LAUNCH_CHECK();
        DevErr he;
        PGCP_TRY(fetch_err(err, &he, s));
        if (he.code) {
            set_error("degenerate source triangle %lld (parent face) in Beltrami computation", (long long)he.index);
            return PGCP_E_SOLVE;
        }
        std::vector<pgcp_solve_stat> st(cur.size());
        int rc = solve_values(b, cur.data(), (int32_t)cur.size(), kval.p, fixed_gid,
                              reinterpret_cast<const double*>(fv.p), nfixed, o, z, st.data(), s);
        if (rc != PGCP_OK) {
            for (size_t q = 0; q < cur.size(); ++q)
                if (st[q].status != PGCP_OK) {
                    set_error("singular linear Beltrami system during repair (submesh %d: status %d, "
                              "relres %.3e, residual %.3e)", cur[q], st[q].status, st[q].relres, st[q].true_res);
                    break;
                }
            return PGCP_E_SOLVE;
        }
        PGCP_TRY(count(false));
        for (int c : cur) {
            iters[c] = it;
            after[c] = hc[c];
            act[c] = hc[c] > 0;
        }
    }
    if (flipped) {  // faces of the listed submeshes still folded
        for (int c = 0; c < b->K; ++c) act[c] = 0;
        for (int c : list) act[c] = 1;
        PGCP_TRY(count(true));
    }
    for (int q = 0; q < n; ++q) {
        const int c = list[q];
        info[4 * q + 0] = before[c];
        info[4 * q + 1] = iters[c];
        info[4 * q + 2] = after[c] == 0;
        info[4 * q + 3] = after[c];
    }
    return PGCP_OK;
}

// lbs_stiffness (assemble.py:124-164) of every submesh for a given per-face
// coefficient, on the Laplacian's CSR pattern
int lbs_stiffness(pgcp_batch* b, const double* z, const double* mu, double* kval, cudaStream_t s) {
    if (!b->has_laplacian) PGCP_TRY(build_laplacian(b, nullptr, s));
    DevBuf<uint8_t> d_act;
    PGCP_TRY(d_act.alloc(b->K, s));
    PGCP_TRY(d_act.fill_bytes(1, s));
    RepairArgs A;
    A.V = b->V.p;
    A.F = b->F.p;
    A.layout = nullptr;
    A.inc_off = b->inc_off.p;
    A.inc = b->inc.p;
    A.face_comp = b->face_comp.p;
    A.vmap = b->vmap.p;
    A.comp_of = b->comp_of_gid.p;
    A.lv_off = b->lv_off.p;
    A.lv_comp = b->lv_comp.p;
    A.lv_gid = b->lv_gid.p;
    A.vert_off = b->vert_off.p;
    A.row_ptr = b->row_ptr.p;
    A.col = b->col.p;
    A.active = d_act.p;
    A.z = reinterpret_cast<const double2*>(z);
    A.cap = 1.0;
    A.mu = reinterpret_cast<const double2*>(mu);
    DevBuf<DevErr> err;
    PGCP_TRY(init_err(err, s));
    k_lbs_rows<<<grid_for(b->sum_n, 128), 128, 0, s>>>(A, b->sum_n, kval, err.p);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY_CUDA(cudaStreamSynchronize(s));
    return PGCP_OK;
}

}  // namespace pgcp
