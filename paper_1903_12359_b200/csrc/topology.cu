// topology.cu -- device partition of a triangle mesh into disk-type submeshes.
//
// Replaces (reference, pure Python):
//   mesh.py:91-111  TriMesh._validate (index range, repeated vertices,
//                   repeated directed edge)
//   mesh.py:146-203 boundary_directed_edges + boundary_loops
//   mesh.py:206-223 validate_topology (chi, loop count)
//   partition.py:48-59  validate_cuts
//   partition.py:94-137 partition_mesh (face adjacency minus cut edges ->
//                   connected components labelled in order of their minimum
//                   face -> sorted vertex maps -> disk check -> boundary cycle)
//
// Everything is integer work over the face/half-edge arrays (HBM bound);
// all outputs are deterministic (atomics only build sets whose order is fixed
// afterwards by sorting or by the stable counting sort).
#include <climits>

#include "batch.cuh"

namespace pgcp {
namespace {

enum : int {
    ERR_FACE_RANGE = 1,
    ERR_FACE_REPEAT = 2,
    ERR_DIRECTED_DUP = 3,
    ERR_VALENCE = 4,
};

// range errors outrank repeated-vertex errors (the reference checks the
// whole index range first): repeats are recorded at index m + f
__global__ void k_validate_faces(const int32_t* __restrict__ F, int64_t m, int64_t n, DevErr* err) {
    GRID_STRIDE(f, m) {
        int a = F[3 * f], b = F[3 * f + 1], c = F[3 * f + 2];
        if (a < 0 || b < 0 || c < 0 || a >= n || b >= n || c >= n) {
            dev_fail(err, ERR_FACE_RANGE, f);
        } else if (a == b || b == c || c == a) {
            dev_fail(err, ERR_FACE_REPEAT, m + f);
        }
    }
}

// int64 face indices -> int32; values outside [0, 2^31) become -1 (reported
// as out of range by the validation)
__global__ void k_faces_i64(const int64_t* __restrict__ src, int32_t* __restrict__ dst, int64_t count) {
    GRID_STRIDE(i, count) {
        int64_t v = src[i];
        dst[i] = (v >= 0 && v < 2147483647ll) ? (int32_t)v : -1;
    }
}

// bounding box (mesh.py:134-138) and degenerate faces (mesh.py:99-104):
// area < 1e-12 * diag^2
__device__ __forceinline__ void atomic_min_d(double* p, double v) {
    unsigned long long* a = reinterpret_cast<unsigned long long*>(p);
    unsigned long long old = *a, assumed;
    do {
        assumed = old;
        if (__longlong_as_double(assumed) <= v) return;
        old = atomicCAS(a, assumed, __double_as_longlong(v));
    } while (old != assumed);
}
__device__ __forceinline__ void atomic_max_d(double* p, double v) {
    unsigned long long* a = reinterpret_cast<unsigned long long*>(p);
    unsigned long long old = *a, assumed;
    do {
        assumed = old;
        if (__longlong_as_double(assumed) >= v) return;
        old = atomicCAS(a, assumed, __double_as_longlong(v));
    } while (old != assumed);
}

__global__ void k_bbox(const double* __restrict__ V, int64_t n, double* bb) {
    __shared__ double red[6][32];
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    GRID_STRIDE(v, n) {
        for (int d = 0; d < 3; ++d) {
            double x = V[3 * v + d];
            lo[d] = fmin(lo[d], x);
            hi[d] = fmax(hi[d], x);
        }
    }
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int d = 0; d < 3; ++d) {
        double a = lo[d], b = hi[d];
        for (int o = 16; o > 0; o >>= 1) {
            a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
            b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
        }
        if (lane == 0) {
            red[d][w] = a;
            red[3 + d][w] = b;
        }
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        int d = threadIdx.x;
        double a = INFINITY, b = -INFINITY;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
            a = fmin(a, red[d][i]);
            b = fmax(b, red[3 + d][i]);
        }
        atomic_min_d(&bb[d], a);
        atomic_max_d(&bb[3 + d], b);
    }
}

__global__ void k_degenerate(const double* __restrict__ V, const int32_t* __restrict__ F, int64_t m,
                             const double* __restrict__ bb, DevErr* err) {
    const double dx = bb[3] - bb[0], dy = bb[4] - bb[1], dz = bb[5] - bb[2];
    const double diag = sqrt((dx * dx + dy * dy) + dz * dz);
    const double lim = 1e-12 * diag * diag;
    GRID_STRIDE(f, m) {
        const double* a = V + 3 * F[3 * f];
        const double* b = V + 3 * F[3 * f + 1];
        const double* c = V + 3 * F[3 * f + 2];
        double ux = b[0] - a[0], uy = b[1] - a[1], uz = b[2] - a[2];
        double vx = c[0] - a[0], vy = c[1] - a[1], vz = c[2] - a[2];
        double cx = uy * vz - uz * vy, cy = uz * vx - ux * vz, cz = ux * vy - uy * vx;
        double area = 0.5 * sqrt((cx * cx + cy * cy) + cz * cz);
        if (area < lim) dev_fail(err, 5, f);
    }
}

__global__ void k_count_inc(const int32_t* __restrict__ F, int64_t nc, int32_t* __restrict__ cnt) {
    GRID_STRIDE(i, nc) { atomicAdd(&cnt[F[i]], 1); }
}

__global__ void k_fill_inc(const int32_t* __restrict__ F, int64_t m, const int64_t* __restrict__ off,
                           int32_t* __restrict__ cursor, int32_t* __restrict__ inc) {
    GRID_STRIDE(i, 3 * m) {
        int v = F[i];
        int pos = atomicAdd(&cursor[v], 1);
        inc[off[v] + pos] = (int32_t)(i / 3);
    }
}

// incident faces of every vertex in increasing face order (deterministic)
__global__ void k_sort_inc(const int64_t* __restrict__ off, int32_t* __restrict__ inc, int64_t n) {
    GRID_STRIDE(v, n) {
        int64_t lo = off[v], hi = off[v + 1];
        for (int64_t i = lo + 1; i < hi; ++i) {
            int32_t x = inc[i];
            int64_t j = i - 1;
            while (j >= lo && inc[j] > x) {
                inc[j + 1] = inc[j];
                --j;
            }
            inc[j + 1] = x;
        }
    }
}

// half-edge h = 3f+c runs F[f][c] -> F[f][(c+1)%3]
__device__ __forceinline__ int he_find(const int32_t* __restrict__ F, const int64_t* __restrict__ off,
                                       const int32_t* __restrict__ inc, int around, int from, int to,
                                       int skip_face) {
    for (int64_t e = off[around]; e < off[around + 1]; ++e) {
        int g = inc[e];
        if (g == skip_face) continue;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (F[3 * g + c] == from && F[3 * g + (c + 1) % 3] == to) return 3 * g + c;
        }
    }
    return -1;
}

__global__ void k_twin(const int32_t* __restrict__ F, int64_t m, const int64_t* __restrict__ off,
                       const int32_t* __restrict__ inc, int32_t* __restrict__ twin, DevErr* err) {
    GRID_STRIDE(h, 3 * m) {
        int f = (int)(h / 3), c = (int)(h % 3);
        int a = F[3 * f + c], b = F[3 * f + (c + 1) % 3];
        // the same directed edge in another face: non-manifold / inconsistent
        if (he_find(F, off, inc, a, a, b, f) >= 0) dev_fail(err, ERR_DIRECTED_DUP, f);
        twin[h] = he_find(F, off, inc, b, b, a, f);
    }
}

__global__ void k_mark_cuts(const int32_t* __restrict__ F, const int64_t* __restrict__ cuts, int64_t ncuts,
                            int64_t n, const int64_t* __restrict__ off, const int32_t* __restrict__ inc,
                            const int32_t* __restrict__ twin, int32_t* __restrict__ mark,
                            uint8_t* __restrict__ he_cut, int* dup_flag, DevErr* nonedge) {
    GRID_STRIDE(i, ncuts) {
        int64_t u = cuts[2 * i], v = cuts[2 * i + 1];
        if (u < 0 || v < 0 || u >= n || v >= n || u == v) {
            dev_fail(nonedge, 1, i);
            continue;
        }
        int h = he_find(F, off, inc, (int)u, (int)u, (int)v, -1);
        if (h < 0) h = he_find(F, off, inc, (int)u, (int)v, (int)u, -1);
        if (h < 0) {
            dev_fail(nonedge, 1, i);
            continue;
        }
        int t = twin[h];
        int canon = (t >= 0 && t < h) ? t : h;
        if (atomicAdd(&mark[canon], 1) > 0) atomicExch(dup_flag, 1);
        he_cut[h] = 1;
        if (t >= 0) he_cut[t] = 1;
    }
}

// ----- union-find over faces (hook the larger root under the smaller: the
// final root of every component is its minimum face index)
__device__ __forceinline__ int uf_find(int* parent, int x) {
    while (true) {
        int p = __ldcg(&parent[x]);
        if (p == x) return x;
        int gp = __ldcg(&parent[p]);
        if (gp != p) parent[x] = gp;  // path halving; only ever points up
        x = p;
    }
}

__global__ void k_uf_init(int* parent, int64_t m) {
    GRID_STRIDE(f, m) parent[f] = (int)f;
}

__global__ void k_uf_union(const int32_t* __restrict__ twin, const uint8_t* __restrict__ he_cut,
                           int64_t m, int* parent) {
    GRID_STRIDE(h, 3 * m) {
        int t = twin[h];
        if (t < 0 || (he_cut && he_cut[h])) continue;
        int f = (int)(h / 3), g = t / 3;
        if (g <= f) continue;
        int a = f, b = g;
        while (true) {
            a = uf_find(parent, a);
            b = uf_find(parent, b);
            if (a == b) break;
            if (a < b) {
                int tmp = a;
                a = b;
                b = tmp;
            }
            if (atomicCAS(&parent[a], a, b) == a) break;
        }
    }
}

__global__ void k_uf_roots(int* parent, int64_t m, int32_t* __restrict__ is_root) {
    GRID_STRIDE(f, m) {
        int r = uf_find(parent, (int)f);
        is_root[f] = (r == (int)f) ? 1 : 0;
    }
}

__global__ void k_face_comp(int* parent, int64_t m, const int64_t* __restrict__ rank,
                            int32_t* __restrict__ face_comp) {
    GRID_STRIDE(f, m) {
        int r = uf_find(parent, (int)f);
        face_comp[f] = (int32_t)rank[r];
    }
}

// ----- local vertices: (parent vertex, submesh) pairs
constexpr int MAX_VCOMP = 64;

__device__ int distinct_comps(const int64_t* __restrict__ off, const int32_t* __restrict__ inc,
                              const int32_t* __restrict__ face_comp, int64_t v, int* buf) {
    int k = 0;
    for (int64_t e = off[v]; e < off[v + 1]; ++e) {
        int c = face_comp[inc[e]];
        bool seen = false;
        for (int j = 0; j < k; ++j) seen |= (buf[j] == c);
        if (!seen) {
            if (k == MAX_VCOMP) return -1;
            // insertion into the sorted prefix
            int j = k - 1;
            while (j >= 0 && buf[j] > c) {
                buf[j + 1] = buf[j];
                --j;
            }
            buf[j + 1] = c;
            ++k;
        }
    }
    return k;
}

__global__ void k_lv_count(const int64_t* __restrict__ off, const int32_t* __restrict__ inc,
                           const int32_t* __restrict__ face_comp, int64_t n, int32_t* __restrict__ cnt,
                           DevErr* err) {
    int buf[MAX_VCOMP];
    GRID_STRIDE(v, n) {
        int k = distinct_comps(off, inc, face_comp, v, buf);
        if (k < 0) {
            dev_fail(err, ERR_VALENCE, v);
            k = 0;
        }
        cnt[v] = k;
    }
}

__global__ void k_lv_fill(const int64_t* __restrict__ off, const int32_t* __restrict__ inc,
                          const int32_t* __restrict__ face_comp, int64_t n, const int64_t* __restrict__ lv_off,
                          int32_t* __restrict__ lv_comp, int32_t* __restrict__ lv_vert) {
    int buf[MAX_VCOMP];
    GRID_STRIDE(v, n) {
        int k = distinct_comps(off, inc, face_comp, v, buf);
        int64_t o = lv_off[v];
        for (int j = 0; j < k; ++j) {
            lv_comp[o + j] = buf[j];
            lv_vert[o + j] = (int32_t)v;
        }
    }
}

__global__ void k_lv_gid(const int32_t* __restrict__ perm, int64_t ne, const int32_t* __restrict__ lv_vert,
                         const int32_t* __restrict__ lv_comp, int32_t* __restrict__ lv_gid,
                         int32_t* __restrict__ vmap, int32_t* __restrict__ comp_of_gid) {
    GRID_STRIDE(p, ne) {
        int e = perm[p];
        lv_gid[e] = (int32_t)p;
        vmap[p] = lv_vert[e];
        comp_of_gid[p] = lv_comp[e];
    }
}

__device__ __forceinline__ int lv_find(const int64_t* __restrict__ lv_off, const int32_t* __restrict__ lv_comp,
                                       const int32_t* __restrict__ lv_gid, int v, int c) {
    for (int64_t e = lv_off[v]; e < lv_off[v + 1]; ++e)
        if (lv_comp[e] == c) return lv_gid[e];
    return -1;
}

// faces per component; consecutive faces mostly share a component, so the
// increments are aggregated per warp (one atomic per distinct component)
__global__ void k_face_count(const int32_t* __restrict__ face_comp, int64_t m, int32_t* __restrict__ fcnt) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t m_round = (m + 31) & ~(int64_t)31;
    for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < m_round; f += stride) {
        const bool ok = f < m;
        const int c = ok ? face_comp[f] : -1;
        const unsigned act = __ballot_sync(0xffffffffu, ok);
        if (ok) {
            const unsigned peers = __match_any_sync(act, c);
            if (lane == __ffs(peers) - 1) atomicAdd(&fcnt[c], __popc(peers));
        }
    }
}

// boundary half-edges of every submesh (twin absent or in another submesh)
// and of the parent mesh (twin absent)
__global__ void k_boundary(const int32_t* __restrict__ F, int64_t m, const int32_t* __restrict__ twin,
                           const int32_t* __restrict__ face_comp, const int64_t* __restrict__ lv_off,
                           const int32_t* __restrict__ lv_comp, const int32_t* __restrict__ lv_gid,
                           int32_t* __restrict__ nxt, int32_t* __restrict__ bcnt, int32_t* __restrict__ start,
                           int32_t* __restrict__ comp_bad, int32_t* __restrict__ pnxt, int32_t* pcount,
                           int32_t* pstart, int32_t* pbad, int32_t* __restrict__ node, int32_t* __restrict__ idx,
                           int32_t* nnode, int32_t* __restrict__ pnode, int32_t* __restrict__ pidx, int64_t n) {
    GRID_STRIDE(h, 3 * m) {
        int f = (int)(h / 3), c = (int)(h % 3);
        int a = F[3 * f + c], b = F[3 * f + (c + 1) % 3];
        int t = twin[h];
        int cf = face_comp[f];
        if (t < 0) {
            int k = atomicAdd(pcount, 1);
            if (atomicCAS(&pnxt[a], -1, b) != -1) atomicExch(pbad, 1);
            atomicMin(pstart, a);
            if (k < n) {
                pnode[k] = a;
                pidx[a] = k;
            }
        }
        if (t < 0 || face_comp[t / 3] != cf) {
            int ga = lv_find(lv_off, lv_comp, lv_gid, a, cf);
            int gb = lv_find(lv_off, lv_comp, lv_gid, b, cf);
            atomicAdd(&bcnt[cf], 1);
            if (atomicCAS(&nxt[ga], -1, gb) != -1) atomicExch(&comp_bad[cf], 1);
            atomicMin(&start[cf], ga);
            int k = atomicAdd(nnode, 1);
            node[k] = ga;
            idx[ga] = k;
        }
    }
}

// ---- parallel boundary walks (pointer jumping instead of sequential walks)
// Component loops: the cycle of every submesh is cut before its smallest
// vertex `start`; list ranking gives every node its distance to the cut, so
// its loop position is (L - 1) - dist. Nodes that never reach the cut lie on
// another loop (the component is then re-walked sequentially by k_walk for
// the reference's diagnostics).
__global__ void k_lr_init(int64_t nn, const int32_t* __restrict__ node, const int32_t* __restrict__ idx,
                          const int32_t* __restrict__ nxt, const int32_t* __restrict__ comp_of_gid,
                          const int32_t* __restrict__ start, int32_t* __restrict__ succ, int32_t* __restrict__ dist,
                          int32_t* __restrict__ comp_flag) {
    GRID_STRIDE(k, nn) {
        int g = node[k];
        int c = comp_of_gid[g];
        int nx = nxt[g];
        int sc = -1;
        if (nx < 0) {
            comp_flag[c] = 1;
        } else if (nx != start[c]) {
            sc = idx[nx];
            if (sc < 0) comp_flag[c] = 1;  // nx has no outgoing boundary edge
        }
        succ[k] = sc;
        dist[k] = sc < 0 ? 0 : 1;
    }
}

__global__ void k_lr_step(int64_t nn, const int32_t* __restrict__ succ_in, const int32_t* __restrict__ dist_in,
                          int32_t* __restrict__ succ_out, int32_t* __restrict__ dist_out) {
    GRID_STRIDE(k, nn) {
        int sc = succ_in[k];
        if (sc >= 0) {
            dist_out[k] = dist_in[k] + dist_in[sc];
            succ_out[k] = succ_in[sc];
        } else {
            dist_out[k] = dist_in[k];
            succ_out[k] = -1;
        }
    }
}

__global__ void k_lr_finish(int64_t nn, const int32_t* __restrict__ node, const int32_t* __restrict__ idx,
                            const int32_t* __restrict__ comp_of_gid, const int32_t* __restrict__ start,
                            const int32_t* __restrict__ succ, const int32_t* __restrict__ dist,
                            const int32_t* __restrict__ bcnt, const int64_t* __restrict__ vert_off,
                            const int64_t* __restrict__ loop_off, const int32_t* __restrict__ comp_bad,
                            int32_t* __restrict__ comp_flag, int32_t* __restrict__ loop) {
    GRID_STRIDE(k, nn) {
        int g = node[k];
        int c = comp_of_gid[g];
        if (comp_bad[c] || comp_flag[c]) continue;
        if (succ[k] >= 0) {  // not on the start's loop
            comp_flag[c] = 1;
            continue;
        }
        int L = dist[idx[start[c]]] + 1;
        if (L != bcnt[c]) {
            comp_flag[c] = 1;
            continue;
        }
        int pos = L - 1 - dist[k];
        loop[loop_off[c] + pos] = (int32_t)(g - vert_off[c]);
    }
}

// parent boundary: every node learns the minimum vertex of its cycle (min
// label pointer jumping on the closed cycles); one loop iff the cycle of the
// smallest boundary vertex holds every boundary edge
__global__ void k_plab_init(int64_t nn, const int32_t* __restrict__ pnode, const int32_t* __restrict__ pidx,
                            const int32_t* __restrict__ pnxt, int32_t* __restrict__ jump, int32_t* __restrict__ lab,
                            int32_t* pbad) {
    GRID_STRIDE(k, nn) {
        int v = pnode[k];
        int nx = pnxt[v];
        int jn = nx < 0 ? -1 : pidx[nx];
        if (jn < 0) {
            atomicExch(pbad, 1);
            jump[k] = (int32_t)k;
        } else {
            jump[k] = jn;
        }
        lab[k] = v;
    }
}

__global__ void k_plab_step(int64_t nn, const int32_t* __restrict__ jump_in, const int32_t* __restrict__ lab_in,
                            int32_t* __restrict__ jump_out, int32_t* __restrict__ lab_out) {
    GRID_STRIDE(k, nn) {
        int jn = jump_in[k];
        lab_out[k] = min(lab_in[k], lab_in[jn]);
        jump_out[k] = jump_in[jn];
    }
}

__global__ void k_plab_finish(int64_t nn, const int32_t* __restrict__ lab, const int32_t* pstart,
                              const int32_t* pcount, const int32_t* pbad, int32_t* on_start,
                              int64_t* __restrict__ out_loops) {
    GRID_STRIDE(k, nn) if (lab[k] == *pstart) atomicAdd(on_start, 1);
}

__global__ void k_plab_result(const int32_t* pcount, const int32_t* pbad, const int32_t* on_start, int64_t n,
                              int64_t* out_loops) {
    if (blockIdx.x || threadIdx.x) return;
    int pb = *pcount;
    if (*pbad || pb > n) *out_loops = -1;
    else if (pb == 0) *out_loops = 0;
    else *out_loops = (*on_start == pb) ? 1 : -2;
}

// one thread per submesh: chi, loop walk from the smallest boundary vertex
__global__ void k_walk(int32_t K, const int64_t* __restrict__ vert_off, const int32_t* __restrict__ fcnt,
                       const int32_t* __restrict__ bcnt, const int32_t* __restrict__ start,
                       const int32_t* __restrict__ nxt, const int64_t* __restrict__ loop_off,
                       int32_t* __restrict__ loop, int32_t* __restrict__ comp_bad, int32_t* __restrict__ chi_out,
                       int32_t* __restrict__ loops_out, uint8_t* __restrict__ seen,
                       const int32_t* __restrict__ comp_flag) {
    GRID_STRIDE(c, K) {
        int64_t nc = vert_off[c + 1] - vert_off[c];
        int64_t mc = fcnt[c], bc = bcnt[c];
        int64_t twoE = 3 * mc + bc;
        int64_t chi = nc - twoE / 2 + mc;
        chi_out[c] = (int32_t)chi;
        int loops = 0;
        bool bad = comp_bad[c] != 0 || (twoE & 1);
        if (!bad && !comp_flag[c]) {
            // single loop already placed by the list ranking (k_lr_finish)
            loops = bc > 0 ? 1 : 0;
            loops_out[c] = loops;
            if (!(chi == 1 && loops == 1)) comp_bad[c] = 1;
            continue;
        }
        for (int64_t q = loop_off[c]; q < loop_off[c] + bc && q < loop_off[c + 1]; ++q) loop[q] = 0;
        if (!bad && bc > 0) {
            int s = start[c];
            int cur = s;
            int64_t j = 0;
            int64_t base = loop_off[c];
            do {
                if (j >= bc) {
                    bad = true;
                    break;
                }
                loop[base + j] = (int32_t)(cur - vert_off[c]);
                seen[cur] = 1;
                ++j;
                cur = nxt[cur];
                if (cur < 0) {
                    bad = true;
                    break;
                }
            } while (cur != s);
            loops = bad ? -1 : 1;
            if (!bad && j != bc) {
                // more loops (validate_topology counts them, mesh.py:190-202):
                // walk every remaining loop from its smallest vertex
                for (int64_t g = vert_off[c]; g < vert_off[c + 1] && !bad; ++g) {
                    if (nxt[g] < 0 || seen[g]) continue;
                    int64_t cur2 = g, guard = 0;
                    do {
                        seen[cur2] = 1;
                        cur2 = nxt[cur2];
                        if (cur2 < 0 || ++guard > bc) {
                            bad = true;
                            break;
                        }
                    } while (cur2 != g);
                    ++loops;
                }
                if (bad) loops = -1;
            }
        } else if (bad) {
            loops = -1;
        }
        loops_out[c] = loops;
        if (bad || !(chi == 1 && loops == 1)) comp_bad[c] = 1;
    }
}

// boundary cycles in parent ids (partition.py:134-135 `used[loop]`)
__global__ void k_cycles(int32_t K, const int64_t* __restrict__ loop_off, const int32_t* __restrict__ loop,
                         const int64_t* __restrict__ vert_off, const int32_t* __restrict__ vmap,
                         int32_t* __restrict__ cyc, int64_t total) {
    GRID_STRIDE(i, total) {
        int lo = 0, hi = K - 1;  // component of loop entry i
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (loop_off[mid] <= i) lo = mid; else hi = mid - 1;
        }
        cyc[i] = vmap[vert_off[lo] + loop[i]];
    }
}


__global__ void k_fill_i32(int32_t* p, int64_t n, int32_t v) {
    GRID_STRIDE(i, n) p[i] = v;
}

__global__ void k_local_faces(const int32_t* __restrict__ F, const int32_t* __restrict__ perm, int64_t m,
                              const int32_t* __restrict__ face_comp, const int64_t* __restrict__ lv_off,
                              const int32_t* __restrict__ lv_comp, const int32_t* __restrict__ lv_gid,
                              const int64_t* __restrict__ vert_off, int32_t* __restrict__ out) {
    GRID_STRIDE(p, m) {
        int f = perm[p];
        int c = face_comp[f];
        for (int j = 0; j < 3; ++j) {
            int g = lv_find(lv_off, lv_comp, lv_gid, F[3 * f + j], c);
            out[3 * p + j] = (int32_t)(g - vert_off[c]);
        }
    }
}

const char* face_err_text(int code) {
    switch (code) {
        case ERR_FACE_RANGE: return "face index out of range";
        case ERR_FACE_REPEAT: return "has repeated vertices";
        case ERR_DIRECTED_DUP: return "inconsistent orientation or non-manifold edge (directed edge repeated)";
        default: return "invalid mesh";
    }
}

int read_err(DevBuf<DevErr>& e, DevErr* h, cudaStream_t s) {
    PGCP_TRY_CUDA(cudaMemcpyAsync(h, e.p, sizeof(DevErr), cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaStreamSynchronize(s));
    return PGCP_OK;
}

int reset_err(DevBuf<DevErr>& e, cudaStream_t s) {
    DevErr h{0, 0, ~0ull, 0};
    PGCP_TRY_CUDA(cudaMemcpyAsync(e.p, &h, sizeof(DevErr), cudaMemcpyHostToDevice, s));
    PGCP_TRY_CUDA(cudaStreamSynchronize(s));  // h is a stack temporary
    return PGCP_OK;
}

}  // namespace

// Parent topology (mesh.py:91-111 validation, vertex -> face incidence,
// half-edge twins): everything that does not depend on the cut set. A batch
// created with PGCP_BATCH_VALIDATE_ONLY stops here; pgcp_batch_create_from
// starts a partition from another batch's topology.
int build_topology(pgcp_batch* b, cudaStream_t s) {
    const int64_t n = b->n, m = b->m;
    const int BT = 256;
    DevBuf<DevErr> err;
    PGCP_TRY(err.alloc(1, s));
    PGCP_TRY(reset_err(err, s));
    DevErr herr;

    // --- parent validation (mesh.py:91-111)
    k_validate_faces<<<grid_for(m, BT), BT, 0, s>>>(b->F.p, m, n, err.p);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY(read_err(err, &herr, s));
    if (herr.code) {
        if (herr.code == ERR_FACE_RANGE)
            set_error("face index out of range [0, %lld)", (long long)n);
        else
            set_error("face %llu has repeated vertices", herr.index - (unsigned long long)m);
        return PGCP_E_MESH;
    }

    // --- degenerate faces against the bounding-box diagonal
    {
        DevBuf<double> bb;
        PGCP_TRY(bb.alloc(6, s));
        double init[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
        PGCP_TRY_CUDA(cudaMemcpyAsync(bb.p, init, sizeof(init), cudaMemcpyHostToDevice, s));
        k_bbox<<<grid_for(n, 256, 296), 256, 0, s>>>(b->V.p, n, bb.p);
        PGCP_LAUNCH_CHECK();
        k_degenerate<<<grid_for(m, 256), 256, 0, s>>>(b->V.p, b->F.p, m, bb.p, err.p);
        PGCP_LAUNCH_CHECK();
        PGCP_TRY(read_err(err, &herr, s));
        if (herr.code) {
            set_error("degenerate face %llu (area below epsilon)", herr.index);
            return PGCP_E_MESH;
        }
    }

    // --- vertex -> face incidence, sorted by face id
    {
        DevBuf<int32_t> cnt;
        PGCP_TRY(cnt.alloc(n, s));
        PGCP_TRY(cnt.zero(s));
        k_count_inc<<<grid_for(3 * m, BT), BT, 0, s>>>(b->F.p, 3 * m, cnt.p);
        PGCP_LAUNCH_CHECK();
        PGCP_TRY(b->inc_off.alloc(n + 1, s));
        PGCP_TRY(exclusive_scan_i32_to_i64(cnt.p, b->inc_off.p, n, s));
        PGCP_TRY(cnt.zero(s));
        PGCP_TRY(b->inc.alloc(3 * m, s));
        k_fill_inc<<<grid_for(3 * m, BT), BT, 0, s>>>(b->F.p, m, b->inc_off.p, cnt.p, b->inc.p);
        PGCP_LAUNCH_CHECK();
        k_sort_inc<<<grid_for(n, BT), BT, 0, s>>>(b->inc_off.p, b->inc.p, n);
        PGCP_LAUNCH_CHECK();
    }

    // --- half-edge twins + repeated directed edges
    PGCP_TRY(b->twin.alloc(3 * m, s));
    k_twin<<<grid_for(3 * m, BT), BT, 0, s>>>(b->F.p, m, b->inc_off.p, b->inc.p, b->twin.p, err.p);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY(read_err(err, &herr, s));
    if (herr.code) {
        set_error("%s", face_err_text(herr.code));
        return PGCP_E_MESH;
    }

    b->has_topology = true;
    return PGCP_OK;
}

int build_components(pgcp_batch* b, const int64_t* cuts, int64_t ncuts, bool no_cuts, cudaStream_t s) {
    const int64_t n = b->n, m = b->m;
    const int BT = 256;
    DevBuf<DevErr> err;
    PGCP_TRY(err.alloc(1, s));
    PGCP_TRY(reset_err(err, s));
    DevErr herr;

    // --- cut edges (partition.py:48-59)
    PGCP_TRY(b->he_cut.alloc(3 * m, s));
    PGCP_TRY(b->he_cut.zero(s));
    if (!no_cuts && ncuts > 0) {
        DevBuf<int32_t> mark, dup;
        PGCP_TRY(mark.alloc(3 * m, s));
        PGCP_TRY(mark.zero(s));
        PGCP_TRY(dup.alloc(1, s));
        PGCP_TRY(dup.zero(s));
        k_mark_cuts<<<grid_for(ncuts, BT), BT, 0, s>>>(b->F.p, cuts, ncuts, n, b->inc_off.p, b->inc.p,
                                                      b->twin.p, mark.p, b->he_cut.p, dup.p, err.p);
        PGCP_LAUNCH_CHECK();
        int hdup = 0;
        PGCP_TRY(fetch_scalar(dup.p, &hdup, s));
        PGCP_TRY(read_err(err, &herr, s));
        if (hdup) {
            set_error("duplicate cut edges");
            return PGCP_E_PARTITION;
        }
        if (herr.code) {
            int64_t pair[2] = {-1, -1};
            PGCP_TRY_CUDA(cudaMemcpyAsync(pair, cuts + 2 * herr.index, sizeof(pair), cudaMemcpyDeviceToHost, s));
            PGCP_TRY_CUDA(cudaStreamSynchronize(s));
            int64_t lo = pair[0] < pair[1] ? pair[0] : pair[1];
            int64_t hi = pair[0] < pair[1] ? pair[1] : pair[0];
            set_error("cut pair (%lld, %lld) is not a mesh edge", (long long)lo + 1, (long long)hi + 1);
            return PGCP_E_PARTITION;
        }
    }

    // --- connected components of the face graph minus cut edges
    {
        DevBuf<int> parent;
        DevBuf<int32_t> is_root;
        DevBuf<int64_t> rank;
        PGCP_TRY(parent.alloc(m, s));
        PGCP_TRY(is_root.alloc(m, s));
        PGCP_TRY(rank.alloc(m + 1, s));
        k_uf_init<<<grid_for(m, BT), BT, 0, s>>>(parent.p, m);
        PGCP_LAUNCH_CHECK();
        k_uf_union<<<grid_for(3 * m, BT), BT, 0, s>>>(b->twin.p, no_cuts ? nullptr : b->he_cut.p, m, parent.p);
        PGCP_LAUNCH_CHECK();
        k_uf_roots<<<grid_for(m, BT), BT, 0, s>>>(parent.p, m, is_root.p);
        PGCP_LAUNCH_CHECK();
        PGCP_TRY(exclusive_scan_i32_to_i64(is_root.p, rank.p, m, s));
        PGCP_TRY(b->face_comp.alloc(m, s));
        k_face_comp<<<grid_for(m, BT), BT, 0, s>>>(parent.p, m, rank.p, b->face_comp.p);
        PGCP_LAUNCH_CHECK();
        int64_t K = 0;
        PGCP_TRY(fetch_scalar(rank.p + m, &K, s));
        b->K = (int32_t)K;
    }
    const int32_t K = b->K;
    if (K <= 0) {
        set_error("mesh has no faces");
        return PGCP_E_MESH;
    }

    // --- local vertices, grouped by submesh with sorted parent ids
    DevBuf<int32_t> lv_vert, perm;
    {
        DevBuf<int32_t> cnt;
        PGCP_TRY(cnt.alloc(n, s));
        k_lv_count<<<grid_for(n, BT), BT, 0, s>>>(b->inc_off.p, b->inc.p, b->face_comp.p, n, cnt.p, err.p);
        PGCP_LAUNCH_CHECK();
        PGCP_TRY(b->lv_off.alloc(n + 1, s));
        PGCP_TRY(exclusive_scan_i32_to_i64(cnt.p, b->lv_off.p, n, s));
        PGCP_TRY(fetch_scalar(b->lv_off.p + n, &b->sum_n, s));
        PGCP_TRY(read_err(err, &herr, s));
        if (herr.code) {
            set_error("vertex %llu touches more than %d submeshes", herr.index, MAX_VCOMP);
            return PGCP_E_PARTITION;
        }
    }
    const int64_t E = b->sum_n;
    PGCP_TRY(b->lv_comp.alloc(E, s));
    PGCP_TRY(lv_vert.alloc(E, s));
    k_lv_fill<<<grid_for(n, BT), BT, 0, s>>>(b->inc_off.p, b->inc.p, b->face_comp.p, n, b->lv_off.p,
                                           b->lv_comp.p, lv_vert.p);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY(perm.alloc(E, s));
    PGCP_TRY(b->vert_off.alloc(K + 1, s));
    PGCP_TRY(stable_counting_sort(b->lv_comp.p, E, K, perm.p, b->vert_off.p, s));
    PGCP_TRY(b->lv_gid.alloc(E, s));
    PGCP_TRY(b->vmap.alloc(E, s));
    PGCP_TRY(b->comp_of_gid.alloc(E, s));
    k_lv_gid<<<grid_for(E, BT), BT, 0, s>>>(perm.p, E, lv_vert.p, b->lv_comp.p, b->lv_gid.p, b->vmap.p,
                                          b->comp_of_gid.p);
    PGCP_LAUNCH_CHECK();

    // --- boundaries, topology, loops
    DevBuf<int32_t> fcnt, bcnt, start, bad, chi, loops, pnxt, pscal;
    PGCP_TRY(fcnt.alloc(K, s));
    PGCP_TRY(fcnt.zero(s));
    PGCP_TRY(bcnt.alloc(K, s));
    PGCP_TRY(bcnt.zero(s));
    PGCP_TRY(start.alloc(K, s));
    PGCP_TRY(bad.alloc(K, s));
    PGCP_TRY(bad.zero(s));
    PGCP_TRY(chi.alloc(K, s));
    PGCP_TRY(loops.alloc(K, s));
    PGCP_TRY(pnxt.alloc(n, s));
    PGCP_TRY(pscal.alloc(5, s));  // count, start, bad, nodes, on_start
    PGCP_TRY(b->nxt.alloc(E, s));
    DevBuf<int32_t> node, idx, pnode, pidx;
    PGCP_TRY(node.alloc(3 * m, s));
    PGCP_TRY(idx.alloc(E, s));
    PGCP_TRY(pnode.alloc(n, s));
    PGCP_TRY(pidx.alloc(n, s));
    PGCP_TRY(idx.fill_bytes(0xff, s));
    PGCP_TRY(pidx.fill_bytes(0xff, s));
    k_fill_i32<<<grid_for(K, BT), BT, 0, s>>>(start.p, K, INT_MAX);
    k_fill_i32<<<grid_for(E, BT), BT, 0, s>>>(b->nxt.p, E, -1);
    k_fill_i32<<<grid_for(n, BT), BT, 0, s>>>(pnxt.p, n, -1);
    {
        int32_t init[5] = {0, INT_MAX, 0, 0, 0};
        PGCP_TRY_CUDA(cudaMemcpyAsync(pscal.p, init, sizeof(init), cudaMemcpyHostToDevice, s));
        PGCP_TRY_CUDA(cudaStreamSynchronize(s));
    }
    k_face_count<<<grid_for(m, BT), BT, 0, s>>>(b->face_comp.p, m, fcnt.p);
    PGCP_LAUNCH_CHECK();
    k_boundary<<<grid_for(3 * m, BT), BT, 0, s>>>(b->F.p, m, b->twin.p, b->face_comp.p, b->lv_off.p,
                                                b->lv_comp.p, b->lv_gid.p, b->nxt.p, bcnt.p, start.p, bad.p,
                                                pnxt.p, pscal.p, pscal.p + 1, pscal.p + 2, node.p, idx.p,
                                                pscal.p + 3, pnode.p, pidx.p, n);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY(b->loop_off.alloc(K + 1, s));
    PGCP_TRY(exclusive_scan_i32_to_i64(bcnt.p, b->loop_off.p, K, s));
    PGCP_TRY(fetch_scalar(b->loop_off.p + K, &b->sum_nb, s));
    PGCP_TRY(b->loop.alloc(b->sum_nb, s));
    PGCP_TRY(b->loop.zero(s));  // entries of non-disk components may stay unwalked
    DevBuf<uint8_t> seen;
    PGCP_TRY(seen.alloc(E, s));
    PGCP_TRY(seen.zero(s));
    DevBuf<int32_t> cflag;
    PGCP_TRY(cflag.alloc(K, s));
    PGCP_TRY(cflag.zero(s));
    int rounds = 1;
    while ((1ll << rounds) < b->sum_nb + 2) ++rounds;
    if (b->sum_nb > 0) {
        DevBuf<int32_t> sa, da, sb, db;
        PGCP_TRY(sa.alloc(b->sum_nb, s));
        PGCP_TRY(da.alloc(b->sum_nb, s));
        PGCP_TRY(sb.alloc(b->sum_nb, s));
        PGCP_TRY(db.alloc(b->sum_nb, s));
        k_lr_init<<<grid_for(b->sum_nb, BT), BT, 0, s>>>(b->sum_nb, node.p, idx.p, b->nxt.p, b->comp_of_gid.p,
                                                        start.p, sa.p, da.p, cflag.p);
        PGCP_LAUNCH_CHECK();
        for (int r = 0; r < rounds; ++r) {
            k_lr_step<<<grid_for(b->sum_nb, BT), BT, 0, s>>>(b->sum_nb, sa.p, da.p, sb.p, db.p);
            PGCP_LAUNCH_CHECK();
            std::swap(sa.p, sb.p);
            std::swap(da.p, db.p);
        }
        k_lr_finish<<<grid_for(b->sum_nb, BT), BT, 0, s>>>(b->sum_nb, node.p, idx.p, b->comp_of_gid.p, start.p,
                                                          sa.p, da.p, bcnt.p, b->vert_off.p, b->loop_off.p, bad.p,
                                                          cflag.p, b->loop.p);
        PGCP_LAUNCH_CHECK();
    }
    k_walk<<<grid_for(K, 64), 64, 0, s>>>(K, b->vert_off.p, fcnt.p, bcnt.p, start.p, b->nxt.p, b->loop_off.p,
                                         b->loop.p, bad.p, chi.p, loops.p, seen.p, cflag.p);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY(b->cyc.alloc(b->sum_nb, s));
    if (b->sum_nb > 0) {
        k_cycles<<<grid_for(b->sum_nb, 256), 256, 0, s>>>(K, b->loop_off.p, b->loop.p, b->vert_off.p, b->vmap.p,
                                                         b->cyc.p, b->sum_nb);
        PGCP_LAUNCH_CHECK();
    }
    DevBuf<int64_t> ploops;
    PGCP_TRY(ploops.alloc(1, s));
    {
        // parent boundary cycles: at most n nodes (more means a broken boundary)
        int32_t hpc = 0;
        PGCP_TRY(fetch_scalar(pscal.p, &hpc, s));
        const int64_t pn = std::min<int64_t>(hpc, n);
        if (pn > 0) {
            DevBuf<int32_t> ja, la, jb, lb;
            PGCP_TRY(ja.alloc(pn, s));
            PGCP_TRY(la.alloc(pn, s));
            PGCP_TRY(jb.alloc(pn, s));
            PGCP_TRY(lb.alloc(pn, s));
            k_plab_init<<<grid_for(pn, BT), BT, 0, s>>>(pn, pnode.p, pidx.p, pnxt.p, ja.p, la.p, pscal.p + 2);
            PGCP_LAUNCH_CHECK();
            int pr = 1;
            while ((1ll << pr) < pn + 2) ++pr;
            for (int r = 0; r < pr; ++r) {
                k_plab_step<<<grid_for(pn, BT), BT, 0, s>>>(pn, ja.p, la.p, jb.p, lb.p);
                PGCP_LAUNCH_CHECK();
                std::swap(ja.p, jb.p);
                std::swap(la.p, lb.p);
            }
            k_plab_finish<<<grid_for(pn, BT), BT, 0, s>>>(pn, la.p, pscal.p + 1, pscal.p, pscal.p + 2, pscal.p + 4,
                                                         ploops.p);
            PGCP_LAUNCH_CHECK();
        }
        k_plab_result<<<1, 32, 0, s>>>(pscal.p, pscal.p + 2, pscal.p + 4, n, ploops.p);
        PGCP_LAUNCH_CHECK();
    }

    // --- host copies of the small per-submesh tables
    b->h_vert_off.resize(K + 1);
    b->h_loop_off.resize(K + 1);
    b->h_comp_chi.resize(K);
    b->h_comp_loops.resize(K);
    std::vector<int32_t> hbad(K), hp(3);
    PGCP_TRY_CUDA(cudaMemcpyAsync(b->h_vert_off.data(), b->vert_off.p, (K + 1) * sizeof(int64_t),
                                  cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(b->h_loop_off.data(), b->loop_off.p, (K + 1) * sizeof(int64_t),
                                  cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(b->h_comp_chi.data(), chi.p, K * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(b->h_comp_loops.data(), loops.p, K * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(hbad.data(), bad.p, K * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(hp.data(), pscal.p, 3 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    int64_t hploops = 0;
    PGCP_TRY_CUDA(cudaMemcpyAsync(&hploops, ploops.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaStreamSynchronize(s));
    // parent topology (mesh.py:206-223): chi = n - E + m with 2E = 3m + b
    int64_t pb = hp[0];
    b->parent_chi = n - (3 * m + pb) / 2 + m;
    b->parent_loops = hploops;
    b->bad_comp = -1;
    for (int c = 0; c < K; ++c) {
        if (hbad[c]) {
            b->bad_comp = c;
            break;
        }
    }
    return PGCP_OK;
}

int local_faces(pgcp_batch* b, int64_t* face_off, int32_t* faces, cudaStream_t s) {
    const int64_t m = b->m;
    DevBuf<int32_t> perm;
    DevBuf<int64_t> off;
    PGCP_TRY(perm.alloc(m, s));
    PGCP_TRY(off.alloc(b->K + 1, s));
    PGCP_TRY(stable_counting_sort(b->face_comp.p, m, b->K, perm.p, off.p, s));
    k_local_faces<<<grid_for(m, 256), 256, 0, s>>>(b->F.p, perm.p, m, b->face_comp.p, b->lv_off.p, b->lv_comp.p,
                                                   b->lv_gid.p, b->vert_off.p, faces);
    PGCP_LAUNCH_CHECK();
    PGCP_TRY_CUDA(cudaMemcpyAsync(face_off, off.p, (b->K + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaStreamSynchronize(s));
    return PGCP_OK;
}

int build_partition(pgcp_batch* b, const int64_t* cuts, int64_t ncuts, bool no_cuts, cudaStream_t s) {
    PGCP_TRY(build_topology(b, s));
    return build_components(b, cuts, ncuts, no_cuts, s);
}

}  // namespace pgcp

extern "C" PGCP_API int pgcp_faces_from_i64(const int64_t* src, int32_t* dst, int64_t count, void* stream) {
    if (count < 0 || (count > 0 && (!src || !dst))) {
        pgcp::set_error("pgcp_faces_from_i64: invalid arguments");
        return PGCP_E_INVALID;
    }
    if (count == 0) return PGCP_OK;
    pgcp::k_faces_i64<<<pgcp::grid_for(count, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(src, dst, count);
    PGCP_LAUNCH_CHECK();
    return PGCP_OK;
}
