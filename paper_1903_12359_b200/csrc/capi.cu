// capi.cu -- extern "C" entry points of libpgcp_b200.so (include/pgcp_b200.h).
#include <algorithm>
#include <cstdlib>

#include "batch.cuh"

using namespace pgcp;

namespace {

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Scratch buffers are stream-ordered allocations from the device's default
// pool. Keep freed blocks cached in the pool (release threshold = max): with
// the default threshold of 0 every stream synchronisation hands the memory
// back to the driver and the next call maps it again.
void keep_pool(int dev) {
    static bool done[64] = {false};
    if (dev < 0 || dev >= 64 || done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        // map the pool's working set once (PGCP_POOL_RESERVE_GB, default 8):
        // growing it later (mapping memory while other threads allocate and
        // launch) stalls the driver for milliseconds
        const char* e = getenv("PGCP_POOL_RESERVE_GB");
        const double gb = e ? atof(e) : 8.0;
        size_t free_b = 0, total_b = 0;
        if (gb > 0 && cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
            const size_t want = std::min<size_t>((size_t)(gb * 1e9), free_b / 4);
            void* p = nullptr;
            int cur = 0;
            cudaGetDevice(&cur);
            cudaSetDevice(dev);
            if (cudaMallocAsync(&p, want, 0) == cudaSuccess) {
                cudaFreeAsync(p, 0);
                cudaStreamSynchronize(0);
            }
            cudaSetDevice(cur);
        }
    }
    cudaGetLastError();
    done[dev] = true;
}

int set_device_of(const void* ptr) {
    if (!ptr) return PGCP_OK;
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, ptr);
    if (e != cudaSuccess || at.type != cudaMemoryTypeDevice) {
        cudaGetLastError();
        set_error("expected a CUDA device pointer");
        return PGCP_E_INVALID;
    }
    PGCP_TRY_CUDA(cudaSetDevice(at.device));
    keep_pool(at.device);
    return PGCP_OK;
}

}  // namespace

extern "C" {

int pgcp_abi_version(void) { return PGCP_ABI_VERSION; }

const char* pgcp_last_error(void) { return get_error(); }

unsigned long long pgcp_launch_count(void) { return pgcp::launch_count(); }

int pgcp_batch_last_solve(const pgcp_batch* b, int which, double* out, int nout) {
    if (!b || !out || which < 0 || which > 1) {
        set_error("pgcp_batch_last_solve: invalid arguments");
        return PGCP_E_INVALID;
    }
    double v[19];
    pgcp::solve_summary(b, which, v);
    for (int i = 0; i < nout && i < 19; ++i) out[i] = v[i];
    return PGCP_OK;
}

int pgcp_batch_create(const double* V, const int32_t* F, int64_t n, int64_t m, const int64_t* cuts, int64_t ncuts,
                      uint32_t flags, void* stream, pgcp_batch** out) {
    if (!out || !V || !F || n <= 0 || m <= 0 || ncuts < 0 || (ncuts > 0 && !cuts)) {
        set_error("pgcp_batch_create: invalid arguments");
        return PGCP_E_INVALID;
    }
    *out = nullptr;
    PGCP_TRY(set_device_of(V));
    cudaStream_t s = as_stream(stream);
    pgcp_batch* b = new pgcp_batch();
    cudaGetDevice(&b->device);
    b->n = n;
    b->m = m;
    int st = b->V.alloc(3 * n, s);
    if (st == PGCP_OK) st = b->F.alloc(3 * m, s);
    if (st == PGCP_OK) {
        cudaError_t e1 = cudaMemcpyAsync(b->V.p, V, 3 * n * sizeof(double), cudaMemcpyDeviceToDevice, s);
        cudaError_t e2 = cudaMemcpyAsync(b->F.p, F, 3 * m * sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
        if (e1 != cudaSuccess || e2 != cudaSuccess) {
            set_error("pgcp_batch_create: copy failed: %s", cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
            st = PGCP_E_CUDA;
        }
    }
    if (st == PGCP_OK)
        st = (flags & PGCP_BATCH_VALIDATE_ONLY)
                 ? build_topology(b, s)
                 : build_partition(b, cuts, ncuts, (flags & PGCP_BATCH_NO_CUTS) != 0, s);
    if (st != PGCP_OK) {
        free_system(b->sys[0]);
        free_system(b->sys[1]);
        delete b;
        return st;
    }
    *out = b;
    return PGCP_OK;
}

int pgcp_batch_create_from(const pgcp_batch* base, const int64_t* cuts, int64_t ncuts, uint32_t flags, void* stream,
                           pgcp_batch** out) {
    if (!out || !base || !base->has_topology || ncuts < 0 || (ncuts > 0 && !cuts)) {
        set_error("pgcp_batch_create_from: invalid arguments");
        return PGCP_E_INVALID;
    }
    *out = nullptr;
    PGCP_TRY_CUDA(cudaSetDevice(base->device));
    cudaStream_t s = as_stream(stream);
    pgcp_batch* b = new pgcp_batch();
    b->device = base->device;
    b->n = base->n;
    b->m = base->m;
    const int64_t n = b->n, m = b->m;
    auto copy = [&](void* dst, const void* src, size_t bytes) -> int {
        cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) {
            set_error("pgcp_batch_create_from: copy failed: %s", cudaGetErrorString(e));
            return PGCP_E_CUDA;
        }
        return PGCP_OK;
    };
    int st = b->V.alloc(3 * n, s);
    if (st == PGCP_OK) st = b->F.alloc(3 * m, s);
    if (st == PGCP_OK) st = b->inc_off.alloc(n + 1, s);
    if (st == PGCP_OK) st = b->inc.alloc(3 * m, s);
    if (st == PGCP_OK) st = b->twin.alloc(3 * m, s);
    if (st == PGCP_OK) st = copy(b->V.p, base->V.p, 3 * n * sizeof(double));
    if (st == PGCP_OK) st = copy(b->F.p, base->F.p, 3 * m * sizeof(int32_t));
    if (st == PGCP_OK) st = copy(b->inc_off.p, base->inc_off.p, (n + 1) * sizeof(int64_t));
    if (st == PGCP_OK) st = copy(b->inc.p, base->inc.p, 3 * m * sizeof(int32_t));
    if (st == PGCP_OK) st = copy(b->twin.p, base->twin.p, 3 * m * sizeof(int32_t));
    if (st == PGCP_OK) {
        b->has_topology = true;
        st = build_components(b, cuts, ncuts, (flags & PGCP_BATCH_NO_CUTS) != 0, s);
    }
    if (st != PGCP_OK) {
        delete b;
        return st;
    }
    *out = b;
    return PGCP_OK;
}

int pgcp_batch_destroy(pgcp_batch* b) {
    if (!b) return PGCP_OK;
    cudaSetDevice(b->device);
    free_system(b->sys[0]);
    free_system(b->sys[1]);
    delete b;
    return PGCP_OK;
}

int pgcp_batch_release_solvers(pgcp_batch* b, int which) {
    if (!b) {
        set_error("pgcp_batch_release_solvers: null batch");
        return PGCP_E_INVALID;
    }
    PGCP_TRY_CUDA(cudaSetDevice(b->device));
    for (int k = 0; k < 2; ++k)
        if (which & (1 << k)) {
            free_system(b->sys[k]);
            b->sys[k] = nullptr;
        }
    return PGCP_OK;
}

int pgcp_batch_info(const pgcp_batch* b, int64_t* info, int ninfo) {
    if (!b || !info) {
        set_error("pgcp_batch_info: null argument");
        return PGCP_E_INVALID;
    }
    int64_t v[PGCP_INFO_COUNT] = {0};
    v[PGCP_INFO_K] = b->K;
    v[PGCP_INFO_SUM_N] = b->sum_n;
    v[PGCP_INFO_SUM_NB] = b->sum_nb;
    v[PGCP_INFO_NNZ_L] = b->nnz;
    v[PGCP_INFO_PARENT_CHI] = b->parent_chi;
    v[PGCP_INFO_PARENT_LOOPS] = b->parent_loops;
    v[PGCP_INFO_N] = b->n;
    v[PGCP_INFO_M] = b->m;
    v[PGCP_INFO_BAD_COMP] = b->bad_comp;
    if (b->bad_comp >= 0) {
        v[9] = b->h_comp_chi[b->bad_comp];
        v[10] = b->h_comp_loops[b->bad_comp];
    }
    for (int i = 0; i < ninfo && i < PGCP_INFO_COUNT; ++i) info[i] = v[i];
    return PGCP_OK;
}

int pgcp_batch_array(const pgcp_batch* b, int which, void** ptr, int64_t* count) {
    if (!b || !ptr || !count) {
        set_error("pgcp_batch_array: null argument");
        return PGCP_E_INVALID;
    }
    switch (which) {
        case PGCP_ARR_FACE_COMP: *ptr = b->face_comp.p; *count = b->m; break;
        case PGCP_ARR_VERT_OFF: *ptr = b->vert_off.p; *count = b->K + 1; break;
        case PGCP_ARR_VMAP: *ptr = b->vmap.p; *count = b->sum_n; break;
        case PGCP_ARR_LOOP_OFF: *ptr = b->loop_off.p; *count = b->K + 1; break;
        case PGCP_ARR_LOOP: *ptr = b->loop.p; *count = b->sum_nb; break;
        case PGCP_ARR_L_ROWPTR: *ptr = b->row_ptr.p; *count = b->has_laplacian ? b->sum_n + 1 : 0; break;
        case PGCP_ARR_L_COL: *ptr = b->col.p; *count = b->has_laplacian ? b->nnz : 0; break;
        case PGCP_ARR_L_VAL: *ptr = b->val.p; *count = b->has_laplacian ? b->nnz : 0; break;
        case PGCP_ARR_W3: *ptr = b->w3.p; *count = b->w3.p ? 3 * b->m : 0; break;
        case PGCP_ARR_PINS: *ptr = b->pins.p; *count = b->pins.p ? 2 * (int64_t)b->K : 0; break;
        case PGCP_ARR_CYCLES: *ptr = b->cyc.p; *count = b->sum_nb; break;
        default:
            set_error("pgcp_batch_array: unknown array id %d", which);
            return PGCP_E_INVALID;
    }
    return PGCP_OK;
}

int pgcp_batch_local_faces(pgcp_batch* b, int64_t* face_off, int32_t* faces, void* stream) {
    if (!b || !face_off || !faces) {
        set_error("pgcp_batch_local_faces: null argument");
        return PGCP_E_INVALID;
    }
    PGCP_TRY_CUDA(cudaSetDevice(b->device));
    return local_faces(b, face_off, faces, as_stream(stream));
}

int pgcp_batch_laplacian(pgcp_batch* b, int64_t* clamped, void* stream) {
    if (!b) {
        set_error("pgcp_batch_laplacian: null batch");
        return PGCP_E_INVALID;
    }
    PGCP_TRY_CUDA(cudaSetDevice(b->device));
    return build_laplacian(b, clamped, as_stream(stream));
}

int pgcp_batch_default_pins(pgcp_batch* b, void* stream) {
    if (!b) {
        set_error("pgcp_batch_default_pins: null batch");
        return PGCP_E_INVALID;
    }
    PGCP_TRY_CUDA(cudaSetDevice(b->device));
    return default_pins(b, as_stream(stream));
}

int pgcp_batch_flatten(pgcp_batch* b, const int32_t* comps, int32_t ncomp, const int32_t* pins,
                       const double* targets, const pgcp_solve_opts* opts, double* z, pgcp_solve_stat* stats,
                       void* stream) {
    if (!b || !z) {
        set_error("pgcp_batch_flatten: null argument");
        return PGCP_E_INVALID;
    }
    PGCP_TRY_CUDA(cudaSetDevice(b->device));
    cudaStream_t s = as_stream(stream);
    if (!b->has_laplacian) PGCP_TRY(build_laplacian(b, nullptr, s));
    return solve_flatten(b, comps, ncomp, pins, targets, opts, z, stats, s);
}

int pgcp_batch_harmonic(pgcp_batch* b, const int32_t* comps, int32_t ncomp, const int32_t* fixed_gid,
                        const double* fixed_val, int64_t nfixed, const pgcp_solve_opts* opts, double* z,
                        pgcp_solve_stat* stats, void* stream) {
    if (!b || !z || nfixed < 0 || (nfixed > 0 && (!fixed_gid || !fixed_val))) {
        set_error("pgcp_batch_harmonic: invalid arguments");
        return PGCP_E_INVALID;
    }
    PGCP_TRY_CUDA(cudaSetDevice(b->device));
    cudaStream_t s = as_stream(stream);
    if (!b->has_laplacian) PGCP_TRY(build_laplacian(b, nullptr, s));
    return solve_harmonic(b, comps, ncomp, fixed_gid, fixed_val, nfixed, opts, z, stats, s);
}

int pgcp_batch_harmonic_prepare(pgcp_batch* b, const int32_t* comps, int32_t ncomp, const int32_t* fixed_gid,
                                int64_t nfixed, const pgcp_solve_opts* opts, void* stream) {
    if (!b || nfixed < 0 || (nfixed > 0 && !fixed_gid)) {
        set_error("pgcp_batch_harmonic_prepare: invalid arguments");
        return PGCP_E_INVALID;
    }
    PGCP_TRY_CUDA(cudaSetDevice(b->device));
    cudaStream_t s = as_stream(stream);
    if (!b->has_laplacian) PGCP_TRY(build_laplacian(b, nullptr, s));
    return prepare_harmonic(b, comps, ncomp, fixed_gid, nfixed, opts, s);
}

int pgcp_batch_harmonic_solve(pgcp_batch* b, const double* fixed_val, int64_t nfixed, const pgcp_solve_opts* opts,
                              double* z, pgcp_solve_stat* stats, void* stream) {
    if (!b || !z || nfixed < 0 || (nfixed > 0 && !fixed_val)) {
        set_error("pgcp_batch_harmonic_solve: invalid arguments");
        return PGCP_E_INVALID;
    }
    PGCP_TRY_CUDA(cudaSetDevice(b->device));
    return finish_harmonic(b, fixed_val, nfixed, opts, z, stats, as_stream(stream));
}

int pgcp_batch_export_system(pgcp_batch* b, int which, int32_t comp, int64_t* dims, int32_t* indptr,
                             int32_t* indices, double* data, double* rhs, void* stream) {
    if (!b || !dims) {
        set_error("pgcp_batch_export_system: null argument");
        return PGCP_E_INVALID;
    }
    PGCP_TRY_CUDA(cudaSetDevice(b->device));
    return export_system(b, which, comp, dims, indptr, indices, data, rhs, as_stream(stream));
}

int pgcp_batch_conformal_energy(pgcp_batch* b, const double* z, double* energy, void* stream) {
    if (!b || !z || !energy) {
        set_error("pgcp_batch_conformal_energy: null argument");
        return PGCP_E_INVALID;
    }
    PGCP_TRY_CUDA(cudaSetDevice(b->device));
    return conformal_energy(b, z, energy, as_stream(stream));
}

int pgcp_face_layout(const double* V, const int32_t* F, int64_t m, double* layout, void* stream) {
    if (m < 0 || (m > 0 && (!V || !F || !layout))) {
        set_error("pgcp_face_layout: invalid arguments");
        return PGCP_E_INVALID;
    }
    PGCP_TRY(set_device_of(V));
    return face_layout(V, F, m, layout, as_stream(stream));
}

int pgcp_beltrami(const double* src, const int32_t* src_faces, const double* tgt, const int32_t* tgt_faces,
                  int64_t m, double* mu, int64_t* first_degenerate, void* stream) {
    if (m < 0 || (m > 0 && (!src || !tgt || !mu))) {
        set_error("pgcp_beltrami: invalid arguments");
        return PGCP_E_INVALID;
    }
    PGCP_TRY(set_device_of(src));
    return beltrami_per_face(src, src_faces, tgt, tgt_faces, m, mu, first_degenerate, as_stream(stream));
}

int pgcp_batch_lbs_stiffness(pgcp_batch* b, const double* z, const double* mu, double* kval, void* stream) {
    if (!b || !z || !mu || !kval) {
        set_error("pgcp_batch_lbs_stiffness: invalid arguments");
        return PGCP_E_INVALID;
    }
    PGCP_TRY_CUDA(cudaSetDevice(b->device));
    return lbs_stiffness(b, z, mu, kval, as_stream(stream));
}

int pgcp_batch_qc_repair(pgcp_batch* b, const int32_t* comps, int32_t ncomp, const double* layout,
                         const int32_t* fixed_gid, int64_t nfixed, int32_t max_iter, double cap,
                         const pgcp_solve_opts* opts, double* z, int32_t* info, uint8_t* flipped, void* stream) {
    if (!b || !z || !info || ncomp < 0 || nfixed < 0 || (nfixed > 0 && !fixed_gid) || max_iter < 0 ||
        !(cap > 0.0 && cap < 1.0)) {
        set_error("pgcp_batch_qc_repair: invalid arguments");
        return PGCP_E_INVALID;
    }
    PGCP_TRY_CUDA(cudaSetDevice(b->device));
    return qc_repair(b, comps, ncomp, layout, fixed_gid, nfixed, max_iter, cap, opts, z, info, flipped,
                     as_stream(stream));
}

}  // extern "C"
