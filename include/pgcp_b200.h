/*
 * pgcp_b200.h -- C ABI of the B200-native PGCP hot path (libpgcp_b200.so).
 *
 * The reference (`/root/reference/pkg/src/pgcp`) is pure Python: its only
 * "plugin seam" is the Python function surface re-exported in
 * `pkg/src/pgcp/__init__.py:7-26` plus the per-subdomain batch seam
 * `pipeline._run_tasks` (`pipeline.py:105-109`). This header is the native
 * boundary under the drop-in Python package `paper_1903_12359_b200`, which
 * binds it with ctypes. Every entry point names the
 * reference code it replaces.
 *
 * Conventions
 *   - every function returns an int status (PGCP_OK or a PGCP_E_* code);
 *     pgcp_last_error() returns the thread-local message of the last failure;
 *   - pointers documented "device" are CUDA device pointers, "host" are host;
 *   - `stream` is a cudaStream_t passed as void*; all device work of a call is
 *     enqueued on it. Calls that must report data-dependent sizes or errors
 *     synchronise that stream before returning (documented per call);
 *   - complex values are interleaved (re, im) doubles (numpy complex128);
 *   - no PyTorch types cross this boundary.
 */
#ifndef PGCP_B200_H
#define PGCP_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define PGCP_API __attribute__((visibility("default")))
#else
#define PGCP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define PGCP_ABI_VERSION 2

/* status codes -> Python exceptions (paper_1903_12359_b200/_native.py) */
#define PGCP_OK 0
#define PGCP_E_INVALID 1    /* bad argument                       -> ValueError      */
#define PGCP_E_MESH 2       /* mesh.py:15 MeshError                                   */
#define PGCP_E_PARTITION 3  /* partition.py:21 PartitionError                         */
#define PGCP_E_SOLVE 4      /* flatten.py:24 SolveError (contract violation)          */
#define PGCP_E_NOCONV 5     /* SolveError: PCG did not reach rtol within maxit         */
#define PGCP_E_WELD 6       /* welding.py:35 WeldError                                */
#define PGCP_E_CUDA 7       /* CUDA runtime failure                  -> RuntimeError    */
#define PGCP_E_VALIDATION 8 /* pipeline.py:32 ValidationError                         */

typedef struct pgcp_batch pgcp_batch;

PGCP_API int pgcp_abi_version(void);
PGCP_API const char* pgcp_last_error(void);
/* number of kernels this library has launched in the process */
PGCP_API unsigned long long pgcp_launch_count(void);
/* diagnostics: the direct solver's workspace cache on the current device --
 * out[0] slots, out[1] cached bytes, out[2] slot (re)allocations since load,
 * out[3] host ms spent in them (cudaFree + cudaMalloc) */
PGCP_API int pgcp_workspace_stats(double* out, int nout);

/* -------------------------------------------------------------------------
 * Batch of disk-type submeshes of one parent mesh, device resident.
 *
 * pgcp_batch_create replaces partition.py:94-137 (partition_mesh: face
 * adjacency minus cut edges -> connected components ordered by minimum face,
 * sorted vertex maps, disk-type check) and mesh.py:144-173 (boundary_loops:
 * walk from the smallest boundary vertex, surface on the left). It also
 * evaluates the parent mesh topology of mesh.py:206-223 (validate_topology).
 *   V     device, n*3 float64     F     device, m*3 int32
 *   cuts  device, ncuts*2 int64 parent vertex pairs (NULL iff ncuts == 0)
 *   flags PGCP_BATCH_NO_CUTS: single domain = the whole mesh (pipeline.py:143-150)
 * Synchronises `stream`. Errors: PGCP_E_MESH (bad indices, non-manifold or
 * inconsistently oriented edges, pinched boundaries), PGCP_E_PARTITION
 * (duplicate/non-edge cuts, non-disk component).
 */
#define PGCP_BATCH_NO_CUTS 1u
/* PGCP_BATCH_VALIDATE_ONLY: validate the parent mesh (mesh.py:91-111: face
 * indices, repeated vertices, degenerate faces, repeated directed edges) and
 * build its incidence and half-edge twins only; no submeshes (K = 0). The
 * TriMesh constructor's check; partitions start from it with
 * pgcp_batch_create_from. */
#define PGCP_BATCH_VALIDATE_ONLY 2u
PGCP_API int pgcp_batch_create(const double* V, const int32_t* F, int64_t n, int64_t m,
                      const int64_t* cuts, int64_t ncuts, uint32_t flags,
                      void* stream, pgcp_batch** out);
/* A partition of base's mesh (pgcp_batch_create without re-validating the
 * mesh and without rebuilding its incidence and twins). flags as above
 * (PGCP_BATCH_NO_CUTS). */
PGCP_API int pgcp_batch_create_from(const pgcp_batch* base, const int64_t* cuts, int64_t ncuts, uint32_t flags,
                                    void* stream, pgcp_batch** out);
PGCP_API int pgcp_batch_destroy(pgcp_batch* b);
/* Free the batch's last flatten (bit 0 of which) and/or harmonic (bit 1)
 * solver systems -- factors, fronts, workspaces -- once their results are
 * consumed (stream-ordered; pgcp_batch_last_solve then reports zeros). */
PGCP_API int pgcp_batch_release_solvers(pgcp_batch* b, int which);

/* host int64 info[PGCP_INFO_COUNT] */
#define PGCP_INFO_K 0            /* number of submeshes                          */
#define PGCP_INFO_SUM_N 1        /* total local vertices (seam copies counted)   */
#define PGCP_INFO_SUM_NB 2       /* total boundary-loop vertices                 */
#define PGCP_INFO_NNZ_L 3        /* total nnz of the per-submesh Laplacians      */
#define PGCP_INFO_PARENT_CHI 4   /* Euler characteristic of the parent mesh      */
#define PGCP_INFO_PARENT_LOOPS 5 /* parent boundary loops (-2: "two or more")    */
#define PGCP_INFO_N 6
#define PGCP_INFO_M 7
#define PGCP_INFO_BAD_COMP 8     /* first non-disk component (-1 if none)        */
#define PGCP_INFO_COUNT 16
PGCP_API int pgcp_batch_info(const pgcp_batch* b, int64_t* info, int ninfo);

/* device pointer and element count of an internal array */
#define PGCP_ARR_FACE_COMP 0   /* int32 [m]       parent face -> submesh            */
#define PGCP_ARR_VERT_OFF 1    /* int64 [K+1]     local-vertex offsets              */
#define PGCP_ARR_VMAP 2        /* int32 [sum_n]   local -> parent vertex (sorted)   */
#define PGCP_ARR_LOOP_OFF 3    /* int64 [K+1]     boundary-loop offsets             */
#define PGCP_ARR_LOOP 4        /* int32 [sum_nb]  loop, local indices               */
#define PGCP_ARR_L_ROWPTR 5    /* int64 [sum_n+1] CSR rows (global, concatenated)   */
#define PGCP_ARR_L_COL 6       /* int32 [nnz]     CSR columns, LOCAL indices        */
#define PGCP_ARR_L_VAL 7       /* f64   [nnz]                                      */
#define PGCP_ARR_W3 8          /* f64   [3m]      half-cotangent per face corner    */
#define PGCP_ARR_PINS 9        /* int32 [2K]      default pins (local)              */
#define PGCP_ARR_CYCLES 10     /* int32 [sum_nb]  boundary cycles, parent ids       */
PGCP_API int pgcp_batch_array(const pgcp_batch* b, int which, void** ptr, int64_t* count);

/* Local faces of every submesh, faces in increasing parent-face order
 * (partition.py:121-126 `remap[mesh.faces[fidx]]`).
 *   face_off host int64 [K+1]; faces device int32 [m*3]. Synchronises. */
PGCP_API int pgcp_batch_local_faces(pgcp_batch* b, int64_t* face_off, int32_t* faces, void* stream);

/* K1 + K2: per-face cotangent weights (flatten.py:39-57) and the canonical
 * CSR cotangent Laplacian of every submesh (flatten.py:61: rows sorted,
 * duplicates summed, structural zeros kept). PGCP_E_MESH on a zero-area face.
 * clamped (host, may be NULL) receives the number of |cot| > 1e8 clamps. */
PGCP_API int pgcp_batch_laplacian(pgcp_batch* b, int64_t* clamped, void* stream);

/* Default pins of every submesh (flatten.py:113-122, sequential arclength
 * sum). Written to the PGCP_ARR_PINS array. */
PGCP_API int pgcp_batch_default_pins(pgcp_batch* b, void* stream);

/* Solver controls and per-submesh results */
typedef struct {
    double rtol;        /* stop when ||r|| <= rtol ||b|| (recurrence residual)   */
    double contract_tol;/* residual contract of flatten.py:170-173 (1e-10)        */
    int32_t maxit;      /* per-submesh iteration cap (PCG)                       */
    int32_t cluster;    /* CTAs per submesh (0 = auto; PCG)                      */
    int32_t solver;     /* PGCP_SOLVER_*: 0 = default (direct unless maxit > 0
                           or PGCP_SOLVER=pcg), 1 = direct, 2 = PCG            */
    int32_t reserved;
} pgcp_solve_opts;

#define PGCP_SOLVER_DEFAULT 0
#define PGCP_SOLVER_DIRECT 1  /* batched multifrontal Cholesky (direct.cu)       */
#define PGCP_SOLVER_PCG 2     /* batched two-level PCG, one cluster per submesh  */

typedef struct {
    int32_t iters;      /* PCG iterations                                        */
    int32_t status;     /* PGCP_OK / PGCP_E_NOCONV / PGCP_E_SOLVE                 */
    double relres;      /* recurrence ||r||/||b||                                 */
    double true_res;    /* ||A x - b|| recomputed                                 */
    double bnorm;       /* ||b||                                                  */
    double xnorm;       /* ||x||                                                  */
} pgcp_solve_stat;

/* DNCP free-boundary flattening of the listed submeshes (flatten.py:125-188):
 * C_ff x = -C_f,fixed t solved as the equivalent complex Hermitian system
 * (L + 2i M_xy) restricted to the non-pinned vertices, batched fp64 Jacobi
 * PCG, one CTA cluster per submesh.
 *   comps    host int32 [ncomp] submesh ids (NULL: all)
 *   pins     host int32 [2*ncomp] local pins (NULL: default pins)
 *   targets  host f64 [4] = (t0.re, t0.im, t1.re, t1.im)
 *   z        device complex [sum_n] (written for the listed submeshes)
 *   stats    host [ncomp]
 * Synchronises. */
PGCP_API int pgcp_batch_flatten(pgcp_batch* b, const int32_t* comps, int32_t ncomp,
                       const int32_t* pins, const double* targets,
                       const pgcp_solve_opts* opts, double* z,
                       pgcp_solve_stat* stats, void* stream);

/* Dirichlet harmonic extension (assemble.py:23-50) for the listed submeshes.
 *   fixed_gid  device int32 [nfixed] global local-vertex ids held fixed
 *   fixed_val  device complex [nfixed]
 * Unknowns are the remaining local vertices of each listed submesh.
 * Synchronises. */
PGCP_API int pgcp_batch_harmonic(pgcp_batch* b, const int32_t* comps, int32_t ncomp,
                        const int32_t* fixed_gid, const double* fixed_val, int64_t nfixed,
                        const pgcp_solve_opts* opts, double* z,
                        pgcp_solve_stat* stats, void* stream);

/* The harmonic solve in two calls: _prepare builds everything that does not
 * depend on the fixed values (unknown numbering, sliced ELL, Jacobi scaling,
 * coarse space; synchronises `stream`), _solve takes the values (same order
 * as fixed_gid), forms the right-hand side and runs the PCG. Lets a caller
 * overlap the preparation with the computation of the values (the weld).
 * pgcp_batch_harmonic = _prepare + _solve. */
PGCP_API int pgcp_batch_harmonic_prepare(pgcp_batch* b, const int32_t* comps, int32_t ncomp,
                                         const int32_t* fixed_gid, int64_t nfixed, const pgcp_solve_opts* opts,
                                         void* stream);
PGCP_API int pgcp_batch_harmonic_solve(pgcp_batch* b, const double* fixed_val, int64_t nfixed,
                                       const pgcp_solve_opts* opts, double* z, pgcp_solve_stat* stats, void* stream);

/* Summary of the last flatten (0) / harmonic (1) solve: out[0] PCG kernel
 * time in ms (CUDA events on the launch stream), [1] total iterations,
 * [2] max iterations, [3] sum over submeshes of iterations x the device
 * kernel's bytes per iteration, [4] stored entries, [5]
 * unknown rows, [6] CTAs per cluster, [7] submeshes, [8] sum over
 * submeshes of iterations x SURVEY §8(d)'s 12 z + 4 (r + 1) for the
 * reference's CSR system (C_ff / L_II), [9] coarse-space setup ms. */
PGCP_API int pgcp_batch_last_solve(const pgcp_batch* b, int which, double* out, int nout);

/* Exported solver systems for pattern parity (flatten.py:160-166 C_ff and
 * assemble.py:40 L_II), one submesh, CSR with int32 indptr/indices as scipy
 * builds them. which = 0: C_ff of the last flatten (real 2n-4 form, exact
 * zeros dropped as csr_binop does); 1: L_II of the last harmonic solve.
 * Two-call protocol: pass NULL buffers to get (rows, nnz) in dims. */
PGCP_API int pgcp_batch_export_system(pgcp_batch* b, int which, int32_t comp, int64_t* dims,
                             int32_t* indptr, int32_t* indices, double* data,
                             double* rhs, void* stream);

/* Energy of embeddings: per submesh E_D - A (flatten.py:89-110).
 * z device complex [sum_n]; energy host f64 [K]. Synchronises. */
PGCP_API int pgcp_batch_conformal_energy(pgcp_batch* b, const double* z, double* energy, void* stream);

/* -------------------------------------------------------------------------
 * Quasi-conformal fold-over repair (assemble.py:53-217)
 */
/* face_layout (assemble.py:53-67): isometric 2D corners of every face, corner
 * 0 at the origin, corner 1 on the positive real axis.
 *   V device f64 [3n]; F device int32 [3m]; layout device complex [3m]. */
PGCP_API int pgcp_face_layout(const double* V, const int32_t* F, int64_t m, double* layout, void* stream);

/* beltrami_per_face (assemble.py:74-92) of the piecewise-linear map src -> tgt.
 * src/tgt are device complex per-vertex coordinates indexed through
 * src_faces/tgt_faces (device int32 [3m]), or per-face corner arrays
 * [3m] when the face pointer is NULL. mu device complex [m] (fz == 0 -> inf).
 * A degenerate source triangle -> PGCP_E_SOLVE with its index in
 * *first_degenerate (host, optional). Synchronises. */
PGCP_API int pgcp_beltrami(const double* src, const int32_t* src_faces, const double* tgt, const int32_t* tgt_faces,
                           int64_t m, double* mu, int64_t* first_degenerate, void* stream);

/* lbs_stiffness (assemble.py:124-164): linear-element stiffness of the
 * operator with Beltrami coefficient mu on the embedding z (absolute face
 * areas), for every submesh, on the batch Laplacian's CSR pattern
 * (PGCP_ARR_L_ROWPTR / PGCP_ARR_L_COL).
 *   z device complex [sum_n]; mu device complex [m] per parent face;
 *   kval device f64 [nnz]. Synchronises. */
PGCP_API int pgcp_batch_lbs_stiffness(pgcp_batch* b, const double* z, const double* mu, double* kval, void* stream);

/* qc_correct (assemble.py:174-217) of the listed submeshes, batched, in place:
 * while a submesh has faces with signed area <= 0 (at most max_iter times):
 * mu = capped Beltrami coefficient of embedding -> layout, K = linear
 * Beltrami stiffness (lbs_stiffness, assemble.py:124-164, on the Laplacian's
 * pattern), solve K_ff u = -K_f,fixed g with the held values g = z[fixed].
 * The reference calls it per submesh after the harmonic solve
 * (pipeline.py:88-102).
 *   comps     host int32 [ncomp] (NULL: all submeshes)
 *   layout    device complex [3m] per parent face, or NULL: face_layout of V
 *   fixed_gid device int32 [nfixed] held local vertices (boundary loops)
 *   z         device complex [sum_n] embeddings, updated in place
 *   info      host int32 [4*ncomp]: flips before, iterations, cleared, flips after
 *   flipped   device uint8 [m] (optional): parent faces of the listed
 *             submeshes still folded at the end
 * Synchronises. PGCP_E_SOLVE on a degenerate embedded triangle or a failed
 * solve ("singular linear Beltrami system during repair"). */
PGCP_API int pgcp_batch_qc_repair(pgcp_batch* b, const int32_t* comps, int32_t ncomp, const double* layout,
                                  const int32_t* fixed_gid, int64_t nfixed, int32_t max_iter, double cap,
                                  const pgcp_solve_opts* opts, double* z, int32_t* info, uint8_t* flipped,
                                  void* stream);

/* -------------------------------------------------------------------------
 * Boundary welding (welding.py:512-842), device resident.
 *
 * A map log is an array of records (welding.py:236-509):
 *   kind 0 Mobius       p[0..7] = a, b, c, d; flags bit0 = axis; bits 8..15 =
 *                       number of pins; pin k: p[8+4k..11+4k] = (z, w), side in
 *                       flags bits 16+8k..23+8k (int8)
 *   kind 1 SqrtRatio    p[0..3] = z0, z1; flags low byte = branch (int8)
 *   kind 2 Open         p[0..1] = xi, p[2..3] = Re/|xi|^2, Im/|xi|^2; branch
 *   kind 3 Close        p[0] = ai, p[1] = bi, p[2] = c, p[3] = d
 *   kind 4 SquareMobius p[0..1] = q (infinity allowed)
 */
typedef struct {
    int32_t kind;
    int32_t flags;
    double p[16];
} pgcp_rec;

/* Whole weld schedule on tracked boundary values (pipeline.py:172-213 and
 * partial_weld / closed_weld, welding.py:640-763). One CTA per weld builds the
 * two logs from the shared arc (phase 1); every other point of the two
 * components replays its side's log (phase 2). Welds on disjoint components
 * run concurrently (schedule levels).
 *   tv      device complex [slots]  tracked values, updated in place
 *   info    host int32 [nsteps*6]   k, closed, na, nb, comp_a, comp_b
 *   src     host int32              slot ids of a_cycle then b_cycle, per step
 *   wb_off  host int64 [nsteps+1];  wb host int32 [2*total] (slot, code):
 *           code bits 0..23 arc position + 1 (0: replay), bit 24 arc from b,
 *           bit 25 / 26 cycle point of a / b, bit 31 replay the b log
 *   out     host f64 [nsteps*8]     seam error, seam residual, area of the
 *           welded a arc, status, nrec_a, nrec_b, level, record offset
 *   recs    host pgcp_rec [recs_cap] (optional) all logs
 * Synchronises. PGCP_E_WELD names the first failing step. */
PGCP_API int pgcp_weld_schedule_run(double* tv, int32_t nsteps, const int32_t* info, const int32_t* src,
                                    const int64_t* wb_off, const int32_t* wb, double hard_tol, double* out,
                                    pgcp_rec* recs, int64_t recs_cap, void* stream);

/* The same in two calls, so that the host-side preparation of a schedule
 * (levels, launch-order descriptors, write-back lists, device buffers and
 * their uploads: ~0.4 ms on cfg 2) can run before the tracked values exist --
 * pipeline.py prepares on the planning thread while the flatten runs.
 *   prepare  arguments as pgcp_weld_schedule_run; uploads on `stream`; the
 *            host arrays may be released when it returns; *handle owns the
 *            device buffers
 *   execute  runs the prepared schedule on tv, once, on `stream` (ordered after
 *            the preparing stream by an event); out / recs as above.
 *            Synchronises.
 *   free     releases the handle (after execute has returned, or unused). */
PGCP_API int pgcp_weld_schedule_prepare(int32_t nsteps, const int32_t* info, const int32_t* src, const int64_t* wb_off,
                                        const int32_t* wb, void* stream, void** handle);
PGCP_API int pgcp_weld_schedule_execute(void* handle, double* tv, double hard_tol, double* out, pgcp_rec* recs,
                                        int64_t recs_cap, void* stream);
PGCP_API void pgcp_weld_schedule_free(void* handle);

/* apply_log: replay nrec host records on device points (in/out) with
 * optional int8 side tags. Synchronises; PGCP_E_WELD on NaN. */
PGCP_API int pgcp_weld_replay(const pgcp_rec* recs, int32_t nrec, double* pts, int8_t* sides, int64_t npts,
                              void* stream);

/* geodesic_to_circle of the polygon tv[src[0..n)] (host src): orientation
 * fix (pipeline.py:218-222), interior point, zip, Cayley, centring.
 *   circ device complex [n] (per src entry); recs host [cap];
 *   meta host f64 [8]: nrec, err, idx, aux, circle error, interior. */
PGCP_API int pgcp_weld_geodesic(const double* tv, const int32_t* src, int32_t n, const double* interior,
                                double* circ, pgcp_rec* recs, int32_t cap, double* meta, void* stream);

/* intermediate_form (welding.py:578-602): zip points 0..k of the n device
 * points (in place) onto the imaginary half-axis of `branch` (+1: +i,
 * -1: -i), then send point 0 to infinity. sides device int8 [n] (out);
 * recs host [cap >= k + 1], *nrec_out records. PGCP_E_WELD with the
 * reference's message on a failed zip. Synchronises. */
PGCP_API int pgcp_weld_intermediate(double* pts, int8_t* sides, int32_t n, int32_t k, int32_t branch,
                                    pgcp_rec* recs, int32_t cap, int32_t* nrec_out, void* stream);

/* polygon_interior_point of tv[src] (host src), optionally reversed. */
PGCP_API int pgcp_polygon_interior(const double* tv, const int32_t* src, int32_t n, int reverse, double* out,
                                   void* stream);

/* z[idx[i]] = add + 1/(z[idx[i]] - sub): sphere-mode exterior inversion
 * (pipeline.py:254, 263). idx device int32 or NULL. */
PGCP_API int pgcp_inv_shift(double* z, const int32_t* idx, int64_t n, double add_re, double add_im,
                            double sub_re, double sub_im, void* stream);

/* device int64 face indices -> int32 (values outside [0, 2^31) become -1,
 * which pgcp_batch_create reports as "face index out of range"); lets
 * TriMesh upload the reference's int64 faces without a host-side cast */
PGCP_API int pgcp_faces_from_i64(const int64_t* src, int32_t* dst, int64_t count, void* stream);

/* dst[i] = src[idx[i]] / dst[idx[i]] = src[i] for complex arrays */
PGCP_API int pgcp_gather_complex(const double* src, const int32_t* idx, double* dst, int64_t n, void* stream);
PGCP_API int pgcp_scatter_complex(const double* src, const int32_t* idx, double* dst, int64_t n, void* stream);

/* -------------------------------------------------------------------------
 * Stitch and metrics
 */
/* stitch_global (assemble.py:286-337): average the seam copies of every
 * parent vertex in submesh order, seam spread / scale check, sphere finish
 * (stereographic_inverse(conj(z)) normalised), disk circle check, flips.
 *   z       device complex [sum_n] per-submesh embeddings (local order)
 *   mode    0 free, 1 disk, 2 sphere
 *   coords  device complex [n]; sphere device f64 [3n] (mode 2)
 *   prov    device int32 [n]; flip device uint8 [m]
 *   stats   host f64 [8]: seam_max, scale, circle dev, flips, status
 * Synchronises; PGCP_E_SOLVE on a failed check. */
PGCP_API int pgcp_batch_stitch(pgcp_batch* b, const double* z, int mode, double hard_tol, double circle_tol,
                               double* coords, double* sphere, int32_t* prov, uint8_t* flip, double* stats,
                               void* stream);

/* Sharded form (one rank of a multi-GPU run, dist.py): flips are counted
 * only over faces with face_mask[f] != 0 (this rank's submeshes); NULL mask =
 * every face. */
PGCP_API int pgcp_batch_stitch_ex(pgcp_batch* b, const double* z, int mode, double hard_tol, double circle_tol,
                                  const uint8_t* face_mask, double* coords, double* sphere, int32_t* prov,
                                  uint8_t* flip, double* stats, void* stream);

/* One rank's share of a batch (dist.py): face_mask (device uint8 [m]) = 1
 * on the faces of the listed submeshes; own_vertices (device int32 [n]
 * capacity) = the parent vertices with a copy in one of them, ascending;
 * *n_own their count. Synchronises. */
PGCP_API int pgcp_batch_shard_maps(pgcp_batch* b, const int32_t* comps, int32_t ncomp, uint8_t* face_mask,
                                   int32_t* own_vertices, int64_t* n_own, void* stream);

/* Caller-supplied reduction over the ranks of a sharded run: combine
 * `count` elements of the device buffer `buf` (dtype PGCP_RED_F64 / U32 /
 * U64, op PGCP_RED_SUM / MAX) in place across ranks, ordered on `stream`
 * (e.g. an NCCL all-reduce issued from Python). Returns 0 on success. */
#define PGCP_RED_F64 0
#define PGCP_RED_U32 1
#define PGCP_RED_U64 2
#define PGCP_RED_SUM 0
#define PGCP_RED_MAX 1
typedef int (*pgcp_reduce_fn)(void* buf, int64_t count, int dtype, int op, void* user, void* stream);

/* distortion_report (metrics.py:31-176): per-corner angular distortion,
 * per-face area log ratio, their summaries (mean, population sd, median,
 * IQR with numpy's linear interpolation on exact order statistics), and the
 * 0.1-degree histogram of |d|.
 *   coords  device complex [n] (planar) or f64 [3n] (mode_sphere = 1)
 *   d       device f64 [3m]; valid device uint8 [3m]
 *   summary host f64 [PGCP_SUMMARY_COUNT] (see metrics.cu)
 *   hist    host uint64 [hist_cap] (skipped if too small). Synchronises. */
#define PGCP_SUMMARY_COUNT 16
PGCP_API int pgcp_distortion(const double* V, const int32_t* F, int64_t n, int64_t m, const double* coords,
                             int mode_sphere, double* d, uint8_t* valid, double* summary, uint64_t* hist,
                             int64_t hist_cap, void* stream);
/* Sharded distortion_report: this rank measures the faces with
 * face_mask[f] != 0; every sum, radix-select histogram (8-bit digits) and
 * histogram count goes through `reduce`, so all ranks return the summary of
 * the whole mesh. summary[14] = bytes passed to `reduce`. */
PGCP_API int pgcp_distortion_ex(const double* V, const int32_t* F, int64_t n, int64_t m, const double* coords,
                                int mode_sphere, const uint8_t* face_mask, pgcp_reduce_fn reduce, void* user,
                                double* d, uint8_t* valid, double* summary, uint64_t* hist, int64_t hist_cap,
                                void* stream);

/* corner_angles / corner_angles_sphere (metrics.py:31-58): per-corner angle
 * and degeneracy flag of every face.
 *   points  device: kind 0 complex [n], 1 f64 [2n], 2 f64 [3n], 3 unit-sphere f64 [3n]
 *           (edges projected on the corner's tangent plane)
 *   ang     device f64 [3m]; bad device uint8 [3m] (a zero-length edge) */
PGCP_API int pgcp_corner_angles(const double* points, int kind, const int32_t* F, int64_t m, double* ang,
                                uint8_t* bad, void* stream);

/* area_distortion (metrics.py:89-104): per face the log of the ratio of the
 * normalised parametric and original areas; zero-area faces invalid (d = 0).
 *   coords device complex [n] or f64 [3n] (mode_sphere); d f64 [m]; valid uint8 [m] */
PGCP_API int pgcp_area_distortion(const double* V, const int32_t* F, int64_t n, int64_t m, const double* coords,
                                  int mode_sphere, double* d, uint8_t* valid, void* stream);

/* Measurement kernel (bench.py): stream buf[0, bytes) `reps` times with
 * L2-only 16-byte loads; bytes x reps / time = attainable L2 read bandwidth. */
PGCP_API int pgcp_l2_probe(const void* buf, int64_t bytes, int32_t reps, unsigned long long* sink, void* stream);

/* Measurement kernel (bench.py): FP64 FMA throughput, 8 independent chains
 * per thread over `iters` steps; flops = 16 x iters x *threads_out. */
PGCP_API int pgcp_fp64_probe(int32_t iters, double* sink, int64_t* threads_out, void* stream);

/* host-side weld-schedule planner (partition.py:236-324): see planner.cpp */
PGCP_API int pgcp_plan_weld_schedule(const int64_t* cyc, const int64_t* cyc_off, int32_t K,
                            const int64_t* cuts, int64_t ncuts, int mode_sphere,
                            const int32_t* pairs, int32_t npairs,
                            int64_t* out_meta, int64_t* out_idx, int64_t out_cap,
                            int64_t* out_len);

#ifdef __cplusplus
}
#endif
#endif /* PGCP_B200_H */
