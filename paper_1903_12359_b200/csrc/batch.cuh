// batch.cuh -- the device-resident batch of submeshes behind pgcp_batch.
//
// HBM layout (all arrays concatenated over submeshes, offsets in int64):
//   parent      V[n*3] f64, F[m*3] i32 (copies owned by the batch)
//   topology    inc_off[n+1], inc[3m]      vertex -> incident faces, sorted
//               twin[3m]                   half-edge 3f+c -> opposite half-edge or -1
//               he_cut[3m]                 half-edge lies on a cut edge
//               face_comp[m]               submesh of every parent face
//   local       vert_off[K+1], vmap[sum_n] submesh-local vertices (sorted parent ids)
//   vertices    lv_off[n+1], lv_gid[...]   parent vertex -> its local-vertex ids
//   loops       loop_off[K+1], loop[sum_nb] (local indices, from the smallest
//               boundary vertex, surface on the left); nxt[sum_n]
//   Laplacian   w3[3m] half-cot per corner; row_ptr[sum_n+1] (i64), col (local
//               i32), val f64 -- canonical CSR rows of every submesh
#pragma once

#include "common.cuh"

struct pgcp_batch {
    int device = 0;
    int64_t n = 0, m = 0;
    int32_t K = 0;
    int64_t sum_n = 0, sum_nb = 0, nnz = 0;
    int64_t parent_chi = 0, parent_loops = 0, bad_comp = -1;
    bool has_laplacian = false;
    bool has_topology = false;  // incidence and twins built (validation passed)

    pgcp::DevBuf<double> V;
    pgcp::DevBuf<int32_t> F;
    pgcp::DevBuf<int64_t> inc_off, lv_off;
    pgcp::DevBuf<int32_t> inc, twin, face_comp;
    pgcp::DevBuf<uint8_t> he_cut;
    pgcp::DevBuf<int64_t> vert_off, loop_off;
    pgcp::DevBuf<int32_t> vmap, lv_comp, lv_gid, loop, nxt, comp_of_gid;
    std::vector<int32_t> h_comp_chi, h_comp_loops;
    pgcp::DevBuf<int32_t> pins;
    pgcp::DevBuf<int32_t> cyc;  // boundary cycles in parent ids (loop order)
    pgcp::DevBuf<double> w3;
    pgcp::DevBuf<int64_t> row_ptr;
    pgcp::DevBuf<int32_t> col;
    pgcp::DevBuf<double> val;

    std::vector<int64_t> h_vert_off, h_loop_off;

    // last DNCP (0) and harmonic (1) solver systems (pcg.cu SolveSystem)
    void* sys[2] = {nullptr, nullptr};
    std::vector<int32_t> last_flat_pins;  // 2 local pins per solved slot
};

namespace pgcp {
// topology.cu
int build_partition(pgcp_batch* b, const int64_t* cuts, int64_t ncuts, bool no_cuts, cudaStream_t s);
int build_topology(pgcp_batch* b, cudaStream_t s);
int build_components(pgcp_batch* b, const int64_t* cuts, int64_t ncuts, bool no_cuts, cudaStream_t s);
int local_faces(pgcp_batch* b, int64_t* face_off, int32_t* faces, cudaStream_t s);
// laplace.cu
int build_laplacian(pgcp_batch* b, int64_t* clamped, cudaStream_t s);
int default_pins(pgcp_batch* b, cudaStream_t s);
int conformal_energy(pgcp_batch* b, const double* z, double* energy, cudaStream_t s);
// pcg.cu
int solve_flatten(pgcp_batch* b, const int32_t* comps, int32_t ncomp, const int32_t* pins,
                  const double* targets, const pgcp_solve_opts* o, double* z, pgcp_solve_stat* st,
                  cudaStream_t s);
int prepare_harmonic(pgcp_batch* b, const int32_t* comps, int32_t ncomp, const int32_t* fixed_gid, int64_t nfixed,
                     const pgcp_solve_opts* o, cudaStream_t s);
int finish_harmonic(pgcp_batch* b, const double* fixed_val, int64_t nfixed, const pgcp_solve_opts* o, double* z,
                    pgcp_solve_stat* st, cudaStream_t s);
int solve_harmonic(pgcp_batch* b, const int32_t* comps, int32_t ncomp, const int32_t* fixed_gid,
                   const double* fixed_val, int64_t nfixed, const pgcp_solve_opts* o, double* z,
                   pgcp_solve_stat* st, cudaStream_t s);
int solve_values(pgcp_batch* b, const int32_t* comps, int32_t ncomp, const double* vals, const int32_t* fixed_gid,
                 const double* fixed_val, int64_t nfixed, const pgcp_solve_opts* o, double* z, pgcp_solve_stat* st,
                 cudaStream_t s);
void free_system(void* p);
void solve_summary(const pgcp_batch* b, int which, double* out8);
unsigned long long launch_count();
int export_system(pgcp_batch* b, int which, int32_t comp, int64_t* dims, int32_t* indptr,
                  int32_t* indices, double* data, double* rhs, cudaStream_t s);
// repair.cu
int face_layout(const double* V, const int32_t* F, int64_t m, double* out, cudaStream_t s);
int beltrami_per_face(const double* src, const int32_t* sf, const double* tgt, const int32_t* tf, int64_t m,
                      double* mu, int64_t* first_degenerate, cudaStream_t s);
int lbs_stiffness(pgcp_batch* b, const double* z, const double* mu, double* kval, cudaStream_t s);
int qc_repair(pgcp_batch* b, const int32_t* comps, int32_t ncomp, const double* layout, const int32_t* fixed_gid,
              int64_t nfixed, int32_t max_iter, double cap, const pgcp_solve_opts* o, double* z, int32_t* info,
              uint8_t* flipped, cudaStream_t s);
// metrics.cu
int stitch(pgcp_batch* b, const double* z, double* coords, double* stats, cudaStream_t s);
}  // namespace pgcp
