// direct.cuh -- batched multifrontal Cholesky of the per-subdomain systems
// (see direct.cu). Internal interface between pcg.cu's SolveSystem and the
// direct solver; not part of the C ABI.
#pragma once

#include <vector>

#include "batch.cuh"

namespace pgcp {

// the Jacobi-scaled system of a solve, as pcg.cu builds it (rows in unknown
// order within every slot, no coarse reordering)
struct DirectInput {
    int32_t nslot = 0;
    const int32_t* comps = nullptr;   // device: slot -> submesh
    const int64_t* sv_off = nullptr;  // device: slot -> first compact vertex
    const int64_t* sl_off = nullptr;  // device: slot -> first slice
    std::vector<int64_t> h_sl_off;    // host copies
    std::vector<int64_t> h_nu;        // unknowns per slot
    const int32_t* rowsrc = nullptr;  // row -> compact vertex (-1: padding)
    const int64_t* sl_ptr = nullptr;  // paired sliced ELL (off-diagonals, unit diagonal implied)
    int64_t nnz_ell = 0;              // stored ELL entries (padding included)
    const int32_t* col = nullptr;
    const double* val = nullptr;
    const uint32_t* sl_mask = nullptr;  // coupling rows (DNCP)
    const int2* cpl = nullptr;
    const double2* cplc = nullptr;
    bool cplx = false;                // complex Hermitian (DNCP coupling) vs real symmetric
    const uint8_t* onloop = nullptr;  // per row: boundary-loop vertex (DNCP: order the loop last)
};

struct DirectFactor;

// internal status: a front outgrew the kernels' bounds (the caller solves
// with PCG instead); never returned through the C ABI
constexpr int DIRECT_FALLBACK = 100;

// nested dissection, symbolic analysis and numeric factorization (PGCP_OK,
// a CUDA error, or DIRECT_FALLBACK); per-slot nonpositive pivots are
// reported through direct_slot_status
int direct_factor(pgcp_batch* b, const DirectInput& in, DirectFactor** out, cudaStream_t s);
// x (rows) = A^-1 b (rows), Jacobi-scaled space; padding rows get 0
int direct_solve(DirectFactor* F, const double2* b_rows, double2* x_rows, cudaStream_t s);
void direct_free(DirectFactor* F);
// boundary-last DNCP factor: its interior block is the Dirichlet system's factor
bool direct_is_boundary_last(const DirectFactor* F);
// x_h = L_II^-1 b_h with that interior block (h2f: Dirichlet row -> DNCP row)
int direct_solve_interior(DirectFactor* F, const int32_t* h2f, int64_t rows_h, const double2* b_h, double2* x_h,
                          cudaStream_t s);
// last factorization: [nodes, levels, max front, real FMAs of the factorization,
// factor ms (ordering + symbolic + numeric), last solve ms, front storage
// bytes, unknowns, numeric-phase ms]
void direct_stats(const DirectFactor* F, double* out9);
// per-slot pivot failure flags of the last factorization (host copy)
const std::vector<int32_t>& direct_slot_status(const DirectFactor* F);

}  // namespace pgcp
