/* hodg_b200 -- C ABI of the B200 (sm_100a) DG Euler residual library.
 *
 * Drop-in boundary for the reference's hot path (arXiv 2209.01877, package
 * `hodg`).  Each entry point replaces one piece of the reference's kernel
 * seam, cited below:
 *
 *   hodg_face_flux      <- _KERNELS[dtype].flux_pass     hodg/dg.py:240-351
 *                          (wrapper face_flux_pass       hodg/dg.py:594-621)
 *   hodg_elem_stage     <- _KERNELS[dtype].rhs_pass      hodg/dg.py:353-460
 *                          fused with _axpy_state / _combine_state
 *                                                        hodg/timestepping.py:165-180
 *                          (wrapper accumulate_rhs       hodg/dg.py:624-649)
 *   hodg_local_dt       <- _dt_pass / local_dt_field     hodg/timestepping.py:105-147
 *   hodg_min_reduce_f64 <- min_reduce                    hodg/timestepping.py:150-162
 *   hodg_residual_l2    <- residual_l2                   hodg/timestepping.py:208-211
 *   hodg_rcm            <- cuthill_mckee / rcm           hodg/renumber.py:171-208
 *   hodg_err_decode     <- _raise_face_error / _raise_cell_error
 *                                                        hodg/dg.py:537-546
 *
 * Conventions (inherited from the reference seam):
 *  - plain pointers and sizes; every buffer is DEVICE memory owned by the
 *    caller; the library never allocates on the hot path;
 *  - calls are asynchronous on the given stream (cudaStream_t passed as
 *    void*); kernels never fail on inadmissible states, they record the
 *    first (smallest) offending face / cell id in a device error word
 *    (uint32[4], reset with hodg_err_reset) that the host reads once per step;
 *  - return value: HODG_OK, HODG_EINVAL (bad argument), HODG_ECUDA (launch
 *    error), HODG_ENODEV (no sm_100 device).
 *
 * Data layout in HBM (N elements, F faces, nb modes, 5 variables):
 *  - state / residual: (N, 5, nb) float64, row stride rs = 5*nb rounded up
 *    to an even count, in the reference-element monomial basis (see
 *    DESIGN.md; hodg_modal_transform converts to/from the reference's
 *    physical Taylor basis);
 *  - face flux buffer: (F, hodg_face_record_stride) at kernel precision,
 *    record = H[v][q] (the reference's FaceFluxBuffer.inviscid,
 *    hodg/dg.py:86-92, transposed) padded to 16 bytes;
 *  - geometry: see hodg_mesh_desc.
 */
#ifndef HODG_B200_H
#define HODG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HODG_OK 0
#define HODG_EINVAL 2
#define HODG_ECUDA 3
#define HODG_ENODEV 4
#define HODG_ETOPOLOGY 5 /* hodg_mesh_setup: non-manifold face / zero-area face / degenerate element */

/* boundary kinds, hodg/physics.py:47-50 */
#define HODG_BC_INTERIOR 0
#define HODG_BC_FAR_FIELD 1
#define HODG_BC_SLIP_WALL 2
#define HODG_BC_NO_SLIP_WALL 3

#define HODG_FLUX_ROE 0
#define HODG_FLUX_LLF 1

/* kernel precision: 64 = FP64 everywhere; 32 = FP32 traces / flux /
 * quadrature with FP64 state, accumulation, mass solve and RK update */
#define HODG_PREC_F64 64
#define HODG_PREC_MIXED 32

/* element geometry record, 16 doubles per element, stored tile-major (see
 * hodg_elem_tile): fields Jinv[9] row-major, fc[4] = sgn*area/vol, h, vol, pad */
#define HODG_EGEO_FIELDS 16
#define HODG_ECONV_STRIDE 18 /* A = J/h [9], A^-1 [9] (modal transforms) */

typedef struct {
    int64_t n_elems;
    int64_t n_faces;
    int order;        /* 0..3 */
    int flux_kind;    /* HODG_FLUX_ROE | HODG_FLUX_LLF */
    double gamma;
    double qinf[5];   /* far-field state (conserved) */
    const double* egeo;      /* tile-major (ceil(N/T), 16, T), T = hodg_elem_tile(order) */
    const double* econv;     /* (N, 18) */
    const int32_t* efaces;   /* tile-major (ceil(N/T), 4, T): face id of local face s (opposite vertex s) */
    const int32_t* fcells;   /* (F, 2) left, right (-1 at boundary) */
    const int32_t* finfo;    /* (F,) slotL | slotR << 2 | bc << 4 */
    const double* fnrm;      /* (F, 4) unit normal left->right, pad */
} hodg_mesh_desc;

typedef struct hodg_mesh hodg_mesh;

/* RK stage: out = a*u0 + b*(us + dt*R(us))       (combine = 0)
 *           out = 0.5*((u0 + us) + dt*R(us))      (combine = 1, Heun final stage)
 *           no state update                       (combine = -1, residual only) */
typedef struct {
    const double* us;   /* stage state (N, rs) */
    const double* u0;   /* RK base state, may be NULL when combine == 0 and a == 0 */
    double* out;        /* new state; may alias us (never u0 unless u0 == us is dead) */
    double* res;        /* residual dU/dt (N, rs), NULL to skip */
    double a, b;
    int combine;
    int dt_is_vector;        /* dt: device scalar (0) or per-element vector (1) */
    const double* dt;
    double* norm_partial;    /* (n_blocks, 5) partial sums of vol*res_0^2, NULL to skip */
    unsigned long long* dt_next;   /* atomic min of the new state's CFL dt (double bits), NULL to skip */
    double* dt_vec_out;      /* per-element CFL dt of the new state, NULL to skip */
    unsigned long long* dt_reset;  /* set to +inf by this launch (another step's dt slot), NULL to skip */
    double cfl;
    float* out32;            /* mixed precision: FP32 shadow of out (row stride hodg_state32_row_stride), NULL to skip */
} hodg_stage_args;

int hodg_version(void);
int hodg_device_ok(void);
int hodg_mesh_create(const hodg_mesh_desc* desc, hodg_mesh** out);
int hodg_mesh_destroy(hodg_mesh* mesh);
int hodg_state_row_stride(int order);  /* rs */
int hodg_n_basis(int order);
int hodg_n_face_points(int order);
int hodg_n_vol_points(int order);
/* elements per element-kernel tile: egeo / efaces are stored tile-major,
 * egeo[(e / T) * 16 T + field * T + e % T], efaces[(e / T) * 4 T + s * T + e % T],
 * padded to whole tiles */
int hodg_elem_tile(int order);
/* per-face record stride (values of the kernel precision) of the face flux
 * buffer: 5 x nqf values H[v][q] padded to 16 bytes */
int hodg_face_record_stride(int order, int prec);
int64_t hodg_stage_blocks(const hodg_mesh* mesh, int prec); /* rows of norm_partial */

int hodg_face_flux(const hodg_mesh* mesh, int prec, const double* state, void* face_buf, uint32_t* err,
                   void* stream);
/* faces [f_begin, f_end) only: lets a partitioned run evaluate interior
 * faces while the halo exchange is in flight, then the partition faces.
 * interior_only = 1 promises every face in the range has a right element
 * and selects the kernel variant without the boundary-state code. */
int hodg_face_flux_range(const hodg_mesh* mesh, int prec, const double* state, void* face_buf, int64_t f_begin,
                         int64_t f_end, int interior_only, uint32_t* err, void* stream);
int hodg_elem_stage(const hodg_mesh* mesh, int prec, const void* face_buf, const hodg_stage_args* args,
                    uint32_t* err, void* stream);

/* Element-slot record layout (the stepper's fused path; same values as
 * face_buf, different placement): block e holds the records of element e's
 * four faces, slot-major, 5 x NQF values each ([slot][var][qp]), at stride
 * hodg_elem_record_stride(order) = 20 NQF + 1 values for the CTA element
 * kernel (odd: conflict-free per-element smem reads) or 20 NQF + 2 for the
 * warp-group kernel (P1, and P2 when built with it); a tile of
 * hodg_elem_tile(order) blocks is a 16-byte multiple at either precision,
 * fetched with one TMA bulk copy.  The face kernel stores each
 * face's record into the blocks of both neighbours (owned elements only:
 * id < n_elems), so the element kernel needs no per-face gather.  Buffer:
 * hodg_elem_record_len(mesh, prec) values at the kernel precision. */
int hodg_elem_record_stride(int order);
int64_t hodg_elem_record_len(const hodg_mesh* mesh, int prec);
int hodg_face_flux_range_es(const hodg_mesh* mesh, int prec, const double* state, void* elem_buf, int64_t f_begin,
                            int64_t f_end, int interior_only, uint32_t* err, void* stream);
int hodg_elem_stage_es(const hodg_mesh* mesh, int prec, const void* elem_buf, const hodg_stage_args* args,
                       uint32_t* err, void* stream);
/* Mixed precision: an FP32 shadow of the stage state -- rows of
 * hodg_state32_row_stride(order) floats (16-byte rows), written by the element
 * kernel next to the FP64 state (hodg_stage_args.out32) -- that the face
 * kernel reads instead of converting each FP64 row at every (face, side).
 * The traces are bitwise those of the FP64-row mixed kernel (the same
 * FP64 -> FP32 rounding, done once per row).  No reference counterpart:
 * the reference's mixed mode stores the whole state in FP32
 * (hodg/precision.py:105-110). */
int hodg_state32_row_stride(int order);
int hodg_state_to_f32(const hodg_mesh* mesh, const double* rows, int64_t n_rows, float* rows32, void* stream);
int hodg_face_flux_range32(const hodg_mesh* mesh, const float* state32, void* face_buf, int64_t f_begin,
                           int64_t f_end, int interior_only, uint32_t* err, void* stream);
int hodg_face_flux_range32_es(const hodg_mesh* mesh, const float* state32, void* elem_buf, int64_t f_begin,
                              int64_t f_end, int interior_only, uint32_t* err, void* stream);
int hodg_local_dt(const hodg_mesh* mesh, const double* state, double cfl, double* dt_vec_out,
                  unsigned long long* dt_min, uint32_t* err, void* stream);
int hodg_norm_finalize(const double* partial, int64_t n_blocks, double* out5, void* stream);
/* Diagnostics (no reference counterpart): the last CUDA runtime / driver
 * error code a kernel launcher saw, and where (*site: 1 shared-memory
 * attribute, 2 tensor-map encode, 3 launch, 4 error after the launch). */
int hodg_last_error(int* site);
int hodg_residual_l2(const hodg_mesh* mesh, const double* res, double* scratch, double* out5, void* stream);
int hodg_min_reduce_f64(const double* x, int64_t n, double* scratch, double* out, void* stream);
int hodg_dt_fill(unsigned long long* slot, double value, void* stream);
int hodg_modal_transform(const hodg_mesh* mesh, int to_reference, const double* in, double* out, void* stream);
int hodg_err_reset(uint32_t* err, void* stream);
/* decode a host copy of the error word: returns 0 (ok), 1 face, 2 volume cell, 3 cell mean; *id = first id */
int hodg_err_decode(const uint32_t* err_host, int64_t* id);

/* Device Reverse Cuthill-McKee (bit-exact with hodg/renumber.py:171-208).
 * indptr (n+1), indices (2E) int64 CSR, neighbour lists ascending (as
 * AdjacencyGraph.from_edges builds them).  forward[old] = new,
 * inverse[new] = old.  work: caller-provided device scratch of
 * hodg_rcm_work_bytes(n, nnz) bytes. */
int64_t hodg_rcm_work_bytes(int64_t n, int64_t nnz);
int hodg_rcm(int64_t n, const int64_t* indptr, const int64_t* indices, int64_t* forward, int64_t* inverse,
             void* work, void* stream);

/* Device mesh setup (csrc/setup.cu): connectivity
 * by sorted face keys and the per-face / per-element geometry of
 * paper_2209_01877_b200/mesh.py:build_tet_mesh on the GPU, same numbering
 * (face id = rank of its first traversal, element-major slot order; the
 * first traverser is the left element; slot f is the face opposite sorted
 * vertex f).  Inputs (device): X (n_nodes, 3) float64, tets (n_elems, 4)
 * int32 with each row ascending.  Outputs (device, sized for the upper bound
 * F <= 4 n_elems): face_cells (F,2), face_slots (F,2) int8, face_nodes (F,3),
 * face_normal (F,3), face_area (F,), cell_faces / cell_fsign /
 * cell_neighbors (n,4), cell_volume (n,), cell_centroid (n,3), cell_h (n,);
 * *n_faces_out = F.  Synchronous (reads F back).  HODG_ETOPOLOGY with
 * *n_faces_out = -1 non-manifold, -2 zero-area face, -3 degenerate element.
 * Limits: n_nodes < 2^21 (64-bit packed key), 4 n_elems < 2^31. */
int64_t hodg_mesh_setup_work_bytes(int64_t n_elems);
int hodg_mesh_setup(int64_t n_nodes, int64_t n_elems, const double* X, const int32_t* tets, int32_t* face_cells,
                    int8_t* face_slots, int32_t* face_nodes, double* face_normal, double* face_area,
                    int32_t* cell_faces, int8_t* cell_fsign, int32_t* cell_neighbors, double* cell_volume,
                    double* cell_centroid, double* cell_h, int64_t* n_faces_out, void* work, void* stream);

/* Element geometry records on the GPU (the device
 * twin of paper_2209_01877_b200/geometry.py:compute_geometry, which replaces
 * the reference's per-cell tables, hodg/geometry.py:120-220).  Inputs
 * (device): X (n_nodes, 3), tets (n, 4) ascending rows, cell_volume, cell_h
 * (n,), face_area (F,), cell_faces (n, 4), cell_fsign (n, 4) int8 -- the
 * hodg_mesh_setup outputs.  Outputs: egeo tile-major (ceil(n/T), 16, T) with
 * T = hodg_elem_tile(order) (zero padded here), econv (n, 18); flag is one
 * device int32 of scratch.  Synchronous.  HODG_ETOPOLOGY: a degenerate
 * element (zero Jacobian determinant). */
int hodg_element_records(int64_t n_elems, int order, const double* X, const int32_t* tets, const double* cell_volume,
                         const double* cell_h, const double* face_area, const int32_t* cell_faces,
                         const int8_t* cell_fsign, double* egeo, double* econv, int32_t* flag, void* stream);

/* Multi-GPU plumbing (csrc/halo.cu).
 *
 * hodg_partition_rcb: host function.  Part id per point by recursive
 * coordinate bisection of (n, 3) float64 points: split along the first axis
 * of maximal extent, order by (coordinate, index), the first child takes
 * (size * floor(k/2)) / k points.  Bit-exact with
 * paper_2209_01877_b200/partition.py:rcb_partition and oracle/partition.py
 * (the reference is single-node; METIS-free by design).
 *
 * hodg_halo_*: the per-stage ghost-row exchange over NCCL point-to-point.
 * hodg_halo_unique_id fills a 128-byte ncclUniqueId on one rank (the caller
 * broadcasts it); hodg_halo_create is collective over the ranks: it builds
 * the NCCL communicator and uploads the plan -- per peer, the local rows to
 * send (concatenated in peer order, host or device int32) and the first
 * local ghost row / count to receive.  hodg_halo_exchange packs the send
 * rows (one kernel) and posts the grouped sends and receives on `stream`;
 * ghost rows land directly in `state` ((rows, rs) float64, device).  NCCL is
 * taken from the process's libnccl.so.2 at run time. */
int hodg_partition_rcb(int64_t n, const double* points, int nparts, int32_t* part);
typedef struct hodg_halo hodg_halo;
int hodg_halo_unique_id(void* id128);
int hodg_halo_create(int nranks, int rank, const void* id128, int npeers, const int32_t* peers,
                     const int64_t* send_count, const int32_t* send_rows, const int64_t* recv_first,
                     const int64_t* recv_count, int rs, hodg_halo** out);
int hodg_halo_exchange(hodg_halo* halo, double* state, void* stream);
/* in-place all-reduce on the halo's communicator (stream-ordered, so a
 * distributed step captures into one CUDA graph): kind 0 = int64 MIN (the dt
 * slot, positive doubles as bit patterns: exact), kind 1 = float64 SUM. */
int hodg_halo_allreduce(hodg_halo* halo, void* buf, int64_t count, int kind, void* stream);
int hodg_halo_destroy(hodg_halo* halo);

/* 2D table-driven path: the reference's own discretisation (triangles and
 * bilinear quads, 4 variables, per-cell quadrature tables of
 * hodg/geometry.py:120-220) with the argument lists of the reference kernels
 * (device pointers; arrays at the kernel precision `prec` unless typed):
 *   hodg2d_flux_pass  <- flux_pass (Euler)     hodg/dg.py:240-351
 *   hodg2d_rhs_pass   <- rhs_pass (Euler)      hodg/dg.py:353-460
 *   hodg2d_dt_pass    <- _dt_pass              hodg/timestepping.py:105-134
 *   hodg2d_axpy       <- _axpy_state           hodg/timestepping.py:165-171
 *   hodg2d_combine    <- _combine_state        hodg/timestepping.py:174-180
 * and the viscous (ivis = 1, BR1) kernels of the same table:
 *   hodg2d_qhat_pass     <- qhat_pass            hodg/dg.py:114-162
 *   hodg2d_aux_pass      <- aux_pass             hodg/dg.py:164-238
 *   hodg2d_flux_pass_ns  <- flux_pass, ivis = 1  hodg/dg.py:240-351
 *   hodg2d_rhs_pass_ns   <- rhs_pass, ivis = 1   hodg/dg.py:353-460
 * (aux is (n_cells, 2, 4, nb) at the state precision, minv of aux_pass too;
 * the reference's scratch arrays live in registers).
 * Error flags are the reference's uint8 per-face / per-cell arrays. */
int hodg2d_flux_pass(int prec, int64_t n_faces, int nqf, int nb, const void* coeffs, const void* fbL, const void* fbR,
                     const int32_t* face_cells, const int8_t* bc_code, const void* fnx, const void* fny,
                     const void* qinf, double gamma, int flux_kind, void* finv, uint8_t* errf, void* stream);
int hodg2d_rhs_pass(int prec, int64_t n_cells, int nb, int nqv, int nqf, int maxf, const void* coeffs,
                    const void* finv, const void* vol_w, const void* vol_basis, const void* vol_gx,
                    const void* vol_gy, const int8_t* cell_nfaces, const int32_t* cell_faces,
                    const int8_t* cell_fsign, const void* face_w, const void* fbL, const void* fbR,
                    const double* minv64, double gamma, double* res, uint8_t* errc, void* stream);
int hodg2d_qhat_pass(int prec, int64_t n_faces, int nqf, int nb, const void* coeffs, const void* fbL, const void* fbR,
                     const int32_t* face_cells, const int8_t* bc_code, const void* fnx, const void* fny,
                     const void* qinf, double gamma, void* qhat, uint8_t* errf, void* stream);
int hodg2d_aux_pass(int prec, int64_t n_cells, int nb, int nqv, int nqf, int maxf, const void* coeffs,
                    const void* qhat, const void* vol_w, const void* vol_basis, const void* vol_gx,
                    const void* vol_gy, const int8_t* cell_nfaces, const int32_t* cell_faces,
                    const int8_t* cell_fsign, const void* face_w, const void* fbL, const void* fbR, const void* fnx,
                    const void* fny, const void* minv, void* aux, void* stream);
int hodg2d_flux_pass_ns(int prec, int64_t n_faces, int nqf, int nb, const void* coeffs, const void* aux,
                        const void* fbL, const void* fbR, const int32_t* face_cells, const int8_t* bc_code,
                        const void* fnx, const void* fny, const void* qinf, double gamma, double Rgas, double mu,
                        double Pr, void* finv, void* fvis, void* fqhat, uint8_t* errf, void* stream);
int hodg2d_rhs_pass_ns(int prec, int64_t n_cells, int nb, int nqv, int nqf, int maxf, const void* coeffs,
                       const void* aux, const void* finv, const void* fvis, const void* vol_w, const void* vol_basis,
                       const void* vol_gx, const void* vol_gy, const int8_t* cell_nfaces, const int32_t* cell_faces,
                       const int8_t* cell_fsign, const void* face_w, const void* fbL, const void* fbR,
                       const double* minv64, double gamma, double Rgas, double mu, double Pr, double* res,
                       uint8_t* errc, void* stream);
int hodg2d_dt_pass(int prec, int64_t n_cells, int nb, const void* coeffs, const double* basis_mean, const double* h,
                   double gamma, double mu, double cfl, int order, double* out, uint8_t* errc, void* stream);
int hodg2d_axpy(int prec, int64_t n_cells, int per_cell, const void* u, const double* r, const double* dtc, void* out,
                void* stream);
int hodg2d_combine(int prec, int64_t n_cells, int per_cell, const void* u, const void* u1, const double* r1,
                   const double* dtc, void* out, void* stream);

/* point evaluations of the device interface flux and boundary state
 * (roe_flux / boundary_state, hodg/physics.py:436-479): qL, qR, q (n, 5),
 * normals (n, 3), qf (5); ok[i] = 0 where the reference returns ok = 0 */
int hodg_point_flux(int prec, int64_t n, const void* qL, const void* qR, const void* normals, double gamma,
                    int flux_kind, void* out, uint8_t* ok, void* stream);
int hodg_point_bstate(int prec, int64_t n, int kind, const void* q, const void* normals, const void* qf, double gamma,
                      void* out, void* stream);

/* device face re-sort of apply_permutation (hodg/renumber.py:224-231):
 * order[k] = old id of the k-th face by (min, max) new incident element id
 * then old id; new_lr (F, 2) int64 = new left / right (-1 -> left), work of
 * hodg_face_sort_work_bytes(F) bytes */
int64_t hodg_face_sort_work_bytes(int64_t n_faces);
int hodg_face_sort(int64_t n_faces, int64_t n_cells, const int64_t* new_lr, int64_t* order, void* work, void* stream);

/* number of kernels this library launched since load (for gpu_launches) */
int64_t hodg_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* HODG_B200_H */
