/*
 * qwb200.h — C ABI of the B200 (sm_100a) quantum-walk inner core, libqwb200.so.
 *
 * This is the drop-in boundary that replaces the CPU linear-algebra backend of
 * the reference `qwalk` 0.1.0 (the Neblina-bridge analogue) and
 * the numpy bodies of its operator builders, step loops and reducers.  Every
 * entry point names the reference interface it replaces as
 * `file:line` under /root/reference/pkg/src/qwalk/.
 *
 * Conventions
 *  - Plain C types only: pointers, sizes, doubles.  No torch types.
 *  - All array arguments are DEVICE pointers owned by the caller, unless the
 *    name ends in `_host`.  Complex128 is `qwb_z` = {re, im}, 16 bytes,
 *    layout-identical to numpy/torch complex128.
 *  - Every call is stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 *    default stream).  Calls that return a host scalar synchronise `stream`.
 *  - Return value: QWB_OK (0) or a status code; the message is available from
 *    qwb_last_error().  Status codes map 1:1 onto the reference's exception
 *    classes (errors.py:9-104); see QWB_E_* below.
 *  - Arithmetic contract: results are bitwise equal to the reference's numpy
 *    arithmetic (products `values * x[cols]` with numpy's FMA complex multiply,
 *    row sums with numpy's pairwise `add.reduceat` order, |z| with numpy's SIMD
 *    cabs).  See DESIGN.md §Numerics.
 *  - A context is used by one host thread at a time (mirrors Engine,
 *    backend.py:259-267).
 */
#ifndef QWB200_H
#define QWB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.py class each maps to) ------------------------ */
#define QWB_OK                        0
#define QWB_E_DIMENSION               1   /* DimensionMismatch            errors.py:27  */
#define QWB_E_NONFINITE               2   /* NonFiniteEntry               errors.py:36  */
#define QWB_E_NOT_ON_DEVICE           3   /* NotOnDevice                  errors.py:31  */
#define QWB_E_ENGINE_STOPPED          4   /* EngineStopped                errors.py:23  */
#define QWB_E_ALREADY_STOPPED         5   /* AlreadyStopped               errors.py:19  */
#define QWB_E_UNSUPPORTED             6   /* UnsupportedEngineKind        errors.py:15  */
#define QWB_E_SERIES_NOT_CONVERGED    7   /* SeriesNotConverged           errors.py:80  */
#define QWB_E_MARKED_OUT_OF_RANGE     8   /* MarkedVertexOutOfRange       errors.py:76  */
#define QWB_E_PERSISTENT_SHIFT        9   /* UnsupportedGraphForPersistentShift errors.py:93 */
#define QWB_E_INVALID_ARGUMENT       10   /* ValueError                                  */
#define QWB_E_CUDA                   20   /* CUDA runtime failure (QuantumWalkError)      */
#define QWB_E_NCCL                   21   /* reserved: multi-GPU transport failure        */
#define QWB_E_OUT_OF_MEMORY          22   /* device allocation failed                     */

/* graph families (graphs.py:115-159) */
#define QWB_FAMILY_GENERIC    0
#define QWB_FAMILY_CYCLE      1
#define QWB_FAMILY_LINE       2
#define QWB_FAMILY_GRID       3
#define QWB_FAMILY_HYPERCUBE  4

/* shifts (coined.py:54) */
#define QWB_SHIFT_FLIPFLOP    0
#define QWB_SHIFT_PERSISTENT  1
#define QWB_SHIFT_NONE        2   /* identity: builds the coin C alone (grover_coin) */

typedef struct qwb_ctx qwb_ctx;
typedef struct { double re, im; } qwb_z;

/* ---- engine lifecycle: init_engine / stop_engine (backend.py:291-314) --- */
int         qwb_init(int device, qwb_ctx** out);
int         qwb_shutdown(qwb_ctx* ctx);
const char* qwb_last_error(const qwb_ctx* ctx);   /* ctx may be NULL: thread-local */
const char* qwb_version(void);
int         qwb_device_count(int* count_host);

/* ---- graph builders (graphs.py:115-159, bit-exact int64 CSR) ------------
 * Two-phase: call with col == NULL to fill row_offsets[n+1] and *nnz_host,
 * then again with col sized *nnz_host.  params: cycle/line {n},
 * grid {nx, ny, periodic}, hypercube {dim}.                                  */
int qwb_family_adjacency(qwb_ctx* ctx, int family, const int64_t* params_host,
                         int64_t* row_offsets, int64_t* col, int64_t* nnz_host,
                         void* stream);

/* ---- coined operator builder U = S C with the -I oracle ------------------
 * replaces coined.evolution_operator / grover_coin / apply_marked_policy /
 * _shift_targets (coined.py:164-238) and csr_from_triplets (backend.py:195-236).
 * adj_*: graph adjacency CSR (sorted, int64).  marked: sorted unique vertex ids
 * (device, may be NULL when n_marked == 0).  shift: QWB_SHIFT_*; family/params
 * are needed for the persistent shift only.  Two-phase like above:
 * u_col == NULL -> fill u_row_offsets[n_arcs+1] and *nnz_host.              */
int qwb_coined_operator(qwb_ctx* ctx, int64_t n, const int64_t* adj_offs,
                        const int64_t* adj_col, const int64_t* marked, int64_t n_marked,
                        int shift, int family, const int64_t* params_host,
                        int64_t* u_row_offsets, int32_t* u_col, qwb_z* u_val,
                        int64_t* nnz_host, void* stream);

/* src[r] = k with S e_k = e_r for the shift permutation S (flip-flop: the
 * reverse arc, coined.py:96-101, 222-227; persistent: coined.py:104-146;
 * NONE: identity).  The permutation CSR of flip_flop_shift / persistent_shift
 * is then rows r -> single column src[r].                                    */
int qwb_shift_sources(qwb_ctx* ctx, int64_t n, const int64_t* adj_offs, const int64_t* adj_col,
                      int shift, int family, const int64_t* params_host, int64_t* src,
                      void* stream);

/* ---- Hamiltonian H = -gamma A - sum_M |v><v| (ctqw.py:84-98) -------------
 * h_row_offsets[n+1], h_col/h_val[nnz_adj + n_marked]; marked sorted unique. */
int qwb_hamiltonian(qwb_ctx* ctx, int64_t n, const int64_t* adj_offs, const int64_t* adj_col,
                    double gamma, const int64_t* marked, int64_t n_marked,
                    int64_t* h_row_offsets, int32_t* h_col, qwb_z* h_val, void* stream);

/* ||M||_inf = max_i sum_j |M_ij| with numpy's cabs + pairwise row sums
 * (ctqw.py:112-120).                                                         */
int qwb_inf_norm(qwb_ctx* ctx, int64_t n_rows, const int64_t* row_offsets, const qwb_z* val,
                 double* result_host, void* stream);

/* generic host-assembled CSR upload helper: int64 -> int32 column indices,
 * with the structural checks of CsrMatrix.validate (backend.py:130-147).     */
int qwb_csr_prepare(qwb_ctx* ctx, int64_t n_rows, int64_t n_cols, const int64_t* row_offsets,
                    const int64_t* col64, const qwb_z* val, int64_t nnz, int32_t* col32,
                    void* stream);

/* ---- CSR SpMV y = M x (backend.matvec_mul / _csr_rows, backend.py:394-430) */
int qwb_spmv(qwb_ctx* ctx, int64_t n_rows, const int64_t* row_offsets, const int32_t* col,
             const qwb_z* val, const qwb_z* x, qwb_z* y, void* stream);

/* Repeated SpMV: the coined.simulate loop (coined.py:263-272).  Writes
 * snapshots U^{k_j} psi0 for the non-decreasing step counts k_host[0..n_snap)
 * into snaps[j * n_rows ...].  Small operators run the whole loop in one
 * persistent CTA with the state in shared memory.  scratch: 2*n_rows + 1 qwb_z
 * (the second vector starts at an even offset).  Any pointer alignment is
 * accepted; 32-B aligned val / scratch take the 256-bit load path. */
int qwb_csr_run(qwb_ctx* ctx, int64_t n_rows, const int64_t* row_offsets, const int32_t* col,
                const qwb_z* val, const qwb_z* psi0, const int64_t* k_host, int64_t n_snap,
                qwb_z* snaps, qwb_z* scratch, void* stream);

/* ---- matrix-free periodic lattice (nx, ny >= 3), flip-flop or persistent --
 * Internal state layout: four direction planes [D, L, R, U] of nx*ny qwb_z
 * each ("planes").  Conversions to/from the reference arc order are exact
 * permutations.  marked_bits: bitmap over vertices (NULL = none).           */
/* marked-vertex bitmap bits[(n+31)/32] from a device list (range-checked:
 * QWB_E_MARKED_OUT_OF_RANGE, coined.py:79-81 / ctqw.py:79-81).               */
int qwb_marked_bitmap(qwb_ctx* ctx, int64_t n, const int64_t* marked, int64_t n_marked,
                      uint32_t* bits, void* stream);
int qwb_lattice_to_planes(qwb_ctx* ctx, int64_t nx, int64_t ny, const qwb_z* arcs, qwb_z* planes,
                          void* stream);
int qwb_lattice_from_planes(qwb_ctx* ctx, int64_t nx, int64_t ny, const qwb_z* planes, qwb_z* arcs,
                            void* stream);
/* Run `steps` coined steps ping-ponging between a (input) and b.  On return
 * *final_in_b_host says where the result is.  The marked set is passed both as
 * the device bitmap and as the sorted host list (marked_host[n_marked]).  On
 * lattices >= 64 x 64, T = 4 steps are fused per HBM pass (temporally blocked
 * tile kernel, lattice_tb.cu; remainder steps one at a time).  If trace !=
 * NULL, trace[s*n_trace+j] (n_trace <= 8) receives p(trace_vertices_host[j])
 * of the state BEFORE step s (s < steps), fused into the step kernels
 * (coined.probability_distribution semantics).                               */
int qwb_lattice_run(qwb_ctx* ctx, int64_t nx, int64_t ny, int shift, const uint32_t* marked_bits,
                    const int64_t* marked_host, int64_t n_marked, qwb_z* a, qwb_z* b, int64_t steps,
                    const int64_t* trace_vertices_host, int n_trace, double* trace,
                    int* final_in_b_host, void* stream);
/* Coined steps fused per HBM pass by qwb_lattice_run for this lattice (0 =
 * one step per launch) and how an untraced run launches it (2 = one
 * persistent dataflow launch for the whole run, 1 = one tile launch per T
 * steps).  Environment overrides: QWB_LATTICE_T, QWB_LATTICE_SHAPE,
 * QWB_LATTICE_FLOW.                                                          */
int qwb_lattice_fused_depth(int64_t nx, int64_t ny, int64_t n_marked, int* depth_host, int* kind_host);
/* One step with an optional fused full distribution p of the INPUT state.    */
int qwb_lattice_step(qwb_ctx* ctx, int64_t nx, int64_t ny, int shift, const uint32_t* marked_bits,
                     const qwb_z* in, qwb_z* out, double* prob_in, void* stream);
/* p[v] of a planes state (coined.py:275-294).                                */
int qwb_lattice_probability(qwb_ctx* ctx, int64_t nx, int64_t ny, const qwb_z* planes, double* p,
                            void* stream);

/* ---- multi-GPU: y-slabs of one periodic lattice, NCCL halo exchange -------
 * (no reference counterpart: its only parallelism is the in-process row-block
 * pool, backend.py:426-430; multi-GPU is future work in PAPER.md:499-501).
 * A rank owns global rows [y0, y0+ny_local) (ny_local >= 2) of an nx x ny
 * torus; its planes buffers hold 4 x nx x (ny_local + 2) qwb_z (one extra row
 * each side).  Arc arrays passed to the slab conversions hold only the owned
 * rows' arcs, i.e. the contiguous range [4*nx*y0, 4*nx*(y0+ny_local)) of the
 * reference arc order.  Results are bitwise equal to the single-GPU run.     */
int qwb_slab_to_planes(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local,
                       const qwb_z* arcs, qwb_z* planes, void* stream);
int qwb_slab_from_planes(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local,
                         const qwb_z* planes, qwb_z* arcs, void* stream);
int qwb_slab_probability(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local,
                         const qwb_z* planes, double* p, void* stream);
/* one step without exchange; part 0 = all owned rows, 1 = first+last, 2 = interior */
int qwb_slab_step(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local, int shift,
                  const uint32_t* marked_bits, const qwb_z* in, qwb_z* out, int part, void* stream);
/* Fused (temporally blocked) slabs: G = qwb_slab_ghost_rows(...) ghost rows
 * each side, G = m T with T = qwb_slab_depth() (6), m = QWB_SLAB_GHOST_MULT (4 while
 * G <= 32) and G <= the thinnest slab; 0: not available, use the 1-extra-row functions
 * above.  Planes hold 4 x nx x (ny_local + 2G) qwb_z, owned rows are local
 * rows [G, G+ny_local).
 * qwb_slab_run_fused: per NCCL exchange of g = jT state rows per plane with
 * each y-neighbour (j = m, fewer at the end), j launches of the temporally
 * blocked kernel over the owned rows extended by (j-1)T, ..., T, 0 rows each
 * side; the last < T steps as single pull steps (1-row exchange).  The same
 * arithmetic as one GPU: bitwise equal.                                       */
int qwb_slab_ghost_rows(int64_t nx, int64_t ny, int64_t ny_local, int64_t n_marked, int* ghost_host);
/* T, the coined steps per temporally blocked slab launch                     */
int qwb_slab_depth(int* depth_host);
int qwb_slab_to_planes_g(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local, int64_t ghost,
                         const qwb_z* arcs, qwb_z* planes, void* stream);
int qwb_slab_from_planes_g(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local, int64_t ghost,
                           const qwb_z* planes, qwb_z* arcs, void* stream);
int qwb_slab_probability_g(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local, int64_t ghost,
                           const qwb_z* planes, double* p, void* stream);
/* one launch without exchange: nsteps = T (temporally blocked, over the owned
 * rows extended by ext rows each side; ghost - ext >= T) or 1 (pull step, ext 0) */
int qwb_slab_advance_local(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local, int64_t ghost,
                           int shift, const uint32_t* marked_bits, const int64_t* marked_host, int64_t n_marked,
                           const qwb_z* in, qwb_z* out, int nsteps, int ext, void* stream);
int qwb_slab_run_fused(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local, int64_t ghost,
                       int shift, const uint32_t* marked_bits, const int64_t* marked_host, int64_t n_marked,
                       qwb_z* a, qwb_z* b, int64_t steps, int rank_below, int rank_above, int* final_in_b_host,
                       void* stream);
/* single-device emulation of the ghost-row exchange (g rows) between nslabs slabs (tests) */
int qwb_slab_ghost_exchange_local(qwb_ctx* ctx, int64_t nx, int64_t ghost, int g, const int64_t* ny_local_host,
                                  qwb_z* const* planes_host, int nslabs, void* stream);
/* single-device emulation of the per-step exchange between nslabs slabs (tests) */
int qwb_slab_exchange_local(qwb_ctx* ctx, int64_t nx, int shift, const int64_t* ny_local_host,
                            qwb_z* const* planes_host, int nslabs, void* stream);
/* Halo exchange of a row-partitioned CSR operator (generic graphs; the row
 * ranges and index lists come from distributed.csr_partition).  x_ext =
 * [own entries (n_local) | halo]; for peer i (peers_host[i], ascending): send
 * x_ext[send_idx[send_off[i] .. send_off[i+1])] (device int64 indices) and
 * receive recv_off[i+1] - recv_off[i] entries into x_ext[n_local + recv_off[i]
 * ..], one NCCL group.  send_buf: send_off[npeers] qwb_z.  The step itself is
 * qwb_spmv on the local rows (columns renumbered into x_ext).               */
int qwb_csr_halo_exchange(qwb_ctx* ctx, int64_t n_local, qwb_z* x_ext, const int64_t* send_idx,
                          const int64_t* send_off_host, const int64_t* recv_off_host, const int* peers_host,
                          int npeers, qwb_z* send_buf, void* stream);
/* NCCL communicator (one per rank; id: 128 bytes from rank 0, broadcast by the caller) */
int qwb_comm_unique_id(void* id_out_host);
int qwb_comm_init(qwb_ctx* ctx, const void* id_host, int nranks, int rank);
int qwb_comm_destroy(qwb_ctx* ctx);
/* `steps` steps with the boundary rows computed first, their exchange on a
 * comm stream overlapped with the interior rows.  marked_bits is a GLOBAL
 * vertex bitmap (NULL = none).                                                */
int qwb_slab_run(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local, int shift,
                 const uint32_t* marked_bits, qwb_z* a, qwb_z* b, int64_t steps, int rank_below,
                 int rank_above, int* final_in_b_host, void* stream);

/* ---- reducers -------------------------------------------------------------
 * coined: p[v] = sum over v's arc span of |psi|^2 (coined.py:275-294)
 * ctqw:   p = |psi|^2                              (ctqw.py:205-212)          */
int qwb_prob_arcs(qwb_ctx* ctx, int64_t n, const int64_t* tail_offsets, const qwb_z* psi,
                  double* p, void* stream);
int qwb_prob_abs2(qwb_ctx* ctx, int64_t n, const qwb_z* psi, double* p, void* stream);

/* ---- BLAS-1 (backend.py:433-464) ------------------------------------------ */
int qwb_axpy(qwb_ctx* ctx, int64_t n, qwb_z alpha, const qwb_z* x, const qwb_z* y, qwb_z* out,
             void* stream);                                   /* out = y + alpha x */
int qwb_scale(qwb_ctx* ctx, int64_t n, qwb_z alpha, const qwb_z* x, qwb_z* out, void* stream);
int qwb_dot(qwb_ctx* ctx, int64_t n, const qwb_z* x, const qwb_z* y, qwb_z* result_host,
            void* stream);                                    /* conj(x) . y       */
int qwb_norm(qwb_ctx* ctx, int64_t n, const qwb_z* x, double* result_host, void* stream);
/* _check_finite (backend.py:60-62): *all_finite_host = 1 iff no NaN/Inf.     */
int qwb_check_finite(qwb_ctx* ctx, int64_t n_doubles, const double* x, int* all_finite_host,
                     void* stream);

/* ---- continuous-time walk: evolve_state (ctqw.py:123-171) ----------------
 * psi (in/out, device, n entries) <- [T_s(tau H)]^substeps psi, where each
 * sub-step sums Taylor terms term_k = (-i tau / k) H term_{k-1} until
 * ||term_k|| <= floor (= tol * ||psi_in||), at most max_terms per sub-step
 * (else QWB_E_SERIES_NOT_CONVERGED).  The caller computes substeps and tau
 * exactly as ctqw.py:149-150 does.  terms_host (nullable, [substeps]) gets
 * the term count of each sub-step.  work: 3*n qwb_z.                         */
int qwb_taylor_evolve_csr(qwb_ctx* ctx, int64_t n, const int64_t* row_offsets, const int32_t* col,
                          const qwb_z* val, qwb_z* psi, qwb_z* work, int64_t substeps, double tau,
                          double floor, int max_terms, int* terms_host, void* stream);
/* matrix-free H = -gamma A(hypercube dim) - sum_M |v><v| (marked_bits bitmap). */
int qwb_taylor_evolve_hypercube(qwb_ctx* ctx, int dim, double gamma, const uint32_t* marked_bits,
                                qwb_z* psi, qwb_z* work, int64_t substeps, double tau, double floor,
                                int max_terms, int* terms_host, void* stream);
/* Sharded matrix-free hypercube evolve (no reference counterpart; SURVEY
 * §8(e) C4): 2^log2_shards ranks, rank r (ctx->rank, NCCL communicator from
 * qwb_comm_init, ctx->nranks == 2^log2_shards) owns the 2^(dim-log2_shards)
 * consecutive vertices whose top log2_shards bits equal r (psi: its local
 * slice).  Per Taylor term the term slice is exchanged with the log2_shards
 * partners r ^ 2^j (NCCL grouped send/recv) and the stop test uses the norm
 * all-gathered over ranks and summed in rank order, so every rank takes the
 * same decision and the state is bitwise the single-GPU one.  marked_bits is
 * the GLOBAL bitmap; floor = tol * ||psi_in|| over the whole state.
 * work: (3 + log2_shards) * 2^(dim-log2_shards) qwb_z.  dim - log2_shards >= 10. */
int qwb_taylor_evolve_hypercube_sharded(qwb_ctx* ctx, int dim, int log2_shards, double gamma,
                                        const uint32_t* marked_bits, qwb_z* psi, qwb_z* work, int64_t substeps,
                                        double tau, double floor, int max_terms, int* terms_host, void* stream);
/* the same decomposition with all 2^log2_shards shards on ONE device (the
 * partner slices are read in place instead of exchanged): psi_host / work_host
 * are host arrays of per-shard device pointers (work: 3 * 2^(dim-log2_shards)). */
int qwb_taylor_evolve_hypercube_shards_local(qwb_ctx* ctx, int dim, int log2_shards, double gamma,
                                             const uint32_t* marked_bits, qwb_z* const* psi_host,
                                             qwb_z* const* work_host, int64_t substeps, double tau, double floor,
                                             int max_terms, int* terms_host, void* stream);
/* one matrix-free hypercube H x (for tests / backend parity). */
int qwb_hypercube_apply(qwb_ctx* ctx, int dim, double gamma, const uint32_t* marked_bits,
                        const qwb_z* x, qwb_z* y, void* stream);

/* ---- distribution sinks (host; reference cli.py:398-432) ----------------
 * Text of a probability record exactly as the reference's JSON / CSV /
 * frames sinks write it (Python float repr: shortest round-trip digits,
 * fixed notation for -4 < decpt <= 16, else d.ddde+XX).  Host-only helpers:
 * no context, no device memory; threads > 1 splits the record.
 * qwb_format_f64_repr: one value into out (>= 32 bytes), returns its length;
 *   json = 1 spells non-finite values NaN / Infinity / -Infinity, else
 *   nan / inf / -inf.
 * qwb_format_json_floats: "p0,p1,...,p{n-1}" (the body of a "p" list,
 *   cli.py:403-405); returns the length, or -1 if cap is too small
 *   (n * 25 bytes always suffices).
 * qwb_format_csv_rows: one line "<prefix><vertex0+i>,<p[i]>\n" per item i (prefix
 *   "k,t," for the csv sink, cli.py:413-416; "" for a frame file, 425-428);
 *   returns the length or -1 (n * (prefix_len + 47) bytes always suffice). */
int qwb_format_f64_repr(double x, int json, char* out);
int64_t qwb_format_json_floats(const double* p, int64_t n, char* out, int64_t cap, int threads);
int64_t qwb_format_csv_rows(const double* p, int64_t n, int64_t vertex0, const char* prefix, int64_t prefix_len,
                            char* out, int64_t cap, int threads);

#ifdef __cplusplus
}
#endif
#endif /* QWB200_H */
