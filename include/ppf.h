/*
 * ppf.h -- polynomially preconditioned f(A)b, C ABI of the B200 hot path.
 *
 * Method: Frommer, Ramirez-Hidalgo, Schweitzer, Tsolakis, "Polynomial
 * preconditioning for the action of the matrix square root and inverse square
 * root" (arXiv 2401.06684).  Citations "P:n" are lines of that paper's
 * PAPER.md; "Qn" are the readings listed in DESIGN.md §3.
 *
 *   Algorithm 1: c = q(A)s, v_1 = c/||c||; for j = 1..m:
 *     u = A v_j, y = q(A)u, w = q(A)y (three stages);
 *     orthogonalise w against v_1..v_j (H_m upper Hessenberg);
 *     h_{j+1,j} = ||w||, v_{j+1} = w/h_{j+1,j};
 *   f_m = V_m (H_m^{-1/2} e_1 ||c||)
 *   with s = b for f(z) = z^{-1/2} and s = A b for f(z) = z^{1/2}.
 *
 * Conventions shared by every entry point
 *   - Every function returns ppf_status; no C++ exception crosses the ABI.
 *     PPF_OK = 0.  On any other status ppf_last_error() (thread-local) holds a
 *     one-line description.  Output arguments are untouched on failure.
 *   - Scalars are double (PPF_R64) or interleaved (re, im) double pairs
 *     (PPF_C128, C99 double _Complex layout).
 *   - Index arrays are 0-based int64.  A matrix is given as this rank's
 *     contiguous row slab [row0, row0 + n_local) of a global n_global x n_global
 *     matrix in CSR form with GLOBAL column indices sorted within each row.
 *   - "device" pointers are CUDA device memory owned by the caller (PyTorch
 *     allocations), valid for the duration of the call and of the stream work it
 *     enqueues.  Device vectors and scratch must be 16-byte aligned (they are
 *     moved as 128-bit pairs and by bulk copies; PPF_EINVAL otherwise, e.g. for
 *     a float64 view starting at an odd element); 256-byte alignment (what
 *     the PyTorch allocator returns) is recommended.  The library never calls cudaMalloc or
 *     cudaFree (one exception: the peer window of ppf_mat_peer_window, which a
 *     CUDA IPC export needs as an allocation of its own); size-query functions
 *     say how much the caller must provide.
 *     "host" pointers are ordinary host memory, only read/written during the
 *     call (the library copies what it needs).
 *   - Vectors passed to ppf_run are this rank's slab (n_local entries).
 *   - Work is enqueued on the context's CUDA stream.  A context is not
 *     thread-safe: use one per host thread.
 */
#ifndef PPF_H_
#define PPF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PPF_ABI_VERSION 3

typedef enum {
  PPF_OK = 0,
  PPF_EINVAL = 1,          /* invalid argument (see ppf_last_error) */
  PPF_ECUDA = 2,           /* CUDA runtime error */
  PPF_ENCCL = 3,           /* NCCL error */
  PPF_EWORKSPACE = 4,      /* caller-provided buffer too small */
  PPF_EBRANCH = 5,         /* a node / eigenvalue of H_m lies on (-inf, 0], or the
                              positivity certificate of q failed */
  PPF_EDENSE = 6,          /* host dense eigen/Schur iteration did not converge */
  PPF_ESTATE = 7           /* object used in the wrong state / mismatched objects */
} ppf_status;

typedef enum { PPF_R64 = 0, PPF_C128 = 1 } ppf_dtype;
typedef enum {
  PPF_INVSQRT = 0,     /* A^{-1/2} b */
  PPF_SQRT = 1,        /* A^{1/2} b = A^{-1/2}(A b) */
  PPF_INVSQRT_SQ = 2,  /* (A^2)^{-1/2} b: the Krylov operator is A^2, applied as two mat-vecs
                          with the given A; q approximates z^{-1/2} on spec(A^2) */
  PPF_SIGN = 3         /* sign(A) b = A (A^2)^{-1/2} b */
} ppf_func;
typedef enum {
  PPF_LANCZOS = 0,        /* Hermitian A: three-term recurrence, all basis vectors kept (reading Q8) */
  PPF_ARNOLDI_CGS2 = 1,   /* general A: classical Gram-Schmidt with one reorthogonalisation */
  PPF_LANCZOS_2PASS = 2   /* Hermitian A, two-pass: pass 1 assembles H_m keeping
                             3 basis vectors, pass 2 regenerates them to form f_m */
} ppf_krylov;
typedef enum {
  PPF_PREC_LEFT = 0,      /* Algorithm 1: Krylov space of A q(A)^2 from q(A)s */
  PPF_PREC_RIGHT = 1      /* Algorithm 2: from s; f_m = Y_m (H_m^{-1/2} e_1 ||s||),
                             y_j = q(A) v_j stored (one-pass) or f_m = q(A) V_m (...) (two-pass) */
} ppf_precond;
typedef enum { PPF_STOP_FIXED_M = 0, PPF_STOP_EST = 1, PPF_STOP_TRUE_ERR = 2 } ppf_stop;
typedef enum { PPF_CONVERGED = 0, PPF_MAX_ITER = 1, PPF_BREAKDOWN = 2 } ppf_term;
typedef enum { PPF_POLY_CHEBYSHEV = 0, PPF_POLY_NEWTON = 1 } ppf_poly_kind;
typedef enum { PPF_FMT_SELL = 0, PPF_FMT_CSR = 1 } ppf_format;
/* device layout of the diagonal block's entries (ppf_plan_encoding) */
typedef enum {
  PPF_ENC_EXPLICIT = 0, /* 32-bit column indices + dtype values */
  PPF_ENC_DELTA16 = 1,  /* 16-bit column deltas + per-slice-column base + dtype values */
  PPF_ENC_PAIR8 = 2     /* one 8-bit code per entry into a table of <= 256 (col - row, value) pairs */
} ppf_encoding;

typedef struct ppf_ctx ppf_ctx;
typedef struct ppf_plan ppf_plan;
typedef struct ppf_mat ppf_mat;
typedef struct ppf_poly ppf_poly;

const char* ppf_status_string(int status);
const char* ppf_last_error(void);
int ppf_abi_version(void);

/* ----------------------------------------------------------------------------
 * Context: one per GPU / rank.
 * ppf_nccl_unique_id: writes 128 bytes (an ncclUniqueId) to host `out128`; call
 *   on rank 0 and broadcast the bytes (e.g. torch.distributed) to the others.
 * ppf_ctx_create: device = CUDA ordinal; cuda_stream = cudaStream_t to enqueue
 *   on (NULL = the legacy default stream).  nranks > 1 with id128 (the
 *   broadcast unique id) initialises an NCCL communicator; nranks > 1 with
 *   id128 == NULL creates a context WITHOUT a communicator whose halo exchange
 *   is done by the caller through ppf_halo_pack / ppf_halo_buffers /
 *   ppf_spmv_local (testing the sharded SpMV in one process), through a host
 *   transport (ppf_ctx_set_transport) or through peer memory
 *   (ppf_mat_peer_window / ppf_mat_peer_connect); with none of these ppf_run
 *   and ppf_spmv return PPF_ESTATE.  nranks == 1 ignores id128.
 * ------------------------------------------------------------------------- */
ppf_status ppf_nccl_unique_id(void* out128);
/* Host transport (nranks > 1 without NCCL): the caller moves the halo and sums
 * the reductions itself, e.g. over torch.distributed/gloo -- used to verify the
 * sharded algorithm with several processes on one device.  The library stages
 * through pinned host memory and synchronises the stream around each call:
 *   exchange(user, send, send_counts, recv, recv_counts): send holds this
 *     rank's packed boundary entries, per-peer segments in peer order,
 *     send_counts[p] doubles each (complex: 2 per entry); fill recv likewise
 *     (recv_counts[p] doubles from peer p, peer order);
 *   allreduce_sum(user, buf, count): in-place sum over all ranks.
 * Both return 0 on success (anything else -> PPF_ENCCL).  The function
 * pointers must stay valid for the context's lifetime; NULL clears. */
typedef struct {
  void* user;
  int (*exchange)(void* user, const double* send, const int64_t* send_counts, double* recv,
                  const int64_t* recv_counts);
  int (*allreduce_sum)(void* user, double* buf, int64_t count);
} ppf_transport;
ppf_status ppf_ctx_set_transport(ppf_ctx* ctx, const ppf_transport* transport);
/* ppf_ctx_set_graphs: with left preconditioning (one-pass, one rank, profiling
 * off) ppf_run captures the step's q(A)q(A) chain -- its 2 deg fused SpMV
 * launches between fixed buffers -- once as a CUDA graph and replays it every
 * step (default on).  Results are bitwise identical either way. */
ppf_status ppf_ctx_set_graphs(ppf_ctx* ctx, int on);
ppf_status ppf_ctx_create(int device, int rank, int nranks, const void* id128,
                          void* cuda_stream, ppf_ctx** out);
void ppf_ctx_destroy(ppf_ctx* ctx);

/* ----------------------------------------------------------------------------
 * Operator A (layer L0).  Host-only planning, then upload.
 *
 * ppf_plan_create: host-side conversion of this rank's CSR slab into the
 *   device layout.  row_bounds[nranks+1] gives every rank's first row
 *   (row_bounds[0] = 0, row_bounds[nranks] = n_global, nondecreasing); this
 *   rank owns [row_bounds[rank], row_bounds[rank+1]).  row_ptr[n_local+1]
 *   (row_ptr[0] = 0, nondecreasing), col[nnz] (global, sorted per row, in
 *   [0, n_global)), val[nnz] (dtype scalars).  format: PPF_FMT_SELL uses
 *   SELL-C-sigma with slice height `sell_C` (32 or 64 for R64, 32 for C128) and
 *   row-sorting window `sell_sigma` (1 = no sorting, else a multiple of
 *   sell_C); PPF_FMT_CSR ignores both.  Columns owned by this rank go to the
 *   diagonal block, others to the off-diagonal (halo) block.  Needs no GPU.
 * ppf_plan_device_bytes: bytes of device memory ppf_mat_create needs.
 * ppf_plan_halo_count / ppf_plan_halo_recv: the global indices this rank must
 *   receive from rank `peer` before each SpMV (sorted, unique).
 * ppf_plan_set_halo_send: the local row indices this rank sends to `peer`
 *   (what `peer` reported as its recv list for us, minus row_bounds[rank]);
 *   the caller exchanges the lists (e.g. torch.distributed) -- host logic only.
 * ppf_mat_create: uploads the plan into device_buf (>= ppf_plan_device_bytes)
 *   on the context stream; the plan may be destroyed afterwards.
 * ppf_spmv: y = A x on this rank's slab (x, y device, n_local entries),
 *   including the halo exchange; for tests and benchmarks.
 * ------------------------------------------------------------------------- */
ppf_status ppf_plan_create(ppf_dtype dtype, int64_t n_global, int nranks, int rank,
                           const int64_t* row_bounds, const int64_t* row_ptr,
                           const int64_t* col, const void* val, ppf_format format,
                           int sell_C, int sell_sigma, ppf_plan** out);
ppf_status ppf_plan_device_bytes(const ppf_plan* plan, size_t* bytes);
ppf_status ppf_plan_info(const ppf_plan* plan, int64_t* n_local, int64_t* nnz,
                         int64_t* stored_entries, int64_t* halo_total);
/* ppf_plan_index_bits: 32, or 16 when the SELL diagonal block (complex C = 32,
 * fp64 C = 64; no sigma sorting) stores its column indices as 16-bit deltas
 * relative to the row (per slice-column base;
 * chosen by ppf_plan_create whenever every slice-column spans <= 65535 --
 * stencils do -- unless the environment sets PPF_IDX16=0). */
ppf_status ppf_plan_index_bits(const ppf_plan* plan, int* bits);
/* ppf_plan_encoding: the layout ppf_mat_create will upload (ppf_encoding) and,
 * for PPF_ENC_PAIR8, the table size (*ntab, else 0; either pointer may be
 * NULL).  ppf_plan_create picks the narrowest lossless layout available:
 *   PPF_ENC_PAIR8 for SELL-64 fp64 without sorting (sell_C = 64,
 *     sell_sigma = 1) when the diagonal block's stored entries, padding
 *     included, take at most 256 distinct (column - row, value) pairs -- a
 *     banded matrix with constant diagonals, i.e. a constant-coefficient
 *     stencil (the paper's Laplacian and convection-diffusion operators,
 *     P:419): 1 byte per entry instead of 10-12 (an entry-dictionary
 *     generalisation of value-indexed CSR; the multiply-adds are the same, in
 *     the same order, as with the explicit layout);
 *   else PPF_ENC_DELTA16 where ppf_plan_index_bits reports 16;
 *   else PPF_ENC_EXPLICIT.
 * The environment variable PPF_PAIR8=0 (PPF_IDX16=0) at plan time disables
 * the pair codes (the deltas).  ppf_plan_set_encoding selects a wider layout
 * than the one chosen (PPF_EINVAL if `enc` is not available for this plan);
 * call it before ppf_plan_device_bytes / ppf_mat_create.  ppf_plan_index_bits
 * reports the layout in force: 8 (pair codes), 16 or 32. */
ppf_status ppf_plan_encoding(const ppf_plan* plan, int* enc, int* ntab);
ppf_status ppf_plan_set_encoding(ppf_plan* plan, int enc);
/* ppf_plan_slice_schedule: the order in which the pair-code SpMV (P:131-146's
 * mat-vec on PPF_ENC_PAIR8) hands SELL slices to thread blocks: warp w of block
 * b takes slice out[8 b + w] (-1: none).  Blocks are tiles of slices whose rows
 * gather from one another (the pair table's two smallest |column - row| >= 64,
 * a stencil's +-N and +-N^2 neighbours), so their x gathers share L1 lines;
 * every slice appears exactly once.  Scheduling only: results are bitwise
 * those of the in-order launch.  *count = number of entries (a multiple of 8;
 * 0 = slices in order, 8 per block: no pair codes, no far offsets, fewer than
 * 64 slices, or PPF_SELLP_TILE=0 at plan time; PPF_SELLP_TILE=TYxTZ with
 * TY * TZ = 8 picks the tile).  `out` (host, may be NULL) receives
 * min(cap, *count) entries. */
ppf_status ppf_plan_slice_schedule(const ppf_plan* plan, int32_t* out, int64_t cap,
                                   int64_t* count);
ppf_status ppf_plan_halo_count(const ppf_plan* plan, int peer, int64_t* count);
ppf_status ppf_plan_halo_recv(const ppf_plan* plan, int peer, int64_t* global_idx);
ppf_status ppf_plan_set_halo_send(ppf_plan* plan, int peer, int64_t count,
                                  const int64_t* local_rows);
void ppf_plan_destroy(ppf_plan* plan);

ppf_status ppf_mat_create(ppf_ctx* ctx, const ppf_plan* plan, void* device_buf,
                          size_t bytes, ppf_mat** out);
ppf_status ppf_spmv(ppf_ctx* ctx, ppf_mat* A, const void* x, void* y);
void ppf_mat_destroy(ppf_mat* A);
/* ppf_mat_set_split: warps per SELL slice of the SpMV kernels:
 *   1, 2, 4 or 8 splits each slice's entry columns over that many warps whose
 *   partial sums are added in part order in shared memory; 0 restores the
 *   automatic choice made by ppf_mat_create (enough warp tasks for >= ~8 waves
 *   of resident warps).  Results differ only by summation order.  CSR: no-op.
 *   *applied (may be NULL) receives the value now in force.  PPF_EINVAL for
 *   other values. */
ppf_status ppf_mat_set_split(ppf_mat* A, int sell_ks, int* applied);
/* Pieces of the sharded SpMV, for callers that move the halo
 * themselves: ppf_halo_pack gathers this rank's boundary entries of x (device)
 * into the send buffer; ppf_halo_buffers returns the device send / receive
 * buffers (per-peer segments in peer order, lengths from the plan's lists:
 * send segment of peer p = the rows set by ppf_plan_set_halo_send(p), receive
 * segment of peer p = ppf_plan_halo_recv(p)); ppf_spmv_local computes y = A x
 * from the local x and the CURRENT receive buffer (diagonal block + halo block)
 * without communicating. */
ppf_status ppf_halo_pack(ppf_ctx* ctx, ppf_mat* A, const void* x);
ppf_status ppf_halo_buffers(ppf_mat* A, void** send, void** recv);
ppf_status ppf_spmv_local(ppf_ctx* ctx, ppf_mat* A, const void* x, void* y);

/* ----------------------------------------------------------------------------
 * Peer-memory communication (SURVEY §8(e) "B200-native alternative for halos":
 * direct peer loads/stores over NVLink instead of NCCL).  With a connected
 * window, every halo exchange and every reduction of ppf_run / ppf_spmv on A
 * goes through peer memory: a push kernel gathers this rank's boundary entries
 * of x and STORES them straight into each neighbour's receive slot (NVLink
 * writes, double-buffered by exchange epoch), then bumps the neighbour's arrival
 * counter (system-scope atomic after a system fence); the neighbour's stream
 * waits for the counter (cuStreamWaitValue32, GEQ -- a front-end wait, no
 * spinning kernel) before its halo block.  The push runs on a communication
 * stream concurrently with the diagonal-block SpMV.  Reductions: each rank
 * stores its partial sums into slot `rank` of every rank's window and bumps
 * their counters; after the wait every rank sums the slots in RANK ORDER, so
 * the reduced values are bit-identical on all ranks and from run to run (the
 * deterministic variant of SURVEY §8(e)).  No NCCL communicator is needed.
 *
 * ppf_mat_peer_window: allocates this rank's window (device memory owned by
 *   the library -- an IPC export needs an allocation base -- freed with A:
 *   counters, 2 x nranks reduction slots, 2 receive slots of halo_total
 *   entries) and writes a PPF_PEER_DESC_BYTES descriptor to host `desc`
 *   (CUDA IPC handle, process id + a random per-process nonce, receive
 *   offsets and counts per peer).
 *   The matrix must be sharded (nranks > 1, 1 < nranks <= PPF_PEER_MAX_RANKS)
 *   with its send lists set.  The caller all-gathers the descriptors.
 * ppf_mat_peer_connect: `descs` = nranks descriptors in rank order (host).
 *   Maps every peer window: cudaIpcOpenMemHandle for another process, the
 *   pointer itself for a rank of the same process (several contexts on one
 *   device, used by the tests).  Checks that every peer's receive count from
 *   this rank equals this rank's send count to it; PPF_EINVAL otherwise.
 *   All ranks must then issue the same sequence of ppf_run / ppf_spmv calls
 *   on A (the exchange epochs pair up by order).  ppf_mat_peer_connect(A, NULL)
 *   returns A to the context's NCCL / host transport.  Connecting force-loads
 *   every kernel of the library (lazy module loading would otherwise load a
 *   kernel at its first launch, which waits for the device -- possibly for a
 *   stream parked in a peer wait).  For the same reason query the workspace
 *   sizes (ppf_workspace_bytes / ppf_ritz_workspace_bytes, which also size the
 *   pinned host staging) and allocate before the ranks start a run: device or
 *   pinned allocation in the middle of one synchronises the device.
 * ------------------------------------------------------------------------- */
#define PPF_PEER_DESC_BYTES 2048
#define PPF_PEER_MAX_RANKS 64
ppf_status ppf_mat_peer_window(ppf_mat* A, void* desc);
ppf_status ppf_mat_peer_connect(ppf_mat* A, const void* descs);

/* ----------------------------------------------------------------------------
 * Preconditioning polynomial q ~ z^{-1/2} (layer L1), a host object.
 *
 * ppf_poly_chebyshev (reading Q2): the degree-`deg` Chebyshev
 *   interpolant of z^{-1/2} at the deg+1 first-kind points of [a, b]
 *   (= the coefficient integrals of P:329 by (deg+1)-point Gauss-Chebyshev
 *   quadrature).  Certificate: q > 0 at z_k = a + (b-a)k/1000, k = 0..1000,
 *   else PPF_EBRANCH.  Requires 0 < a < b, 0 <= deg <= 256.
 * ppf_poly_ritz_newton: runs deg+1 Arnoldi steps with A started
 *   from `start` (device, n_local entries; "started with the vector b"),
 *   takes the Ritz values (eigenvalues of H_{deg+1}), rejects any on
 *   (-inf, 0] (PPF_EBRANCH), Leja-orders them (max modulus first, then
 *   greedy max sum log|theta - chosen|, ties to the smaller index after sorting
 *   by (Re, Im)) and forms the divided differences of z^{-1/2}.  `work` is
 *   device scratch of at least ppf_ritz_workspace_bytes.  Complex operators:
 *   any nodes off (-inf, 0]; real operators: real nodes, or conjugate pairs in
 *   the real-pair form.
 * ppf_poly_import: kind CHEBYSHEV: ab = {a, b}, coef = deg+1 doubles, nodes
 *   ignored.  kind NEWTON: coef = deg+1 complex divided differences, nodes =
 *   deg+1 complex Leja-ordered nodes, ab ignored.  No certificate is applied.
 *   A Newton polynomial is applied to a PPF_R64 operator only if all its nodes
 *   and divided differences are real (exactly zero imaginary parts); the Ritz
 *   construction on a PPF_R64 operator with complex (conjugate-pair) Ritz
 *   values returns the real-pair form (ppf_poly_set_newton_eval mode 2).
 * ppf_poly_export: the same layout (caller buffers of deg+1 entries; query deg
 *   first with coef = nodes = NULL).
 * ppf_poly_eval: q at `npts` complex points (host, interleaved) -> host out.
 * ------------------------------------------------------------------------- */
ppf_status ppf_poly_chebyshev(double a, double b, int deg, ppf_poly** out);
ppf_status ppf_ritz_workspace_bytes(ppf_ctx* ctx, const ppf_mat* A, int deg, size_t* bytes);
ppf_status ppf_poly_ritz_newton(ppf_ctx* ctx, ppf_mat* A, const void* start, int deg,
                                void* work, size_t work_bytes, ppf_poly** out);
/* The same for the Ritz values of A^power (power 1 or 2; power 2 = the operator
 * of PPF_INVSQRT_SQ / PPF_SIGN, two mat-vecs per Arnoldi step); with
 * harmonic != 0 the nodes are the harmonic Ritz values, the eigenvalues of
 * H_d + h_{d+1,d}^2 H_d^{-*} e_d e_d^* (P:357-367). */
ppf_status ppf_poly_ritz_newton_pow(ppf_ctx* ctx, ppf_mat* A, const void* start, int deg,
                                    int power, int harmonic, void* work, size_t work_bytes,
                                    ppf_poly** out);
/* ppf_poly_contour_ls (§5.3): the least-squares polynomial of degree
 *   deg for z^{-1/2} on the discretised contour `points` (npts complex, host,
 *   interleaved; npts > deg + 1; no point on (-inf, 0]): Arnoldi on
 *   diag(points) from ones/sqrt(npts), alpha = P^H z^{-1/2}.  Stored in Newton
 *   form on deg+1 Leja-ordered contour points (the interpolant of a degree-deg
 *   polynomial is the polynomial), applied by the fused Newton-Horner chain.
 *   min_re_q (may be NULL) = min Re q over the points; <= 0 gives PPF_EBRANCH
 *   (the certificate of P:401-403). */
ppf_status ppf_poly_contour_ls(const double* points, int npts, int deg, double* min_re_q,
                               ppf_poly** out);
/* ppf_contour_from_ritz (Q29): a contour
 *   for ppf_poly_contour_ls from Ritz values theta (ntheta complex, host,
 *   interleaved): their convex hull (collinear values: the segment there and
 *   back), densified in steps <= step, the parts closer to 0 than r_min
 *   replaced by the arc |z| = r_min (then resampled uniformly).  Writes *npts
 *   points to `points` (cap complex entries; query with points = NULL).
 *   PPF_EBRANCH if the hull surrounds 0. */
ppf_status ppf_contour_from_ritz(const double* theta, int ntheta, double r_min, double step,
                                 int cap, double* points, int* npts);
/* ppf_poly_certify: the branch certificate of the preconditioned method --
 *   q must not vanish where ((q(A))^2)^{1/2} = q(A) is needed: q > 0 on the
 *   spectral interval for a Chebyshev q (checked at the points of
 *   P:420), Re q > 0 on the contour for a least-squares q.
 *   pts: npts host points, PPF_R64 (npts doubles) or PPF_C128 (npts
 *   interleaved (re, im) pairs); pts == NULL (Chebyshev q only) checks the
 *   default grid z_k = a + (b-a)k/1000, k = 0..1000.  *min_re_q (may be NULL)
 *   receives min Re q over the points (NaN if q is NaN anywhere); the status is
 *   PPF_EBRANCH unless that minimum is > 0.  ppf_poly_chebyshev and
 *   ppf_poly_contour_ls apply it before returning a polynomial.  Host only. */
ppf_status ppf_poly_certify(const ppf_poly* q, const void* pts, int npts, int dtype,
                            double* min_re_q);
ppf_status ppf_poly_import(int kind, int deg, const double* ab, const void* coef,
                           const void* nodes, ppf_poly** out);
ppf_status ppf_poly_export(const ppf_poly* q, int* kind, int* deg, double* ab,
                           void* coef, void* nodes);
ppf_status ppf_poly_eval(const ppf_poly* q, int npts, const double* z, double* out);
/* y = q(A) x on the device (x, y device, n_local entries, distinct), the fused
 * SpMV chain of the hot path (Clenshaw P:332 / Newton-Horner P:354): exactly
 * deg SpMV launches.  `work` is device scratch of ppf_poly_apply_bytes. */
ppf_status ppf_poly_apply_bytes(ppf_ctx* ctx, const ppf_mat* A, size_t* bytes);
ppf_status ppf_poly_apply(ppf_ctx* ctx, ppf_mat* A, const ppf_poly* q, const void* x, void* y,
                          void* work, size_t work_bytes);
/* ppf_poly_set_newton_eval: how the device applies a Newton-form q.
 *   mode 0 (default): Horner, w = (A - theta_j) w + dd_j v (the paper's "Horner-type
 *   scheme"); mode 1: the forward Newton basis p_{j+1} = (A - theta_j) p_j with
 *   sum dd_j p_j accumulated as a second output of each SpMV (one more vector
 *   stream per launch), numerically preferable when spec(A) extends far beyond
 *   the nodes (Q28).  Same deg SpMV launches.  Chebyshev: ignored.
 *   mode 2: the real conjugate-pair form for a real operator (nodes closed
 *   under conjugation): Leja order with each complex node followed by its
 *   conjugate, real basis P_{j+1} = (A - Re th_j) P_j [+ (Im th)^2 P_{j-1} for
 *   the second of a pair], real coefficients -- all in real arithmetic; the
 *   nodes/dd are reordered (ppf_poly_export shows the new order).  The Ritz
 *   construction on a PPF_R64 operator selects it when Ritz values are complex.
 *   PPF_EINVAL if the nodes are not conjugate-symmetric. */
ppf_status ppf_poly_set_newton_eval(ppf_poly* q, int mode);
void ppf_poly_destroy(ppf_poly* q);

/* ----------------------------------------------------------------------------
 * The run (layers L2-L5): Algorithm 1, f(H_m) on the host, x = V_m y_m.
 *
 * opts.func / krylov / precond: see enums.  q == NULL selects the plain
 *   (unpreconditioned, d = 1) method: the Krylov space of A from s ("d = 1
 *   corresponds to an unpreconditioned method"); precond is then ignored.
 *   m_max >= 1 (<= 1024).  stop:
 *   FIXED_M   run exactly m_max steps (unless breakdown);
 *   EST       stop at the first checkpoint m with the paper's estimate
 *             ||f_m - f_{m-k}|| / ||f_m|| <= tol, k = check_every.
 *             Left / plain: = ||[y_{m-k};0] - y_m|| / ||y_m|| (V orthonormal).
 *             Right, one-pass: formed from the iterates Y_m y_m on the device
 *             (Y_m is not orthonormal).  Right, two-pass: the
 *             coefficient difference is used as a proxy (DESIGN.md readings);
 *   TRUE_ERR  stop at the first checkpoint with ||f_m - x_ref|| / ||x_ref|| <= tol
 *             (x_ref device, n_local entries; for calibrating m*, reading Q11;
 *             for PPF_SIGN f_m is the (A^2)^{-1/2} b iterate, before the final A);
 *             not available with PPF_LANCZOS_2PASS (PPF_EINVAL).
 * ppf_workspace_bytes: device scratch `work` needed by ppf_run for these
 *   (A, q, opts); it holds V (m_max+1 columns; 4 for PPF_LANCZOS_2PASS), Y
 *   (m_max columns, right preconditioning one-pass only), 5-6 n-vectors and
 *   reduction scratch.
 * ppf_run: b, x device (n_local entries).  Enqueues everything on the context
 *   stream and returns once x has been enqueued; the report is valid on return.
 * ppf_run_host: the same with b_host / x_host host buffers; the H2D copy of b
 *   and the D2H copy of x go through the library (pinned staging) and the call
 *   returns with x_host filled.
 * ppf_history: per-checkpoint records of the last run (count <= cap).
 * ppf_hessenberg: the last run's (m+1) x m matrix H (column-major, leading
 *   dimension ld >= m+1, dtype scalars) and ||c||.  Query m with H = NULL.
 * ------------------------------------------------------------------------- */
typedef struct {
  int func;            /* ppf_func */
  int krylov;          /* ppf_krylov */
  int m_max;
  int stop;            /* ppf_stop */
  double tol;
  int check_every;     /* k >= 1 */
  const void* x_ref;   /* device, TRUE_ERR only */
  double breakdown_rtol;
  int record_history;
  int precond;         /* ppf_precond (ABI 2) */
} ppf_opts;

typedef struct {
  int iterations;              /* m of the returned f_m */
  int term;                    /* ppf_term */
  long long mvms;              /* products with A (P:455 unit), incl. c = q(A)s, A b; for
                                  PPF_INVSQRT_SQ / PPF_SIGN 2 per application of A^2 (Table 2's
                                  unit) plus 1 for the final A f (SIGN) */
  long long inner_products;     /* norms included, ||c|| not */
  double est;                  /* last estimate (NaN if none) */
  double err;                  /* last true error (NaN unless TRUE_ERR) */
  double beta0;                /* ||c|| */
  double seconds_total;        /* host wall time of the call */
  double seconds_host_dense;   /* host time in f(H_m) evaluations */
  long long kernel_launches;   /* kernels this call launched */
  double seconds_device;       /* device time of the call's stream work (ABI 3): CUDA events
                                  recorded on the context stream before the first and after
                                  the last enqueued operation (H2D / D2H of ppf_run_host
                                  included) */
} ppf_report;

ppf_status ppf_workspace_bytes(ppf_ctx* ctx, const ppf_mat* A, const ppf_poly* q,
                               const ppf_opts* opts, size_t* bytes);
ppf_status ppf_run(ppf_ctx* ctx, ppf_mat* A, const ppf_poly* q, const ppf_opts* opts,
                   const void* b, void* x, void* work, size_t work_bytes, ppf_report* rep);
ppf_status ppf_run_host(ppf_ctx* ctx, ppf_mat* A, const ppf_poly* q, const ppf_opts* opts,
                        const void* b_host, void* x_host, void* work, size_t work_bytes,
                        ppf_report* rep);
ppf_status ppf_history(ppf_ctx* ctx, int cap, int* count, int* m, double* est, double* err,
                       long long* mvms);
ppf_status ppf_hessenberg(ppf_ctx* ctx, int ld, void* H, int* m, double* beta0);

/* Optional device timing of the hot-path kernels: with profiling on, every
 * kernel launch of ppf_run / ppf_poly_apply / ppf_poly_ritz_newton is
 * bracketed by CUDA events on the context stream; per class the library
 * accumulates launches, device milliseconds and ALGORITHMIC bytes (the minimum
 * HBM traffic of that launch: SpMV (s+4) nnz + s n (x, out, [z], [u]);
 * CGS sweeps (ncols + 1 or 2) s n).
 * cls: 0 = SpMV / fused chain steps, 1 = orthogonalisation (CGS2, Lanczos,
 * scaling), 2 = other (norms, combine).  ppf_profile_enable resets. */
ppf_status ppf_profile_enable(ppf_ctx* ctx, int on);
ppf_status ppf_profile_read(ppf_ctx* ctx, int cls, long long* launches, double* ms,
                            double* bytes);

/* ----------------------------------------------------------------------------
 * Host dense kernel (layer L4, K10), exposed for tests:
 * y = beta0 * H^{-1/2} e_1 for an m x m matrix H (column-major, leading
 * dimension ld, dtype scalars), principal branch.  hermitian != 0: H is taken
 * as symmetric tridiagonal (diagonal and first subdiagonal read) and solved by
 * a tridiagonal eigendecomposition; else complex Schur -> triangular square
 * root -> triangular solve.  PPF_EBRANCH if an eigenvalue is on
 * (-inf, 0].  y: m dtype scalars (host).
 * ------------------------------------------------------------------------- */
ppf_status ppf_dense_invsqrt_e1(ppf_dtype dtype, int m, const void* H, int ld, double beta0,
                                int hermitian, void* y);

#ifdef __cplusplus
}
#endif

#endif /* PPF_H_ */
