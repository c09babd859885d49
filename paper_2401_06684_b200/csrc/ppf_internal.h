// Internal declarations of the ppf library (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <complex>
#include <string>
#include <vector>

#include "../../include/ppf.h"

#ifndef PPF_HD
#ifdef __CUDACC__
#define PPF_HD __host__ __device__ __forceinline__
#else
#define PPF_HD inline
#endif
#endif

namespace ppf {

// ---------------------------------------------------------------------------
// Scalar types: double (PPF_R64) and an interleaved complex (PPF_C128).
// ---------------------------------------------------------------------------
struct alignas(16) cplx {
  double re, im;
};

PPF_HD double s_real(double a) { return a; }
PPF_HD double s_real(cplx a) { return a.re; }
PPF_HD double s_conj(double a) { return a; }
PPF_HD cplx s_conj(cplx a) { return {a.re, -a.im}; }
PPF_HD double s_add(double a, double b) { return a + b; }
PPF_HD cplx s_add(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
PPF_HD double s_sub(double a, double b) { return a - b; }
PPF_HD cplx s_sub(cplx a, cplx b) { return {a.re - b.re, a.im - b.im}; }
PPF_HD double s_mul(double a, double b) { return a * b; }
PPF_HD cplx s_mul(cplx a, cplx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
// a*b + c
PPF_HD double s_fma(double a, double b, double c) { return fma(a, b, c); }
PPF_HD cplx s_fma(cplx a, cplx b, cplx c) {
  return {fma(a.re, b.re, fma(-a.im, b.im, c.re)), fma(a.re, b.im, fma(a.im, b.re, c.im))};
}
// conj(a)*b + c
PPF_HD double s_cfma(double a, double b, double c) { return fma(a, b, c); }
PPF_HD cplx s_cfma(cplx a, cplx b, cplx c) {
  return {fma(a.re, b.re, fma(a.im, b.im, c.re)), fma(a.re, b.im, fma(-a.im, b.re, c.im))};
}
PPF_HD double s_abs2(double a) { return a * a; }
PPF_HD double s_abs2(cplx a) { return a.re * a.re + a.im * a.im; }
PPF_HD double s_scale(double a, double s) { return a * s; }
PPF_HD cplx s_scale(cplx a, double s) { return {a.re * s, a.im * s}; }
template <typename T> PPF_HD T s_zero();
template <> PPF_HD double s_zero<double>() { return 0.0; }
template <> PPF_HD cplx s_zero<cplx>() { return {0.0, 0.0}; }
template <typename T> PPF_HD T s_from(double re, double im);
template <> PPF_HD double s_from<double>(double re, double) { return re; }
template <> PPF_HD cplx s_from<cplx>(double re, double im) { return {re, im}; }
template <typename T> PPF_HD constexpr int n_doubles() { return sizeof(T) / sizeof(double); }

using zc = std::complex<double>;

// ---------------------------------------------------------------------------
// Errors
// ---------------------------------------------------------------------------
struct Error {
  ppf_status st;
  std::string msg;
};
[[noreturn]] void fail(ppf_status st, const std::string& msg);
void set_last_error(const std::string& msg);
void cuda_check(cudaError_t e, const char* what);
#define PPF_CUDA(call) ::ppf::cuda_check((call), #call)
#define PPF_REQUIRE(cond, msg) \
  do {                         \
    if (!(cond)) ::ppf::fail(PPF_EINVAL, msg); \
  } while (0)
// device vectors and scratch are read and written as 128-bit pairs (double2,
// complex128) and fed to cp.async.bulk: 16-byte alignment is required
#define PPF_REQUIRE_ALIGNED(p, name) \
  PPF_REQUIRE((reinterpret_cast<uintptr_t>(p) & 15) == 0, name " must be 16-byte aligned")

// ---------------------------------------------------------------------------
// Matrix layout
// ---------------------------------------------------------------------------
// SELL-C-sigma: slice s covers (permuted) local rows [s*C, s*C + C); its
// entries start at slice_ptr[s] (a multiple of C) and are stored
// [k][row-in-slice]: entry k of row r is at slice_ptr[s] + k*C + (r - s*C).
// Padding entries have val = 0 and col = the first row of the slice.
// CSR: row_ptr (int64) / col (int32) / val.
// Columns of the diagonal block are LOCAL indices; the off-diagonal (halo)
// block is a compact CSR over the rows that touch other ranks, columns index
// the halo receive buffer.
struct HostBlock {
  int64_t rows = 0;
  int64_t nslices = 0;
  std::vector<int64_t> ptr;    // SELL slice_ptr [nslices+1] or CSR row_ptr [rows+1]
  std::vector<int32_t> col;
  std::vector<double> val;     // n_doubles per entry
  std::vector<int32_t> perm;   // SELL sigma > 1: perm[pos] = original local row
  // SELL (C = 32, or C = 64 fp64; no sorting) with 16-bit column deltas
  // (round 2): column of entry (slice s, column k, slot t, row r = C s + t) =
  // r + cb[ptr[s]/C + k] + d16[ptr[s] + C k + t]; padding entries carry delta 0
  // (val 0).  Empty unless every (s, k) spans <= 65535 in (col - row).
  std::vector<uint16_t> d16;
  std::vector<int32_t> cb;
  // SELL-64 fp64 (no sorting) with dictionary-coded entries (round 2, "pair
  // codes"): entry (s, k, t) of row r = C s + t is the pair
  // (tab_off[c], tab_val[c]) with c = code8[(pptr[s] & ~511) + 512 (k / 8) +
  // 16 (t / 2) + 2 (k mod 8) + t mod 2] (lane-major chunks of 8 columns): column
  // r + tab_off[c] (clamped to the last row for the padding pair (0, +0.0)),
  // value tab_val[c].  Empty unless the block's entries (padding included)
  // take <= 256 distinct (col - row, value bits) pairs.
  std::vector<int64_t> pptr;   // pair codes' slice pointers (multiples of 512) | slice width
  std::vector<uint8_t> code8;
  std::vector<int32_t> tab_off;
  std::vector<double> tab_val;
  // slice schedule of the pair-code SpMV (optional): warp w of block b takes
  // slice sched[8 b + w] (-1: none).  Blocks are (y, z) tiles of slices whose
  // rows are each other's far neighbours (the pair table's two smallest
  // offsets >= C), so their x gathers meet in the SM's L1; empty = slices in
  // order, 8 per block.  Scheduling only: results are bitwise the same.
  std::vector<int32_t> sched;
};

struct HostHalo {
  std::vector<int32_t> rows;     // local rows with off-rank columns
  std::vector<int64_t> ptr;      // [rows.size()+1]
  std::vector<int32_t> col;      // index into the recv buffer
  std::vector<double> val;
};

}  // namespace ppf

struct ppf_plan {
  ppf_dtype dtype;
  int64_t n_global, row0, n_local, nnz;
  int nranks, rank;
  std::vector<int64_t> bounds;
  ppf_format fmt;
  int C, sigma;
  int enc = PPF_ENC_EXPLICIT;   // device layout of the diagonal block (ppf_encoding)
  ppf::HostBlock diag;
  ppf::HostHalo halo;
  std::vector<std::vector<int64_t>> recv;   // per peer: global indices received (sorted)
  std::vector<int64_t> recv_off;            // per peer offset into the recv buffer
  std::vector<std::vector<int64_t>> send;   // per peer: local rows to send
  bool sends_set = false;
};

namespace ppf {
struct PeerState;
}

struct ppf_mat {
  ppf_ctx* ctx;
  ppf_dtype dtype;
  ppf_format fmt;
  int64_t n_global, row0, n_local, nnz, stored;
  int C, sigma;
  int nranks, rank;
  int64_t nslices;
  const int64_t* d_ptr;     // slice_ptr or row_ptr
  const int32_t* d_col;
  const void* d_val;
  const int32_t* d_perm;    // null unless sigma > 1
  const uint16_t* d_d16 = nullptr;  // 16-bit column deltas (SELL), with d_cb
  const int32_t* d_cb = nullptr;    // per (slice, column) base offset (col - row)
  const uint8_t* d_code8 = nullptr; // pair codes (SELL-64 fp64), with d_tab_off / d_tab_val
  const int32_t* d_tab_off = nullptr;
  const double* d_tab_val = nullptr;
  int ntab = 0;
  // host copy of a small pair table (ntab <= 32): passed to sellp_kernel by
  // value, so its lookups go through the constant cache, not the L1 data pipe
  double h_tab_val[32] = {};
  int h_tab_off[32] = {};
  // codes uploaded pre-multiplied by 16 (tables of <= 16 pairs): each code byte
  // is then the byte offset of its 16-B record, one PRMT from the code word
  bool code_scaled = false;
  const int32_t* d_sched = nullptr;  // slice schedule (see HostBlock::sched), 8 per block
  int sched_blocks = 0;
  int csr_group;            // lanes per row for the CSR kernel
  int sell_ks;              // warps per SELL slice (1, 2, 4, 8), see auto_sell_ks
  int64_t sell_heavy = 0;   // leading slices given a whole block each (see sell_heavy_prefix)
  // halo (nranks > 1)
  int64_t halo_rows, halo_nnz, halo_total, send_total;
  const int32_t* d_halo_rows;
  const int64_t* d_halo_ptr;
  const int32_t* d_halo_col;
  const void* d_halo_val;
  void* d_recv;             // halo_total scalars
  void* d_send;             // send_total scalars
  const int32_t* d_send_idx;
  std::vector<int64_t> recv_count, recv_off, send_count, send_off;  // per peer
  ppf::PeerState* peer = nullptr;  // peer-memory window (peer.cu), null unless requested
};

struct ppf_poly {
  int kind;                         // ppf_poly_kind
  int deg;
  double a, b;                      // Chebyshev interval
  std::vector<double> c;            // Chebyshev coefficients c_0..c_deg
  std::vector<ppf::zc> nodes, dd;   // Newton form (Leja order)
  int newton_eval = 0;              // 0: Horner, 1: forward Newton basis, 2: real pairs
  std::vector<double> rp_a, rp_b2, rp_c;  // real-pair form (real_pair_form)
};

namespace ppf {

struct HistRec {
  int m;
  double est, err;
  long long mvms;
};

}  // namespace ppf

struct ppf_ctx {
  int device, rank, nranks;
  cudaStream_t stream;
  void* nccl_comm;            // ncclComm_t when nranks > 1
  // halo exchange overlap (nranks > 1 with a communicator): the NCCL
  // send/recv runs on comm_stream while the diagonal-block SpMV runs on
  // `stream`; ev_pack / ev_halo order the two streams
  cudaStream_t comm_stream;
  cudaEvent_t ev_pack, ev_halo;
  // host transport (ppf_ctx_set_transport) instead of NCCL
  bool has_transport = false;
  ppf_transport transport{};
  void* t_host = nullptr;      // pinned staging for halo send + recv / reductions
  size_t t_host_bytes = 0;
  int num_sms;
  // pinned host staging for H columns and y
  void* h_pinned;
  size_t h_pinned_bytes;
  cudaEvent_t ev;
  cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr;  // timing events: ppf_report.seconds_device
  void* res_ctl = nullptr;     // mapped pinned control block of the resident step loop
  size_t res_ctl_bytes = 0;
  // last run
  std::vector<ppf::HistRec> hist;
  std::vector<double> lastH;  // (m+1) x m, n_doubles per entry, column-major ld = m+1
  int last_m;
  double last_beta0;
  ppf_dtype last_dtype;
  long long launches;
  // optional per-kernel-class timing with CUDA events on the context stream
  int profile;
  int use_graphs = 1;         // CUDA-graph replay of the step's q(A)q(A) chain (ppf_ctx_set_graphs)
  cudaStream_t cap_stream = nullptr;  // private stream the chain is captured on
  std::vector<cudaEvent_t> prof_pool;
  struct ProfAcc {
    long long launches;
    double ms, bytes;
  } prof[3];  // 0 = SpMV (fused chain steps), 1 = orthogonalisation, 2 = other
};

namespace ppf {

// ---------------------------------------------------------------------------
// Host dense routines (dense.cpp)
// ---------------------------------------------------------------------------
// y = beta0 * T^{-1/2} e1 for symmetric tridiagonal T (diag d[m], offdiag e[m-1]).
void tridiag_invsqrt_e1(int m, const double* d, const double* e, double beta0, double* y);
// Complex Schur H = Q T Q^H of a general m x m matrix (column-major, ld = m).
struct CRot {  // a logged plane rotation of the complex Schur sweep (columns k, k+1)
  int k;
  double c;
  zc s;
};
void complex_schur(int m, std::vector<zc>& H, std::vector<zc>& Q, std::vector<CRot>* log = nullptr);
// y = beta0 * H^{-1/2} e1 via Schur -> triangular sqrt -> solve.
void general_invsqrt_e1(int m, const std::vector<zc>& H, double beta0, std::vector<zc>& y);
// y = beta0 * H^{-1/2} e1 for a REAL upper Hessenberg H (column-major, ld ldh):
// real Schur (Francis double shift) -> quasi-triangular square root -> solve.
void real_invsqrt_e1(int m, const double* H, int ldh, double beta0, double* y);
// f with H^H f = e_{m-1} (harmonic Ritz values)
std::vector<zc> solve_dense_adjoint_ed(int m, const std::vector<zc>& H);
// Eigenvalues of a general complex m x m matrix (column-major).
std::vector<zc> eigenvalues(int m, std::vector<zc> H);

// ---------------------------------------------------------------------------
// Polynomials (poly.cpp)
// ---------------------------------------------------------------------------
void chebyshev_coefficients(double a, double b, int deg, std::vector<double>& c);
double chebyshev_eval(const ppf_poly& q, double z);
zc poly_eval(const ppf_poly& q, zc z);
double certify_min_re(const ppf_poly& q, const void* pts, int npts, int dtype);
std::vector<zc> leja_order(const std::vector<zc>& nodes);
std::vector<zc> divided_differences_invsqrt(const std::vector<zc>& nodes);
void real_pair_form(ppf_poly& q);
std::vector<zc> ritz_polygon(const std::vector<zc>& theta, double r_min, double step);
void contour_ls_newton(const std::vector<zc>& z, int deg, std::vector<zc>& nodes,
                       std::vector<zc>& dd, double& min_re);

// ---------------------------------------------------------------------------
// Device kernels (kernels.cu): host-side launchers
// ---------------------------------------------------------------------------
struct Epi {          // out = s_ax*(A x) + s_x*xe + s_z*z + s_u*u
  double s_ax[2], s_x[2], s_z[2], s_u[2];
  const void* z;      // may be null (s_z ignored)
  const void* u;      // may be null (s_u ignored)
  const void* xe = nullptr;  // null: xe = x (the SpMV input); set for A = Q^2 chains
  // optional second output (forward Newton basis, Newton-eval mode 1):
  //   acc = (acc_init ? s_acc0*xe : acc) + s_acc*out
  void* acc = nullptr;
  double s_acc[2] = {0.0, 0.0}, s_acc0[2] = {0.0, 0.0};
  bool acc_init = false;
};

int auto_sell_ks(const ppf_mat* m, int num_sms);
void launch_spmv(ppf_mat* A, const void* x, void* out, const Epi& e, cudaStream_t st);
void launch_halo_pack(ppf_mat* A, const void* x, cudaStream_t st);
// the second output of an Epi with acc set, from a completed `out` (x: the SpMV input)
void launch_acc(ppf_mat* A, const void* x, const void* out, const Epi& e, cudaStream_t st);
// recv: the receive buffer to read (null: A->d_recv)
void launch_halo_apply(ppf_mat* A, void* out, const double* s_ax, cudaStream_t st,
                       const void* recv = nullptr, const unsigned* recv_sel = nullptr);
const void* kernels_module_symbol();
// peer.cu: the peer-memory exchange (ppf_mat_peer_window / _connect)
void peer_destroy(PeerState* p);
bool peer_active(const ppf_mat* A);
// force-load every kernel of the library (multi-rank contexts): under lazy
// module loading a first launch waits for the device, which a rank blocked in
// a collective or a peer wait would turn into a cross-rank stall
void preload_kernels();
void peer_halo_begin(ppf_ctx* ctx, ppf_mat* A, const void* x, cudaStream_t st);
// returns the receive slots' base; *sel = the device word whose parity picks the slot
const void* peer_halo_wait(ppf_ctx* ctx, ppf_mat* A, cudaStream_t st, const unsigned** sel);
void peer_halo_done(ppf_ctx* ctx, ppf_mat* A, cudaStream_t st);
void peer_allreduce(ppf_ctx* ctx, ppf_mat* A, double* raw, int nv, cudaStream_t st);
// run.cpp: the sharded SpMV with communication/compute overlap
void halo_spmv(ppf_ctx* ctx, ppf_mat* A, const void* x, void* out, const Epi& e,
               cudaStream_t st = nullptr);
bool poly_fits(const ppf_poly* q, ppf_dtype dt);

struct RedScratch {   // reduction scratch (device)
  double* partials;   // [max_blocks * max_vals * 2]
  unsigned* counter;  // zero-initialised, self-resetting
  int max_blocks;
  // multi-rank: when non-null the last block stores the rank-local sums here
  // (no finalisation); the caller allreduces them and calls launch_finalize
  double* raw = nullptr;
};
enum { FIN_NORM = 0, FIN_SQRT = 1, FIN_COEF = 2, FIN_SUBNORM = 3, FIN_LZ1 = 4, FIN_LZ2 = 5 };
void launch_finalize(int op, int nv, int nd, const double* raw, void* o0, void* o1, void* o2,
                     const void* ci, cudaStream_t st);
// dst = alpha * src (alpha read from device double *alpha_dev if non-null, else alpha_host)
void launch_scale(ppf_dtype dt, int64_t n, const void* src, void* dst, const double* alpha_dev,
                  double alpha_host, cudaStream_t st);
// res[0] = ||v||^2 partial -> nrm_out[0] = ||v||, nrm_out[1] = 1/||v||
void launch_norm(ppf_dtype dt, int64_t n, const void* v, double* nrm_out, RedScratch& rs, int grid,
                 cudaStream_t st);
// CGS kernels on V (ld = ldv, columns 0..ncols-1), w (in place).
//   mode 0: coef_out[0:ncols] = V^H w
//   mode 1: w -= V coef_in ; coef_out = V^H w ; H[:,j] = coef_in + coef_out
//   mode 2: w -= V coef_in ; H[j+1,j] = ||w||, inv[0] = 1/||w||
// resident step loop (kernels.cu): mapped host control block and the chain
constexpr int RES_MAX_ROWS = 4096;
constexpr int RES_AHEAD = 4;
constexpr unsigned long long RES_WAIT_NS = 200000;  // the device's longest wait for the host
struct ResCtl {
  int stop;      // host -> device: stop before the next step
  int acked;     // host -> device: steps the host has decided (the device runs <= RES_AHEAD past)
  int done;      // device -> host: steps completed (H columns 0..done-1 written)
  int pad;
  double beta0;  // device -> host: ||c||
  double H[1];   // device -> host: H columns, (ldh x (m_max+1)) scalars, column-major
};
struct ResCallSpec {
  const void* x;
  void* out;
  Epi e;
};
bool resident_fits(const ppf_mat* A);
size_t resident_call_bytes(ppf_dtype dt);
void resident_pack_calls(ppf_dtype dt, const std::vector<ResCallSpec>& spec, void* dst);
void launch_resident(ppf_mat* A, void* V, int64_t ldv, void* U, void* W, void* H, int ldh,
                     int m_max, int lanczos, const double* beta0_dev, ResCtl* ctl_dev,
                     const void* calls_dev, int ncalls, int ahead, cudaStream_t st);
int launch_cgs(ppf_dtype dt, int mode, int64_t n, const void* V, int64_t ldv, int ncols, void* w,
                const void* coef_in, void* coef_out, void* Hcol, void* Hsub, double* inv,
                RedScratch& rs, int grid, cudaStream_t st);
// Lanczos: phase 1: w -= beta_prev * vprev (if vprev); alpha = v^H w -> Hdiag (real part kept)
//          phase 2: w -= alpha v; beta = ||w|| -> Hsub, Hsup; inv = 1/beta
void launch_lanczos(ppf_dtype dt, int phase, int64_t n, const void* v, const void* vprev,
                    const double* beta_prev, void* w, void* Hdiag, void* Hsub, void* Hsup,
                    double* inv, RedScratch& rs, int grid, cudaStream_t st);
// two-pass Lanczos pass 2: w <- (w - alpha v - beta_prev vprev) * inv_beta; x += ycoef * w
void launch_lanczos_regen(ppf_dtype dt, int64_t n, void* w, const void* v, const void* vprev,
                          double alpha, double beta_prev, double inv_beta, double ycoef, void* x,
                          cudaStream_t st);
// x = V y (y device, ncols entries)
void launch_combine(ppf_dtype dt, int64_t n, const void* V, int64_t ldv, int ncols, const void* y,
                    void* x, cudaStream_t st);
// out[0] = ||a - b||, out[1] = ||b||
void launch_diffnorm(ppf_dtype dt, int64_t n, const void* a, const void* b, double* out,
                     RedScratch& rs, int grid, cudaStream_t st);

}  // namespace ppf
