// The run (layers L2-L5): Algorithm 1 of the paper on the device,
// f(H_m) on the host, x = V_m y_m on the device.
//
// Per step j (0-based; basis column j is v_{j+1} of the paper):
//   u = A v_j                      -> U            (1 SpMV)
//   y = q(A) u                     -> Y            (deg fused SpMV launches)
//   w = q(A) y                     -> V[:, j+1]    (deg fused SpMV launches)
//   orthogonalise w in place (Lanczos: 2 fused sweeps; CGS2: 3 fused sweeps)
//   v_{j+1} = w / h_{j+1,j}        (scale)
// H lives on the device; the host reads it only at checkpoints (estimate /
// true error) and at the end.  q(A) is the Clenshaw recurrence (P:332,
// reading Q4) or the Newton-Horner scheme, each SpMV's epilogue
// carrying the recurrence's vector updates.
#include <atomic>
#include <thread>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstring>
#include <deque>
#include <future>
#include <utility>

#include "ppf_internal.h"

namespace ppf {

namespace {

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

// Workspace shape: which bases the run keeps.
enum { WS_RIGHT = 1,     // right preconditioning, one-pass: Y_m (m_max columns)
       WS_TWOPASS = 2,   // two-pass Lanczos: V = {v_1, ring of 3}, + accumulator XA
       WS_SQUARE = 4,    // operator A = Q^2: + the intermediate Q x (TSQ)
       WS_GRAPH = 8 };   // CUDA-graph step: + the fixed output W2 of the captured q(A)q(A) chain

struct WsLayout {
  int64_t ldv;       // leading dimension of V and vector length (padded)
  int ldh;           // leading dimension of H
  int vcols;         // columns of V
  size_t V, Yb, U, Y, T0, T1, T2, XA, TSQ, W2, H, hbuf, gbuf, ybuf, ybuf2, scal, partials,
      counter, raw, total;
  int max_blocks;
  int max_vals;
};

WsLayout ws_layout(int64_t n, ppf_dtype dt, int m_max, int num_sms, int shape = 0) {
  const size_t sc = dt == PPF_R64 ? 8 : 16;
  WsLayout L{};
  L.ldv = (n + 63) & ~int64_t(63);
  L.ldh = m_max + 2;
  L.max_blocks = std::max(8 * num_sms, 256);
  L.max_vals = (m_max + 2) * 2;
  L.vcols = (shape & WS_TWOPASS) ? 4 : m_max + 1;
  size_t o = 0;
  const size_t vec = al256(size_t(L.ldv) * sc);
  L.V = o;
  o += vec * size_t(L.vcols);
  L.Yb = o;
  if (shape & WS_RIGHT) o += vec * size_t(m_max);
  L.U = o;
  o += vec;
  L.Y = o;
  o += vec;
  L.T0 = o;
  o += vec;
  L.T1 = o;
  o += vec;
  L.T2 = o;
  o += vec;
  L.XA = o;
  if (shape & WS_TWOPASS) o += vec;
  L.TSQ = o;
  if (shape & WS_SQUARE) o += vec;
  L.W2 = o;
  if (shape & WS_GRAPH) o += vec;
  L.H = o;
  o += al256(size_t(L.ldh) * (m_max + 1) * sc);
  L.hbuf = o;
  o += al256(size_t(m_max + 2) * sc);
  L.gbuf = o;
  o += al256(size_t(m_max + 2) * sc);
  L.ybuf = o;
  o += al256(size_t(m_max + 2) * sc);
  L.ybuf2 = o;
  o += al256(size_t(m_max + 2) * sc);
  L.scal = o;
  o += 256;
  L.partials = o;
  o += al256(size_t(L.max_blocks) * L.max_vals * 8);
  L.counter = o;
  o += 256;
  L.raw = o;
  o += al256(size_t(L.max_vals) * 8);
  L.total = o;
  return L;
}

}  // namespace

// a polynomial the operator's arithmetic can apply: Chebyshev always, Newton on
// a real operator only with real nodes and divided differences
bool poly_fits(const ppf_poly* q, ppf_dtype dt) {
  if (q->kind == PPF_POLY_CHEBYSHEV || dt == PPF_C128 || q->newton_eval == 2) return true;
  for (size_t i = 0; i < q->nodes.size(); ++i)
    if (q->nodes[i].imag() != 0.0 || q->dd[i].imag() != 0.0) return false;
  return true;
}

namespace {

bool squared(const ppf_opts* o) { return o->func == PPF_INVSQRT_SQ || o->func == PPF_SIGN; }

int ws_shape(const ppf_poly* q, const ppf_opts* o) {
  int s = squared(o) ? WS_SQUARE : 0;
  if (o->krylov == PPF_LANCZOS_2PASS) s |= WS_TWOPASS;
  else if (q && o->precond == PPF_PREC_RIGHT) s |= WS_RIGHT;
  // left-preconditioned one-pass steps can replay their q(A)q(A) chain as a CUDA graph
  if (q && q->deg >= 1 && o->precond == PPF_PREC_LEFT && o->krylov != PPF_LANCZOS_2PASS)
    s |= WS_GRAPH;
  return s;
}

// scalar slots (doubles) in the scal area
enum { S_BETA0 = 0, S_INV0 = 1, S_INV = 2, S_ERR = 4, S_REF = 5 };

// Halo exchange of the packed boundary entries: one grouped
// NCCL send/recv per peer with a non-empty list, on stream `cs`.
void halo_sendrecv(ppf_ctx* ctx, ppf_mat* A, cudaStream_t cs) {
  auto comm = static_cast<ncclComm_t>(ctx->nccl_comm);
  if (!comm) fail(PPF_ESTATE, "nranks > 1 needs a context with an NCCL communicator");
  const size_t sc = A->dtype == PPF_R64 ? 8 : 16;
  const int nd = int(sc / 8);
  if (ncclGroupStart() != ncclSuccess) fail(PPF_ENCCL, "ncclGroupStart");
  for (int p = 0; p < A->nranks; ++p) {
    if (A->send_count[p])
      if (ncclSend(static_cast<char*>(A->d_send) + A->send_off[p] * sc, A->send_count[p] * nd,
                   ncclDouble, p, comm, cs) != ncclSuccess)
        fail(PPF_ENCCL, "ncclSend");
    if (A->recv_count[p])
      if (ncclRecv(static_cast<char*>(A->d_recv) + A->recv_off[p] * sc, A->recv_count[p] * nd,
                   ncclDouble, p, comm, cs) != ncclSuccess)
        fail(PPF_ENCCL, "ncclRecv");
  }
  if (ncclGroupEnd() != ncclSuccess) fail(PPF_ENCCL, "ncclGroupEnd");
}

}  // namespace

// The sharded SpMV, out = epilogue(A x) on this rank's slab, with the halo
// exchange overlapped by the diagonal-block product:
//   stream:       pack boundary entries of x -> [ev_pack] ........ diag-block SpMV + epilogue -> wait ev_halo -> halo block
//   comm_stream:             wait ev_pack -> NCCL send/recv -> [ev_halo]
// The halo block adds s_ax * A_offdiag x_halo to out (the epilogue is linear
// in A x, so the split is exact).  Buffer reuse is ordered by the streams:
// the next pack (stream) follows this halo block, which followed ev_halo.
// pinned host staging of the host transport, grown on demand
static double* transport_stage(ppf_ctx* ctx, size_t bytes) {
  if (ctx->t_host_bytes < bytes) {
    PPF_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->t_host) PPF_CUDA(cudaFreeHost(ctx->t_host));
    ctx->t_host = nullptr;
    ctx->t_host_bytes = 0;
    PPF_CUDA(cudaHostAlloc(&ctx->t_host, bytes, cudaHostAllocDefault));
    ctx->t_host_bytes = bytes;
  }
  return static_cast<double*>(ctx->t_host);
}

// the halo exchange through the caller's host transport (no overlap: a
// verification path, see ppf_ctx_set_transport)
static void halo_transport(ppf_ctx* ctx, ppf_mat* A, const void* x) {
  cudaStream_t st = ctx->stream;
  const size_t sc = A->dtype == PPF_R64 ? 8 : 16;
  const int nd = int(sc / 8);
  launch_halo_pack(A, x, st);
  double* hs = transport_stage(ctx, size_t(A->send_total + A->halo_total) * sc + 64);
  double* hr = hs + size_t(A->send_total) * nd;
  if (A->send_total)
    PPF_CUDA(cudaMemcpyAsync(hs, A->d_send, size_t(A->send_total) * sc, cudaMemcpyDeviceToHost, st));
  PPF_CUDA(cudaStreamSynchronize(st));
  std::vector<int64_t> scount(A->nranks), rcount(A->nranks);
  for (int p = 0; p < A->nranks; ++p) {
    scount[p] = A->send_count[p] * nd;
    rcount[p] = A->recv_count[p] * nd;
  }
  if (ctx->transport.exchange(ctx->transport.user, hs, scount.data(), hr, rcount.data()) != 0)
    fail(PPF_ENCCL, "transport exchange failed");
  if (A->halo_total)
    PPF_CUDA(cudaMemcpyAsync(A->d_recv, hr, size_t(A->halo_total) * sc, cudaMemcpyHostToDevice, st));
  PPF_CUDA(cudaStreamSynchronize(st));  // the staging is reused by the next call
}

void halo_spmv(ppf_ctx* ctx, ppf_mat* A, const void* x, void* out, const Epi& e,
               cudaStream_t st_in) {
  // st_in: the stream of the caller's SpMV sequence (a capture stream while the
  // step's chain is recorded as a CUDA graph), else the context's
  cudaStream_t st = st_in ? st_in : ctx->stream;
  if (peer_active(A)) {
    // peer memory (peer.cu): push on the comm stream || diagonal block here
    const bool comm = A->send_total || A->halo_total;
    if (comm) peer_halo_begin(ctx, A, x, st);
    Epi ed = e;
    ed.acc = nullptr;
    launch_spmv(A, x, out, ed, st);
    const unsigned* sel = nullptr;
    const void* recv = comm ? peer_halo_wait(ctx, A, st, &sel) : nullptr;
    if (A->halo_rows) launch_halo_apply(A, out, e.s_ax, st, recv, sel);
    if (comm) peer_halo_done(ctx, A, st);
    if (e.acc) launch_acc(A, x, out, e, st);
    return;
  }
  if (ctx->has_transport) {
    halo_transport(ctx, A, x);
    Epi ed = e;
    ed.acc = nullptr;
    launch_spmv(A, x, out, ed, st);
    if (A->halo_rows) launch_halo_apply(A, out, e.s_ax, st);
    if (e.acc) launch_acc(A, x, out, e, st);
    return;
  }
  if (A->send_total || A->halo_total) {
    if (!ctx->nccl_comm)
      fail(PPF_ESTATE, "nranks > 1 needs an NCCL communicator, a transport or a peer window");
    launch_halo_pack(A, x, st);
    PPF_CUDA(cudaEventRecord(ctx->ev_pack, st));
    PPF_CUDA(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_pack, 0));
    halo_sendrecv(ctx, A, ctx->comm_stream);
    PPF_CUDA(cudaEventRecord(ctx->ev_halo, ctx->comm_stream));
  }
  Epi ed = e;
  ed.acc = nullptr;  // the second output needs the complete out: after the halo block
  launch_spmv(A, x, out, ed, st);
  if (A->send_total || A->halo_total) PPF_CUDA(cudaStreamWaitEvent(st, ctx->ev_halo, 0));
  if (A->halo_rows) launch_halo_apply(A, out, e.s_ax, st);
  if (e.acc) launch_acc(A, x, out, e, st);
}

// Grow the context's pinned host staging to `need` bytes.  Pinned allocation
// and release synchronise the device, so the workspace queries call this
// ahead of a run: a sharded run on peer memory must not stall here while a
// neighbour's stream waits for this rank (peer.cu).
void ensure_pinned(ppf_ctx* ctx, size_t need) {
  if (ctx->h_pinned_bytes >= need) return;
  PPF_CUDA(cudaStreamSynchronize(ctx->stream));
  PPF_CUDA(cudaFreeHost(ctx->h_pinned));
  ctx->h_pinned = nullptr;
  ctx->h_pinned_bytes = 0;
  PPF_CUDA(cudaHostAlloc(&ctx->h_pinned, need, cudaHostAllocDefault));
  ctx->h_pinned_bytes = need;
}

size_t pinned_need(const WsLayout& L, int m_max, size_t sc) {
  return al256(size_t(L.ldh) * (m_max + 1) * sc + 64) + 2 * al256(size_t(m_max + 2) * 16);
}

namespace {

struct Runner {
  ppf_ctx* ctx;
  ppf_mat* A;
  const ppf_poly* q;  // may be null for the plain (Ritz setup) operator
  ppf_dtype dt;
  int64_t n;
  size_t sc;
  WsLayout L;
  char* w;
  cudaStream_t st;
  RedScratch rs;
  int grid_vec, grid_cgs;
  long long launches = 0;
  bool dist = false;  // row-slab sharded over nranks > 1 (NCCL)

  // multi-rank: allreduce the rank-local sums a reduction kernel left in rs.raw,
  // then finalise them (sqrt, H entries, 1/norm) on the device; no-op on 1 rank.
  void reduce_fin(int op, int nv, void* o0, void* o1, void* o2, const void* ci) {
    if (!dist) return;
    if (peer_active(A)) {
      peer_allreduce(ctx, A, rs.raw, nv, st);
    } else if (ctx->has_transport) {
      double* hb = transport_stage(ctx, size_t(nv) * 8 + 64);
      PPF_CUDA(cudaMemcpyAsync(hb, rs.raw, size_t(nv) * 8, cudaMemcpyDeviceToHost, st));
      PPF_CUDA(cudaStreamSynchronize(st));
      if (ctx->transport.allreduce_sum(ctx->transport.user, hb, nv) != 0)
        fail(PPF_ENCCL, "transport allreduce failed");
      PPF_CUDA(cudaMemcpyAsync(rs.raw, hb, size_t(nv) * 8, cudaMemcpyHostToDevice, st));
      PPF_CUDA(cudaStreamSynchronize(st));
    } else if (ncclAllReduce(rs.raw, rs.raw, size_t(nv), ncclDouble, ncclSum,
                             static_cast<ncclComm_t>(ctx->nccl_comm), st) != ncclSuccess) {
      fail(PPF_ENCCL, "ncclAllReduce");
    }
    timed(2, 0.0, [&] { launch_finalize(op, nv, int(sc / 8), rs.raw, o0, o1, o2, ci, st); });
  }

  bool right = false;    // Algorithm 2 (y_j = q(A) v_j first, w = A q(A) y_j)
  bool twopass = false;  // V is {v_1, ring of 3}

  Runner(ppf_ctx* c, ppf_mat* a, const ppf_poly* qq, int m_max, void* work, size_t bytes,
         int shape = 0, bool right_prec = false)
      : ctx(c), A(a), q(qq), dt(a->dtype), n(a->n_local) {
    sc = dt == PPF_R64 ? 8 : 16;
    L = ws_layout(n, dt, m_max, c->num_sms, shape);
    right = right_prec && q;
    twopass = shape & WS_TWOPASS;
    if (!work || bytes < L.total) fail(PPF_EWORKSPACE, "workspace too small");
    if (reinterpret_cast<uintptr_t>(work) & 255) fail(PPF_EINVAL, "workspace not 256-B aligned");
    w = static_cast<char*>(work);
    st = c->stream;
    rs.partials = reinterpret_cast<double*>(w + L.partials);
    rs.counter = reinterpret_cast<unsigned*>(w + L.counter);
    rs.max_blocks = L.max_blocks;
    dist = A->nranks > 1;
    if (dist) {
      if (!c->nccl_comm && !c->has_transport && !peer_active(A))
        fail(PPF_ESTATE, "nranks > 1 needs an NCCL communicator, a transport or a peer window");
      rs.raw = reinterpret_cast<double*>(w + L.raw);
    }
    grid_vec = std::min(L.max_blocks, 4 * c->num_sms);
    grid_cgs = std::min(L.max_blocks, c->num_sms);  // persistent CGS kernel: one CTA per SM
    PPF_CUDA(cudaMemsetAsync(w + L.counter, 0, 256, st));
    PPF_CUDA(cudaMemsetAsync(w + L.H, 0, size_t(L.ldh) * (m_max + 1) * sc, st));
    // pinned host staging: H (and beta0), then two coefficient-vector slots;
    // grown on demand (the context keeps the largest)
    stage_h = al256(size_t(L.ldh) * (m_max + 1) * sc + 64);
    stage_y = al256(size_t(m_max + 2) * 16);
    ensure_pinned(ctx, stage_h + 2 * stage_y);
  }
  size_t stage_h = 0, stage_y = 0;

  void* V(int j) { return w + L.V + size_t(j) * al256(size_t(L.ldv) * sc); }
  void* Yb(int j) { return w + L.Yb + size_t(j) * al256(size_t(L.ldv) * sc); }
  // basis vectors of step j: v_j (source), w -> v_{j+1} (destination), v_{j-1}
  void* vsrc(int j) { return twopass ? V(1 + j % 3) : V(j); }
  void* vdst(int j) { return twopass ? V(1 + (j + 1) % 3) : V(j + 1); }
  void* vprv(int j) { return j == 0 ? nullptr : (twopass ? V(1 + (j + 2) % 3) : V(j - 1)); }
  void* vec(size_t off) { return w + off; }
  void* Hp(int i, int j) { return w + L.H + (size_t(i) + size_t(j) * L.ldh) * sc; }
  double* scal(int i) { return reinterpret_cast<double*>(w + L.scal) + i; }

  // ----- recording of a step's SpMV sequence (for look-ahead enqueueing) -----
  struct Call {
    const void* x;
    void* out;
    Epi e;
    bool scale;   // out = c * x (degree-0 polynomial) instead of an SpMV
    double c;
    bool graph = false;  // replay the captured q(A)q(A) chain (U -> W2)
  };
  std::vector<Call>* rec = nullptr;

  void play(const Call& c) {
    if (c.graph) {
      run_graph();
      return;
    }
    if (c.scale)
      timed(2, 2.0 * n * sc, [&] { launch_scale(dt, n, c.x, c.out, nullptr, c.c, st); });
    else
      spmv_now(c.x, c.out, c.e);
  }

  // the SpMV / scale sequence of step j (w = Op v_j), not launched
  std::vector<Call> record_step(int j) {
    std::vector<Call> v;
    rec = &v;
    op_apply(j);
    rec = nullptr;
    return v;
  }

  // ----- SpMV with halo exchange (nranks > 1) -----
  // A x with its fused epilogue.  power == 2 (A = Q^2): two
  // launches, t = Q x, then out = s_ax Q t + s_x x + s_z z + s_u u -- the
  // epilogue's x term reads the chain vector x, not the launch input t.
  int power = 1;
  void spmv(const void* x, void* out, const Epi& e) {
    if (power == 2) {
      spmv1(x, vec(L.TSQ), epi(1.0, 0.0, 0.0, nullptr, 0.0, nullptr));
      Epi e2 = e;
      if (!e2.xe) e2.xe = x;
      spmv1(vec(L.TSQ), out, e2);
      return;
    }
    spmv1(x, out, e);
  }
  void spmv1(const void* x, void* out, const Epi& e) {
    if (rec) {
      rec->push_back({x, out, e, false, 0.0});
      return;
    }
    spmv_now(x, out, e);
  }

  void spmv_now(const void* x, void* out, const Epi& e) {
    // algorithmic bytes: values + column indices once, x gathered once, out
    // written once, z and u streamed once
    // (index bytes per entry: 4, or 2 + 4/C with the 16-bit column deltas;
    // with the pair codes one byte per entry carries column and value)
    const double idxb = A->d_d16 ? 2.0 + 4.0 / double(A->C) : 4.0;
    const double entb = A->d_code8 ? 1.0 : double(sc) + idxb;
    const double bytes = entb * double(A->nnz) +
                         double(sc) * double(n) * (2 + (e.z ? 1 : 0) + (e.u ? 1 : 0));
    if (A->nranks > 1) {
      // pack + overlapped exchange + diagonal block + halo block; timed as one
      // unit (its device time includes any exposed communication)
      launches += (A->send_total ? 1 : 0) + (A->halo_rows ? 1 : 0) +
                  ((peer_active(A) && (A->send_total || A->halo_total)) ? 1 : 0);
      timed(0, bytes, [&] { halo_spmv(ctx, A, x, out, e, st); });
      return;
    }
    timed(0, bytes, [&] { launch_spmv(A, x, out, e, st); });
  }

  static Epi epi(zc sax, zc sx, zc sz, const void* z, zc su, const void* u) {
    Epi e;
    e.s_ax[0] = sax.real();
    e.s_ax[1] = sax.imag();
    e.s_x[0] = sx.real();
    e.s_x[1] = sx.imag();
    e.s_z[0] = sz.real();
    e.s_z[1] = sz.imag();
    e.s_u[0] = su.real();
    e.s_u[1] = su.imag();
    e.z = z;
    e.u = u;
    return e;
  }

  // out = c * in (complex c allowed for C128)
  void lincomb(const void* in, void* out, zc c) {
    // a SpMV-free scaled copy: reuse the SpMV epilogue would need A; use scale
    if (c.imag() != 0.0 && dt == PPF_R64) fail(PPF_EINVAL, "complex coefficient on a real operator");
    if (c.imag() == 0.0) {
      if (rec) {
        rec->push_back({in, out, Epi{}, true, c.real()});
        return;
      }
      timed(2, 2.0 * n * sc, [&] { launch_scale(dt, n, in, out, nullptr, c.real(), st); });
    } else {
      fail(PPF_EINVAL, "degree-0 complex Newton polynomial not supported");
    }
  }

  // out = q(A) in.  T0..T2 rotation buffers; in/out distinct from them.
  void apply_q(const void* in, void* out) {
    void* T[3] = {vec(L.T0), vec(L.T1), vec(L.T2)};
    const int d = q->deg;
    if (q->kind == PPF_POLY_CHEBYSHEV) {
      const double alpha = 2.0 / (q->b - q->a), beta = -(q->a + q->b) / (q->b - q->a);
      const std::vector<double>& c = q->c;
      if (d == 0) {
        lincomb(in, out, c[0]);
        return;
      }
      if (d == 1) {  // out = Ahat(c1 u) + c0 u
        spmv(in, out, epi(alpha * c[1], beta * c[1] + c[0], 0.0, nullptr, 0.0, nullptr));
        return;
      }
      // b_{d-1} = 2 Ahat (c_d u) + c_{d-1} u
      spmv(in, T[0], epi(2.0 * alpha * c[d], 2.0 * beta * c[d] + c[d - 1], 0.0, nullptr, 0.0,
                         nullptr));
      // index of buffers holding b_{i+1} (cur) and b_{i+2} (prev); b_d = c_d u is implicit
      int cur = 0, prev = -1;
      for (int i = d - 2; i >= 1; --i) {
        int nxt = 0;
        while (nxt == cur || nxt == prev) ++nxt;
        if (prev < 0)  // b_{i+2} = b_d = c_d u
          spmv(T[cur], T[nxt], epi(2.0 * alpha, 2.0 * beta, 0.0, nullptr, c[i] - c[d], in));
        else
          spmv(T[cur], T[nxt], epi(2.0 * alpha, 2.0 * beta, -1.0, T[prev], c[i], in));
        prev = cur;
        cur = nxt;
      }
      // out = Ahat b_1 - b_2 + c_0 u
      if (prev < 0)
        spmv(T[cur], out, epi(alpha, beta, 0.0, nullptr, c[0] - c[d], in));
      else
        spmv(T[cur], out, epi(alpha, beta, -1.0, T[prev], c[0], in));
    } else if (q->newton_eval == 2) {
      // real conjugate-pair form (real_pair_form): P_0 = v, P_{j+1} =
      // (A - a_j) P_j [+ b_j^2 P_{j-1}], out = sum c_j P_j carried as the
      // SpMV's second output -- real arithmetic for a real operator whose
      // Ritz values come in complex pairs; three rotating buffers
      const auto& ra = q->rp_a;
      const auto& rb = q->rp_b2;
      const auto& rc = q->rp_c;
      if (d == 0) {
        lincomb(in, out, rc[0]);
        return;
      }
      const void* pm1 = nullptr;  // P_{j-1}
      const void* pj = in;        // P_j
      for (int j = 0; j < d; ++j) {
        void* dst = T[j % 3];
        Epi e = epi(1.0, -ra[j], rb[j], rb[j] != 0.0 ? pm1 : nullptr, 0.0, nullptr);
        e.acc = out;
        e.s_acc[0] = rc[j + 1];
        if (j == 0) {
          e.acc_init = true;
          e.s_acc0[0] = rc[0];
        }
        spmv(pj, dst, e);
        pm1 = pj;
        pj = dst;
      }
    } else if (q->newton_eval == 1) {
      // forward Newton basis: p_0 = v, p_{j+1} = (A - theta_j) p_j,
      // out = sum_j dd_j p_j accumulated by the SpMV's second output (the
      // first step initialises out = dd_0 v + dd_1 p_1); the basis is
      // numerically preferable to Horner when spec(A) reaches far beyond the
      // nodes (the graph Laplacian, Q28)
      const auto& dd = q->dd;
      const auto& th = q->nodes;
      if (d == 0) {
        lincomb(in, out, dd[0]);
        return;
      }
      const void* src = in;
      for (int j = 0; j < d; ++j) {
        void* dst = T[j % 2];
        Epi e = epi(1.0, -th[j], 0.0, nullptr, 0.0, nullptr);
        e.acc = out;
        e.s_acc[0] = dd[j + 1].real();
        e.s_acc[1] = dd[j + 1].imag();
        if (j == 0) {
          e.acc_init = true;
          e.s_acc0[0] = dd[0].real();
          e.s_acc0[1] = dd[0].imag();
        }
        spmv(src, dst, e);
        src = dst;
      }
    } else {
      // Horner on the Newton form: w = dd_d v; w = (A - theta_j) w + dd_j v, j = d-1..0
      const auto& dd = q->dd;
      const auto& th = q->nodes;
      if (d == 0) {
        lincomb(in, out, dd[0]);
        return;
      }
      if (d == 1) {
        spmv(in, out, epi(dd[1], -th[0] * dd[1] + dd[0], 0.0, nullptr, 0.0, nullptr));
        return;
      }
      spmv(in, T[0], epi(dd[d], -th[d - 1] * dd[d] + dd[d - 1], 0.0, nullptr, 0.0, nullptr));
      int cur = 0;
      for (int j = d - 2; j >= 1; --j) {
        const int nxt = (cur + 1) % 2;
        spmv(T[cur], T[nxt], epi(1.0, -th[j], 0.0, nullptr, dd[j], in));
        cur = nxt;
      }
      spmv(T[cur], out, epi(1.0, -th[0], 0.0, nullptr, dd[0], in));
    }
  }

  // w = Op v_j into vdst(j).  Op = A (q == null, plain method);
  // left (Alg 1 line 4): u = A v_j, y = q(A)u, w = q(A)y;
  // right (Alg 2 line 4): y_j = q(A)v_j (kept in Y_m one-pass), u = q(A)y_j, w = A u.
  void op_apply(int j) {
    const Epi plain = epi(1.0, 0.0, 0.0, nullptr, 0.0, nullptr);
    if (!q) {
      spmv(vsrc(j), vdst(j), plain);
    } else if (right) {
      void* yj = twopass ? vec(L.Y) : Yb(j);
      apply_q(vsrc(j), yj);
      apply_q(yj, vec(L.U));
      spmv(vec(L.U), vdst(j), plain);
    } else if (use_graph) {
      spmv(vsrc(j), vec(L.U), plain);
      if (rec)
        rec->push_back({nullptr, nullptr, Epi{}, false, 0.0, true});
      else
        run_graph();
    } else {
      spmv(vsrc(j), vec(L.U), plain);
      apply_q(vec(L.U), vec(L.Y));
      apply_q(vec(L.Y), vdst(j));
    }
  }

  // ----- CUDA graph of the step's q(A) q(A) chain (left preconditioning) -----
  // Its 2 deg (x power) SpMV launches always read U and write W2 through the
  // same buffers, so one capture serves every step: each step is then one
  // plain SpMV (v_j -> U), one graph launch and the orthogonalisation, which
  // takes w from W2 and writes v_{j+1}.  Launch-bound steps (C1, C2, small
  // n) lose most of their per-kernel host cost and inter-kernel gaps.
  bool use_graph = false;
  cudaGraphExec_t gexec = nullptr;
  long long graph_kernels = 0;
  void run_graph() {
    if (!gexec) {
      // capture on the context's private stream (the caller's may be the
      // legacy default stream, which cannot capture); replay on the caller's
      if (!ctx->cap_stream) PPF_CUDA(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
      const long long before = launches;
      cudaStream_t user = st;
      cudaGraph_t g = nullptr;
      st = ctx->cap_stream;
      PPF_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      try {
        apply_q(vec(L.U), vec(L.Y));
        apply_q(vec(L.Y), vec(L.W2));
      } catch (...) {
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        st = user;
        throw;
      }
      PPF_CUDA(cudaStreamEndCapture(st, &g));
      st = user;
      PPF_CUDA(cudaGraphInstantiate(&gexec, g, 0));
      PPF_CUDA(cudaGraphDestroy(g));
      graph_kernels = launches - before;
      launches = before;
    }
    PPF_CUDA(cudaGraphLaunch(gexec, st));
    launches += graph_kernels;
  }
  ~Runner() {
    if (gexec) cudaGraphExecDestroy(gexec);
  }
  // where step j's w = Op v_j lands: W2 with the graph, else v_{j+1} itself
  void* wbuf(int j) { return use_graph ? vec(L.W2) : vdst(j); }

  void orthogonalise(int j, bool lanczos) {
    const double vb = double(n) * double(sc);
    if (lanczos) {
      const double* bprev = j > 0 ? reinterpret_cast<const double*>(Hp(j, j - 1)) : nullptr;
      timed(1, vb * (j > 0 ? 4 : 3), [&] {
        launch_lanczos(dt, 1, n, vsrc(j), vprv(j), bprev, wbuf(j), Hp(j, j), nullptr, nullptr,
                       nullptr, rs, grid_vec, st);
      });
      reduce_fin(FIN_LZ1, int(sc / 8), Hp(j, j), nullptr, nullptr, nullptr);
      timed(1, vb * 3, [&] {
        launch_lanczos(dt, 2, n, vsrc(j), nullptr, nullptr, wbuf(j), Hp(j, j), Hp(j + 1, j),
                       Hp(j, j + 1), scal(S_INV), rs, grid_vec, st);
      });
      reduce_fin(FIN_LZ2, 1, Hp(j + 1, j), Hp(j, j + 1), scal(S_INV), nullptr);
    } else {
      void* hb = vec(L.hbuf);
      void* gb = vec(L.gbuf);
      // launch_cgs returns the number of kernels it issued (column tiles of 32)
      const int nv = (j + 1) * int(sc / 8);
      timed(1, vb * (j + 2), [&] {
        launches += launch_cgs(dt, 0, n, V(0), L.ldv, j + 1, wbuf(j), nullptr, hb, nullptr,
                               nullptr, nullptr, rs, grid_cgs, st) - 1;
      });
      reduce_fin(FIN_COEF, nv, hb, nullptr, nullptr, nullptr);
      timed(1, vb * (j + 3), [&] {
        launches += launch_cgs(dt, 1, n, V(0), L.ldv, j + 1, wbuf(j), hb, gb, Hp(0, j), nullptr,
                               nullptr, rs, grid_cgs, st) - 1;
      });
      reduce_fin(FIN_COEF, nv, gb, Hp(0, j), nullptr, hb);
      timed(1, vb * (j + 3), [&] {
        launches += launch_cgs(dt, 2, n, V(0), L.ldv, j + 1, wbuf(j), gb, nullptr, nullptr,
                               Hp(j + 1, j), scal(S_INV), rs, grid_cgs, st) - 1;
      });
      reduce_fin(FIN_SUBNORM, 1, Hp(j + 1, j), nullptr, scal(S_INV), nullptr);
    }
    timed(1, vb * 2, [&] { launch_scale(dt, n, wbuf(j), vdst(j), scal(S_INV), 0.0, st); });
  }

  // start: V0 = s/||s||  (||s|| -> scal(S_BETA0))
  void normalise_start() {
    const double vb = double(n) * double(sc);
    timed(2, vb, [&] { launch_norm(dt, n, V(0), scal(S_BETA0), rs, grid_vec, st); });
    reduce_fin(FIN_NORM, 1, scal(S_BETA0), nullptr, nullptr, nullptr);
    timed(2, 2 * vb, [&] { launch_scale(dt, n, V(0), V(0), scal(S_INV0), 0.0, st); });
  }

  // ----- optional event timing per kernel class (ppf_profile_enable) -----
  struct Pend {
    int cls, e0, e1;
    double bytes;
  };
  std::vector<Pend> pend;
  size_t next_ev = 0;

  cudaEvent_t ev_at(size_t i) {
    while (ctx->prof_pool.size() <= i) {
      cudaEvent_t e;
      PPF_CUDA(cudaEventCreate(&e));
      ctx->prof_pool.push_back(e);
    }
    return ctx->prof_pool[i];
  }

  // run f (which launches exactly one kernel), counting it; with profiling on
  // bracket it with events and remember its algorithmic bytes.
  template <typename F> void timed(int cls, double bytes, F&& f) {
    ++launches;
    if (!ctx->profile) {
      f();
      return;
    }
    const int a = int(next_ev);
    PPF_CUDA(cudaEventRecord(ev_at(next_ev++), st));
    f();
    const int b = int(next_ev);
    PPF_CUDA(cudaEventRecord(ev_at(next_ev++), st));
    pend.push_back({cls, a, b, bytes});
  }

  // after the stream has been synchronised
  void flush_prof() {
    for (auto& p : pend) {
      float ms = 0.f;
      PPF_CUDA(cudaEventElapsedTime(&ms, ctx->prof_pool[p.e0], ctx->prof_pool[p.e1]));
      ctx->prof[p.cls].launches += 1;
      ctx->prof[p.cls].ms += ms;
      ctx->prof[p.cls].bytes += p.bytes;
    }
    pend.clear();
    next_ev = 0;
  }

  // copy H[0:rows, 0:cols] (and beta0) to pinned host; wait.
  void fetch_H(int rows, int cols, std::vector<zc>& Hh, double& beta0) {
    fetch_H_async(cols);
    fetch_H_wait(rows, cols, Hh, beta0);
  }

  // enqueue the D2H copy of H[:, 0:cols] and beta0, then an event
  void fetch_H_async(int cols) {
    char* hp = static_cast<char*>(ctx->h_pinned);
    const size_t bytes = size_t(L.ldh) * cols * sc;
    PPF_CUDA(cudaMemcpyAsync(hp, w + L.H, bytes, cudaMemcpyDeviceToHost, st));
    PPF_CUDA(cudaMemcpyAsync(hp + bytes, scal(S_BETA0), 8, cudaMemcpyDeviceToHost, st));
    PPF_CUDA(cudaEventRecord(ctx->ev, st));
  }

  // wait for fetch_H_async (work enqueued after it keeps running)
  void fetch_H_wait(int rows, int cols, std::vector<zc>& Hh, double& beta0) {
    char* hp = static_cast<char*>(ctx->h_pinned);
    const size_t bytes = size_t(L.ldh) * cols * sc;
    PPF_CUDA(cudaEventSynchronize(ctx->ev));
    const double* h = reinterpret_cast<const double*>(hp);
    const int nd = int(sc / 8);
    Hh.assign(size_t(rows) * cols, zc(0.0, 0.0));
    for (int jj = 0; jj < cols; ++jj)
      for (int i = 0; i < rows; ++i) {
        const size_t o = (size_t(i) + size_t(jj) * L.ldh) * nd;
        Hh[size_t(i) + size_t(jj) * rows] = zc(h[o], nd == 2 ? h[o + 1] : 0.0);
      }
    std::memcpy(&beta0, hp + bytes, 8);
  }

  void upload_y(const std::vector<zc>& y, size_t dst_off = size_t(-1), int slot = 0) {
    if (dst_off == size_t(-1)) dst_off = L.ybuf;
    char* hp = static_cast<char*>(ctx->h_pinned) + stage_h + slot * stage_y;
    double* d = reinterpret_cast<double*>(hp);
    const int nd = int(sc / 8);
    for (size_t i = 0; i < y.size(); ++i) {
      d[i * nd] = y[i].real();
      if (nd == 2) d[i * nd + 1] = y[i].imag();
    }
    if (y.size() * sc > stage_y) fail(PPF_EINVAL, "m too large for the coefficient staging buffer");
    PPF_CUDA(cudaMemcpyAsync(w + dst_off, hp, y.size() * sc, cudaMemcpyHostToDevice, st));
  }
};

// y = beta0 * H_m^{-1/2} e1 from the leading m x m block of Hh ((m+1) x m, ld rows)
std::vector<zc> dense_y(const std::vector<zc>& Hh, int rows, int m, double beta0, bool lanczos) {
  std::vector<zc> y(m);
  if (lanczos) {
    std::vector<double> d(m), e(m, 0.0), yy(m);
    for (int i = 0; i < m; ++i) d[i] = Hh[size_t(i) + size_t(i) * rows].real();
    for (int i = 0; i + 1 < m; ++i) e[i] = Hh[size_t(i + 1) + size_t(i) * rows].real();
    tridiag_invsqrt_e1(m, d.data(), e.data(), beta0, yy.data());
    for (int i = 0; i < m; ++i) y[i] = yy[i];
  } else {
    bool real = true;
    for (int jj = 0; jj < m && real; ++jj)
      for (int i = 0; i < m; ++i)
        if (Hh[size_t(i) + size_t(jj) * rows].imag() != 0.0) {
          real = false;
          break;
        }
    if (real) {  // a real operator's Arnoldi matrix: real Schur route (dense.cpp)
      std::vector<double> Hr(size_t(m) * m), yy(m);
      for (int jj = 0; jj < m; ++jj)
        for (int i = 0; i < m; ++i) Hr[size_t(i) + size_t(jj) * m] = Hh[size_t(i) + size_t(jj) * rows].real();
      real_invsqrt_e1(m, Hr.data(), m, beta0, yy.data());
      for (int i = 0; i < m; ++i) y[i] = yy[i];
      return y;
    }
    std::vector<zc> Hm(size_t(m) * m);
    for (int jj = 0; jj < m; ++jj)
      for (int i = 0; i < m; ++i) Hm[size_t(i) + size_t(jj) * m] = Hh[size_t(i) + size_t(jj) * rows];
    general_invsqrt_e1(m, Hm, beta0, y);
  }
  return y;
}

double nrm(const std::vector<zc>& v) {
  double s = 0.0;
  for (auto& x : v) s += std::norm(x);
  return std::sqrt(s);
}

void check_opts(const ppf_opts* o) {
  PPF_REQUIRE(o, "opts is NULL");
  PPF_REQUIRE(o->func == PPF_INVSQRT || o->func == PPF_SQRT || o->func == PPF_INVSQRT_SQ ||
                  o->func == PPF_SIGN,
              "bad func");
  PPF_REQUIRE(o->krylov == PPF_LANCZOS || o->krylov == PPF_ARNOLDI_CGS2 ||
                  o->krylov == PPF_LANCZOS_2PASS,
              "bad krylov");
  PPF_REQUIRE(o->precond == PPF_PREC_LEFT || o->precond == PPF_PREC_RIGHT, "bad precond");
  PPF_REQUIRE(o->m_max >= 1 && o->m_max <= 1024, "m_max out of range [1, 1024]");
  PPF_REQUIRE(o->stop >= 0 && o->stop <= 2, "bad stop");
  PPF_REQUIRE(o->stop == PPF_STOP_FIXED_M || o->tol > 0.0, "tol must be > 0");
  PPF_REQUIRE(o->check_every >= 1 || o->stop == PPF_STOP_FIXED_M, "check_every >= 1");
  PPF_REQUIRE(o->stop != PPF_STOP_TRUE_ERR || o->x_ref, "TRUE_ERR needs x_ref");
  PPF_REQUIRE(o->stop != PPF_STOP_TRUE_ERR || o->krylov != PPF_LANCZOS_2PASS,
              "TRUE_ERR needs the basis: not available with the two-pass method");
}

ppf_status run_impl(ppf_ctx* ctx, ppf_mat* A, const ppf_poly* q, const ppf_opts* o,
                    const void* b, void* x, const void* b_host, void* x_host, void* work,
                    size_t bytes, ppf_report* rep) {
  auto t_start = std::chrono::steady_clock::now();
  PPF_REQUIRE(ctx && A && rep, "NULL argument");
  PPF_REQUIRE(A->ctx == ctx, "matrix belongs to another context");
  check_opts(o);
  PPF_REQUIRE_ALIGNED(work, "work");
  if (o->x_ref) PPF_REQUIRE_ALIGNED(o->x_ref, "x_ref");
  PPF_REQUIRE(!q || poly_fits(q, A->dtype),
              "a Newton polynomial with complex nodes needs a complex operator");
  const bool twopass = o->krylov == PPF_LANCZOS_2PASS;
  const bool lanczos = o->krylov != PPF_ARNOLDI_CGS2;
  const bool right = q && o->precond == PPF_PREC_RIGHT;
  const int deg = q ? q->deg : 0;
  const int power = squared(o) ? 2 : 1;  // A = Q^2 for INVSQRT_SQ / SIGN
  // mvms per preconditioned step (2 per application of Q^2)
  const long long per_step = power * (q ? 2LL * deg + 1 : 1);
  const int m_max = o->m_max;
  const int k = std::max(1, o->check_every);
  const double brt = o->breakdown_rtol > 0.0 ? o->breakdown_rtol : 1e-14;
  Runner R(ctx, A, q, m_max, work, bytes, ws_shape(q, o), right);
  R.power = power;
  // graphs pay most where launches dominate (L2-scale matrices: C1, C2, the
  // graph Laplacian, Table 1's 100^3: C2 deg 20 6.7 -> 4.7 ms) and still trim
  // the inter-kernel gaps at C3/C4 (-0.4..0.6%)
  const bool big = double(A->stored) * double(R.sc + 4) >= 256e6;
  // sharded: the chain's halo exchanges over peer memory are capturable
  // (fixed-value semaphores, peer.cu); the NCCL and host-transport paths
  // launch directly (NCCL's own capture support is not exercised here: the
  // one-GPU tests run NCCL through a stand-in that is not graph-safe)
  R.use_graph = (ws_shape(q, o) & WS_GRAPH) && ctx->use_graphs && !ctx->profile &&
                (A->nranks == 1 || (peer_active(A) && !ctx->has_transport));
  const int64_t n = R.n;
  const size_t vb = size_t(n) * R.sc;
  double t_dense = 0.0;
  ctx->hist.clear();

  PPF_CUDA(cudaEventRecord(ctx->ev_t0, R.st));
  const void* bin = b;
  if (b_host) {
    PPF_CUDA(cudaMemcpyAsync(R.vec(R.L.U), b_host, vb, cudaMemcpyHostToDevice, R.st));
    bin = R.vec(R.L.U);
  }
  // start (Alg 1 line 2 / Alg 2 line 2): s = b or A b; left: c = q(A) s;
  // right / plain: c = s.  v_1 = c / ||c||.
  long long mvms = 0;
  const void* s_vec = bin;
  if (o->func == PPF_SQRT) {
    void* sdst = (right || !q) ? R.V(0) : R.vec(R.L.Y);
    R.spmv(bin, sdst, Runner::epi(1.0, 0.0, 0.0, nullptr, 0.0, nullptr));
    ++mvms;
    s_vec = sdst;
  }
  if (right || !q) {
    if (s_vec != R.V(0))
      PPF_CUDA(cudaMemcpyAsync(R.V(0), s_vec, vb, cudaMemcpyDeviceToDevice, R.st));
  } else {
    R.apply_q(s_vec, R.V(0));
    mvms += (long long)deg * power;
  }
  R.normalise_start();
  if (twopass) PPF_CUDA(cudaMemcpyAsync(R.vsrc(0), R.V(0), vb, cudaMemcpyDeviceToDevice, R.st));
  const long long mvms_start = mvms;

  std::vector<zc> Hh, y, y_prev;
  double beta0 = 0.0;
  int m = 0;
  int term = PPF_MAX_ITER;
  double est = NAN, err = NAN;
  // Look-ahead: at a checkpoint the host waits for H while the first LOOKAHEAD
  // mat-vecs of the next step (which only read v_{j+1}) already run, so the
  // device does not idle during the D2H copy, f(H_m) and the relaunch.  If the
  // run stops there, that work (<= LOOKAHEAD SpMVs) is discarded.  Not with
  // right preconditioning one-pass, whose checkpoint itself uses the device.
  // (with the step graph the second call is the whole chain: for large
  // matrices only the plain SpMV runs ahead, so at most one SpMV is wasted)
  const int LOOKAHEAD = (o->stop == PPF_STOP_EST && !(right && !twopass)) ? ((R.use_graph && big) ? 1 : 2) : 0;
  // the basis the iterate is combined from: V_m, or Y_m (right, one-pass)
  auto basis0 = [&]() -> const void* { return (right && !twopass) ? R.Yb(0) : R.V(0); };
  // Run-ahead: when f(H_m) on the host takes longer than the host waits for
  // H_m (host-bound: small operators, large m, e.g. C2 deg 5 at m = 76), the
  // whole next step -- operator chain AND orthogonalisation, both device-only
  // -- is enqueued before the host waits for H_m, and f(H_m) itself goes to a
  // worker thread (up to kPend checkpoints in flight, decided in order), so
  // the device keeps stepping while the host evaluates.  If the run stops at
  // m, the steps run beyond it are discarded (V_1..V_m, H_m and the counters
  // are untouched by them).  Re-decided from the measured times.
  bool run_ahead = false, ortho_ahead = false;
  // PPF_RUN_AHEAD=1 / 0 forces the mode on / off (tests: results must not
  // depend on it); unset: chosen from the measured times
  const int force_ahead = [] {
    const char* e = std::getenv("PPF_RUN_AHEAD");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  // the decision at checkpoint mc (mbc: m after an early breakdown inside the
  // stride): the estimate from y_{m-k}, the history, the stop test;
  // true = stop, with term set
  auto decide = [&](int mc, int mbc, double hsubc, long long mvmsc, const std::vector<zc>& yc) -> bool {
    if (!y_prev.empty()) {
      if (right && !twopass) {
        // Y_m is not orthonormal: ||f_m - f_{m-k}|| / ||f_m|| from the iterates
        // themselves: T0 = Y_m y_m, T1 = Y_m [y_{m-k}; 0]
        std::vector<zc> yp(yc.size(), zc(0.0, 0.0));
        for (size_t i = 0; i < y_prev.size(); ++i) yp[i] = y_prev[i];
        R.upload_y(yc, R.L.ybuf, 0);
        R.upload_y(yp, R.L.ybuf2, 1);
        R.timed(2, double(vb) * (mbc + 1), [&] {
          launch_combine(R.dt, n, basis0(), R.L.ldv, mbc, R.vec(R.L.ybuf), R.vec(R.L.T0), R.st);
        });
        R.timed(2, double(vb) * (mbc + 1), [&] {
          launch_combine(R.dt, n, basis0(), R.L.ldv, mbc, R.vec(R.L.ybuf2), R.vec(R.L.T1), R.st);
        });
        R.timed(2, 2.0 * vb, [&] {
          launch_diffnorm(R.dt, n, R.vec(R.L.T1), R.vec(R.L.T0), R.scal(S_ERR), R.rs, R.grid_vec,
                          R.st);
        });
        R.reduce_fin(FIN_SQRT, 2, R.scal(S_ERR), nullptr, nullptr, nullptr);
        double e2[2];
        PPF_CUDA(cudaMemcpyAsync(e2, R.scal(S_ERR), 16, cudaMemcpyDeviceToHost, R.st));
        PPF_CUDA(cudaStreamSynchronize(R.st));
        est = e2[0] / e2[1];
      } else {
        std::vector<zc> dlt = yc;
        for (size_t i = 0; i < y_prev.size(); ++i) dlt[i] -= y_prev[i];
        est = nrm(dlt) / nrm(yc);
      }
    }
    y_prev = yc;
    if (o->stop == PPF_STOP_TRUE_ERR) {
      R.upload_y(yc);
      R.timed(2, double(vb) * (mbc + 1), [&] {
        launch_combine(R.dt, n, basis0(), R.L.ldv, mbc, R.vec(R.L.ybuf), R.vec(R.L.T0), R.st);
      });
      R.timed(2, 2.0 * vb, [&] {
        launch_diffnorm(R.dt, n, R.vec(R.L.T0), o->x_ref, R.scal(S_ERR), R.rs, R.grid_vec, R.st);
      });
      R.reduce_fin(FIN_SQRT, 2, R.scal(S_ERR), nullptr, nullptr, nullptr);
      double e2[2];
      PPF_CUDA(cudaMemcpyAsync(e2, R.scal(S_ERR), 16, cudaMemcpyDeviceToHost, R.st));
      PPF_CUDA(cudaStreamSynchronize(R.st));
      err = e2[0] / e2[1];
    }
    if (o->record_history) ctx->hist.push_back({mbc, est, err, mvmsc - (mc - mbc) * per_step});
    if (mbc != mc || hsubc <= brt * beta0) {
      term = PPF_BREAKDOWN;
      return true;
    }
    if (o->stop == PPF_STOP_EST && !std::isnan(est) && est <= o->tol) {
      term = PPF_CONVERGED;
      return true;
    }
    if (o->stop == PPF_STOP_TRUE_ERR && err <= o->tol) {
      term = PPF_CONVERGED;
      return true;
    }
    return false;
  };
  // f(H_m) of checkpoints evaluated on worker threads (run-ahead mode), up to
  // kPend in flight, decided strictly in checkpoint order
  struct Pending {
    int m = 0, mb = 0;
    double hsub = 0.0;
    long long mvms = 0;
    std::future<std::pair<std::vector<zc>, double>> fut;
  };
  constexpr size_t kPend = 4;
  constexpr int kAhead = 5;
  std::deque<Pending> pend;
  double t_wait = 0.0;
  // decide the oldest pending checkpoint; true = the run stops there
  auto resolve_front = [&]() -> bool {
    Pending& p = pend.front();
    auto r = p.fut.get();
    t_dense += r.second;
    run_ahead = A->nranks == 1 && (force_ahead > 0 || (force_ahead < 0 && r.second > t_wait));
    const bool stop = decide(p.m, p.mb, p.hsub, p.mvms, r.first);
    if (stop) {
      m = p.mb;
      y = std::move(r.first);
    }
    pend.pop_front();
    return stop;
  };
  // Resident step loop (small operators; kernels.cu: resident_steps_kernel):
  // one CTA runs the steps back to back while the host decides the
  // checkpoints from H columns it reads out of a mapped block.
  const bool resident = [&] {
    const char* e = std::getenv("PPF_RESIDENT");
    if (e && e[0] == '0') return false;
    return resident_fits(A) && q && q->deg >= 1 && !right && !twopass && power == 1 &&
           (o->stop == PPF_STOP_EST || o->stop == PPF_STOP_FIXED_M) && !ctx->profile;
  }();
  bool resident_done = false;
  if (resident) {
    // the step's q(A)q(A) chain, U -> Y -> W2, as recorded SpMV calls
    std::vector<Runner::Call> chain;
    R.rec = &chain;
    R.apply_q(R.vec(R.L.U), R.vec(R.L.Y));
    R.apply_q(R.vec(R.L.Y), R.vec(R.L.W2));
    R.rec = nullptr;
    bool ok = true;
    std::vector<ResCallSpec> spec;
    for (auto& c : chain) {
      if (c.scale || c.graph) ok = false;
      spec.push_back({c.x, c.out, c.e});
    }
    if (ok) {
      const size_t cb = resident_call_bytes(R.dt);
      const size_t hbytes = size_t(R.L.ldh) * size_t(m_max + 1) * R.sc;
      const size_t calls_off = (sizeof(ResCtl) + hbytes + 255) & ~size_t(255);
      const size_t need = calls_off + spec.size() * cb + 256;
      if (ctx->res_ctl_bytes < need) {
        PPF_CUDA(cudaStreamSynchronize(R.st));
        if (ctx->res_ctl) PPF_CUDA(cudaFreeHost(ctx->res_ctl));
        ctx->res_ctl = nullptr;
        ctx->res_ctl_bytes = 0;
        PPF_CUDA(cudaHostAlloc(&ctx->res_ctl, need, cudaHostAllocMapped));
        ctx->res_ctl_bytes = need;
      }
      char* blk = static_cast<char*>(ctx->res_ctl);
      void* blk_dev = nullptr;
      PPF_CUDA(cudaHostGetDevicePointer(&blk_dev, blk, 0));
      auto* ctl = reinterpret_cast<ResCtl*>(blk);
      volatile int* v_stop = &ctl->stop;
      volatile int* v_acked = &ctl->acked;
      volatile int* v_done = &ctl->done;
      *v_stop = 0;
      *v_done = 0;
      *v_acked = o->stop == PPF_STOP_FIXED_M ? m_max : 0;
      resident_pack_calls(R.dt, spec, blk + calls_off);
      std::atomic_thread_fence(std::memory_order_seq_cst);
      R.timed(0, 0.0, [&] {
        launch_resident(A, R.V(0), R.L.ldv, R.vec(R.L.U), R.vec(R.L.W2), R.Hp(0, 0), R.L.ldh,
                        m_max, lanczos ? 1 : 0, R.scal(S_BETA0), reinterpret_cast<ResCtl*>(blk_dev),
                        static_cast<char*>(blk_dev) + calls_off, int(spec.size()), RES_AHEAD, R.st);
      });
      const int nd = int(R.sc / 8);
      if (o->stop == PPF_STOP_FIXED_M) {
        m = m_max;
      } else {
        int decided = 0;
        bool stopped = false;
        while (!stopped && decided < m_max) {
          const int d = *v_done;
          std::atomic_thread_fence(std::memory_order_acquire);
          if (d <= decided) {
            // the kernel ended early only if it failed: report, do not spin
            const cudaError_t qs = cudaStreamQuery(R.st);
            if (qs != cudaErrorNotReady && *v_done <= decided) {
              PPF_CUDA(qs);
              fail(PPF_ECUDA, "resident step kernel ended before the host's decision");
            }
            std::this_thread::yield();
            continue;
          }
          for (int mm = decided + 1; mm <= d && !stopped; ++mm) {
            m = mm;
            mvms = mvms_start + (long long)mm * per_step;
            decided = mm;
            if (!(mm % k == 0 || mm == m_max)) {
              *v_acked = mm;
              continue;
            }
            beta0 = ctl->beta0;
            Hh.assign(size_t(mm + 1) * mm, zc(0.0, 0.0));
            for (int jj = 0; jj < mm; ++jj)
              for (int i = 0; i <= std::min(mm, jj + 1); ++i) {
                const size_t oo = (size_t(i) + size_t(jj) * R.L.ldh) * nd;
                Hh[size_t(i) + size_t(jj) * (mm + 1)] = zc(ctl->H[oo], nd == 2 ? ctl->H[oo + 1] : 0.0);
              }
            const double hsub = std::abs(Hh[size_t(mm) + size_t(mm - 1) * (mm + 1)]);
            int mb = mm;
            for (int jj = std::max(0, mm - k); jj < mm; ++jj)
              if (std::abs(Hh[size_t(jj + 1) + size_t(jj) * (mm + 1)]) <= brt * beta0) {
                mb = jj + 1;
                break;
              }
            std::vector<zc> Hs = Hh;
            if (mb != mm) {
              std::vector<zc> H2(size_t(mb + 1) * mb);
              for (int jj = 0; jj < mb; ++jj)
                for (int i = 0; i <= mb; ++i) H2[size_t(i) + size_t(jj) * (mb + 1)] = Hh[size_t(i) + size_t(jj) * (mm + 1)];
              Hs = H2;
            }
            auto td = std::chrono::steady_clock::now();
            std::vector<zc> yy = dense_y(Hs, mb + 1, mb, beta0, lanczos);
            t_dense += std::chrono::duration<double>(std::chrono::steady_clock::now() - td).count();
            if (decide(mm, mb, hsub, mvms, yy)) {
              m = mb;
              y = std::move(yy);
              stopped = true;
              *v_stop = 1;
              break;
            }
            *v_acked = mm;
          }
        }
        if (!stopped) *v_stop = 1;
      }
      PPF_CUDA(cudaStreamSynchronize(R.st));
      mvms = mvms_start + (long long)m * per_step;
      resident_done = true;
    }
  }
  if (!resident_done) {
  std::vector<Runner::Call> calls = R.record_step(0);
  size_t played = 0;
  for (int j = 0; j < m_max; ++j) {
    for (; played < calls.size(); ++played) R.play(calls[played]);
    if (!ortho_ahead) R.orthogonalise(j, lanczos);
    ortho_ahead = false;
    m = j + 1;
    mvms += per_step;
    // checkpoints left to worker threads: decide those already finished, and
    // wait for one once the device has been given kAhead steps beyond it (the
    // steps run past a stop are discarded: this bounds them for any k)
    {
      bool stopped = false;
      while (!stopped && !pend.empty() &&
             (m - pend.front().m >= kAhead ||
              pend.front().fut.wait_for(std::chrono::seconds(0)) == std::future_status::ready))
        stopped = resolve_front();
      if (stopped) break;
    }
    const bool check = (o->stop != PPF_STOP_FIXED_M) && (m % k == 0 || m == m_max);
    const bool more = j + 1 < m_max;
    if (!check) {
      if (more) {
        calls = R.record_step(j + 1);
        played = 0;
      }
      continue;
    }
    R.fetch_H_async(m);
    if (more) {
      calls = R.record_step(j + 1);
      played = 0;
      if (run_ahead && LOOKAHEAD > 0) {
        for (; played < calls.size(); ++played) R.play(calls[played]);
        R.orthogonalise(j + 1, lanczos);
        ortho_ahead = true;
      } else {
        for (; played < calls.size() && played < size_t(LOOKAHEAD); ++played) R.play(calls[played]);
      }
    }
    const auto tw = std::chrono::steady_clock::now();
    R.fetch_H_wait(m + 1, m, Hh, beta0);
    t_wait = std::chrono::duration<double>(std::chrono::steady_clock::now() - tw).count();
    const double hsub = std::abs(Hh[size_t(m) + size_t(m - 1) * (m + 1)]);
    // earlier breakdown inside the stride?
    int mb = m;
    for (int jj = std::max(0, m - k); jj < m; ++jj)
      if (std::abs(Hh[size_t(jj + 1) + size_t(jj) * (m + 1)]) <= brt * beta0) {
        mb = jj + 1;
        break;
      }
    std::vector<zc> Hs = Hh;
    if (mb != m) {
      std::vector<zc> H2(size_t(mb + 1) * mb);
      for (int jj = 0; jj < mb; ++jj)
        for (int i = 0; i <= mb; ++i) H2[size_t(i) + size_t(jj) * (mb + 1)] = Hh[size_t(i) + size_t(jj) * (m + 1)];
      Hs = H2;
    }
    // (1) earlier checkpoints left to worker threads are decided first, in
    // order: those already finished, and the oldest while kPend are in flight
    bool stopped = false;
    while (!stopped && !pend.empty() &&
           (pend.size() >= kPend ||
            pend.front().fut.wait_for(std::chrono::seconds(0)) == std::future_status::ready))
      stopped = resolve_front();
    if (stopped) break;
    // (2) this checkpoint on a worker thread while the device runs ahead,
    // unless a breakdown or the last step forces the decision now; a stop
    // found later discards the steps run meanwhile (<= kPend + 1)
    if (run_ahead && more && mb == m && !(hsub <= brt * beta0) && o->stop == PPF_STOP_EST &&
        !(right && !twopass)) {
      Pending p;
      p.m = m;
      p.mb = mb;
      p.hsub = hsub;
      p.mvms = mvms;
      p.fut = std::async(std::launch::async, [Hs, mb, beta0, lanczos]() {
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<zc> yy = dense_y(Hs, mb + 1, mb, beta0, lanczos);
        return std::make_pair(std::move(yy), std::chrono::duration<double>(
                                                 std::chrono::steady_clock::now() - t0).count());
      });
      pend.push_back(std::move(p));
      continue;
    }
    while (!stopped && !pend.empty()) stopped = resolve_front();
    if (stopped) break;
    auto td = std::chrono::steady_clock::now();
    y = dense_y(Hs, mb + 1, mb, beta0, lanczos);
    const double t_this = std::chrono::duration<double>(std::chrono::steady_clock::now() - td).count();
    t_dense += t_this;
    // one rank only: the decision comes from host timings, and the ranks'
    // collectives must pair up (every rank has to run the same steps)
    run_ahead = A->nranks == 1 && (force_ahead > 0 || (force_ahead < 0 && t_this > t_wait));
    if (decide(m, mb, hsub, mvms, y)) {
      m = mb;
      break;
    }
  }
  }
  // final H, y_m
  R.fetch_H(m + 1, m, Hh, beta0);
  if (o->stop == PPF_STOP_FIXED_M) {
    for (int jj = 0; jj < m; ++jj)
      if (std::abs(Hh[size_t(jj + 1) + size_t(jj) * (m + 1)]) <= brt * beta0) {
        const int mb = jj + 1;
        std::vector<zc> H2(size_t(mb + 1) * mb);
        for (int c = 0; c < mb; ++c)
          for (int i = 0; i <= mb; ++i) H2[size_t(i) + size_t(c) * (mb + 1)] = Hh[size_t(i) + size_t(c) * (m + 1)];
        Hh = H2;
        m = mb;
        term = PPF_BREAKDOWN;
        break;
      }
  }
  if (int(y.size()) != m || o->stop == PPF_STOP_FIXED_M) {
    auto td = std::chrono::steady_clock::now();
    y = dense_y(Hh, m + 1, m, beta0, lanczos);
    t_dense += std::chrono::duration<double>(std::chrono::steady_clock::now() - td).count();
  }
  void* xo = x_host ? R.vec(R.L.Y) : x;
  // sign(Q) b = Q f: f goes to U (free once the steps are done), then one SpMV
  void* fo = o->func == PPF_SIGN ? R.vec(R.L.U) : xo;
  long long mv_total = mvms_start + (long long)m * per_step;
  if (!twopass) {
    // Alg 1 line 11 / Alg 2 line 11: f_m = V_m y_m or Y_m y_m
    R.upload_y(y);
    R.timed(2, double(vb) * (m + 1), [&] {
      launch_combine(R.dt, n, basis0(), R.L.ldv, m, R.vec(R.L.ybuf), fo, R.st);
    });
  } else {
    // two-pass, pass 2: regenerate v_2..v_m with the pass-1
    // coefficients (host scalars, no inner products) and accumulate
    // x~ = V_m y_m; right preconditioning: f_m = q(A) x~.
    void* acc = R.vec(R.L.XA);  // (xo may be the left path's intermediate buffer L.Y)
    auto alpha = [&](int jj) { return Hh[size_t(jj) + size_t(jj) * (m + 1)].real(); };
    auto beta = [&](int jj) { return Hh[size_t(jj + 1) + size_t(jj) * (m + 1)].real(); };
    PPF_CUDA(cudaMemcpyAsync(R.vsrc(0), R.V(0), vb, cudaMemcpyDeviceToDevice, R.st));
    R.timed(2, 2.0 * vb, [&] { launch_scale(R.dt, n, R.V(0), acc, nullptr, y[0].real(), R.st); });
    for (int j = 0; j + 1 < m; ++j) {
      std::vector<Runner::Call> cs = R.record_step(j);
      for (auto& c : cs) R.play(c);
      R.timed(1, double(vb) * (j > 0 ? 6 : 5), [&] {
        launch_lanczos_regen(R.dt, n, R.vdst(j), R.vsrc(j), R.vprv(j), alpha(j),
                             j > 0 ? beta(j - 1) : 0.0, 1.0 / beta(j), y[size_t(j + 1)].real(), acc,
                             R.st);
      });
    }
    mv_total += (long long)(m - 1) * per_step;
    if (right) {
      R.apply_q(acc, fo);
      mv_total += (long long)deg * power;
    } else {
      PPF_CUDA(cudaMemcpyAsync(fo, acc, vb, cudaMemcpyDeviceToDevice, R.st));
    }
  }
  if (o->func == PPF_SIGN) {
    R.power = 1;
    R.spmv(fo, xo, Runner::epi(1.0, 0.0, 0.0, nullptr, 0.0, nullptr));
    mv_total += 1;
  }
  if (x_host) PPF_CUDA(cudaMemcpyAsync(x_host, xo, vb, cudaMemcpyDeviceToHost, R.st));
  // (also: the host staging for y must not be reused before its copy is done)
  PPF_CUDA(cudaEventRecord(ctx->ev_t1, R.st));
  PPF_CUDA(cudaEventSynchronize(ctx->ev_t1));
  float dev_ms = 0.0f;
  PPF_CUDA(cudaEventElapsedTime(&dev_ms, ctx->ev_t0, ctx->ev_t1));
  R.flush_prof();
  // keep H for ppf_hessenberg
  ctx->last_m = m;
  ctx->last_beta0 = beta0;
  ctx->last_dtype = R.dt;
  const int nd = int(R.sc / 8);
  ctx->lastH.assign(size_t(m + 1) * m * nd, 0.0);
  for (int jj = 0; jj < m; ++jj)
    for (int i = 0; i <= m; ++i) {
      const zc v = Hh[size_t(i) + size_t(jj) * (m + 1)];
      const size_t oo = (size_t(i) + size_t(jj) * (m + 1)) * nd;
      ctx->lastH[oo] = v.real();
      if (nd == 2) ctx->lastH[oo + 1] = v.imag();
    }
  ctx->launches += R.launches;
  if (ctx->nccl_comm && A->nranks > 1) {
    // NCCL reports communication failures asynchronously (SURVEY §8(b) errors)
    ncclResult_t as = ncclSuccess;
    if (ncclCommGetAsyncError(static_cast<ncclComm_t>(ctx->nccl_comm), &as) != ncclSuccess ||
        as != ncclSuccess)
      fail(PPF_ENCCL, "NCCL communicator reported an asynchronous error");
  }
  rep->iterations = m;
  rep->term = term;
  rep->mvms = mv_total;
  rep->inner_products = lanczos ? 2LL * m : (long long)m * m + 2LL * m;
  rep->est = est;
  rep->err = err;
  rep->beta0 = beta0;
  rep->seconds_host_dense = t_dense;
  rep->kernel_launches = R.launches;
  rep->seconds_device = 1e-3 * double(dev_ms);
  rep->seconds_total =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  return PPF_OK;
}

}  // namespace
}  // namespace ppf

using namespace ppf;

#define PPF_API_BEGIN try {
#define PPF_API_END                               \
  return PPF_OK;                                  \
  }                                               \
  catch (const ppf::Error& e) {                   \
    ppf::set_last_error(e.msg);                   \
    return e.st;                                  \
  }                                               \
  catch (...) {                                   \
    ppf::set_last_error("unknown C++ exception"); \
    return PPF_EINVAL;                            \
  }

extern "C" {

ppf_status ppf_workspace_bytes(ppf_ctx* ctx, const ppf_mat* A, const ppf_poly* q,
                               const ppf_opts* o, size_t* bytes) {
  PPF_API_BEGIN
  PPF_REQUIRE(ctx && A && bytes, "NULL argument");
  check_opts(o);
  const WsLayout L = ws_layout(A->n_local, A->dtype, o->m_max, ctx->num_sms, ws_shape(q, o));
  *bytes = L.total;
  ensure_pinned(ctx, pinned_need(L, o->m_max, A->dtype == PPF_R64 ? 8 : 16));
  PPF_API_END
}

ppf_status ppf_run(ppf_ctx* ctx, ppf_mat* A, const ppf_poly* q, const ppf_opts* o, const void* b,
                   void* x, void* work, size_t bytes, ppf_report* rep) {
  PPF_API_BEGIN
  PPF_REQUIRE(b && x, "NULL b/x");
  PPF_REQUIRE_ALIGNED(b, "b");
  PPF_REQUIRE_ALIGNED(x, "x");
  return run_impl(ctx, A, q, o, b, x, nullptr, nullptr, work, bytes, rep);
  PPF_API_END
}

ppf_status ppf_run_host(ppf_ctx* ctx, ppf_mat* A, const ppf_poly* q, const ppf_opts* o,
                        const void* b_host, void* x_host, void* work, size_t bytes,
                        ppf_report* rep) {
  PPF_API_BEGIN
  PPF_REQUIRE(b_host && x_host, "NULL b_host/x_host");
  return run_impl(ctx, A, q, o, nullptr, nullptr, b_host, x_host, work, bytes, rep);
  PPF_API_END
}

ppf_status ppf_history(ppf_ctx* ctx, int cap, int* count, int* m, double* est, double* err,
                       long long* mvms) {
  PPF_API_BEGIN
  PPF_REQUIRE(ctx && count, "NULL argument");
  const int nh = int(ctx->hist.size());
  *count = nh;
  for (int i = 0; i < nh && i < cap; ++i) {
    if (m) m[i] = ctx->hist[i].m;
    if (est) est[i] = ctx->hist[i].est;
    if (err) err[i] = ctx->hist[i].err;
    if (mvms) mvms[i] = ctx->hist[i].mvms;
  }
  PPF_API_END
}

ppf_status ppf_hessenberg(ppf_ctx* ctx, int ld, void* H, int* m, double* beta0) {
  PPF_API_BEGIN
  PPF_REQUIRE(ctx, "NULL ctx");
  const int mm = ctx->last_m;
  if (m) *m = mm;
  if (beta0) *beta0 = ctx->last_beta0;
  if (H) {
    PPF_REQUIRE(ld >= mm + 1, "ld < m+1");
    const int nd = ctx->last_dtype == PPF_R64 ? 1 : 2;
    double* h = static_cast<double*>(H);
    for (int j = 0; j < mm; ++j)
      for (int i = 0; i <= mm; ++i)
        for (int d = 0; d < nd; ++d)
          h[(size_t(i) + size_t(j) * ld) * nd + d] = ctx->lastH[(size_t(i) + size_t(j) * (mm + 1)) * nd + d];
  }
  PPF_API_END
}

ppf_status ppf_ritz_workspace_bytes(ppf_ctx* ctx, const ppf_mat* A, int deg, size_t* bytes) {
  PPF_API_BEGIN
  PPF_REQUIRE(ctx && A && bytes && deg >= 0 && deg < 255, "bad arguments");
  const WsLayout L = ws_layout(A->n_local, A->dtype, deg + 1, ctx->num_sms, WS_SQUARE);
  *bytes = L.total;
  ensure_pinned(ctx, pinned_need(L, deg + 1, A->dtype == PPF_R64 ? 8 : 16));
  PPF_API_END
}

// Ritz values of H_d from d = deg+1 Arnoldi steps with A^power,
// Leja order, divided differences.
ppf_status ppf_poly_ritz_newton_pow(ppf_ctx* ctx, ppf_mat* A, const void* start, int deg,
                                    int power, int harmonic, void* work, size_t bytes,
                                    ppf_poly** out) {
  PPF_API_BEGIN
  PPF_REQUIRE(ctx && A && start && out, "NULL argument");
  PPF_REQUIRE(deg >= 0 && deg < 255, "deg out of range");
  PPF_REQUIRE(power == 1 || power == 2, "power must be 1 or 2");
  PPF_REQUIRE_ALIGNED(start, "start");
  PPF_REQUIRE_ALIGNED(work, "work");
  const int d = deg + 1;
  Runner R(ctx, A, nullptr, d, work, bytes, WS_SQUARE);
  R.power = power;
  PPF_CUDA(cudaMemcpyAsync(R.V(0), start, size_t(R.n) * R.sc, cudaMemcpyDeviceToDevice, R.st));
  R.normalise_start();
  for (int j = 0; j < d; ++j) {
    R.op_apply(j);
    R.orthogonalise(j, false);
  }
  std::vector<zc> Hh;
  double beta0;
  R.fetch_H(d + 1, d, Hh, beta0);
  R.flush_prof();
  ctx->launches += R.launches;
  std::vector<zc> Hd(size_t(d) * d);
  for (int j = 0; j < d; ++j)
    for (int i = 0; i < d; ++i) Hd[size_t(i) + size_t(j) * d] = Hh[size_t(i) + size_t(j) * (d + 1)];
  if (harmonic) {
    // H~_d = H_d + |h_{d+1,d}|^2 f e_d^T with H_d^H f = e_d
    const zc hs = Hh[size_t(d) + size_t(d - 1) * (d + 1)];
    std::vector<zc> f = solve_dense_adjoint_ed(d, Hd);
    for (int i = 0; i < d; ++i) Hd[size_t(i) + size_t(d - 1) * d] += std::norm(hs) * f[i];
  }
  std::vector<zc> theta = eigenvalues(d, Hd);
  bool pairs = false;
  if (A->dtype == PPF_R64) {
    // a real operator runs the chain in real arithmetic: real Ritz values are
    // used as they are; complex ones come in conjugate pairs and get the
    // real-pair form (real_pair_form) below
    for (auto& t : theta) {
      if (std::abs(t.imag()) > 1e-12 * std::abs(t))
        pairs = true;
      else
        t = zc(t.real(), 0.0);
    }
  }
  for (auto& t : theta)
    if (std::abs(t.imag()) <= 1e-13 * std::max(std::abs(t), 1e-300) && t.real() <= 0.0)
      fail(PPF_EBRANCH, "Ritz value on the branch cut (-inf, 0]");
  auto* q = new ppf_poly();
  q->kind = PPF_POLY_NEWTON;
  q->deg = deg;
  q->a = q->b = 0.0;
  q->nodes = leja_order(theta);
  q->dd = divided_differences_invsqrt(q->nodes);
  if (pairs) {
    try {
      real_pair_form(*q);
    } catch (...) {
      delete q;
      throw;
    }
  }
  *out = q;
  PPF_API_END
}

ppf_status ppf_poly_ritz_newton(ppf_ctx* ctx, ppf_mat* A, const void* start, int deg, void* work,
                                size_t bytes, ppf_poly** out) {
  return ppf_poly_ritz_newton_pow(ctx, A, start, deg, 1, 0, work, bytes, out);
}

}  // extern "C"

extern "C" ppf_status ppf_spmv(ppf_ctx* ctx, ppf_mat* A, const void* x, void* y) {
  try {
    PPF_REQUIRE(ctx && A && x && y, "NULL argument");
    PPF_REQUIRE(A->ctx == ctx, "matrix belongs to another context");
    PPF_REQUIRE_ALIGNED(x, "x");
    PPF_REQUIRE_ALIGNED(y, "y");
    ppf::Epi e{};
    e.s_ax[0] = 1.0;
    if (A->nranks > 1) {
      ppf::halo_spmv(ctx, A, x, y, e);
      ctx->launches += 1 + (A->send_total ? 1 : 0) + (A->halo_rows ? 1 : 0) +
                       ((ppf::peer_active(A) && (A->send_total || A->halo_total)) ? 1 : 0);
      return PPF_OK;
    }
    ppf::launch_spmv(A, x, y, e, ctx->stream);
    ctx->launches += 1;
    return PPF_OK;
  } catch (const ppf::Error& e) {
    ppf::set_last_error(e.msg);
    return e.st;
  } catch (...) {
    ppf::set_last_error("unknown C++ exception");
    return PPF_EINVAL;
  }
}

extern "C" ppf_status ppf_poly_apply_bytes(ppf_ctx* ctx, const ppf_mat* A, size_t* bytes) {
  try {
    PPF_REQUIRE(ctx && A && bytes, "NULL argument");
    *bytes = ppf::ws_layout(A->n_local, A->dtype, 1, ctx->num_sms).total;
    return PPF_OK;
  } catch (const ppf::Error& e) {
    ppf::set_last_error(e.msg);
    return e.st;
  }
}

extern "C" ppf_status ppf_poly_apply(ppf_ctx* ctx, ppf_mat* A, const ppf_poly* q, const void* x,
                                     void* y, void* work, size_t bytes) {
  try {
    PPF_REQUIRE(ctx && A && q && x && y, "NULL argument");
    PPF_REQUIRE(A->ctx == ctx, "matrix belongs to another context");
    PPF_REQUIRE(x != y, "x and y must be distinct");
    PPF_REQUIRE_ALIGNED(x, "x");
    PPF_REQUIRE_ALIGNED(y, "y");
    PPF_REQUIRE_ALIGNED(work, "work");
    PPF_REQUIRE(ppf::poly_fits(q, A->dtype),
                "a Newton polynomial with complex nodes needs a complex operator");
    ppf::Runner R(ctx, A, q, 1, work, bytes);
    R.apply_q(x, y);
    if (ctx->profile) {
      PPF_CUDA(cudaStreamSynchronize(R.st));
      R.flush_prof();
    }
    ctx->launches += R.launches;
    return PPF_OK;
  } catch (const ppf::Error& e) {
    ppf::set_last_error(e.msg);
    return e.st;
  } catch (...) {
    ppf::set_last_error("unknown C++ exception");
    return PPF_EINVAL;
  }
}

extern "C" ppf_status ppf_halo_pack(ppf_ctx* ctx, ppf_mat* A, const void* x) {
  try {
    PPF_REQUIRE(ctx && A && x, "NULL argument");
    PPF_REQUIRE(A->ctx == ctx, "matrix belongs to another context");
    PPF_REQUIRE_ALIGNED(x, "x");
    ppf::launch_halo_pack(A, x, ctx->stream);
    ctx->launches += A->send_total ? 1 : 0;
    return PPF_OK;
  } catch (const ppf::Error& e) {
    ppf::set_last_error(e.msg);
    return e.st;
  }
}

extern "C" ppf_status ppf_halo_buffers(ppf_mat* A, void** send, void** recv) {
  if (!A) {
    ppf::set_last_error("NULL matrix");
    return PPF_EINVAL;
  }
  if (send) *send = A->d_send;
  if (recv) *recv = A->d_recv;
  return PPF_OK;
}

extern "C" ppf_status ppf_spmv_local(ppf_ctx* ctx, ppf_mat* A, const void* x, void* y) {
  try {
    PPF_REQUIRE(ctx && A && x && y, "NULL argument");
    PPF_REQUIRE(A->ctx == ctx, "matrix belongs to another context");
    PPF_REQUIRE_ALIGNED(x, "x");
    PPF_REQUIRE_ALIGNED(y, "y");
    ppf::Epi e{};
    e.s_ax[0] = 1.0;
    ppf::launch_spmv(A, x, y, e, ctx->stream);
    ctx->launches += 1;
    if (A->halo_rows) {
      ppf::launch_halo_apply(A, y, e.s_ax, ctx->stream);
      ctx->launches += 1;
    }
    return PPF_OK;
  } catch (const ppf::Error& e) {
    ppf::set_last_error(e.msg);
    return e.st;
  }
}
