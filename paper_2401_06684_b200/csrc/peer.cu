// Peer-memory communication for the sharded path ("B200-native
// alternative for halos: direct peer loads/stores over NVLink ... reads the
// neighbour's boundary plane in place after a flag or barrier, which avoids
// NCCL launch latency"; include/ppf.h: ppf_mat_peer_window / _connect).
//
// Window of rank r (cudaMalloc, exported with CUDA IPC; byte offsets):
//   OFF_READY_H  u32[p]  semaphore: pushes of sender p into r not yet consumed
//   OFF_FREED_H  u32[q]  semaphore: free receive slots of receiver q for r's
//                        pushes (starts at 2: the receive slots are double-buffered)
//   OFF_READY_R  u32     reduction arrivals: +1 per peer partial stored into r
//   OFF_BLK      u32  last-block ticket of r's own push kernel (local only)
//   OFF_XCOUNT   u32  halo exchanges r has completed (local only); slot = parity
//   OFF_RED      2 slots x nranks x RCAP doubles (slot E&1, row = source rank)
//   halo_off     2 slots x halo_total scalars (slot XCOUNT&1; per-peer segments at
//                r's recv_off, the same layout as the NCCL receive buffer)
// Every rank issues the same exchanges in the same order, so the sender's and
// the receiver's exchange counts -- and with them the slot parity -- agree.
//
// Halo exchange on rank r (one per sharded SpMV), all comparison values FIXED
// (semaphores instead of epochs), so a captured CUDA graph of the step's
// SpMV chain replays correctly (round 2):
//   stream:  [ev_pack] .. diag-block SpMV .. wait ev_halo, wait READY_H[p] >= 1 (each sender p)
//            .. halo block (slot XCOUNT&1) .. consume kernel
//   comm:    wait ev_pack, wait FREED_H[q] >= 1 (each receiver q), push kernel [ev_halo]
// The push kernel stores x[send_idx] into each receiver's slot XCOUNT&1
// (NVLink stores); its last block, after every block's __threadfence_system(),
// takes one slot from each FREED_H[q] and adds 1 to READY_H[r] of each
// receiver.  The consume kernel (after the halo block read the slot) gives the
// arrivals back (READY_H[p] -= 1), returns the slot to each sender (+1 on
// FREED_H[r] in its window) and advances XCOUNT.  The counters are per peer:
// neighbours are not all-to-all, so a fast neighbour can run an exchange ahead
// of a slow one and an aggregate count could be met with one exchange's data
// missing.
//
// Reduction E (allreduce of the rank-local partial sums a reduction kernel left
// in RedScratch::raw): one block stores raw into slot E&1 / row r of every
// rank's window and bumps READY_R of the others; the stream waits READY_R >=
// (nranks-1)*E and sums the rows in rank order 0..nranks-1 (bit-identical on
// every rank).  One aggregate counter suffices here: every rank's put of E+1
// follows its wait of E, which needs every put of E, so no rank's count can run
// an epoch ahead of another's.  Slot reuse is ordered the same way: rank r
// writes slot E&1 of rank q again at epoch E+2, after its own wait of epoch
// E+1, which needs q's store of E+1, which q's stream issues after its sum of E.
//
// Waits are cuStreamWaitValue32 (GEQ) on this rank's OWN window: the stream
// front end blocks, no kernel spins, so ranks that share one device (the
// tests) cannot starve each other of SMs.
#include <cuda.h>
#include <unistd.h>

#include <chrono>
#include <cstring>
#include <random>
#include <string>
#include <thread>

#include "ppf_internal.h"

namespace ppf {

namespace {

constexpr size_t OFF_READY_H = 0, OFF_FREED_H = 4 * PPF_PEER_MAX_RANKS;
constexpr size_t OFF_READY_R = 8 * PPF_PEER_MAX_RANKS, OFF_BLK = OFF_READY_R + 64;
constexpr size_t OFF_XCOUNT = OFF_BLK + 64;
constexpr size_t OFF_RED = 1024;
// reduction row: up to (m_max + 1) complex coefficients (m_max <= 1024) + slack
constexpr int RCAP = 2 * (1024 + 2) + 16;
constexpr uint32_t DESC_MAGIC = 0x50504650u;  // "PFPP"

struct PeerDesc {
  uint32_t magic, version;
  int32_t rank, nranks;
  int64_t pid;
  int64_t nonce;  // random per process: "same process" needs pid AND nonce to match
  uint64_t win;  // device address in the owner's process
  int64_t halo_total;
  int32_t sc, device;
  int64_t win_bytes;
  cudaIpcMemHandle_t ipc;
  int64_t recv_count[PPF_PEER_MAX_RANKS];
  int64_t recv_off[PPF_PEER_MAX_RANKS];
};
static_assert(sizeof(PeerDesc) <= PPF_PEER_DESC_BYTES, "descriptor size");

struct PushEnt {      // one receiver of this rank's boundary entries
  char* dst;          // receiver's slot-0 segment for this rank (slot 1: + stride)
  int64_t stride;     // bytes between the receiver's two slots
  int64_t off, cnt;   // segment [off, off + cnt) of this rank's send list
};

size_t halo_off(int nranks) {
  const size_t red = OFF_RED + size_t(2) * nranks * RCAP * 8;
  return (red + 255) / 256 * 256;
}

// identifies this process among the ranks (pid alone may repeat across hosts
// or containers)
int64_t process_nonce() {
  static const int64_t v = [] {
    std::random_device rd;
    return (int64_t(rd()) << 32) ^ int64_t(rd()) ^ int64_t(getpid());
  }();
  return v;
}

using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

WaitFn wait_fn() {
  static WaitFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &p, 12000, cudaEnableDefault,
                                         &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<WaitFn>(p);
  }();
  if (!fn) fail(PPF_ECUDA, "cuStreamWaitValue32 is not available from the driver");
  return fn;
}

void stream_wait_geq(cudaStream_t st, const void* addr, uint32_t value) {
  CUresult r = wait_fn()(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(addr),
                         value, CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) fail(PPF_ECUDA, "cuStreamWaitValue32 failed");
}

void check_launch(const char* what) { cuda_check(cudaGetLastError(), what); }

template <typename F>
F driver_fn(const char* name, unsigned version) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPointByVersion(name, &p, version, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    fail(PPF_ECUDA, std::string("driver entry point missing: ") + name);
  return reinterpret_cast<F>(p);
}

// Load every kernel of the module that holds `sym` now.  Under lazy module
// loading (the CUDA 12 default) the first launch of a kernel loads it, and a
// load waits for the device: a launch issued while this rank's stream sits in
// a peer wait would block the host until the peer's push arrives -- and the
// peer may be blocked the same way (measured: tools/waitvalue_probe.cu hangs
// without the preload).
void preload_module(const void* sym) {
  using GetModule = CUresult (*)(CUmodule*, CUfunction);
  using Count = CUresult (*)(unsigned*, CUmodule);
  using Enum = CUresult (*)(CUfunction*, unsigned, CUmodule);
  using Load = CUresult (*)(CUfunction);
  cudaFunction_t f;
  PPF_CUDA(cudaGetFuncBySymbol(&f, sym));
  CUmodule mod;
  if (driver_fn<GetModule>("cuFuncGetModule", 12000)(&mod, reinterpret_cast<CUfunction>(f)) !=
      CUDA_SUCCESS)
    fail(PPF_ECUDA, "cuFuncGetModule failed");
  unsigned n = 0;
  if (driver_fn<Count>("cuModuleGetFunctionCount", 12040)(&n, mod) != CUDA_SUCCESS)
    fail(PPF_ECUDA, "cuModuleGetFunctionCount failed");
  std::vector<CUfunction> fns(n);
  if (n && driver_fn<Enum>("cuModuleEnumerateFunctions", 12040)(fns.data(), n, mod) != CUDA_SUCCESS)
    fail(PPF_ECUDA, "cuModuleEnumerateFunctions failed");
  auto load = driver_fn<Load>("cuFuncLoad", 12040);
  for (CUfunction fn : fns)
    if (load(fn) != CUDA_SUCCESS) fail(PPF_ECUDA, "cuFuncLoad failed");
}

// ---------------------------------------------------------------------------
// Kernels
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) peer_push_kernel(
    const T* __restrict__ x, const int32_t* __restrict__ idx, const PushEnt* __restrict__ ent,
    int nent, int64_t total, const unsigned* xcount, unsigned* const* __restrict__ sig, int nto,
    unsigned* blk) {
  const int slot = int(*reinterpret_cast<const volatile unsigned*>(xcount) & 1u);
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    int e = 0;
    while (e + 1 < nent && i >= ent[e + 1].off) ++e;  // nent = neighbours (2 for slabs)
    T* dst = reinterpret_cast<T*>(ent[e].dst + slot * ent[e].stride);
    dst[i - ent[e].off] = x[idx[i]];
  }
  __threadfence_system();  // every thread's peer stores before the block's ticket
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(blk, 1u) == gridDim.x - 1) {
      *blk = 0;  // the next push is stream-ordered after this one
      __threadfence_system();
      // sig[0, nto): READY_H[r] in each receiver's window; sig[nto, 2 nto):
      // this rank's FREED_H[q] of the same receivers (a slot now in use)
      for (int k = 0; k < nto; ++k) atomicSub(sig[nto + k], 1u);
      for (int k = 0; k < nto; ++k) atomicAdd_system(sig[k], 1u);
    }
  }
}

// after the halo block read the receive slot: the arrivals are consumed
// (READY_H[p] -= 1, this rank's window), the slot goes back to every sender
// (FREED_H[r] += 1 in its window), the exchange count advances
__global__ void peer_consume_kernel(unsigned* const* __restrict__ sig, int nfrom,
                                    unsigned* xcount) {
  if (threadIdx.x == 0) {
    // sig[0, nfrom): own READY_H[p]; sig[nfrom, 2 nfrom): FREED_H[r] at each sender p
    for (int k = 0; k < nfrom; ++k) atomicSub(sig[k], 1u);
    __threadfence_system();
    for (int k = 0; k < nfrom; ++k) atomicAdd_system(sig[nfrom + k], 1u);
    *xcount += 1u;
  }
}

// one block: raw -> row `rank` of slot `slot` in every rank's window, then
// one arrival on every other rank
__global__ void __launch_bounds__(256) peer_red_put_kernel(const double* __restrict__ raw, int nv,
                                                           double* const* __restrict__ dst,
                                                           unsigned* const* __restrict__ sig,
                                                           int nranks, int64_t slot_stride,
                                                           int slot) {
  for (int q = 0; q < nranks; ++q) {
    double* d = dst[q] + slot * slot_stride;
    for (int i = threadIdx.x; i < nv; i += blockDim.x) d[i] = raw[i];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 0; q < nranks - 1; ++q) atomicAdd_system(sig[q], 1u);
  }
}

// raw[i] = sum over rows q = 0..nranks-1 of slot `slot`, in rank order
__global__ void __launch_bounds__(256) peer_red_sum_kernel(const double* __restrict__ rows,
                                                           int nranks, int64_t row_stride,
                                                           int nv, double* __restrict__ raw) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < nranks; ++q) s += rows[q * row_stride + i];
    raw[i] = s;
  }
}

}  // namespace

struct PeerState {
  char* win = nullptr;
  size_t win_bytes = 0;
  int nranks = 0, rank = 0, device = 0;
  bool connected = false;
  std::vector<char*> peer;         // mapped windows (own window at [rank])
  std::vector<bool> ipc_opened;
  // device tables: push entries, push signals, reduction destinations + signals
  void* d_tab = nullptr;
  PushEnt* d_ent = nullptr;
  unsigned** d_push_sig = nullptr;   // push: READY_H at receivers, own FREED_H
  unsigned** d_cons_sig = nullptr;   // consume: own READY_H, FREED_H at senders
  double** d_red_dst = nullptr;
  unsigned** d_red_sig = nullptr;
  int nent = 0, n_to = 0, n_from = 0, push_blocks = 1;
  std::vector<unsigned*> wait_ready, wait_freed;  // own counters: READY_H[p], FREED_H[q]
  uint32_t halo_epoch = 0, red_epoch = 0;
  size_t hoff = 0;
};

void peer_destroy(PeerState* p) {
  if (!p) return;
  cudaSetDevice(p->device);
  cudaDeviceSynchronize();  // no push or reduction of ours may still touch a window
  // A receiver's last push signals "consumed" into OUR window; wait (bounded)
  // until every receiver's count has reached the number of exchanges before
  // freeing the window under it (all ranks run the same exchanges).
  if (p->connected && p->halo_epoch > 0) {
    const auto t0 = std::chrono::steady_clock::now();
    for (unsigned* f : p->wait_freed) {   // both slots back from every receiver
      uint32_t v = 0;
      while (cudaMemcpy(&v, f, 4, cudaMemcpyDeviceToHost) == cudaSuccess && v < 2u &&
             std::chrono::steady_clock::now() - t0 < std::chrono::seconds(10))
        std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
  }
  for (size_t q = 0; q < p->peer.size(); ++q)
    if (p->ipc_opened[q]) cudaIpcCloseMemHandle(p->peer[q]);
  if (p->d_tab) cudaFree(p->d_tab);
  if (p->win) cudaFree(p->win);
  delete p;
}

bool peer_active(const ppf_mat* A) { return A->peer && A->peer->connected; }

void preload_kernels() {
  static bool done = false;  // per process; loading is idempotent, so a race is harmless
  if (done) return;
  preload_module(kernels_module_symbol());
  preload_module(reinterpret_cast<const void*>(&peer_red_sum_kernel));
  done = true;
}

static void ensure_comm_objects(ppf_ctx* ctx) {
  if (!ctx->comm_stream)
    PPF_CUDA(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
  if (!ctx->ev_pack) PPF_CUDA(cudaEventCreateWithFlags(&ctx->ev_pack, cudaEventDisableTiming));
  if (!ctx->ev_halo) PPF_CUDA(cudaEventCreateWithFlags(&ctx->ev_halo, cudaEventDisableTiming));
}

// comm stream: push this rank's boundary entries of x into the receivers
// (`st`: the stream the SpMV runs on -- the context's, or a capture stream)
void peer_halo_begin(ppf_ctx* ctx, ppf_mat* A, const void* x, cudaStream_t st) {
  PeerState* P = A->peer;
  cudaStream_t cs = ctx->comm_stream;
  ++P->halo_epoch;  // host count (teardown only)
  PPF_CUDA(cudaEventRecord(ctx->ev_pack, st));
  PPF_CUDA(cudaStreamWaitEvent(cs, ctx->ev_pack, 0));
  for (unsigned* f : P->wait_freed) stream_wait_geq(cs, f, 1u);
  unsigned* blk = reinterpret_cast<unsigned*>(P->win + OFF_BLK);
  const unsigned* xc = reinterpret_cast<const unsigned*>(P->win + OFF_XCOUNT);
  if (A->dtype == PPF_R64)
    peer_push_kernel<double><<<P->push_blocks, 256, 0, cs>>>(
        static_cast<const double*>(x), A->d_send_idx, P->d_ent, P->nent, A->send_total, xc,
        P->d_push_sig, P->n_to, blk);
  else
    peer_push_kernel<double2><<<P->push_blocks, 256, 0, cs>>>(
        static_cast<const double2*>(x), A->d_send_idx, P->d_ent, P->nent, A->send_total, xc,
        P->d_push_sig, P->n_to, blk);
  check_launch("peer_push_kernel");
  PPF_CUDA(cudaEventRecord(ctx->ev_halo, cs));
}

// stream `st`: this rank's push has read x, every sender's entries have
// arrived; returns the receive slots' base (the halo block picks slot
// XCOUNT&1 on the device through *sel)
const void* peer_halo_wait(ppf_ctx* ctx, ppf_mat* A, cudaStream_t st, const unsigned** sel) {
  PeerState* P = A->peer;
  PPF_CUDA(cudaStreamWaitEvent(st, ctx->ev_halo, 0));
  for (unsigned* f : P->wait_ready) stream_wait_geq(st, f, 1u);
  *sel = reinterpret_cast<const unsigned*>(P->win + OFF_XCOUNT);
  return P->win + P->hoff;
}

// stream `st`, after the halo block: arrivals consumed, slots returned
void peer_halo_done(ppf_ctx* ctx, ppf_mat* A, cudaStream_t st) {
  (void)ctx;
  PeerState* P = A->peer;
  peer_consume_kernel<<<1, 32, 0, st>>>(P->d_cons_sig, P->n_from,
                                        reinterpret_cast<unsigned*>(P->win + OFF_XCOUNT));
  check_launch("peer_consume_kernel");
}

// allreduce(sum) of raw[0:nv] over the ranks, deterministic (rank order)
void peer_allreduce(ppf_ctx* ctx, ppf_mat* A, double* raw, int nv, cudaStream_t st) {
  PeerState* P = A->peer;
  if (nv > RCAP) fail(PPF_EINVAL, "peer reduction longer than the window row");
  const uint32_t E = ++P->red_epoch;
  const int slot = int(E & 1u);
  const int64_t slot_stride = int64_t(P->nranks) * RCAP;
  peer_red_put_kernel<<<1, 256, 0, st>>>(raw, nv, P->d_red_dst, P->d_red_sig, P->nranks,
                                         slot_stride, slot);
  check_launch("peer_red_put_kernel");
  stream_wait_geq(st, P->win + OFF_READY_R, uint32_t(P->nranks - 1) * E);
  const double* rows = reinterpret_cast<const double*>(P->win + OFF_RED) + slot * slot_stride;
  peer_red_sum_kernel<<<(nv + 255) / 256, 256, 0, st>>>(rows, P->nranks, RCAP, nv, raw);
  check_launch("peer_red_sum_kernel");
}

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

ppf_status ppf_mat_peer_window(ppf_mat* A, void* desc) {
  PPF_API_BEGIN
  PPF_REQUIRE(A && desc, "NULL argument");
  PPF_REQUIRE(A->nranks > 1 && A->nranks <= PPF_PEER_MAX_RANKS,
              "peer windows need 1 < nranks <= PPF_PEER_MAX_RANKS");
  ppf_ctx* ctx = A->ctx;
  PPF_CUDA(cudaSetDevice(ctx->device));
  if (A->peer) {
    peer_destroy(A->peer);
    A->peer = nullptr;
  }
  auto* P = new PeerState();
  A->peer = P;
  P->nranks = A->nranks;
  P->rank = A->rank;
  P->device = ctx->device;
  const size_t sc = A->dtype == PPF_R64 ? 8 : 16;
  P->hoff = halo_off(A->nranks);
  P->win_bytes = P->hoff + size_t(2) * size_t(A->halo_total) * sc + 256;
  PPF_CUDA(cudaMalloc(&P->win, P->win_bytes));
  PPF_CUDA(cudaMemset(P->win, 0, P->win_bytes));
  PPF_CUDA(cudaDeviceSynchronize());
  PeerDesc d;
  std::memset(&d, 0, sizeof(d));
  d.magic = DESC_MAGIC;
  d.version = 1;
  d.rank = A->rank;
  d.nranks = A->nranks;
  d.pid = int64_t(getpid());
  d.nonce = process_nonce();
  d.win = reinterpret_cast<uint64_t>(P->win);
  d.halo_total = A->halo_total;
  d.sc = int32_t(sc);
  d.device = ctx->device;
  d.win_bytes = int64_t(P->win_bytes);
  PPF_CUDA(cudaIpcGetMemHandle(&d.ipc, P->win));
  for (int p = 0; p < A->nranks; ++p) {
    d.recv_count[p] = A->recv_count[p];
    d.recv_off[p] = A->recv_off[p];
  }
  std::memset(desc, 0, PPF_PEER_DESC_BYTES);
  std::memcpy(desc, &d, sizeof(d));
  PPF_API_END
}

ppf_status ppf_mat_peer_connect(ppf_mat* A, const void* descs) {
  PPF_API_BEGIN
  PPF_REQUIRE(A, "NULL matrix");
  if (!descs) {
    if (A->peer) A->peer->connected = false;
    return PPF_OK;
  }
  PPF_REQUIRE(A->peer && A->peer->win, "call ppf_mat_peer_window first");
  PeerState* P = A->peer;
  PPF_REQUIRE(!P->connected, "window already connected");
  ppf_ctx* ctx = A->ctx;
  PPF_CUDA(cudaSetDevice(ctx->device));
  const int R = A->nranks, me = A->rank;
  const size_t sc = A->dtype == PPF_R64 ? 8 : 16;
  std::vector<PeerDesc> D(R);
  for (int q = 0; q < R; ++q) {
    std::memcpy(&D[q], static_cast<const char*>(descs) + size_t(q) * PPF_PEER_DESC_BYTES,
                sizeof(PeerDesc));
    PPF_REQUIRE(D[q].magic == DESC_MAGIC && D[q].version == 1, "not a peer descriptor");
    PPF_REQUIRE(D[q].rank == q && D[q].nranks == R, "descriptors not in rank order / nranks");
    PPF_REQUIRE(D[q].sc == int32_t(sc), "peers disagree on the scalar type");
    PPF_REQUIRE(D[q].recv_count[me] == A->send_count[q],
                "a peer's receive count from this rank differs from this rank's send list");
  }
  PPF_REQUIRE(D[me].win == reinterpret_cast<uint64_t>(P->win), "own descriptor is stale");
  P->peer.assign(R, nullptr);
  P->ipc_opened.assign(R, false);
  const int64_t mypid = int64_t(getpid()), mynonce = process_nonce();
  for (int q = 0; q < R; ++q) {
    if (q == me) {
      P->peer[q] = P->win;
    } else if (D[q].pid == mypid && D[q].nonce == mynonce) {
      // a rank of this process: its raw pointer is only usable here if it
      // lives on this rank's device (several contexts on one GPU, the tests)
      // or peer access to its device is enabled
      if (D[q].device != ctx->device) {
        int can = 0;
        PPF_CUDA(cudaDeviceCanAccessPeer(&can, ctx->device, D[q].device));
        PPF_REQUIRE(can, "same-process rank on a device without peer access to this one");
        const cudaError_t e = cudaDeviceEnablePeerAccess(D[q].device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError();
        else PPF_CUDA(e);
      }
      P->peer[q] = reinterpret_cast<char*>(D[q].win);
    } else {
      void* p = nullptr;
      PPF_CUDA(cudaIpcOpenMemHandle(&p, D[q].ipc, cudaIpcMemLazyEnablePeerAccess));
      P->peer[q] = static_cast<char*>(p);
      P->ipc_opened[q] = true;
    }
  }
  // push entries (receivers in peer order = this rank's send-list order) and
  // signal targets: READY_H of each receiver, then FREED_H of each sender
  std::vector<PushEnt> ent;
  std::vector<unsigned*> psig, pown, csig, cown;
  for (int q = 0; q < R; ++q)
    if (q != me && A->send_count[q]) {
      const size_t qh = halo_off(R);
      ent.push_back({P->peer[q] + qh + size_t(D[q].recv_off[me]) * sc,
                     int64_t(D[q].halo_total) * int64_t(sc), A->send_off[q], A->send_count[q]});
      psig.push_back(reinterpret_cast<unsigned*>(P->peer[q] + OFF_READY_H) + me);
      pown.push_back(reinterpret_cast<unsigned*>(P->win + OFF_FREED_H) + q);
      P->wait_freed.push_back(reinterpret_cast<unsigned*>(P->win + OFF_FREED_H) + q);
    }
  P->n_to = int(ent.size());
  for (int q = 0; q < R; ++q)
    if (q != me && A->recv_count[q]) {
      cown.push_back(reinterpret_cast<unsigned*>(P->win + OFF_READY_H) + q);
      csig.push_back(reinterpret_cast<unsigned*>(P->peer[q] + OFF_FREED_H) + me);
      P->wait_ready.push_back(reinterpret_cast<unsigned*>(P->win + OFF_READY_H) + q);
    }
  P->n_from = int(cown.size());
  psig.insert(psig.end(), pown.begin(), pown.end());
  cown.insert(cown.end(), csig.begin(), csig.end());
  // both receive slots of every receiver start free
  {
    std::vector<unsigned> two(size_t(R), 2u);
    PPF_CUDA(cudaMemcpy(P->win + OFF_FREED_H, two.data(), size_t(R) * 4, cudaMemcpyHostToDevice));
  }
  P->nent = int(ent.size());
  if (ent.empty()) ent.push_back({nullptr, 0, 0, 0});
  std::vector<double*> rdst(R);
  std::vector<unsigned*> rsig;
  for (int q = 0; q < R; ++q) {
    rdst[q] = reinterpret_cast<double*>(P->peer[q] + OFF_RED) + size_t(me) * RCAP;
    if (q != me) rsig.push_back(reinterpret_cast<unsigned*>(P->peer[q] + OFF_READY_R));
  }
  const size_t b_ent = ent.size() * sizeof(PushEnt), b_ps = (psig.size() + 1) * sizeof(void*),
               b_rd = rdst.size() * sizeof(void*), b_rs = (rsig.size() + 1) * sizeof(void*),
               b_cs = (cown.size() + 1) * sizeof(void*);
  if (P->d_tab) PPF_CUDA(cudaFree(P->d_tab));
  PPF_CUDA(cudaMalloc(&P->d_tab, b_ent + b_ps + b_rd + b_rs + b_cs));
  char* t = static_cast<char*>(P->d_tab);
  P->d_ent = reinterpret_cast<PushEnt*>(t);
  P->d_push_sig = reinterpret_cast<unsigned**>(t + b_ent);
  P->d_red_dst = reinterpret_cast<double**>(t + b_ent + b_ps);
  P->d_red_sig = reinterpret_cast<unsigned**>(t + b_ent + b_ps + b_rd);
  P->d_cons_sig = reinterpret_cast<unsigned**>(t + b_ent + b_ps + b_rd + b_rs);
  if (!cown.empty())
    PPF_CUDA(cudaMemcpy(P->d_cons_sig, cown.data(), cown.size() * sizeof(void*), cudaMemcpyHostToDevice));
  PPF_CUDA(cudaMemcpy(P->d_ent, ent.data(), b_ent, cudaMemcpyHostToDevice));
  if (!psig.empty())
    PPF_CUDA(cudaMemcpy(P->d_push_sig, psig.data(), psig.size() * sizeof(void*), cudaMemcpyHostToDevice));
  PPF_CUDA(cudaMemcpy(P->d_red_dst, rdst.data(), b_rd, cudaMemcpyHostToDevice));
  if (!rsig.empty())
    PPF_CUDA(cudaMemcpy(P->d_red_sig, rsig.data(), rsig.size() * sizeof(void*), cudaMemcpyHostToDevice));
  // enough blocks to stream the boundary planes, few enough that the
  // last-block ticket stays cheap
  P->push_blocks = int(std::min<int64_t>(std::max<int64_t>((A->send_total + 255) / 256, 1),
                                         int64_t(ctx->num_sms) * 2));
  ensure_comm_objects(ctx);
  wait_fn();  // fail now, not inside a run, if the driver lacks stream waits
  preload_kernels();
  P->connected = true;
  PPF_API_END
}
