// TEST INFRASTRUCTURE ONLY -- a stand-in for libnccl.so.2 that lets several
// processes share ONE GPU, so the library's NCCL code path (run.cpp:
// halo_sendrecv on the comm stream overlapped with the diagonal-block SpMV,
// ncclAllReduce of the rank-local reduction partials on the compute stream)
// runs unmodified on a single-GPU box.  Real NCCL refuses two ranks on one
// device.  Never linked into the product libppf.so (build.py builds
// libppf_fakenccl.so from the same objects only for tests/).
//
// Semantics kept from NCCL: every operation is enqueued on its CUDA stream and
// completes in stream order; the sends/receives between a group start/end pair
// progress together (no deadlock when two ranks send to each other); messages
// between a pair of ranks match in issue order; all ranks see bit-identical
// allreduce results.  Mechanism: a stream-ordered device->host copy into pinned
// staging, a host function (cudaLaunchHostFunc) that moves the bytes over Unix
// domain sockets with poll(), a host->device copy.  The host function blocks
// only its own stream; the GPU never waits on another process's kernels.
#include <cuda_runtime.h>
#include <nccl.h>
#include <poll.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <cerrno>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

namespace {

constexpr int kTimeoutMs = 120000;  // a lost peer aborts the process instead of hanging it

[[noreturn]] void die(const char* what) {
  std::fprintf(stderr, "fake_nccl: %s (errno %d)\n", what, errno);
  std::abort();
}

size_t type_bytes(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    case ncclInt64: case ncclUint64: case ncclFloat64: return 8;
    default: return 0;
  }
}

// one point-to-point transfer of `bytes` with `peer` through host staging
struct Xfer {
  int peer;
  bool send;
  void* dev;
  size_t bytes;
  char* host = nullptr;
};

struct Batch {
  ncclComm_t comm;
  std::vector<Xfer> x;
  // allreduce (sum of doubles) instead of point-to-point
  bool allreduce = false;
  size_t count = 0;
  char* stage = nullptr;
  size_t stage_bytes = 0;
  cudaEvent_t done = nullptr;
};

}  // namespace

struct ncclComm {
  int rank = 0, nranks = 1;
  std::vector<int> fd;  // fd[p]: socket to peer p (-1 for self)
  std::string path;
  std::vector<Batch*> live;  // staging in flight, freed once `done` has fired
};

namespace {

thread_local int g_group = 0;
thread_local std::vector<Xfer> g_pending;
thread_local ncclComm_t g_pending_comm = nullptr;
thread_local cudaStream_t g_pending_stream = nullptr;

// move every transfer of `v` to completion, all at once (full duplex, poll)
void progress(ncclComm_t c, std::vector<Xfer>& v) {
  std::vector<size_t> done(v.size(), 0);
  auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    std::vector<pollfd> pf;
    std::vector<int> who;
    for (size_t i = 0; i < v.size(); ++i) {
      if (done[i] == v[i].bytes) continue;
      // one outstanding transfer per (peer, direction): keep issue order
      bool earlier = false;
      for (size_t j = 0; j < i; ++j)
        if (v[j].peer == v[i].peer && v[j].send == v[i].send && done[j] < v[j].bytes) earlier = true;
      if (earlier) continue;
      pf.push_back({c->fd[v[i].peer], short(v[i].send ? POLLOUT : POLLIN), 0});
      who.push_back(int(i));
    }
    if (pf.empty()) return;
    int r = poll(pf.data(), pf.size(), 1000);
    if (r < 0 && errno != EINTR) die("poll");
    for (size_t k = 0; k < pf.size(); ++k) {
      if (!(pf[k].revents & (POLLIN | POLLOUT | POLLHUP | POLLERR))) continue;
      Xfer& t = v[who[k]];
      size_t& d = done[who[k]];
      ssize_t n = t.send ? ::send(pf[k].fd, t.host + d, t.bytes - d, MSG_DONTWAIT | MSG_NOSIGNAL)
                         : ::recv(pf[k].fd, t.host + d, t.bytes - d, MSG_DONTWAIT);
      if (n < 0 && (errno == EAGAIN || errno == EWOULDBLOCK || errno == EINTR)) continue;
      if (n <= 0) die(t.send ? "send to peer failed" : "peer closed the connection");
      d += size_t(n);
    }
    if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(kTimeoutMs))
      die("timed out waiting for a peer");
  }
}

void CUDART_CB host_p2p(void* arg) {
  auto* b = static_cast<Batch*>(arg);
  progress(b->comm, b->x);
}

// every rank sends its vector to every peer, then sums in rank order 0..n-1,
// so all ranks hold bit-identical results
void CUDART_CB host_allreduce(void* arg) {
  auto* b = static_cast<Batch*>(arg);
  ncclComm_t c = b->comm;
  const size_t bytes = b->count * 8;
  std::vector<Xfer> v;
  for (int p = 0; p < c->nranks; ++p) {
    if (p == c->rank) continue;
    v.push_back({p, true, nullptr, bytes, b->stage + size_t(c->rank) * bytes});
    v.push_back({p, false, nullptr, bytes, b->stage + size_t(p) * bytes});
  }
  progress(c, v);
  std::vector<double> sum(b->count, 0.0);
  for (int p = 0; p < c->nranks; ++p) {
    const double* src = reinterpret_cast<const double*>(b->stage + size_t(p) * bytes);
    for (size_t i = 0; i < b->count; ++i) sum[i] += src[i];
  }
  std::memcpy(b->stage + size_t(c->rank) * bytes, sum.data(), bytes);
}

void reap(ncclComm_t c, bool wait) {
  std::vector<Batch*> keep;
  for (Batch* b : c->live) {
    if (wait) cudaEventSynchronize(b->done);
    if (cudaEventQuery(b->done) == cudaSuccess) {
      cudaEventDestroy(b->done);
      cudaFreeHost(b->stage);
      delete b;
    } else {
      keep.push_back(b);
    }
  }
  c->live.swap(keep);
}

ncclResult_t launch(Batch* b, cudaStream_t s) {
  ncclComm_t c = b->comm;
  reap(c, false);
  if (cudaMallocHost(&b->stage, b->stage_bytes ? b->stage_bytes : 8) != cudaSuccess)
    return ncclUnhandledCudaError;
  if (cudaEventCreateWithFlags(&b->done, cudaEventDisableTiming) != cudaSuccess)
    return ncclUnhandledCudaError;
  if (b->allreduce) {
    char* mine = b->stage + size_t(c->rank) * b->count * 8;
    if (cudaMemcpyAsync(mine, b->x[0].dev, b->count * 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaLaunchHostFunc(s, host_allreduce, b) != cudaSuccess ||
        cudaMemcpyAsync(b->x[1].dev, mine, b->count * 8, cudaMemcpyHostToDevice, s) != cudaSuccess)
      return ncclUnhandledCudaError;
  } else {
    size_t off = 0;
    for (auto& t : b->x) {
      t.host = b->stage + off;
      off += t.bytes;
      if (t.send && t.bytes &&
          cudaMemcpyAsync(t.host, t.dev, t.bytes, cudaMemcpyDeviceToHost, s) != cudaSuccess)
        return ncclUnhandledCudaError;
    }
    if (cudaLaunchHostFunc(s, host_p2p, b) != cudaSuccess) return ncclUnhandledCudaError;
    for (auto& t : b->x)
      if (!t.send && t.bytes &&
          cudaMemcpyAsync(t.dev, t.host, t.bytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
        return ncclUnhandledCudaError;
  }
  if (cudaEventRecord(b->done, s) != cudaSuccess) return ncclUnhandledCudaError;
  c->live.push_back(b);
  return ncclSuccess;
}

ncclResult_t flush_group() {
  if (g_pending.empty()) return ncclSuccess;
  auto* b = new Batch();
  b->comm = g_pending_comm;
  b->x.swap(g_pending);
  for (auto& t : b->x) b->stage_bytes += t.bytes;
  return launch(b, g_pending_stream);
}

ncclResult_t p2p(bool send, const void* buf, size_t count, ncclDataType_t dt, int peer,
                 ncclComm_t comm, cudaStream_t s) {
  const size_t tb = type_bytes(dt);
  if (!comm || !tb || peer < 0 || peer >= comm->nranks || peer == comm->rank)
    return ncclInvalidArgument;
  if (!g_pending.empty() && (g_pending_comm != comm || g_pending_stream != s))
    return ncclInvalidUsage;  // one communicator and stream per group (all the library uses)
  g_pending_comm = comm;
  g_pending_stream = s;
  g_pending.push_back({peer, send, const_cast<void*>(buf), count * tb});
  return g_group ? ncclSuccess : flush_group();
}

}  // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  std::memset(id, 0, sizeof(*id));
  std::random_device rd;
  std::snprintf(id->internal, sizeof(id->internal), "/tmp/ppf_fakenccl_%d_%08x", int(getpid()),
                unsigned(rd()));
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* out, int nranks, ncclUniqueId id, int rank) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks || !id.internal[0])
    return ncclInvalidArgument;
  auto* c = new ncclComm();
  c->rank = rank;
  c->nranks = nranks;
  c->fd.assign(nranks, -1);
  c->path = std::string(id.internal) + "." + std::to_string(rank);
  auto addr_of = [&](int r) {
    sockaddr_un a{};
    a.sun_family = AF_UNIX;
    std::snprintf(a.sun_path, sizeof(a.sun_path), "%s.%d", id.internal, r);
    return a;
  };
  // listen first, then connect to every lower rank (completes from the
  // backlog), then accept every higher rank; each side names itself
  int ls = socket(AF_UNIX, SOCK_STREAM, 0);
  sockaddr_un me = addr_of(rank);
  unlink(me.sun_path);
  if (ls < 0 || bind(ls, reinterpret_cast<sockaddr*>(&me), sizeof(me)) != 0 || listen(ls, 256) != 0)
    die("listen");
  for (int p = 0; p < rank; ++p) {
    sockaddr_un a = addr_of(p);
    int s = socket(AF_UNIX, SOCK_STREAM, 0);
    auto t0 = std::chrono::steady_clock::now();
    while (connect(s, reinterpret_cast<sockaddr*>(&a), sizeof(a)) != 0) {
      if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(kTimeoutMs))
        die("connect timed out");
      std::this_thread::sleep_for(std::chrono::milliseconds(10));
      close(s);
      s = socket(AF_UNIX, SOCK_STREAM, 0);
    }
    if (::send(s, &rank, sizeof(rank), MSG_NOSIGNAL) != sizeof(rank)) die("handshake send");
    c->fd[p] = s;
  }
  for (int k = rank + 1; k < nranks; ++k) {
    pollfd pf{ls, POLLIN, 0};
    if (poll(&pf, 1, kTimeoutMs) != 1) die("accept timed out");
    int s = accept(ls, nullptr, nullptr);
    int who = -1;
    if (s < 0 || ::recv(s, &who, sizeof(who), MSG_WAITALL) != sizeof(who) || who <= rank ||
        who >= nranks || c->fd[who] != -1)
      die("handshake recv");
    c->fd[who] = s;
  }
  close(ls);
  unlink(me.sun_path);
  *out = c;
  return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t c) {
  if (!c) return ncclSuccess;
  reap(c, true);
  for (int s : c->fd)
    if (s >= 0) close(s);
  delete c;
  return ncclSuccess;
}

ncclResult_t ncclGroupStart() {
  ++g_group;
  return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
  if (g_group <= 0) return ncclInvalidUsage;
  return --g_group ? ncclSuccess : flush_group();
}

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t dt, int peer, ncclComm_t comm,
                      cudaStream_t s) {
  return p2p(true, buf, count, dt, peer, comm, s);
}

ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t dt, int peer, ncclComm_t comm,
                      cudaStream_t s) {
  return p2p(false, buf, count, dt, peer, comm, s);
}

ncclResult_t ncclAllReduce(const void* sendbuf, void* recvbuf, size_t count, ncclDataType_t dt,
                           ncclRedOp_t op, ncclComm_t comm, cudaStream_t s) {
  if (!comm || dt != ncclFloat64 || op != ncclSum) return ncclInvalidArgument;
  if (g_group) return ncclInvalidUsage;
  auto* b = new Batch();
  b->comm = comm;
  b->allreduce = true;
  b->count = count;
  b->stage_bytes = size_t(comm->nranks) * count * 8;
  b->x.push_back({comm->rank, true, const_cast<void*>(sendbuf), count * 8});
  b->x.push_back({comm->rank, false, recvbuf, count * 8});
  return launch(b, s);
}

const char* ncclGetErrorString(ncclResult_t) { return "fake_nccl error"; }

ncclResult_t ncclCommGetAsyncError(ncclComm_t comm, ncclResult_t* err) {
  if (!comm || !err) return ncclInvalidArgument;
  *err = ncclSuccess;  // failures abort the process (die) instead
  return ncclSuccess;
}

}  // extern "C"
