// C ABI entry points (include/ppf.h): errors, context, operator planning and
// upload, polynomial objects, the host dense kernel.  ppf_run lives in run.cpp.
#include <climits>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>

#include "ppf_internal.h"

// default tile of the pair-code slice schedule (0 x 0: slices in order)
#ifndef PPF_SELLP_TILE_TY
#define PPF_SELLP_TILE_TY 0
#define PPF_SELLP_TILE_TZ 0
#endif

namespace ppf {

static thread_local std::string g_last_error;

void set_last_error(const std::string& msg) { g_last_error = msg; }

[[noreturn]] void fail(ppf_status st, const std::string& msg) { throw Error{st, msg}; }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(PPF_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Warps per SELL slice (kernels.cu sell*_kernel).  KS > 1 only pays when the
// matrix has fewer slices than about two full blocks per SM (then each warp
// task is too long for the machine to fill) and rows are wide enough to
// split; every BASELINE config gets KS = 1 (measured).
int auto_sell_ks(const ppf_mat* m, int num_sms) {
  if (m->fmt != PPF_FMT_SELL || m->nslices == 0) return 1;
  const double width = double(m->stored) / (double(m->nslices) * m->C);
  const double few = 2.0 * num_sms * 8;
  int ks = 1;
  while (ks < 8 && double(m->nslices) * ks < few && width / (2 * ks) >= 8.0) ks *= 2;
  return ks;
}

// Leading slices whose width is >= 2x the mean (and >= 16 entries per lane):
// after a whole-matrix sigma sort (descending row length) these are the
// power-law rows.  One warp per such slice would be the critical path of the
// whole launch (C7: the 239-entry slices, 38.9 us/launch at KS = 1, 20.0 at a
// uniform KS = 4 that idles the short slices' extra warps), so the SELL kernel
// gives each of them a block of 8 warps.  0 when every slice is heavy.
int64_t sell_heavy_prefix(const std::vector<int64_t>& ptr, int C) {
  const int64_t ns = int64_t(ptr.size()) - 1;
  if (ns <= 0) return 0;
  const double mean = double(ptr[ns]) / (double(ns) * C);
  // (C7: 2x/16 -> 17.1 us per SpMV, 4x/32 -> 18.8, 1.5x/12 -> 18.9)
  const double thr = std::max(16.0, 2.0 * mean);
  int64_t h = 0;
  while (h < ns && double(ptr[h + 1] - ptr[h]) / C >= thr) ++h;
  return h == ns ? 0 : h;
}

}  // namespace ppf

using namespace ppf;

#define PPF_API_BEGIN try {
#define PPF_API_END                      \
  return PPF_OK;                         \
  }                                      \
  catch (const ppf::Error& e) {          \
    ppf::set_last_error(e.msg);          \
    return e.st;                         \
  }                                      \
  catch (const std::bad_alloc&) {        \
    ppf::set_last_error("out of host memory"); \
    return PPF_EINVAL;                   \
  }                                      \
  catch (...) {                          \
    ppf::set_last_error("unknown C++ exception"); \
    return PPF_EINVAL;                   \
  }

extern "C" {

const char* ppf_status_string(int st) {
  switch (st) {
    case PPF_OK: return "PPF_OK";
    case PPF_EINVAL: return "PPF_EINVAL";
    case PPF_ECUDA: return "PPF_ECUDA";
    case PPF_ENCCL: return "PPF_ENCCL";
    case PPF_EWORKSPACE: return "PPF_EWORKSPACE";
    case PPF_EBRANCH: return "PPF_EBRANCH";
    case PPF_EDENSE: return "PPF_EDENSE";
    case PPF_ESTATE: return "PPF_ESTATE";
    default: return "PPF_UNKNOWN";
  }
}

const char* ppf_last_error(void) { return g_last_error.c_str(); }
int ppf_abi_version(void) { return PPF_ABI_VERSION; }

// ---------------------------------------------------------------------------
// Context
// ---------------------------------------------------------------------------
ppf_status ppf_nccl_unique_id(void* out128) {
  PPF_API_BEGIN
  PPF_REQUIRE(out128, "out128 is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) fail(PPF_ENCCL, "ncclGetUniqueId failed");
  std::memcpy(out128, &id, 128);
  PPF_API_END
}

ppf_status ppf_ctx_create(int device, int rank, int nranks, const void* id128, void* stream,
                          ppf_ctx** out) {
  PPF_API_BEGIN
  PPF_REQUIRE(out, "out is NULL");
  PPF_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank/nranks");
  PPF_CUDA(cudaSetDevice(device));
  auto* c = new ppf_ctx();
  c->device = device;
  c->rank = rank;
  c->nranks = nranks;
  c->stream = static_cast<cudaStream_t>(stream);
  c->nccl_comm = nullptr;
  c->comm_stream = nullptr;
  c->ev_pack = c->ev_halo = nullptr;
  c->last_m = 0;
  c->last_beta0 = 0.0;
  c->last_dtype = PPF_R64;
  c->launches = 0;
  c->profile = 0;
  for (auto& p : c->prof) p = {0, 0.0, 0.0};
  try {
    PPF_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    c->h_pinned_bytes = size_t(66) * 65 * 16 + 2 * 2048;  // grown by ppf_run for larger m_max
    PPF_CUDA(cudaHostAlloc(&c->h_pinned, c->h_pinned_bytes, cudaHostAllocDefault));
    PPF_CUDA(cudaEventCreateWithFlags(&c->ev, cudaEventDisableTiming));
    PPF_CUDA(cudaEventCreate(&c->ev_t0));
    PPF_CUDA(cudaEventCreate(&c->ev_t1));
    if (nranks > 1) ppf::preload_kernels();
    if (nranks > 1 && id128) {
      ncclUniqueId id;
      std::memcpy(&id, id128, 128);
      ncclComm_t comm;
      if (ncclCommInitRank(&comm, nranks, id, rank) != ncclSuccess)
        fail(PPF_ENCCL, "ncclCommInitRank failed");
      c->nccl_comm = comm;
      PPF_CUDA(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
      PPF_CUDA(cudaEventCreateWithFlags(&c->ev_pack, cudaEventDisableTiming));
      PPF_CUDA(cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming));
    }
  } catch (...) {
    delete c;
    throw;
  }
  *out = c;
  PPF_API_END
}

ppf_status ppf_ctx_set_transport(ppf_ctx* c, const ppf_transport* t) {
  PPF_API_BEGIN
  PPF_REQUIRE(c, "NULL ctx");
  if (!t) {
    c->has_transport = false;
    return PPF_OK;
  }
  PPF_REQUIRE(c->nranks > 1, "a transport needs nranks > 1");
  PPF_REQUIRE(!c->nccl_comm, "context already has an NCCL communicator");
  PPF_REQUIRE(t->exchange && t->allreduce_sum, "NULL transport function");
  c->transport = *t;
  c->has_transport = true;
  PPF_API_END
}

ppf_status ppf_ctx_set_graphs(ppf_ctx* c, int on) {
  PPF_API_BEGIN
  PPF_REQUIRE(c, "NULL ctx");
  c->use_graphs = on ? 1 : 0;
  PPF_API_END
}

ppf_status ppf_profile_enable(ppf_ctx* c, int on) {
  PPF_API_BEGIN
  PPF_REQUIRE(c, "NULL ctx");
  c->profile = on ? 1 : 0;
  for (auto& p : c->prof) p = {0, 0.0, 0.0};
  PPF_API_END
}

ppf_status ppf_profile_read(ppf_ctx* c, int cls, long long* launches, double* ms, double* bytes) {
  PPF_API_BEGIN
  PPF_REQUIRE(c && cls >= 0 && cls < 3, "bad arguments");
  if (launches) *launches = c->prof[cls].launches;
  if (ms) *ms = c->prof[cls].ms;
  if (bytes) *bytes = c->prof[cls].bytes;
  PPF_API_END
}

void ppf_ctx_destroy(ppf_ctx* c) {
  if (!c) return;
  for (auto e : c->prof_pool) cudaEventDestroy(e);
  if (c->nccl_comm) ncclCommDestroy(static_cast<ncclComm_t>(c->nccl_comm));
  if (c->h_pinned) cudaFreeHost(c->h_pinned);
  if (c->t_host) cudaFreeHost(c->t_host);
  if (c->ev) cudaEventDestroy(c->ev);
  if (c->res_ctl) cudaFreeHost(c->res_ctl);
  if (c->ev_t0) cudaEventDestroy(c->ev_t0);
  if (c->ev_t1) cudaEventDestroy(c->ev_t1);
  if (c->ev_pack) cudaEventDestroy(c->ev_pack);
  if (c->ev_halo) cudaEventDestroy(c->ev_halo);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  delete c;
}

// ---------------------------------------------------------------------------
// Slice schedule of the pair-code SpMV (HostBlock::sched).  The pair table's
// offsets say which rows gather from each other: with a1 < a2 the two smallest
// |col - row| >= C (a 3-D stencil's +-N and +-N^2), slices G1 = a1 / C and
// G2 = a2 / C apart are y- and z-neighbours.  A block of 8 warps takes a
// ty x tz tile of such slices (same residue r modulo G1), so most of the +-a1 /
// +-a2 gathers of its rows fall on lines another warp of the block also reads
// (8 consecutive slices of C4 -- two grid lines -- pull 32 quarter-lines of x
// through L1 for their 8; a 4 x 2 tile pulls 20).  Blocks run r fastest, so
// neighbouring blocks still stream neighbouring slices.  PPF_SELLP_TILE =
// "0" (none) | "TYxTZ" (TY * TZ = 8).  Scheduling only.  Measured (one B200,
// SpMV ms per solve, C4 / C3 deg 20): in order 124.8 / 74.5, 4x2 128.4 / 77.5,
// 8x1 129.5 / 79.0, 2x4 129.6 / 77.6 -- the tiles lose the single ascending
// front of the in-order launch and the kernel is not bound by L1 misses, so
// the default (PPF_SELLP_TILE_TY = 0) is no schedule.
// ---------------------------------------------------------------------------
static void build_slice_schedule(HostBlock& B, int C) {
  B.sched.clear();
  int ty = PPF_SELLP_TILE_TY, tz = PPF_SELLP_TILE_TZ;
  if (const char* ev = std::getenv("PPF_SELLP_TILE")) {
    if (ev[0] == '0') return;
    int a = 0, b = 0;
    if (std::sscanf(ev, "%dx%d", &a, &b) == 2 && a > 0 && b > 0 && a * b == 8) {
      ty = a;
      tz = b;
    }
  }
  if (ty <= 0) return;
  std::vector<int64_t> far;
  for (int32_t o : B.tab_off) {
    const int64_t a = o < 0 ? -int64_t(o) : int64_t(o);
    if (a >= C) far.push_back(a);
  }
  std::sort(far.begin(), far.end());
  far.erase(std::unique(far.begin(), far.end()), far.end());
  const int64_t ns = B.nslices;
  if (far.empty() || ns < 64) return;
  const int64_t G1 = std::max<int64_t>(1, (far[0] + C / 2) / C);
  int64_t G2 = ns;   // one plane: a 2-D stencil, tiles of 8 along y
  for (size_t i = 1; i < far.size(); ++i) {
    const int64_t g = (far[i] + C / 2) / C;
    if (g >= 2 * G1 * ty) {
      G2 = std::min(g, ns);
      break;
    }
  }
  if (G2 >= ns) {
    ty = 8;
    tz = 1;
  }
  const int64_t nz = (ns + G2 - 1) / G2, ny = (G2 + G1 - 1) / G1;
  B.sched.reserve(size_t(ns + ns / 8));
  for (int64_t zt = 0; zt * tz < nz; ++zt)
    for (int64_t yt = 0; yt * ty < ny; ++yt)
      for (int64_t r = 0; r < G1; ++r) {
        int32_t blk[8];
        bool any = false;
        for (int wz = 0; wz < tz; ++wz)
          for (int wy = 0; wy < ty; ++wy) {
            const int64_t z = zt * tz + wz, y = yt * ty + wy, in = y * G1 + r;
            const int64_t sl = z * G2 + in;
            const bool ok = z < nz && y < ny && in < G2 && sl < ns;
            blk[wz * ty + wy] = ok ? int32_t(sl) : -1;
            any |= ok;
          }
        if (any) B.sched.insert(B.sched.end(), blk, blk + 8);
      }
}

// ---------------------------------------------------------------------------
// Plan: host conversion CSR slab -> device layout (diag block SELL or CSR,
// off-rank columns into a compact halo CSR).
// ---------------------------------------------------------------------------
ppf_status ppf_plan_create(ppf_dtype dtype, int64_t n_global, int nranks, int rank,
                           const int64_t* row_bounds, const int64_t* row_ptr, const int64_t* col,
                           const void* val, ppf_format format, int sell_C, int sell_sigma,
                           ppf_plan** out) {
  PPF_API_BEGIN
  PPF_REQUIRE(out, "out is NULL");
  PPF_REQUIRE(dtype == PPF_R64 || dtype == PPF_C128, "bad dtype");
  PPF_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank/nranks");
  PPF_REQUIRE(row_bounds && row_ptr, "NULL row_bounds/row_ptr");
  PPF_REQUIRE(n_global >= 1 && n_global < (int64_t(1) << 31), "n_global out of range");
  PPF_REQUIRE(row_bounds[0] == 0 && row_bounds[nranks] == n_global, "row_bounds must span [0, n)");
  for (int r = 0; r < nranks; ++r)
    PPF_REQUIRE(row_bounds[r] <= row_bounds[r + 1], "row_bounds not nondecreasing");
  const int64_t row0 = row_bounds[rank], n_local = row_bounds[rank + 1] - row0;
  PPF_REQUIRE(n_local >= 1, "empty row slab");
  PPF_REQUIRE(row_ptr[0] == 0, "row_ptr[0] != 0");
  for (int64_t i = 0; i < n_local; ++i)
    PPF_REQUIRE(row_ptr[i + 1] >= row_ptr[i], "row_ptr not monotone");
  const int64_t nnz = row_ptr[n_local];
  PPF_REQUIRE(nnz == 0 || (col && val), "NULL col/val");
  PPF_REQUIRE(nnz < (int64_t(1) << 40), "nnz too large");
  for (int64_t i = 0; i < n_local; ++i)
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      PPF_REQUIRE(col[k] >= 0 && col[k] < n_global, "column index out of range");
      PPF_REQUIRE(k == row_ptr[i] || col[k] > col[k - 1], "columns not strictly sorted in a row");
    }
  PPF_REQUIRE(format == PPF_FMT_SELL || format == PPF_FMT_CSR, "bad format");
  if (format == PPF_FMT_SELL) {
    PPF_REQUIRE(sell_C == 32 || (sell_C == 64 && dtype == PPF_R64),
                "sell_C must be 32 (or 64 for R64)");
    PPF_REQUIRE(sell_sigma >= 1, "sell_sigma >= 1");
    PPF_REQUIRE(sell_sigma == 1 || (sell_sigma % sell_C == 0 && sell_C == 32),
                "sell_sigma must be 1 or a multiple of C (C = 32 when sorting)");
  }
  const int ND = dtype == PPF_R64 ? 1 : 2;
  const double* v = static_cast<const double*>(val);

  auto* p = new ppf_plan();
  std::unique_ptr<ppf_plan> guard(p);
  p->dtype = dtype;
  p->n_global = n_global;
  p->row0 = row0;
  p->n_local = n_local;
  p->nnz = nnz;
  p->nranks = nranks;
  p->rank = rank;
  p->bounds.assign(row_bounds, row_bounds + nranks + 1);
  p->fmt = format;
  p->C = format == PPF_FMT_SELL ? sell_C : 1;
  p->sigma = format == PPF_FMT_SELL ? sell_sigma : 1;
  p->recv.assign(nranks, {});
  p->send.assign(nranks, {});
  const int64_t row1 = row0 + n_local;
  auto owner = [&](int64_t g) {
    return int(std::upper_bound(p->bounds.begin(), p->bounds.end(), g) - p->bounds.begin()) - 1;
  };
  // diagonal-block row lengths and halo needs
  std::vector<int64_t> dlen(n_local, 0);
  int64_t halo_nnz = 0;
  for (int64_t i = 0; i < n_local; ++i)
    for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      if (col[k] >= row0 && col[k] < row1)
        ++dlen[i];
      else {
        ++halo_nnz;
        p->recv[owner(col[k])].push_back(col[k]);
      }
    }
  p->recv_off.assign(nranks + 1, 0);
  for (int r = 0; r < nranks; ++r) {
    auto& rv = p->recv[r];
    std::sort(rv.begin(), rv.end());
    rv.erase(std::unique(rv.begin(), rv.end()), rv.end());
    p->recv_off[r + 1] = p->recv_off[r] + int64_t(rv.size());
  }
  // halo block
  if (halo_nnz) {
    auto& H = p->halo;
    H.ptr.push_back(0);
    for (int64_t i = 0; i < n_local; ++i) {
      bool any = false;
      for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
        if (col[k] >= row0 && col[k] < row1) continue;
        const int o = owner(col[k]);
        const auto& rv = p->recv[o];
        const int64_t pos = std::lower_bound(rv.begin(), rv.end(), col[k]) - rv.begin();
        H.col.push_back(int32_t(p->recv_off[o] + pos));
        for (int d = 0; d < ND; ++d) H.val.push_back(v[k * ND + d]);
        any = true;
      }
      if (any) {
        H.rows.push_back(int32_t(i));
        H.ptr.push_back(int64_t(H.col.size()));
      }
    }
  }
  // diagonal block
  auto& B = p->diag;
  B.rows = n_local;
  if (format == PPF_FMT_CSR) {
    B.ptr.assign(n_local + 1, 0);
    for (int64_t i = 0; i < n_local; ++i) B.ptr[i + 1] = B.ptr[i] + dlen[i];
    B.col.resize(B.ptr[n_local]);
    B.val.resize(size_t(B.ptr[n_local]) * ND);
    for (int64_t i = 0; i < n_local; ++i) {
      int64_t o = B.ptr[i];
      for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
        if (col[k] < row0 || col[k] >= row1) continue;
        B.col[o] = int32_t(col[k] - row0);
        for (int d = 0; d < ND; ++d) B.val[size_t(o) * ND + d] = v[k * ND + d];
        ++o;
      }
    }
  } else {
    const int C = p->C;
    std::vector<int32_t> perm(n_local);
    for (int64_t i = 0; i < n_local; ++i) perm[i] = int32_t(i);
    if (p->sigma > 1) {
      for (int64_t w0 = 0; w0 < n_local; w0 += p->sigma) {
        const int64_t w1 = std::min<int64_t>(n_local, w0 + p->sigma);
        std::stable_sort(perm.begin() + w0, perm.begin() + w1,
                         [&](int32_t a, int32_t b) { return dlen[a] > dlen[b]; });
      }
      B.perm = perm;
    }
    B.nslices = (n_local + C - 1) / C;
    B.ptr.assign(B.nslices + 1, 0);
    for (int64_t s = 0; s < B.nslices; ++s) {
      int64_t w = 0;
      for (int64_t pp = s * C; pp < std::min<int64_t>(n_local, (s + 1) * C); ++pp)
        w = std::max(w, dlen[perm[pp]]);
      B.ptr[s + 1] = B.ptr[s] + w * C;
    }
    const int64_t stored = B.ptr[B.nslices];
    B.col.assign(stored, 0);
    B.val.assign(size_t(stored) * ND, 0.0);
    for (int64_t s = 0; s < B.nslices; ++s) {
      const int64_t w = (B.ptr[s + 1] - B.ptr[s]) / C;
      const int32_t pad_col = perm[s * C];
      for (int lane = 0; lane < C; ++lane) {
        const int64_t pp = s * C + lane;
        int64_t k = 0;
        if (pp < n_local) {
          const int64_t i = perm[pp];
          for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
            if (col[e] < row0 || col[e] >= row1) continue;
            const int64_t idx = B.ptr[s] + k * C + lane;
            B.col[idx] = int32_t(col[e] - row0);
            for (int d = 0; d < ND; ++d) B.val[size_t(idx) * ND + d] = v[e * ND + d];
            ++k;
          }
        }
        for (; k < w; ++k) B.col[B.ptr[s] + k * C + lane] = pad_col;
      }
    }
    // 16-bit column deltas (SELL-64, fp64, no sorting): per (slice s, column k)
    // a base offset b = min over the slice's real entries of (col - row); each
    // entry stores col - row - b in 16 bits.  Relative to the row, a stencil's
    // k-th entries of one slice differ only by where the boundary shifts them
    // (C4, N = 256: offsets within one (s, k) span at most N^2 - 1 = 65535),
    // so the index stream shrinks from 4 to 2 + 4/64 bytes per entry (C4: 12
    // -> 10.06 bytes per stored entry).  If any (s, k) spans more than 65535
    // the plan keeps 32-bit indices.  PPF_IDX16=0 keeps them always.
    const char* e16 = std::getenv("PPF_IDX16");
    // (complex SELL-32 and fp64 SELL-64: the bandwidth-bound layouts; on the
    // fp64 SELL-32 operators -- small, L2-resident, latency-bound -- the extra
    // base load per entry cost more than the bytes saved: C2 deg 5 8.8 -> 9.6 ms)
    if (((C == 32 && p->dtype == PPF_C128) || (C == 64 && p->dtype == PPF_R64)) &&
        p->sigma <= 1 && !(e16 && e16[0] == '0') && stored > 0) {
      std::vector<int32_t> cb(size_t(stored / C));
      std::vector<uint16_t> d16(size_t(stored), 0);
      bool ok = true;
      for (int64_t s = 0; s < B.nslices && ok; ++s) {
        const int64_t w = (B.ptr[s + 1] - B.ptr[s]) / C;
        for (int64_t k = 0; k < w && ok; ++k) {
          int64_t lo = INT64_MAX, hi = INT64_MIN;
          for (int lane = 0; lane < C; ++lane) {
            const int64_t pp = s * C + lane;
            if (pp >= n_local || k >= dlen[pp]) continue;   // padding
            const int64_t off = int64_t(B.col[B.ptr[s] + k * C + lane]) - pp;
            lo = std::min(lo, off);
            hi = std::max(hi, off);
          }
          if (lo == INT64_MAX) lo = hi = 0;   // all padding (delta 0: col = row)
          if (hi - lo > 65535) {
            ok = false;
            break;
          }
          cb[size_t(B.ptr[s] / C + k)] = int32_t(lo);
          for (int lane = 0; lane < C && ok; ++lane) {
            const int64_t pp = s * C + lane;
            const size_t idx = size_t(B.ptr[s] + k * C + lane);
            if (pp < n_local && k < dlen[pp]) {
              d16[idx] = uint16_t(int64_t(B.col[idx]) - pp - lo);
              continue;
            }
            // padding (val 0): delta 0; the kernel clamps every decoded column
            // to [0, n), so the x it reads there is in bounds
            d16[idx] = 0;
          }
        }
      }
      if (ok) {
        B.cb.swap(cb);
        B.d16.swap(d16);
        p->enc = PPF_ENC_DELTA16;
      }
    }
    // Pair codes (SELL-64 fp64, no sorting): every stored entry, padding
    // included, becomes an 8-bit index into a table of (col - row, value)
    // pairs when there are at most 256 distinct pairs -- the constant
    // diagonals of a constant-coefficient stencil (C3: 7 pairs + the padding
    // pair, C4: 7 + 1).  1 byte per entry instead of 10.06 (deltas) or 12
    // (explicit); the kernel takes the pair from shared memory and does the
    // same multiply-adds in the same order.  Padding is the pair (0, +0.0):
    // column = row (clamped to the last row in the kernel), value 0, as the
    // delta layout's padding.  PPF_PAIR8=0 keeps the wider layouts.
    const char* ep = std::getenv("PPF_PAIR8");
    if (C == 64 && p->dtype == PPF_R64 && p->sigma <= 1 && !(ep && ep[0] == '0') && stored > 0) {
      // open-addressing table keyed by (offset, value bits); 1024 slots for
      // at most 256 keys
      constexpr int SLOTS = 1024;
      std::vector<int> slot(SLOTS, -1);
      std::vector<int32_t> toff;
      std::vector<double> tval;
      std::vector<uint64_t> tbits;
      std::vector<uint8_t> code(size_t(stored), 0);
      bool ok = true;
      auto code_of = [&](int64_t off, double v) -> int {
        uint64_t bits;
        std::memcpy(&bits, &v, 8);
        uint64_t h = (uint64_t(off) * 0x9E3779B97F4A7C15ull) ^ (bits * 0xC2B2AE3D27D4EB4Full);
        h ^= h >> 29;
        for (int probe = 0; probe < SLOTS; ++probe) {
          const int sl = int((h + uint64_t(probe)) & (SLOTS - 1));
          const int c = slot[sl];
          if (c < 0) {
            if (toff.size() == 256) return -1;
            slot[sl] = int(toff.size());
            toff.push_back(int32_t(off));
            tval.push_back(v);
            tbits.push_back(bits);
            return slot[sl];
          }
          if (toff[c] == off && tbits[c] == bits) return c;
        }
        return -1;
      };
      // Lane-major chunks: slice s's codes start at pptr[s] (a multiple of
      // 512) and come in chunks of 8 columns; in chunk c, the 16 bytes at
      // 16 l hold column k = 8 c + j of rows 2l, 2l + 1 at bytes 2j, 2j + 1
      // -- one 16-B load gives a lane all its codes of 8 columns.  pptr[s]
      // carries the slice width w (< 512) in its low 9 bits.
      std::vector<int64_t> pptr(B.nslices + 1, 0);
      for (int64_t s = 0; s < B.nslices; ++s) {
        const int64_t w = (B.ptr[s + 1] - B.ptr[s]) / C;
        if (w >= 512) ok = false;
        pptr[s + 1] = pptr[s] + 512 * ((w + 7) / 8);
      }
      if (ok) code.assign(size_t(pptr[B.nslices]), 0);
      for (int64_t s = 0; s < B.nslices && ok; ++s) {
        const int64_t w = (B.ptr[s + 1] - B.ptr[s]) / C;
        for (int64_t k = 0; k < w && ok; ++k) {
          for (int lane = 0; lane < C; ++lane) {
            const int64_t pp = s * C + lane;
            const size_t idx = size_t(B.ptr[s] + k * C + lane);
            const bool real = pp < n_local && k < dlen[pp];
            const int c = real ? code_of(int64_t(B.col[idx]) - pp, B.val[idx]) : code_of(0, 0.0);
            if (c < 0) {
              ok = false;
              break;
            }
            code[size_t(pptr[s] + 512 * (k / 8) + 16 * (lane / 2) + 2 * (k % 8) + (lane % 2))] =
                uint8_t(c);
          }
        }
      }
      if (ok) {
        for (int64_t s = 0; s < B.nslices; ++s) pptr[s] |= (B.ptr[s + 1] - B.ptr[s]) / C;
        B.pptr.swap(pptr);
        B.code8.swap(code);
        B.tab_off.swap(toff);
        B.tab_val.swap(tval);
        p->enc = PPF_ENC_PAIR8;
        build_slice_schedule(B, C);
      }
    }
  }
  p->sends_set = (nranks == 1);
  *out = guard.release();
  PPF_API_END
}

ppf_status ppf_plan_slice_schedule(const ppf_plan* p, int32_t* out, int64_t cap, int64_t* count) {
  PPF_API_BEGIN
  PPF_REQUIRE(p && count, "NULL argument");
  PPF_REQUIRE(cap >= 0, "negative capacity");
  const std::vector<int32_t> none;
  const std::vector<int32_t>& sc = p->enc == PPF_ENC_PAIR8 ? p->diag.sched : none;
  *count = int64_t(sc.size());
  if (out)
    for (int64_t i = 0; i < cap && i < *count; ++i) out[i] = sc[size_t(i)];
  PPF_API_END
}

ppf_status ppf_plan_index_bits(const ppf_plan* p, int* bits) {
  PPF_API_BEGIN
  PPF_REQUIRE(p && bits, "NULL argument");
  *bits = p->enc == PPF_ENC_PAIR8 ? 8 : p->enc == PPF_ENC_DELTA16 ? 16 : 32;
  PPF_API_END
}

ppf_status ppf_plan_encoding(const ppf_plan* p, int* enc, int* ntab) {
  PPF_API_BEGIN
  PPF_REQUIRE(p, "NULL plan");
  if (enc) *enc = p->enc;
  if (ntab) *ntab = p->enc == PPF_ENC_PAIR8 ? int(p->diag.tab_off.size()) : 0;
  PPF_API_END
}

ppf_status ppf_plan_set_encoding(ppf_plan* p, int enc) {
  PPF_API_BEGIN
  PPF_REQUIRE(p, "NULL plan");
  const bool avail = enc == PPF_ENC_EXPLICIT ||
                     (enc == PPF_ENC_DELTA16 && !p->diag.d16.empty()) ||
                     (enc == PPF_ENC_PAIR8 && !p->diag.code8.empty());
  PPF_REQUIRE(avail, "encoding not available for this plan");
  p->enc = enc;
  PPF_API_END
}

ppf_status ppf_plan_halo_count(const ppf_plan* p, int peer, int64_t* count) {
  PPF_API_BEGIN
  PPF_REQUIRE(p && count && peer >= 0 && peer < p->nranks, "bad arguments");
  *count = int64_t(p->recv[peer].size());
  PPF_API_END
}

ppf_status ppf_plan_halo_recv(const ppf_plan* p, int peer, int64_t* idx) {
  PPF_API_BEGIN
  PPF_REQUIRE(p && peer >= 0 && peer < p->nranks, "bad arguments");
  PPF_REQUIRE(idx || p->recv[peer].empty(), "idx is NULL");
  std::copy(p->recv[peer].begin(), p->recv[peer].end(), idx);
  PPF_API_END
}

ppf_status ppf_plan_set_halo_send(ppf_plan* p, int peer, int64_t count, const int64_t* rows) {
  PPF_API_BEGIN
  PPF_REQUIRE(p && peer >= 0 && peer < p->nranks && count >= 0, "bad arguments");
  PPF_REQUIRE(peer != p->rank || count == 0, "cannot send to self");
  PPF_REQUIRE(count == 0 || rows, "rows is NULL");
  for (int64_t i = 0; i < count; ++i)
    PPF_REQUIRE(rows[i] >= 0 && rows[i] < p->n_local, "send row out of range");
  p->send[peer].assign(rows, rows + count);
  p->sends_set = true;
  PPF_API_END
}

static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

struct Layout {
  size_t ptr, col, cb, val, sched, perm, hrows, hptr, hcol, hval, recv, send, sidx, total;
};

static Layout layout_of(const ppf_plan* p) {
  const size_t sc = p->dtype == PPF_R64 ? 8 : 16;
  Layout L{};
  size_t o = 0;
  L.ptr = o;
  o += al256(p->diag.ptr.size() * 8);
  L.col = o;   // 32-bit indices, or the 16-bit deltas + per-(slice, column) bases,
               // or the pair codes + the pair table's offsets (L.cb) and values (L.val)
  if (p->enc == PPF_ENC_PAIR8) {
    o += al256(p->diag.code8.size());
    L.cb = o;
    o += al256(p->diag.tab_off.size() * 4);
    L.val = o;
    o += al256(p->diag.tab_val.size() * 8);
    L.sched = o;
    o += al256(p->diag.sched.size() * 4);
  } else {
    if (p->enc == PPF_ENC_EXPLICIT) {
      o += al256(p->diag.col.size() * 4);
      L.cb = o;
    } else {
      o += al256(p->diag.d16.size() * 2);
      L.cb = o;
      o += al256(p->diag.cb.size() * 4);
    }
    L.val = o;
    o += al256(p->diag.col.size() * sc);
  }
  L.perm = o;
  o += al256(p->diag.perm.size() * 4);
  L.hrows = o;
  o += al256(p->halo.rows.size() * 4);
  L.hptr = o;
  o += al256(p->halo.ptr.size() * 8);
  L.hcol = o;
  o += al256(p->halo.col.size() * 4);
  L.hval = o;
  o += al256(p->halo.col.size() * sc);
  int64_t recv_total = p->recv_off.empty() ? 0 : p->recv_off.back();
  int64_t send_total = 0;
  for (auto& s : p->send) send_total += int64_t(s.size());
  L.recv = o;
  o += al256(size_t(recv_total) * sc);
  L.send = o;
  o += al256(size_t(send_total) * sc);
  L.sidx = o;
  o += al256(size_t(send_total) * 4);
  L.total = o;
  return L;
}

ppf_status ppf_plan_device_bytes(const ppf_plan* p, size_t* bytes) {
  PPF_API_BEGIN
  PPF_REQUIRE(p && bytes, "NULL argument");
  *bytes = layout_of(p).total;
  PPF_API_END
}

ppf_status ppf_plan_info(const ppf_plan* p, int64_t* n_local, int64_t* nnz, int64_t* stored,
                         int64_t* halo_total) {
  PPF_API_BEGIN
  PPF_REQUIRE(p, "NULL plan");
  if (n_local) *n_local = p->n_local;
  if (nnz) *nnz = p->nnz;
  if (stored) *stored = int64_t(p->diag.col.size()) + int64_t(p->halo.col.size());
  if (halo_total) *halo_total = p->recv_off.empty() ? 0 : p->recv_off.back();
  PPF_API_END
}

void ppf_plan_destroy(ppf_plan* p) { delete p; }

ppf_status ppf_mat_create(ppf_ctx* ctx, const ppf_plan* p, void* buf, size_t bytes,
                          ppf_mat** out) {
  PPF_API_BEGIN
  PPF_REQUIRE(ctx && p && out, "NULL argument");
  PPF_REQUIRE(p->nranks == ctx->nranks && p->rank == ctx->rank, "plan/context rank mismatch");
  PPF_REQUIRE(p->sends_set, "halo send lists not set (ppf_plan_set_halo_send)");
  const Layout L = layout_of(p);
  PPF_REQUIRE(buf && bytes >= L.total, "device buffer too small");
  PPF_REQUIRE((reinterpret_cast<uintptr_t>(buf) & 255) == 0, "device buffer not 256-B aligned");
  const size_t sc = p->dtype == PPF_R64 ? 8 : 16;
  char* b = static_cast<char*>(buf);
  cudaStream_t st = ctx->stream;
  auto up = [&](size_t off, const void* src, size_t n) {
    if (n) PPF_CUDA(cudaMemcpyAsync(b + off, src, n, cudaMemcpyHostToDevice, st));
  };
  // (pair codes: their own slice pointers, width in the low bits)
  up(L.ptr, (p->enc == PPF_ENC_PAIR8 ? p->diag.pptr : p->diag.ptr).data(), p->diag.ptr.size() * 8);
  // (pair codes of a table of <= 16 pairs go up pre-multiplied by 16, see
  // ppf_mat::code_scaled; PPF_SELLP_SCALED=0 keeps them as indices)
  const char* scv = std::getenv("PPF_SELLP_SCALED");
  const bool scaled = p->enc == PPF_ENC_PAIR8 && p->diag.tab_off.size() <= 16 && !(scv && scv[0] == '0');
  std::vector<uint8_t> code16;
  if (scaled) {
    code16.resize(p->diag.code8.size());
    for (size_t i = 0; i < code16.size(); ++i) code16[i] = uint8_t(p->diag.code8[i] << 4);
  }
  if (p->enc == PPF_ENC_PAIR8) {
    up(L.col, scaled ? code16.data() : p->diag.code8.data(), p->diag.code8.size());
    up(L.cb, p->diag.tab_off.data(), p->diag.tab_off.size() * 4);
    up(L.val, p->diag.tab_val.data(), p->diag.tab_val.size() * 8);
    up(L.sched, p->diag.sched.data(), p->diag.sched.size() * 4);
  } else {
    if (p->enc == PPF_ENC_EXPLICIT) {
      up(L.col, p->diag.col.data(), p->diag.col.size() * 4);
    } else {
      up(L.col, p->diag.d16.data(), p->diag.d16.size() * 2);
      up(L.cb, p->diag.cb.data(), p->diag.cb.size() * 4);
    }
    up(L.val, p->diag.val.data(), p->diag.col.size() * sc);
  }
  up(L.perm, p->diag.perm.data(), p->diag.perm.size() * 4);
  up(L.hrows, p->halo.rows.data(), p->halo.rows.size() * 4);
  up(L.hptr, p->halo.ptr.data(), p->halo.ptr.size() * 8);
  up(L.hcol, p->halo.col.data(), p->halo.col.size() * 4);
  up(L.hval, p->halo.val.data(), p->halo.col.size() * sc);
  std::vector<int32_t> sidx;
  auto* m = new ppf_mat();
  m->send_count.assign(p->nranks, 0);
  m->send_off.assign(p->nranks + 1, 0);
  m->recv_count.assign(p->nranks, 0);
  m->recv_off.assign(p->recv_off.begin(), p->recv_off.end());
  for (int r = 0; r < p->nranks; ++r) {
    m->recv_count[r] = int64_t(p->recv[r].size());
    m->send_count[r] = int64_t(p->send[r].size());
    m->send_off[r + 1] = m->send_off[r] + m->send_count[r];
    for (int64_t x : p->send[r]) sidx.push_back(int32_t(x));
  }
  up(L.sidx, sidx.data(), sidx.size() * 4);
  PPF_CUDA(cudaStreamSynchronize(st));
  m->ctx = ctx;
  m->dtype = p->dtype;
  m->fmt = p->fmt;
  m->n_global = p->n_global;
  m->row0 = p->row0;
  m->n_local = p->n_local;
  m->nnz = p->nnz;
  m->stored = int64_t(p->diag.col.size());
  m->C = p->C;
  m->sigma = p->sigma;
  m->nranks = p->nranks;
  m->rank = p->rank;
  m->nslices = p->diag.nslices;
  m->d_ptr = reinterpret_cast<const int64_t*>(b + L.ptr);
  m->d_col = nullptr;
  m->d_val = nullptr;
  if (p->enc == PPF_ENC_PAIR8) {
    m->d_code8 = reinterpret_cast<const uint8_t*>(b + L.col);
    m->d_tab_off = reinterpret_cast<const int32_t*>(b + L.cb);
    m->d_tab_val = reinterpret_cast<const double*>(b + L.val);
    m->ntab = int(p->diag.tab_off.size());
    m->code_scaled = scaled;
    if (!p->diag.sched.empty()) {
      m->d_sched = reinterpret_cast<const int32_t*>(b + L.sched);
      m->sched_blocks = int(p->diag.sched.size() / 8);
    }
    for (int i = 0; i < m->ntab && i < 32; ++i) {
      m->h_tab_val[i] = p->diag.tab_val[size_t(i)];
      m->h_tab_off[i] = p->diag.tab_off[size_t(i)];
    }
  } else {
    if (p->enc == PPF_ENC_EXPLICIT) {
      m->d_col = reinterpret_cast<const int32_t*>(b + L.col);
    } else {
      m->d_d16 = reinterpret_cast<const uint16_t*>(b + L.col);
      m->d_cb = reinterpret_cast<const int32_t*>(b + L.cb);
    }
    m->d_val = b + L.val;
  }
  m->d_perm = p->diag.perm.empty() ? nullptr : reinterpret_cast<const int32_t*>(b + L.perm);
  {
    const double avg = double(m->stored) / double(std::max<int64_t>(1, p->n_local));
    // lanes per CSR row: the largest power of two <= avg/12 (each lane keeps
    // >= ~12 entries in flight; measured: 7-entry stencil rows 1 lane 5.6 TB/s
    // vs 8 lanes 1.7; the 49-entry Wilson rows 4 lanes 5.4 vs 32 lanes 3.0)
    int g = 1;
    while (g < 32 && 2.0 * g <= avg / 12.0) g *= 2;
    m->csr_group = g;
  }
  m->sell_ks = auto_sell_ks(m, ctx->num_sms);
  if (m->fmt == PPF_FMT_SELL && m->C == 32) m->sell_heavy = sell_heavy_prefix(p->diag.ptr, m->C);
  m->halo_rows = int64_t(p->halo.rows.size());
  m->halo_nnz = int64_t(p->halo.col.size());
  m->halo_total = p->recv_off.empty() ? 0 : p->recv_off.back();
  m->send_total = int64_t(sidx.size());
  m->d_halo_rows = reinterpret_cast<const int32_t*>(b + L.hrows);
  m->d_halo_ptr = reinterpret_cast<const int64_t*>(b + L.hptr);
  m->d_halo_col = reinterpret_cast<const int32_t*>(b + L.hcol);
  m->d_halo_val = b + L.hval;
  m->d_recv = b + L.recv;
  m->d_send = b + L.send;
  m->d_send_idx = reinterpret_cast<const int32_t*>(b + L.sidx);
  *out = m;
  PPF_API_END
}

void ppf_mat_destroy(ppf_mat* m) {
  if (!m) return;
  if (m->peer) ppf::peer_destroy(m->peer);
  delete m;
}

ppf_status ppf_mat_set_split(ppf_mat* A, int ks, int* applied) {
  PPF_API_BEGIN
  PPF_REQUIRE(A, "NULL matrix");
  PPF_REQUIRE(ks == 0 || ks == 1 || ks == 2 || ks == 4 || ks == 8, "sell_ks not in {0,1,2,4,8}");
  if (A->fmt == PPF_FMT_SELL) A->sell_ks = ks ? ks : auto_sell_ks(A, A->ctx->num_sms);
  if (applied) *applied = A->fmt == PPF_FMT_SELL ? A->sell_ks : 1;
  PPF_API_END
}

// ---------------------------------------------------------------------------
// Polynomials
// ---------------------------------------------------------------------------
ppf_status ppf_poly_chebyshev(double a, double b, int deg, ppf_poly** out) {
  PPF_API_BEGIN
  PPF_REQUIRE(out, "out is NULL");
  PPF_REQUIRE(std::isfinite(a) && std::isfinite(b) && 0.0 < a && a < b, "need 0 < a < b");
  PPF_REQUIRE(deg >= 0 && deg <= 256, "deg out of range [0, 256]");
  auto* q = new ppf_poly();
  std::unique_ptr<ppf_poly> g(q);
  q->kind = PPF_POLY_CHEBYSHEV;
  q->deg = deg;
  q->a = a;
  q->b = b;
  chebyshev_coefficients(a, b, deg, q->c);
  // positivity certificate on z_k = a + (b-a)k/1000
  if (!(certify_min_re(*q, nullptr, 0, PPF_R64) > 0.0))
    fail(PPF_EBRANCH, "Chebyshev q is not positive on [a, b]");
  *out = g.release();
  PPF_API_END
}

ppf_status ppf_poly_certify(const ppf_poly* q, const void* pts, int npts, int dtype,
                            double* min_re_q) {
  PPF_API_BEGIN
  PPF_REQUIRE(q, "NULL polynomial");
  PPF_REQUIRE(dtype == PPF_R64 || dtype == PPF_C128, "bad dtype");
  PPF_REQUIRE(npts >= 0 && (npts == 0 || pts), "bad points");
  PPF_REQUIRE(pts || q->kind == PPF_POLY_CHEBYSHEV,
              "default points exist only for a Chebyshev q (its interval [a, b])");
  const double mn = certify_min_re(*q, pts, pts ? npts : 0, dtype);
  if (min_re_q) *min_re_q = mn;
  if (!(mn > 0.0)) fail(PPF_EBRANCH, "certificate failed: Re q <= 0 at a point");
  PPF_API_END
}

ppf_status ppf_poly_import(int kind, int deg, const double* ab, const void* coef,
                           const void* nodes, ppf_poly** out) {
  PPF_API_BEGIN
  PPF_REQUIRE(out && coef, "NULL argument");
  PPF_REQUIRE(deg >= 0 && deg <= 256, "deg out of range");
  auto* q = new ppf_poly();
  std::unique_ptr<ppf_poly> g(q);
  q->kind = kind;
  q->deg = deg;
  if (kind == PPF_POLY_CHEBYSHEV) {
    PPF_REQUIRE(ab && ab[0] < ab[1], "bad interval");
    q->a = ab[0];
    q->b = ab[1];
    const double* c = static_cast<const double*>(coef);
    q->c.assign(c, c + deg + 1);
  } else if (kind == PPF_POLY_NEWTON) {
    PPF_REQUIRE(nodes, "nodes is NULL");
    const double* c = static_cast<const double*>(coef);
    const double* nd = static_cast<const double*>(nodes);
    for (int i = 0; i <= deg; ++i) {
      q->dd.push_back(zc(c[2 * i], c[2 * i + 1]));
      q->nodes.push_back(zc(nd[2 * i], nd[2 * i + 1]));
    }
  } else {
    fail(PPF_EINVAL, "bad poly kind");
  }
  *out = g.release();
  PPF_API_END
}

ppf_status ppf_poly_export(const ppf_poly* q, int* kind, int* deg, double* ab, void* coef,
                           void* nodes) {
  PPF_API_BEGIN
  PPF_REQUIRE(q, "NULL poly");
  if (kind) *kind = q->kind;
  if (deg) *deg = q->deg;
  if (q->kind == PPF_POLY_CHEBYSHEV) {
    if (ab) {
      ab[0] = q->a;
      ab[1] = q->b;
    }
    if (coef) std::copy(q->c.begin(), q->c.end(), static_cast<double*>(coef));
  } else {
    double* c = static_cast<double*>(coef);
    double* nd = static_cast<double*>(nodes);
    for (int i = 0; i <= q->deg; ++i) {
      if (c) {
        c[2 * i] = q->dd[i].real();
        c[2 * i + 1] = q->dd[i].imag();
      }
      if (nd) {
        nd[2 * i] = q->nodes[i].real();
        nd[2 * i + 1] = q->nodes[i].imag();
      }
    }
  }
  PPF_API_END
}

ppf_status ppf_poly_eval(const ppf_poly* q, int npts, const double* z, double* out) {
  PPF_API_BEGIN
  PPF_REQUIRE(q && npts >= 0 && (npts == 0 || (z && out)), "bad arguments");
  for (int i = 0; i < npts; ++i) {
    const zc r = poly_eval(*q, zc(z[2 * i], z[2 * i + 1]));
    out[2 * i] = r.real();
    out[2 * i + 1] = r.imag();
  }
  PPF_API_END
}

ppf_status ppf_poly_contour_ls(const double* points, int npts, int deg, double* min_re_q,
                               ppf_poly** out) {
  PPF_API_BEGIN
  PPF_REQUIRE(points && out, "NULL argument");
  PPF_REQUIRE(deg >= 0 && deg <= 256 && npts > deg + 1, "need 0 <= deg <= 256 and npts > deg + 1");
  std::vector<zc> z(npts);
  for (int i = 0; i < npts; ++i) {
    z[i] = zc(points[2 * i], points[2 * i + 1]);
    PPF_REQUIRE(std::isfinite(z[i].real()) && std::isfinite(z[i].imag()), "non-finite point");
    if (std::abs(z[i].imag()) <= 1e-14 * std::abs(z[i]) && z[i].real() <= 0.0)
      fail(PPF_EBRANCH, "contour point on the branch cut (-inf, 0]");
  }
  auto* q = new ppf_poly();
  double mr = 0.0;
  try {
    contour_ls_newton(z, deg, q->nodes, q->dd, mr);
  } catch (...) {
    delete q;
    throw;
  }
  q->kind = PPF_POLY_NEWTON;
  q->deg = deg;
  q->a = q->b = 0.0;
  // certificate of P:401-403 on the stored (Newton) form q applies, through
  // ppf_poly_certify's evaluation; the least-squares fit's own values agree
  // to rounding (mr)
  (void)mr;
  double mc = 0.0;
  try {
    mc = certify_min_re(*q, points, npts, PPF_C128);
  } catch (...) {
    delete q;
    throw;
  }
  if (min_re_q) *min_re_q = mc;
  if (!(mc > 0.0)) {
    delete q;
    fail(PPF_EBRANCH, "Re q <= 0 at a contour point (certificate of P:401-403)");
  }
  *out = q;
  PPF_API_END
}

ppf_status ppf_contour_from_ritz(const double* theta, int ntheta, double r_min, double step,
                                 int cap, double* points, int* npts) {
  PPF_API_BEGIN
  PPF_REQUIRE(theta && npts && ntheta >= 2, "need >= 2 Ritz values");
  PPF_REQUIRE(r_min > 0.0 && step > 0.0, "need r_min > 0 and step > 0");
  std::vector<zc> th(ntheta);
  for (int i = 0; i < ntheta; ++i) th[i] = zc(theta[2 * i], theta[2 * i + 1]);
  std::vector<zc> z = ritz_polygon(th, r_min, step);
  *npts = int(z.size());
  if (points) {
    PPF_REQUIRE(cap >= int(z.size()), "points buffer too small (query npts with points = NULL)");
    for (size_t i = 0; i < z.size(); ++i) {
      points[2 * i] = z[i].real();
      points[2 * i + 1] = z[i].imag();
    }
  }
  PPF_API_END
}

ppf_status ppf_poly_set_newton_eval(ppf_poly* q, int mode) {
  PPF_API_BEGIN
  PPF_REQUIRE(q, "NULL polynomial");
  PPF_REQUIRE(mode >= 0 && mode <= 2,
              "mode must be 0 (Horner), 1 (forward Newton basis) or 2 (real conjugate pairs)");
  if (mode == 2) {
    PPF_REQUIRE(q->kind == PPF_POLY_NEWTON, "real-pair form needs a Newton polynomial");
    real_pair_form(*q);  // reorders nodes, recomputes dd, sets newton_eval = 2
  } else {
    q->newton_eval = mode;
  }
  PPF_API_END
}

void ppf_poly_destroy(ppf_poly* q) { delete q; }

// ---------------------------------------------------------------------------
// Host dense kernel
// ---------------------------------------------------------------------------
ppf_status ppf_dense_invsqrt_e1(ppf_dtype dtype, int m, const void* H, int ld, double beta0,
                                int hermitian, void* y) {
  PPF_API_BEGIN
  PPF_REQUIRE(H && y && m >= 1 && ld >= m, "bad arguments");
  const int ND = dtype == PPF_R64 ? 1 : 2;
  const double* h = static_cast<const double*>(H);
  double* yo = static_cast<double*>(y);
  if (hermitian) {
    std::vector<double> d(m), e(m, 0.0), yy(m);
    for (int i = 0; i < m; ++i) d[i] = h[(size_t(i) + size_t(i) * ld) * ND];
    for (int i = 0; i + 1 < m; ++i) e[i] = h[(size_t(i + 1) + size_t(i) * ld) * ND];
    tridiag_invsqrt_e1(m, d.data(), e.data(), beta0, yy.data());
    for (int i = 0; i < m; ++i) {
      yo[i * ND] = yy[i];
      if (ND == 2) yo[i * ND + 1] = 0.0;
    }
  } else if (ND == 1) {  // real Hessenberg: the real Schur route
    std::vector<double> yy(m);
    real_invsqrt_e1(m, h, ld, beta0, yy.data());
    for (int i = 0; i < m; ++i) yo[i] = yy[i];
  } else {
    std::vector<zc> A(size_t(m) * m), yy;
    for (int j = 0; j < m; ++j)
      for (int i = 0; i < m; ++i) {
        const size_t o = (size_t(i) + size_t(j) * ld) * ND;
        A[size_t(i) + size_t(j) * m] = zc(h[o], ND == 2 ? h[o + 1] : 0.0);
      }
    general_invsqrt_e1(m, A, beta0, yy);
    for (int i = 0; i < m; ++i) {
      yo[i * ND] = yy[i].real();
      if (ND == 2) yo[i * ND + 1] = yy[i].imag();
    }
  }
  PPF_API_END
}

}  // extern "C"
