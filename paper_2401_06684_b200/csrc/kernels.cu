// Device kernels of the hot path, sm_100a.
//
// Everything here is HBM-bandwidth bound (SURVEY §8(d) roofline: 0.17-0.5
// flop/byte), so the kernels are organised around coalesced streams:
//  * SpMV (K1) with the polynomial recurrences fused into the epilogue (K2
//    Clenshaw, K3 Newton-Horner): one pass over A per degree, P:136/P:332/P:354.
//    SELL-C-sigma (one row per lane, C = 32, or two rows per lane as 128-bit
//    double2/int2 loads, C = 64) and a CSR kernel (G lanes per row).
//  * CGS2 (K5/K6/K7): three fused tall-skinny sweeps over V, warps own columns,
//    V values are held in registers between the update and the projection.
//  * Lanczos (K8), combine x = V y (K9), norms.
// Reductions are deterministic: per-block partials, then the last block to
// arrive sums them in block order (fixed tree), independent of timing.
#include <atomic>
#include <set>
#include <mutex>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <type_traits>
#include <utility>

#include "ppf_internal.h"

namespace ppf {

namespace {

constexpr unsigned FULL = 0xffffffffu;

template <typename T> struct EpiT {
  T s_ax, s_x, s_z, s_u;
  const T* z;
  const T* u;
  const T* xe;  // vector of the s_x term: the SpMV input, or Epi::xe (squared operator)
  T* acc;       // second output (ACC kernels): acc = (acc_init ? s_acc0 xe : acc) + s_acc out
  T s_acc, s_acc0;
  bool acc_init;
};

template <typename T> EpiT<T> to_epi(const Epi& e, const void* x) {
  EpiT<T> r;
  r.s_ax = s_from<T>(e.s_ax[0], e.s_ax[1]);
  r.s_x = s_from<T>(e.s_x[0], e.s_x[1]);
  r.s_z = s_from<T>(e.s_z[0], e.s_z[1]);
  r.s_u = s_from<T>(e.s_u[0], e.s_u[1]);
  r.z = static_cast<const T*>(e.z);
  r.u = static_cast<const T*>(e.u);
  r.xe = static_cast<const T*>(e.xe ? e.xe : x);
  r.acc = static_cast<T*>(e.acc);
  r.s_acc = s_from<T>(e.s_acc[0], e.s_acc[1]);
  r.s_acc0 = s_from<T>(e.s_acc0[0], e.s_acc0[1]);
  r.acc_init = e.acc_init;
  return r;
}

__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }
__device__ __forceinline__ cplx ldg(const cplx* p) {
  double2 v = __ldg(reinterpret_cast<const double2*>(p));
  return {v.x, v.y};
}

// Loads whose issue order is pinned (asm volatile is not reordered against
// other asm volatile): the SpMV loops issue a whole batch of loads before the
// first use.  The matrix streams (values, indices) are read once, so they
// bypass L1 (L1::no_allocate) and leave it to the x gathers.
__device__ __forceinline__ int ld_stream(const int32_t* p) {
  int r;
  asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ int ld_stream(const uint16_t* p) {
  unsigned short r;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(r) : "l"(p));
  return int(r);
}
__device__ __forceinline__ uint4 ld_stream_u4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ double ld_stream(const double* p) {
  double r;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ cplx ld_stream(const cplx* p) {
  const double2 v = ld_stream(reinterpret_cast<const double2*>(p));
  return {v.x, v.y};
}
// gather of x (cached in L1: stencil neighbours of adjacent rows share lines)
__device__ __forceinline__ double ld_gather(const double* p) {
  double r;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ cplx ld_gather(const cplx* p) {
  double2 r;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return {r.x, r.y};
}

// Programmatic dependent launch (PDL): an SpMV launched with
// cudaLaunchAttributeProgrammaticStreamSerialization lets its blocks start as
// soon as every block of the previous kernel has started (pdl_release at the
// top of every SELL kernel), i.e. during the previous kernel's drain, when
// SMs fall idle one by one.  Such a block prefetches its slice of the matrix
// (read-only, independent of the previous kernel) into L2, then pdl_wait()s
// for the previous grid to complete and its stores to be visible before it
// touches x or the epilogue vectors or writes anything.
__device__ __forceinline__ void pdl_release() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2::evict_normal [%0];" ::"l"(p));
}

template <typename T>
__device__ __forceinline__ T epilogue(const EpiT<T>& e, T ax, const T* __restrict__ x, int64_t row,
                                      bool has_x) {
  T r = s_mul(e.s_ax, ax);
  if (has_x) r = s_fma(e.s_x, ldg(e.xe + row), r);
  if (e.z) r = s_fma(e.s_z, ldg(e.z + row), r);
  if (e.u) r = s_fma(e.s_u, ldg(e.u + row), r);
  return r;
}

// second output of the forward-Newton-basis chain: acc += s_acc * r
template <typename T>
__device__ __forceinline__ void acc_update(const EpiT<T>& e, int64_t row, T r) {
  const T base = e.acc_init ? s_mul(e.s_acc0, ldg(e.xe + row)) : e.acc[row];
  e.acc[row] = s_fma(e.s_acc, r, base);
}

// ---------------------------------------------------------------------------
// SELL-C-sigma SpMV + fused epilogue.  KS warps per slice, one row per lane.
//
// KS > 1 splits a slice's entry columns k = 0..w-1 into KS contiguous parts,
// one per warp of the same block; the parts' partial sums meet in shared
// memory and the part-0 warp adds them in part order (deterministic) and runs
// the epilogue.  Every warp load is still one contiguous 32-entry row of the
// slice (512 B of complex values + 128 B of indices).  KS multiplies the warp
// tasks for matrices with very few slices; the automatic choice is KS = 1
// for every BASELINE config (measured on C5: KS = 1/2/4 -> 6.51/6.21/5.69
// TB/s, the block barrier costs more than the smaller last wave saves).
//
// The loop body issues U = 4 entries' index loads, then their value loads and
// x gathers, then the FMAs.  With __launch_bounds__(256, 3) ptxas keeps the
// batch in registers (80 for complex); left at 32 registers it interleaves one
// entry's loads with the previous FMA, and C5's 49-entry complex rows were
// latency-bound at 5.2 TB/s (ncu: 36% "mem busy", 60 warps/SM active) instead
// of 6.5 TB/s.
// ---------------------------------------------------------------------------
template <typename T, int KS, bool PERM, bool ACC = false, bool IDX16 = false>
__global__ void __launch_bounds__(256, sizeof(T) == 16 ? 3 : 1) sell1_kernel(int64_t nslices, int64_t n,
                                                    const int64_t* __restrict__ sptr,
                                                    const int32_t* __restrict__ col,
                                                    const T* __restrict__ val,
                                                    const T* __restrict__ x, T* __restrict__ out,
                                                    EpiT<T> e, bool has_x,
                                                    const int32_t* __restrict__ perm,
                                                    int64_t nheavy,
                                                    const uint16_t* __restrict__ d16 = nullptr,
                                                    const int32_t* __restrict__ cbase = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // the first nheavy slices (the longest rows after a whole-matrix sigma sort)
  // get a whole block each, 8 warps splitting their entry columns; the rest
  // KS warps per slice
  const bool heavy = blockIdx.x < nheavy;
  const int nw = blockDim.x >> 5;
  const int64_t slice = heavy ? int64_t(blockIdx.x)
                              : nheavy + (int64_t(blockIdx.x) - nheavy) * (nw / KS) + warp / KS;
  const int parts = heavy ? nw : KS;
  const int part = heavy ? warp : warp % KS;
  const bool live = slice < nslices;
  T acc = s_zero<T>();
  if (live) {
    const int64_t base = sptr[slice];
    const int w = int((sptr[slice + 1] - base) >> 5);
    const int k0 = part * w / parts, k1 = (part + 1) * w / parts;
    const int32_t* cp = col + base + lane;
    const T* vp = val + base + lane;
    if constexpr (IDX16) {
      // column = row + base(s, k) + 16-bit delta, clamped to [0, n) (padding;
      // see the plan's encoding and sell2_kernel)
      const uint16_t* dp = d16 + base + lane;
      const int32_t* cbp = cbase + (base >> 5);
      const int ri = int(slice * 32 + lane), nm1 = int(n - 1);
      constexpr int U = sizeof(T) == 8 ? 2 : 4;
      int k = k0;
      for (; k + U <= k1; k += U) {
        int c[U];
        T v[U], xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          c[u] = min(max(ri + __ldg(cbp + k + u) + ld_stream(dp + 32 * (k + u)), 0), nm1);
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld_stream(vp + 32 * (k + u));
#pragma unroll
        for (int u = 0; u < U; ++u) xv[u] = ld_gather(x + c[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) acc = s_fma(v[u], xv[u], acc);
      }
      for (; k < k1; ++k) {
        const int c0 = min(max(ri + __ldg(cbp + k) + ld_stream(dp + 32 * k), 0), nm1);
        acc = s_fma(ldg(vp + 32 * k), ldg(x + c0), acc);
      }
    } else if constexpr (sizeof(T) == 8) {
      // fp64: ptxas' own 32-register schedule at full occupancy is faster
      // (as for sell2_kernel; batching measured 4.2 vs 6.2 TB/s on C3, and
      // 3.4 vs 6.1 TB/s on C3 in this C = 32 layout; on C7's gathers: equal)
#pragma unroll 4
      for (int k = k0; k < k1; ++k)
        acc = s_fma(__ldg(vp + 32 * k), __ldg(x + __ldg(cp + 32 * k)), acc);
    } else {
      // complex: batches of U entries -- all U index loads, then the U value
      // loads and the U gathers of x, then the FMAs: U independent loads in
      // flight per lane (left to itself the compiler issues one entry's loads
      // at a time)
      constexpr int U = 4;
      int k = k0;
      for (; k + U <= k1; k += U) {
        int c[U];
        T v[U], xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) c[u] = ld_stream(cp + 32 * (k + u));
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = ld_stream(vp + 32 * (k + u));
#pragma unroll
        for (int u = 0; u < U; ++u) xv[u] = ld_gather(x + c[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) acc = s_fma(v[u], xv[u], acc);
      }
      for (; k < k1; ++k) acc = s_fma(ldg(vp + 32 * k), ldg(x + __ldg(cp + 32 * k)), acc);
    }
  }
  __shared__ T red[8][32];
  if (heavy) {  // block-uniform
    red[warp][lane] = acc;
    __syncthreads();
    if (warp != 0) return;
    for (int p = 1; p < nw; ++p) acc = s_add(acc, red[p][lane]);
  } else if constexpr (KS > 1) {
    red[warp][lane] = acc;
    __syncthreads();
    if (part != 0) return;
#pragma unroll
    for (int p = 1; p < KS; ++p) acc = s_add(acc, red[warp + p][lane]);
  }
  if (!live) return;
  const int64_t pos = slice * 32 + lane;
  if (pos < n) {
    const int64_t row = PERM ? int64_t(perm[pos]) : pos;
    const T r = epilogue(e, acc, x, row, has_x);
    out[row] = r;
    if constexpr (ACC) acc_update(e, row, r);
  }
}

// two rows per lane, 128-bit loads of (val, val) and (col, col); C = 64, fp64;
// KS warps per slice as in sell1_kernel
template <int KS, bool ACC = false, bool IDX16 = false>
__global__ void __launch_bounds__(256) sell2_kernel(int64_t nslices, int64_t n,
                                                    const int64_t* __restrict__ sptr,
                                                    const int32_t* __restrict__ col,
                                                    const double* __restrict__ val,
                                                    const double* __restrict__ x,
                                                    double* __restrict__ out, EpiT<double> e,
                                                    bool has_x, const uint16_t* __restrict__ d16,
                                                    const int32_t* __restrict__ cbase) {
  pdl_release();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t slice = int64_t(blockIdx.x) * (blockDim.x >> 5) / KS + warp / KS;
  const int part = warp % KS;
  const bool live = slice < nslices;
  double a0 = 0.0, a1 = 0.0;
  int64_t base = 0;
  int k0 = 0, k1 = 0;
  if (live) {
    base = sptr[slice];
    const int w = int((sptr[slice + 1] - base) >> 6);
    k0 = part * w / KS;
    k1 = (part + 1) * w / KS;
    // Prefetch the slice's matrix columns into L2 before anything else: all
    // of a warp's matrix lines are requested at once instead of 4 columns at a
    // time by the unrolled loop (C4 309 -> 302 ms, C3 SpMV 6.15 -> 6.30 TB/s;
    // in sell1_kernel it cost C5 13% and C7 9%, so it is sell2-only).  One
    // 128-B line per 8 lanes of values (16 B each) / 16 lanes of indices.
    if ((lane & 7) == 0)
      for (int k = k0; k < k1; ++k) prefetch_l2(val + base + 64 * k + 2 * lane);
    if constexpr (IDX16) {
      // 16-bit deltas: 128 B per column of the slice; the bases: 4 B per column
      if (lane == 0) {
        for (int k = k0; k < k1; ++k) prefetch_l2(d16 + base + 64 * k);
        prefetch_l2(cbase + (base >> 6) + k0);
      }
    } else {
      if ((lane & 15) == 0)
        for (int k = k0; k < k1; ++k) prefetch_l2(col + base + 64 * k + 2 * lane);
    }
  }
  pdl_wait();
  // the slice's rows of the epilogue vectors and of x (its own rows: the
  // diagonal and the +-1 neighbours): one 128-B line per 8 lanes
  if (live && part == 0 && (lane & 7) == 0) {
    const int64_t r0 = slice * 64 + 2 * lane;
    if (r0 < n) {
      prefetch_l2(x + r0);
      if (e.z) prefetch_l2(e.z + r0);
      if (e.u) prefetch_l2(e.u + r0);
      if (has_x && e.xe != x) prefetch_l2(e.xe + r0);
    }
  }
  if (live) {
    const double2* vp = reinterpret_cast<const double2*>(val + base) + lane;
    // (measured: the compiler's own schedule of this loop, at 32 registers
    // and full occupancy, streams C3/C4 at 97-98% of the measured copy
    // bandwidth; the forced batching of sell1_kernel drops it to 72%)
    if constexpr (IDX16) {
      // column = row + base(s, k) + 16-bit delta (the plan's encoding),
      // clamped to [0, n): padding slots (val 0, delta 0) of rows near the
      // ends, and of the lanes past n in the last slice, then read in bounds
      const ushort2* dp = reinterpret_cast<const ushort2*>(d16 + base) + lane;
      const int32_t* cbp = cbase + (base >> 6);
      const int r0i = int(slice * 64 + 2 * lane), nm1 = int(n - 1);
      // (measured and dropped: the slice's bases loaded once and taken by
      // shuffles in the loop -- C4 273 -> 290 ms; the broadcast load per step
      // stays)
#pragma unroll 4
      for (int k = k0; k < k1; ++k) {
        const ushort2 d = __ldg(dp + 32 * k);
        const int cb = __ldg(cbp + k) + r0i;
        const double2 v = __ldg(vp + 32 * k);
        const int c0 = min(max(cb + int(d.x), 0), nm1);
        const int c1 = min(max(cb + 1 + int(d.y), 0), nm1);
        a0 = fma(v.x, __ldg(x + c0), a0);
        a1 = fma(v.y, __ldg(x + c1), a1);
      }
    } else {
      const int2* cp = reinterpret_cast<const int2*>(col + base) + lane;
#pragma unroll 4
      for (int k = k0; k < k1; ++k) {
        const int2 c = __ldg(cp + 32 * k);
        const double2 v = __ldg(vp + 32 * k);
        a0 = fma(v.x, __ldg(x + c.x), a0);
        a1 = fma(v.y, __ldg(x + c.y), a1);
      }
    }
  }
  if constexpr (KS > 1) {
    __shared__ double2 red[8][32];
    red[warp][lane] = make_double2(a0, a1);
    __syncthreads();
    if (part != 0) return;
#pragma unroll
    for (int p = 1; p < KS; ++p) {
      const double2 t = red[warp + p][lane];
      a0 += t.x;
      a1 += t.y;
    }
  }
  if (!live) return;
  const int64_t r0 = slice * 64 + 2 * lane;
  if (r0 + 1 < n) {
    double2 r;
    r.x = e.s_ax * a0;
    r.y = e.s_ax * a1;
    if (has_x) {
      const double2 xv = __ldg(reinterpret_cast<const double2*>(e.xe + r0));
      r.x = fma(e.s_x, xv.x, r.x);
      r.y = fma(e.s_x, xv.y, r.y);
    }
    if (e.z) {
      const double2 zv = __ldg(reinterpret_cast<const double2*>(e.z + r0));
      r.x = fma(e.s_z, zv.x, r.x);
      r.y = fma(e.s_z, zv.y, r.y);
    }
    if (e.u) {
      const double2 uv = __ldg(reinterpret_cast<const double2*>(e.u + r0));
      r.x = fma(e.s_u, uv.x, r.x);
      r.y = fma(e.s_u, uv.y, r.y);
    }
    *reinterpret_cast<double2*>(out + r0) = r;
    if constexpr (ACC) {
      acc_update(e, r0, r.x);
      acc_update(e, r0 + 1, r.y);
    }
  } else if (r0 < n) {
    const double r = epilogue(e, a0, x, r0, has_x);
    out[r0] = r;
    if constexpr (ACC) acc_update(e, r0, r);
  }
}

// ---------------------------------------------------------------------------
// SELL-64 fp64 SpMV + fused epilogue on pair codes (PPF_ENC_PAIR8): entry
// (s, k, t) is the pair (off, val) = table[code], column = row + off.  Lane
// i of the slice's warp takes rows 64 s + 2i and 64 s + 2i + 1, as in
// sell2_kernel (the two gathers of a column fall on the same lines, the
// second an L1 hit); the codes are stored lane-major in chunks of 8 columns
// (ppf_internal.h), so one 16-B load gives the lane its codes of 8 columns
// and all their gathers issue back to back (pair_chunk<NK>, unrolled per
// chunk width, no per-column branch) -- with __launch_bounds__(256, 8) at 32
// registers and full occupancy.  Measured on C4 / C3 deg 20 (ms per solve):
// column-major codes, one 16-bit load per column: 176.4 / 94.8; lane-major
// chunks with a per-column branch: no batching; pair_chunk at 48 registers
// (40 warps/SM): 168.6 / 89.5; at 64: 181.4 / 98.7; at 40: 160.2 / 84.3; at
// 32 (64 warps/SM): 152.5 / 79.8; pair records (value, byte offset) and no
// column clamp outside the last slice: 144.0 / 77.1.  With the first code
// chunk loaded before
// the PDL wait: 155.5 / 84.0 (dropped); with rows i, i + 32 per lane in the
// chunked layout (half the L1 wavefronts per gather): 152.7 / SpMV unchanged
// (dropped).
//
// With 1 byte per entry the matrix is ~18% of the DRAM bytes (C4: 117 of the
// 654 MB per chain SpMV) and DRAM is no longer the bound: at 155-160 us per
// C4 SpMV (4.1 TB/s of DRAM traffic, 1.02x the algorithmic bytes) the L1
// data pipe is 76% busy (the x gathers; a fifth of it the table lookups),
// DRAM 51%, and
// long-scoreboard stalls on the x gathers dominate.  Measured on C4 (ncu, per
// SpMV) and dropped:
//  * rows i and i + 32 per lane (every warp access 32 consecutive rows,
//    fewer L1 wavefronts): L1 hit rate 49 -> 24%, 155 -> 168 us;
//  * one aligned 16-B load of x[c], x[c + 1] where both rows take the same
//    pair at an even column (5 of C4's 7 columns, fewer L1 sectors): the
//    branch cost more than it saved, 160 -> 187 us (and 179 us with
//    diagonal-aligned slots, where the branch never diverges);
//  * two slices per warp (twice the independent loads per loop turn, 40
//    registers): 161 -> 195 us;
//  * a window-staged persistent kernel (producer warp bulk-copying codes,
//    z, u and x as three contiguous windows per 1024-row stage into a 4-deep
//    mbarrier ring, 16 consumer warps working from shared memory): 203 us,
//    consumers waiting on the ring (DRAM 36%);
//  * x staged in shared memory over the block's rows +- one block height
//    (coalesced 16-B loads after the PDL wait), the near pairs' gathers read
//    there through a generic pointer: 161 -> 233 us;
//  * all codes of 8 columns, then all gathers, then the FMAs (64 registers,
//    half the warps): 195 us;
//  * a persistent grid, each CTA walking a contiguous range of slices (L1
//    reuse of the +-1 / +-N neighbours): the far (+-N^2) neighbours' reuse
//    distance across CTAs outgrew L2 -- DRAM reads 0.52 -> 0.96 GB, 227 us.
// A table of at most 32 pairs (C3/C4: 8) is passed by value as a
// __grid_constant__ kernel parameter, so the lookups are indexed constant-
// cache loads off the L1 data pipe (C4 186.2 -> 177.8 ms, C3 deg 20 97.9 ->
// 93.8 ms); larger tables are held in shared memory as (value, offset bits)
// pairs: one 16-B load per lookup, a broadcast where a column's codes agree.
// PPF_SELLP_CTAB=0 forces the shared-memory table.  KS warps per slice as in
// sell2_kernel.  The multiply-adds are the explicit layout's, in its order
// (bitwise-identical results).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ int pair_off(double2 p) { return int(__double_as_longlong(p.y)); }

// one 16-B record per pair: the value, and the column offset in bytes
// (8 * (col - row)), so a lookup is two constant loads at one scaled index
struct PairRec {
  double v;
  int o8;
  int pad;
};
struct PairTab32 {
  PairRec p[32];
};

// a pair's record from its code: an index, or (SC, ppf_mat::code_scaled) the
// record's byte offset (16 x index), so the lookup needs no scaling
template <bool SC>
__device__ __forceinline__ const PairRec& crec(const PairTab32& ct, int e) {
  if constexpr (SC) return *reinterpret_cast<const PairRec*>(reinterpret_cast<const char*>(ct.p) + e);
  else return ct.p[e];
}
template <bool SC>
__device__ __forceinline__ double2 srec(const double2* s_tab, int e) {
  if constexpr (SC) return *reinterpret_cast<const double2*>(reinterpret_cast<const char*>(s_tab) + e);
  else return s_tab[e];
}
// codes of column j (0..7 in the chunk) for the lane's rows 0 and 1: bytes
// 2j, 2j + 1 of the chunk
template <bool SC>
__device__ __forceinline__ void pair_codes(const uint32_t* qw, int j, int& e0, int& e1) {
  if constexpr (SC) {   // one PRMT each (byte into a zeroed word)
    e0 = int(__byte_perm(qw[j >> 1], 0u, (j & 1) ? 0x4442u : 0x4440u));
    e1 = int(__byte_perm(qw[j >> 1], 0u, (j & 1) ? 0x4443u : 0x4441u));
  } else {
    const uint32_t wd = qw[j >> 1] >> (16 * (j & 1));
    e0 = int(wd & 0xffu);
    e1 = int((wd >> 8) & 0xffu);
  }
}

// NK columns of one lane's chunk (codes in q: byte 2j + r = column j, row r):
// all 2 NK gathers, then the FMAs in column order.  TAIL (the last slice):
// columns clamped to n - 1 for the padding pairs of lanes past n; elsewhere
// the gather address is the row's x address plus the pair's byte offset.
template <int NK, bool CT, bool TAIL, bool SC>
__device__ __forceinline__ void pair_chunk(const uint4 q, const double* __restrict__ x, int r0i, int nm1,
                                           const PairTab32& ct, const double2* s_tab, double& a0,
                                           double& a1) {
  const uint32_t qw[4] = {q.x, q.y, q.z, q.w};
  double g0[NK], g1[NK];
  int e0[NK], e1[NK];
  const char* xr = reinterpret_cast<const char*>(x + r0i);
#pragma unroll
  for (int j = 0; j < NK; ++j) {
    pair_codes<SC>(qw, j, e0[j], e1[j]);
    if constexpr (CT && !TAIL) {
      g0[j] = __ldg(reinterpret_cast<const double*>(xr + crec<SC>(ct, e0[j]).o8));
      g1[j] = __ldg(reinterpret_cast<const double*>(xr + 8 + crec<SC>(ct, e1[j]).o8));
    } else {
      const int o0 = CT ? crec<SC>(ct, e0[j]).o8 / 8 : pair_off(srec<SC>(s_tab, e0[j]));
      const int o1 = CT ? crec<SC>(ct, e1[j]).o8 / 8 : pair_off(srec<SC>(s_tab, e1[j]));
      g0[j] = __ldg(x + min(r0i + o0, nm1));
      g1[j] = __ldg(x + min(r0i + 1 + o1, nm1));
    }
  }
#pragma unroll
  for (int j = 0; j < NK; ++j) {
    a0 = fma(CT ? crec<SC>(ct, e0[j]).v : srec<SC>(s_tab, e0[j]).x, g0[j], a0);
    a1 = fma(CT ? crec<SC>(ct, e1[j]).v : srec<SC>(s_tab, e1[j]).x, g1[j], a1);
  }
}

// CT: the table (<= 32 pairs) comes by value as a kernel parameter, so the
// lookups are constant-cache loads (uniform across the warp where a column's
// codes agree) instead of shared-memory loads on the L1 data pipe
template <int KS, bool ACC = false, bool CT = false, bool SC = false>
__global__ void __launch_bounds__(256, 8) sellp_kernel(int64_t nslices, int64_t n,
                                                    const int64_t* __restrict__ sptr,
                                                    const uint8_t* __restrict__ code8,
                                                    const int32_t* __restrict__ tab_off,
                                                    const double* __restrict__ tab_val, int ntab,
                                                    const double* __restrict__ x,
                                                    double* __restrict__ out, EpiT<double> e,
                                                    bool has_x, const __grid_constant__ PairTab32 ct,
                                                    const int32_t* __restrict__ sched) {
  __shared__ double2 s_tab[CT ? 1 : 256];
  pdl_release();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // (KS = 1 with a slice schedule: the block's warps take a tile of slices
  // that gather from each other's rows, api.cpp build_slice_schedule)
  const int64_t slice = (KS == 1 && sched) ? int64_t(__ldg(sched + blockIdx.x * 8 + warp))
                                           : int64_t(blockIdx.x) * (blockDim.x >> 5) / KS + warp / KS;
  const int part = warp % KS;
  const bool live = slice >= 0 && slice < nslices;
  double a0 = 0.0, a1 = 0.0;
  int64_t base = 0;
  int k0 = 0, k1 = 0;
  if (live) {
    const int64_t pe = sptr[slice];   // chunk offset | slice width
    base = pe & ~int64_t(511);
    const int w = int(pe & 511);
    k0 = part * w / KS;
    k1 = (part + 1) * w / KS;
    // the slice's code chunks (512 B per 8 columns) into L2 before the PDL wait
    for (int o = 512 * (k0 / 8) + 128 * lane; o < 512 * ((k1 + 7) / 8); o += 32 * 128)
      prefetch_l2(code8 + base + o);
  }
  if constexpr (!CT) {
    for (int i = threadIdx.x; i < ntab; i += blockDim.x)
      s_tab[i] = make_double2(__ldg(tab_val + i), __longlong_as_double((long long)__ldg(tab_off + i)));
    __syncthreads();
  }
  pdl_wait();
  // the slice's rows of the epilogue vectors and of x: one line per 8 lanes
  if (live && part == 0 && (lane & 7) == 0) {
    const int64_t r0 = slice * 64 + 2 * lane;
    if (r0 < n) {
      prefetch_l2(x + r0);
      if (e.z) prefetch_l2(e.z + r0);
      if (e.u) prefetch_l2(e.u + r0);
      if (has_x && e.xe != x) prefetch_l2(e.xe + r0);
    }
  }
  if (KS == 1 && live) {
    // one 16-B load gives the lane its codes of up to 8 columns, then all
    // their gathers issue back to back (pair_chunk<NK>: no per-column branch)
    const int r0i = int(slice * 64 + 2 * lane), nm1 = int(n - 1);
    const bool tail = slice * 64 + 64 > n;   // warp-uniform
    for (int c = 0; 8 * c < k1; ++c) {
      const uint4 q = ld_stream_u4(code8 + base + 512 * c + 16 * lane);
      const int nk = k1 - 8 * c < 8 ? k1 - 8 * c : 8;
      switch (nk) {
#define PPF_PC(NK)                                                             \
  case NK:                                                                     \
    if (tail) pair_chunk<NK, CT, true, SC>(q, x, r0i, nm1, ct, s_tab, a0, a1); \
    else pair_chunk<NK, CT, false, SC>(q, x, r0i, nm1, ct, s_tab, a0, a1);     \
    break;
        PPF_PC(1) PPF_PC(2) PPF_PC(3) PPF_PC(4) PPF_PC(5) PPF_PC(6) PPF_PC(7) PPF_PC(8)
#undef PPF_PC
      }
    }
  } else if (live) {
    const int r0i = int(slice * 64 + 2 * lane), nm1 = int(n - 1);
    for (int c = k0 / 8; 8 * c < k1; ++c) {
      const uint4 q = ld_stream_u4(code8 + base + 512 * c + 16 * lane);
      const uint32_t qw[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = 8 * c + j;
        if (k < k0 || k >= k1) continue;
        int e0, e1;
        pair_codes<SC>(qw, j, e0, e1);
        if constexpr (CT) {
          const PairRec &r0 = crec<SC>(ct, e0), &r1 = crec<SC>(ct, e1);
          a0 = fma(r0.v, __ldg(x + min(r0i + r0.o8 / 8, nm1)), a0);
          a1 = fma(r1.v, __ldg(x + min(r0i + 1 + r1.o8 / 8, nm1)), a1);
        } else {
          const double2 p0 = srec<SC>(s_tab, e0), p1 = srec<SC>(s_tab, e1);
          a0 = fma(p0.x, __ldg(x + min(r0i + pair_off(p0), nm1)), a0);
          a1 = fma(p1.x, __ldg(x + min(r0i + 1 + pair_off(p1), nm1)), a1);
        }
      }
    }
  }
  if constexpr (KS > 1) {
    __shared__ double2 red[8][32];
    red[warp][lane] = make_double2(a0, a1);
    __syncthreads();
    if (part != 0) return;
#pragma unroll
    for (int p = 1; p < KS; ++p) {
      const double2 t = red[warp + p][lane];
      a0 += t.x;
      a1 += t.y;
    }
  }
  if (!live) return;
  const int64_t r0 = slice * 64 + 2 * lane;
  if (r0 + 1 < n) {
    double2 r;
    r.x = e.s_ax * a0;
    r.y = e.s_ax * a1;
    if (has_x) {
      const double2 xv = __ldg(reinterpret_cast<const double2*>(e.xe + r0));
      r.x = fma(e.s_x, xv.x, r.x);
      r.y = fma(e.s_x, xv.y, r.y);
    }
    if (e.z) {
      const double2 zv = __ldg(reinterpret_cast<const double2*>(e.z + r0));
      r.x = fma(e.s_z, zv.x, r.x);
      r.y = fma(e.s_z, zv.y, r.y);
    }
    if (e.u) {
      const double2 uv = __ldg(reinterpret_cast<const double2*>(e.u + r0));
      r.x = fma(e.s_u, uv.x, r.x);
      r.y = fma(e.s_u, uv.y, r.y);
    }
    *reinterpret_cast<double2*>(out + r0) = r;
    if constexpr (ACC) {
      acc_update(e, r0, r.x);
      acc_update(e, r0 + 1, r.y);
    }
  } else if (r0 < n) {
    const double r = epilogue(e, a0, x, r0, has_x);
    out[r0] = r;
    if constexpr (ACC) acc_update(e, r0, r);
  }
}

// ---------------------------------------------------------------------------
// CSR SpMV + fused epilogue, G lanes per row.
// ---------------------------------------------------------------------------
template <typename T, int G, bool ACC = false>
__global__ void __launch_bounds__(256) csr_kernel(int64_t n, const int64_t* __restrict__ rp,
                                                  const int32_t* __restrict__ col,
                                                  const T* __restrict__ val,
                                                  const T* __restrict__ x, T* __restrict__ out,
                                                  EpiT<T> e, bool has_x) {
  const int64_t gt = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t row = gt / G;
  const int lg = threadIdx.x % G;
  const int lane = threadIdx.x & 31;
  const unsigned mask = (G == 32) ? FULL : (((1u << G) - 1u) << (lane & ~(G - 1)));
  if (row >= n) return;  // whole group exits together
  T acc = s_zero<T>();
  const int64_t end = rp[row + 1];
  for (int64_t k = rp[row] + lg; k < end; k += G) acc = s_fma(ldg(val + k), ldg(x + __ldg(col + k)), acc);
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    if constexpr (sizeof(T) == 8) {
      acc = s_add(acc, __shfl_xor_sync(mask, acc, o));
    } else {
      cplx t;
      t.re = __shfl_xor_sync(mask, reinterpret_cast<cplx&>(acc).re, o);
      t.im = __shfl_xor_sync(mask, reinterpret_cast<cplx&>(acc).im, o);
      acc = s_add(acc, reinterpret_cast<T&>(t));
    }
  }
  if (lg == 0) {
    const T r = epilogue(e, acc, x, row, has_x);
    out[row] = r;
    if constexpr (ACC) acc_update(e, row, r);
  }
}

// halo: out[rows[i]] += s_ax * sum val * recv[col]
// recv_sel (peer memory): the receive slot is chosen on the device, slot
// (*recv_sel & 1) at recv + slot * slot_elems -- so a captured graph replays
// correctly whatever the exchange count
template <typename T>
__global__ void halo_apply_kernel(int64_t nrows, const int32_t* __restrict__ rows,
                                  const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                  const T* __restrict__ val, const T* __restrict__ recv,
                                  T* __restrict__ out, T s_ax, const unsigned* recv_sel,
                                  int64_t slot_elems) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nrows) return;
  if (recv_sel) recv += int64_t(*reinterpret_cast<const volatile unsigned*>(recv_sel) & 1u) * slot_elems;
  T acc = s_zero<T>();
  for (int64_t k = rp[i]; k < rp[i + 1]; ++k) acc = s_fma(ldg(val + k), ldg(recv + col[k]), acc);
  const int64_t r = rows[i];
  out[r] = s_fma(s_ax, acc, out[r]);
}

template <typename T>
__global__ void halo_pack_kernel(int64_t cnt, const int32_t* __restrict__ idx,
                                 const T* __restrict__ x, T* __restrict__ send) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < cnt) send[i] = ldg(x + idx[i]);
}

// ---------------------------------------------------------------------------
// Reduction helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// Block-wide sum of `v` (all threads participate); result valid in thread 0.
__device__ __forceinline__ double block_sum(double v, double* sm) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) sm[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = (lane < int(blockDim.x >> 5)) ? sm[lane] : 0.0;
    r = warp_sum(r);
  }
  return r;
}

// After each block wrote its partials: returns true (block-uniform) in the last
// block to arrive.  Partials written before the call are then visible to it.
__device__ __forceinline__ bool last_block(unsigned* counter) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(counter, 1u);
    am_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (am_last) __threadfence();
  return am_last;
}

// In the last block: sum partials[b * stride + i] over b = 0..nb-1 for i in
// [0, nv) (one warp per value, fixed order), calling f(i, sum) in lane 0.
template <typename F>
__device__ __forceinline__ void reduce_partials(const double* partials, int nb, int stride, int nv,
                                                F f) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int i = w; i < nv; i += nw) {
    double s = 0.0;
    for (int b = lane; b < nb; b += 32) s += __ldcg(partials + int64_t(b) * stride + i);
    s = warp_sum(s);
    if (lane == 0) f(i, s);
  }
}

// ---------------------------------------------------------------------------
// scale / norm / diffnorm / combine
// ---------------------------------------------------------------------------
template <typename T>
__global__ void scale_kernel(int64_t n, const T* __restrict__ src, T* __restrict__ dst,
                             const double* __restrict__ alpha_dev, double alpha_host) {
  const double a = alpha_dev ? *alpha_dev : alpha_host;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = s_scale(ldg(src + i), a);
}

template <typename T>
__global__ void __launch_bounds__(256) norm_kernel(int64_t n, const T* __restrict__ v,
                                                   double* __restrict__ out, double* partials,
                                                   unsigned* counter, double* raw) {
  __shared__ double sm[32];
  double s = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    s += s_abs2(ldg(v + i));
  s = block_sum(s, sm);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
  if (last_block(counter)) {
    reduce_partials(partials, gridDim.x, 1, 1, [&](int, double t) {
      if (raw) {  // multi-rank: rank-local sum, finalised after the allreduce
        raw[0] = t;
      } else {
        const double nrm = sqrt(t);
        out[0] = nrm;
        out[1] = 1.0 / nrm;
      }
      *counter = 0;
    });
  }
}

// Finalisation of a reduction after the cross-rank allreduce of its raw sums
// (op codes FIN_* in ppf_internal.h).
__global__ void finalize_kernel(int op, int nv, int nd, const double* __restrict__ raw,
                                double* o0, double* o1, double* o2, const double* ci) {
  const int i = threadIdx.x;
  switch (op) {
    case FIN_NORM:
      if (i == 0) {
        o0[0] = sqrt(raw[0]);
        o0[1] = 1.0 / o0[0];
      }
      break;
    case FIN_SQRT:
      if (i < nv) o0[i] = sqrt(raw[i]);
      break;
    case FIN_COEF:
      for (int k = i; k < nv; k += blockDim.x) {
        o0[k] = raw[k];
        if (o1) o1[k] = ci[k] + raw[k];
      }
      break;
    case FIN_SUBNORM:
    case FIN_LZ2:
      if (i == 0) {
        const double b = sqrt(raw[0]);
        o0[0] = b;
        if (nd == 2) o0[1] = 0.0;
        if (op == FIN_LZ2) {
          o1[0] = b;
          if (nd == 2) o1[1] = 0.0;
        }
        o2[0] = 1.0 / b;
      }
      break;
    case FIN_LZ1:
      if (i < nd) o0[i] = raw[i];
      break;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) diffnorm_kernel(int64_t n, const T* __restrict__ a,
                                                       const T* __restrict__ b,
                                                       double* __restrict__ out, double* partials,
                                                       unsigned* counter, double* raw) {
  __shared__ double sm[32];
  double s = 0.0, t = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const T bv = ldg(b + i);
    s += s_abs2(s_sub(ldg(a + i), bv));
    t += s_abs2(bv);
  }
  s = block_sum(s, sm);
  t = block_sum(t, sm);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = s;
    partials[2 * blockIdx.x + 1] = t;
  }
  if (last_block(counter)) {
    reduce_partials(partials, gridDim.x, 2, 2, [&](int i, double v) {
      if (raw)
        raw[i] = v;
      else
        out[i] = sqrt(v);
    });
    __syncthreads();
    if (threadIdx.x == 0) *counter = 0;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) combine_kernel(int64_t n, const T* __restrict__ V,
                                                      int64_t ldv, int ncols,
                                                      const T* __restrict__ y, T* __restrict__ x) {
  extern __shared__ double ysm_raw[];
  T* ysm = reinterpret_cast<T*>(ysm_raw);
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) ysm[c] = y[c];
  __syncthreads();
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    T acc = s_zero<T>();
    for (int c = 0; c < ncols; ++c) acc = s_fma(ldg(V + c * ldv + i), ysm[c], acc);
    x[i] = acc;
  }
}

// ---------------------------------------------------------------------------
// CGS2 sweeps (K5/K6/K7) on a column tile [c0, c0+nct) of V, nct <= NC.
//
// Persistent, warp-specialised kernel, one CTA per SM.  The rows are cut into
// chunks of R rows.  A producer warp streams chunk after chunk into a ring of
// S shared-memory stages with bulk async copies (cp.async.bulk, the 1-D TMA
// path): one copy per basis column segment plus one for the w segment
// (R*sizeof(T) contiguous bytes each), issued in parallel by the producer's
// lanes and completing on the stage's "full" mbarrier (expect_tx).  S is as
// deep as ~200 KB of shared memory allows, so every SM keeps 130-200 KB of
// reads in flight whatever nct is.  R consumer threads own one row of the
// chunk each: they read the row's basis values from shared memory once
// (conflict-free: column segments are contiguous), keep them in registers for
// the update and the projection, accumulate their nct projections in
// registers across chunks, and release the stage on its "empty" mbarrier
// (one arrival per consumer warp) -- no block-wide barrier in the loop.
// Flags:
//   UPD : w -= V_tile coef_in_tile          (w written back to global)
//   PROJ: coef_out_tile = V_tile^H w        (after UPD if both)
//   NRM : ||w||^2 -> Hsub = ||w||, inv = 1/||w||
// With PROJ|UPD the finalisation also writes Hcol = coef_in + coef_out.
// Block partials, then the last CTA to arrive sums them in CTA order
// (deterministic).
// ---------------------------------------------------------------------------
constexpr int F_UPD = 1, F_PROJ = 2, F_NRM = 4;
constexpr int CGS_SMEM = 212 * 1024;  // dynamic shared memory per CTA (ring + barriers)

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// ld.shared at a 32-bit shared-window address; volatile: the ring's stages
// are rewritten by the bulk copies between mbarrier waits, so a load must
// never be merged with one from an earlier pass over the same stage
template <typename T> __device__ __forceinline__ T lds_s(uint32_t a);
template <> __device__ __forceinline__ double lds_s<double>(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
template <> __device__ __forceinline__ cplx lds_s<cplx>(uint32_t a) {
  cplx v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.re), "=d"(v.im) : "r"(a));
  return v;
}

// shared-memory read the compiler may not hoist out of the chunk loop (the
// nct coefficients would otherwise occupy registers next to the nct
// accumulators and spill)
__device__ __forceinline__ double lds_nohoist(const double* p) { return *reinterpret_cast<const volatile double*>(p); }
__device__ __forceinline__ cplx lds_nohoist(const cplx* p) {
  const volatile double* q = reinterpret_cast<const volatile double*>(p);
  return {q[0], q[1]};
}

// rows per chunk (per RPT block): 16 consumer warps x 16 rows, two lanes per
// row; complex rows are twice as wide, so 128 rows (8 consumer warps)
template <typename T> __host__ __device__ constexpr int cgs_rows() { return sizeof(T) == 8 ? 256 : 128; }
template <typename T> __host__ __device__ constexpr int cgs_consumers() { return 2 * cgs_rows<T>(); }
// padding after each column segment in shared memory (16 B): the two lanes
// of a row read columns c and c+1 in the same instruction, which must not
// fall in the same bank
template <typename T> __host__ __device__ constexpr int cgs_pad() { return 16 / int(sizeof(T)); }

// RPT blocks per chunk: a stage of ~48 KB whatever nct is, so the per-chunk
// handshake stays small against the chunk's transfer time, and never fewer
// than 2 (>= 4 KB per bulk copy for fp64) while two stages still fit:
// measured on C4, 2-KB copies (RPT = 1) stream at ~5 TB/s, 4-KB and larger
// at 6.9-7.9 TB/s
template <typename T> __host__ __device__ inline int cgs_rpt(int nct) {
  constexpr int R = cgs_rows<T>();
  const int col = R * int(sizeof(T));  // bytes of one column segment per RPT block
  int r = (48 * 1024) / ((nct + 1) * col);
  if (r < 2 && 2 * (nct + 1) * (2 * col + 16) <= CGS_SMEM - 32 * 8) r = 2;
  return r > 16 ? 16 : (r < 1 ? 1 : r);
}
// shared-memory elements of one stage
template <typename T> __host__ __device__ inline int cgs_stage_elems(int nct) {
  return (nct + 1) * (cgs_rows<T>() * cgs_rpt<T>(nct) + cgs_pad<T>());
}
// stages of the ring (2..16)
template <typename T> __host__ __device__ inline int cgs_stages(int nct) {
  const int stage = cgs_stage_elems<T>(nct) * int(sizeof(T));
  int S = (CGS_SMEM - 32 * 8) / stage;
  return S > 16 ? 16 : (S < 2 ? 2 : S);
}

template <typename T, int NC, int FL>
__global__ void __launch_bounds__(cgs_consumers<T>() + 32, 1)
    cgs_kernel(int64_t n, const T* __restrict__ V, int64_t ldv, int nct, T* __restrict__ w,
               const T* __restrict__ coef_in, T* __restrict__ coef_out, T* __restrict__ Hcol,
               T* __restrict__ Hsub, double* __restrict__ inv, double* partials, unsigned* counter,
               double* raw) {
  constexpr int ND = n_doubles<T>();
  constexpr int R = cgs_rows<T>();
  constexpr int NW = cgs_consumers<T>() / 32;  // consumer warps; warp NW is the producer
  constexpr int NCL = NC / 2;                  // columns per lane (c = 2 cc + h)
  constexpr bool UPD = FL & F_UPD, PROJ = FL & F_PROJ, NRM = FL & F_NRM;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(16) T cin[NC];
  __shared__ double red[NW][NC * ND + 1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int S = cgs_stages<T>(nct);
  const int RPT = cgs_rpt<T>(nct);
  const int RC = R * RPT;                       // rows per chunk
  const int CS = RC + cgs_pad<T>();             // column stride in the stage
  const int stage_elems = cgs_stage_elems<T>(nct);
  T* ring = reinterpret_cast<T*>(smem);
  const uint32_t full0 = smem_u32(smem + size_t(S) * stage_elems * sizeof(T));
  const uint32_t empty0 = full0 + 8 * 16;
  const int64_t nchunks = (n + RC - 1) / RC;
  const int64_t nloc = blockIdx.x < nchunks ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // fp64: the coefficients of lane parity h (columns h, h + 2, ...) stored
  // contiguously, read two at a time (16-B shared loads) by the update
  if (UPD)
    for (int c = tid; c < nct; c += blockDim.x) cin[ND == 1 ? (c & 1) * (NC / 2) + (c >> 1) : c] = coef_in[c];
  __syncthreads();

  T acc[NCL];
#pragma unroll
  for (int c = 0; c < NCL; ++c) acc[c] = s_zero<T>();
  double nrm = 0.0;
  const int h = lane & 1;

  if (warp == NW) {
    // ---- producer warp ----
    for (int64_t i = 0; i < nloc; ++i) {
      const int s = int(i % S);
      if (i >= S) mbar_wait(empty0 + 8 * s, uint32_t(((i / S) - 1) & 1));
      const int64_t r0 = (int64_t(blockIdx.x) + i * gridDim.x) * RC;
      const int64_t rows = n - r0 < RC ? n - r0 : RC;
      // whole 16-B units; a ragged fp64 tail reads one padding element of the
      // column (columns are padded to a multiple of 64 entries, ldv >= n + 1)
      const uint32_t bytes = uint32_t((rows * int64_t(sizeof(T)) + 15) & ~int64_t(15));
      const uint32_t full = full0 + 8 * s;
      const uint32_t dst = smem_u32(ring + size_t(s) * stage_elems);
      if (lane == 0) mbar_expect_tx(full, bytes * uint32_t(nct + 1));
      __syncwarp();
      for (int c = lane; c <= nct; c += 32) {
        const T* src = c < nct ? V + int64_t(c) * ldv + r0 : w + r0;
        bulk_g2s(dst + uint32_t(c * CS * sizeof(T)), src, bytes, full);
      }
    }
  } else {
    // ---- consumer warps: lanes (2i, 2i+1) of warp q own row 16 q + i of
    // every RPT block, lane parity h takes the columns c = h, h+2, ... ----
    // Shared-memory operands are addressed as 32-bit shared-window addresses
    // (ld.shared): with generic pointers into the dynamic ring the compiler
    // re-derived the window base for every load, and the per-element column /
    // row predicates were packed into a register and unpacked per use -- the
    // UPD+PROJ sweep issued ~330 instructions per 16-row group for 48 FMAs
    // (ncu: 57% issue-slot busy, consumer-bound at 64.5% of DRAM peak).  Now
    // the row's basis values are loaded once into registers (used by both the
    // update and the projection), and the column / row checks exist only in
    // the variants for a partial column tile (nct < NC) or the last chunk.
    const int lrow = warp * 16 + (lane >> 1);
    const uint32_t ring_u = smem_u32(ring);
    const uint32_t colb = uint32_t(CS * sizeof(T));  // bytes between column segments
    const int ncl_h = (nct - h + 1) >> 1;             // this lane's columns c = 2 cc + h < nct
    const uint32_t cin_u = smem_u32(cin) + uint32_t(h * sizeof(T) * (ND == 1 ? NC / 2 : 1));
    // the warp releases the stage (its "empty" arrival) as soon as it has
    // read the last row block's operands into registers, before that block's
    // arithmetic: the producer can refill the stage while the FMA chains run
    // (with two stages of ~100 KB, holding a stage through the update chain
    // left only one stage in flight for a fifth of the time)
    auto consume = [&](auto colchk_t, auto rowchk_t, uint32_t st_u, int64_t r0, uint32_t empty) {
      constexpr bool COLCHK = decltype(colchk_t)::value, ROWCHK = decltype(rowchk_t)::value;
      bool released = false;
#pragma unroll 1
      for (int k = 0; k < RPT; ++k) {
        const int lr = k * R + lrow;
        const int64_t r = r0 + lr;
        const bool valid = !ROWCHK || r < n;
        if (ROWCHK && !__any_sync(FULL, valid)) break;  // warp-uniform: the shuffles need every lane
        const uint32_t a = st_u + uint32_t(lr * sizeof(T)) + uint32_t(h) * colb;
        T wr = valid ? lds_s<T>(st_u + uint32_t((nct * CS + lr) * sizeof(T))) : s_zero<T>();
        T tv[NCL];
#pragma unroll
        for (int cc = 0; cc < NCL; ++cc)
          tv[cc] = ((!COLCHK || cc < ncl_h) && valid) ? lds_s<T>(a + uint32_t(2 * cc) * colb)
                                                      : s_zero<T>();
        if (k == RPT - 1) {
          __syncwarp();
          if (lane == 0) mbar_arrive(empty);
          released = true;
        }
        if (UPD) {
          // two interleaved partial sums per lane, then the pair's halves
          T s0 = s_zero<T>(), s1 = s_zero<T>();
          if constexpr (ND == 1) {
#pragma unroll
            for (int cc = 0; cc < NCL; cc += 2) {
              if (COLCHK && cc >= ncl_h) continue;
              double c0, c1;
              asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                           : "=d"(c0), "=d"(c1)
                           : "r"(cin_u + uint32_t(cc * sizeof(T))));
              s0 = s_fma(tv[cc], c0, s0);
              if (cc + 1 < NCL && !(COLCHK && cc + 1 >= ncl_h)) s1 = s_fma(tv[cc + 1], c1, s1);
            }
          } else {
#pragma unroll
            for (int cc = 0; cc < NCL; ++cc) {
              if (COLCHK && cc >= ncl_h) continue;
              const T cf = lds_s<T>(cin_u + uint32_t(2 * cc * sizeof(T)));
              if (cc & 1)
                s1 = s_fma(tv[cc], cf, s1);
              else
                s0 = s_fma(tv[cc], cf, s0);
            }
          }
          T sum = s_add(s0, s1);
          if constexpr (ND == 1) {
            sum += __shfl_xor_sync(FULL, sum, 1);
          } else {
            cplx& z = reinterpret_cast<cplx&>(sum);
            z.re += __shfl_xor_sync(FULL, z.re, 1);
            z.im += __shfl_xor_sync(FULL, z.im, 1);
          }
          wr = s_sub(wr, sum);
          if (valid && h == 0) w[r] = wr;
        }
        if (NRM && valid && h == 0) nrm += s_abs2(wr);
        if (PROJ) {
#pragma unroll
          for (int cc = 0; cc < NCL; ++cc) acc[cc] = s_cfma(tv[cc], wr, acc[cc]);
        }
      }
      if (!released) {
        __syncwarp();
        if (lane == 0) mbar_arrive(empty);
      }
    };
    using F_ = std::false_type;
    using T_ = std::true_type;
    for (int64_t i = 0; i < nloc; ++i) {
      const int s = int(i % S);
      mbar_wait(full0 + 8 * s, uint32_t((i / S) & 1));
      const uint32_t st_u = ring_u + uint32_t(size_t(s) * stage_elems * sizeof(T));
      const int64_t r0 = (int64_t(blockIdx.x) + i * gridDim.x) * RC;
      const bool last = r0 + RC > n;
      const uint32_t empty = empty0 + 8 * s;
      if (nct == NC) {
        if (!last) consume(F_{}, F_{}, st_u, r0, empty);
        else consume(F_{}, T_{}, st_u, r0, empty);
      } else {
        if (!last) consume(T_{}, F_{}, st_u, r0, empty);
        else consume(T_{}, T_{}, st_u, r0, empty);
      }
    }
  }

  // block partials (the producer warp contributes zeros)
  if (PROJ) {
    if (warp < NW) {
#pragma unroll
      for (int cc = 0; cc < NCL; ++cc) {
        const double* a = reinterpret_cast<const double*>(&acc[cc]);
#pragma unroll
        for (int d = 0; d < ND; ++d) {
          double v = a[d];
          // sum over the lanes of equal parity: lane 0 -> column 2cc, lane 1 -> 2cc+1
#pragma unroll
          for (int o = 16; o > 1; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
          const int c = 2 * cc + lane;
          if (lane < 2 && c < nct) red[warp][c * ND + d] = v;
        }
      }
    }
    __syncthreads();
    for (int q = tid; q < nct * ND; q += blockDim.x) {
      double v = 0.0;
      for (int k = 0; k < NW; ++k) v += red[k][q];
      partials[int64_t(blockIdx.x) * nct * ND + q] = v;
    }
  }
  if (NRM) {
    __shared__ double smn[32];
    const double v = block_sum(nrm, smn);
    if (tid == 0) partials[blockIdx.x] = v;
  }
  if (last_block(counter)) {
    if (PROJ) {
      reduce_partials(partials, gridDim.x, nct * ND, nct * ND, [&](int q, double v) {
        if (raw) {
          raw[q] = v;
          return;
        }
        reinterpret_cast<double*>(coef_out)[q] = v;
        if (Hcol) reinterpret_cast<double*>(Hcol)[q] = reinterpret_cast<const double*>(coef_in)[q] + v;
      });
    }
    if (NRM) {
      reduce_partials(partials, gridDim.x, 1, 1, [&](int, double v) {
        if (raw) {
          raw[0] = v;
          return;
        }
        const double nr = sqrt(v);
        double* hs = reinterpret_cast<double*>(Hsub);
        hs[0] = nr;
        if (ND == 2) hs[1] = 0.0;
        inv[0] = 1.0 / nr;
      });
    }
    __syncthreads();
    if (tid == 0) *counter = 0;
  }
}

// Lanczos (K8).  phase 1: w -= beta_prev*vprev; alpha = v^H w.
//                phase 2: w -= alpha*v; beta = ||w||.
template <typename T, int PHASE>
__global__ void __launch_bounds__(256) lanczos_kernel(int64_t n, const T* __restrict__ v,
                                                      const T* __restrict__ vprev,
                                                      const double* __restrict__ beta_prev,
                                                      T* __restrict__ w, T* __restrict__ Hdiag,
                                                      T* __restrict__ Hsub, T* __restrict__ Hsup,
                                                      double* __restrict__ inv, double* partials,
                                                      unsigned* counter, double* raw) {
  constexpr int ND = n_doubles<T>();
  __shared__ double sm[32];
  double s0 = 0.0, s1 = 0.0;
  const double bp = (PHASE == 1 && vprev) ? *beta_prev : 0.0;
  T alpha = s_zero<T>();
  if (PHASE == 2) alpha = *Hdiag;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    T wi = w[i];
    const T vi = ldg(v + i);
    if (PHASE == 1) {
      if (vprev) wi = s_sub(wi, s_scale(ldg(vprev + i), bp));
      w[i] = wi;
      const T d = s_cfma(vi, wi, s_zero<T>());
      s0 += s_real(d);
      if (ND == 2) s1 += reinterpret_cast<const cplx&>(d).im;
    } else {
      wi = s_sub(wi, s_mul(alpha, vi));
      w[i] = wi;
      s0 += s_abs2(wi);
    }
  }
  s0 = block_sum(s0, sm);
  if (PHASE == 1 && ND == 2) s1 = block_sum(s1, sm);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = s0;
    partials[2 * blockIdx.x + 1] = s1;
  }
  if (last_block(counter)) {
    if (PHASE == 1) {
      reduce_partials(partials, gridDim.x, 2, ND, [&](int i, double s) {
        if (raw)
          raw[i] = s;
        else
          reinterpret_cast<double*>(Hdiag)[i] = s;
      });
    } else {
      reduce_partials(partials, gridDim.x, 2, 1, [&](int, double s) {
        if (raw) {
          raw[0] = s;
          return;
        }
        const double b = sqrt(s);
        reinterpret_cast<double*>(Hsub)[0] = b;
        reinterpret_cast<double*>(Hsup)[0] = b;
        if (ND == 2) {
          reinterpret_cast<double*>(Hsub)[1] = 0.0;
          reinterpret_cast<double*>(Hsup)[1] = 0.0;
        }
        inv[0] = 1.0 / b;
      });
    }
    __syncthreads();
    if (threadIdx.x == 0) *counter = 0;
  }
}

// Two-pass Lanczos, pass 2: with the pass-1 recurrence
// coefficients known on the host, regenerate the next basis vector from
// w = Op v_j and accumulate the iterate, one sweep:
//   v_{j+1} = (w - alpha v_j - beta_prev v_{j-1}) * inv_beta   (in place in w)
//   x += ycoef * v_{j+1}
template <typename T>
__global__ void __launch_bounds__(256) lanczos_regen_kernel(int64_t n, T* __restrict__ w,
                                                            const T* __restrict__ v,
                                                            const T* __restrict__ vprev,
                                                            double alpha, double beta_prev,
                                                            double inv_beta, double ycoef,
                                                            T* __restrict__ x) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    T t = s_sub(w[i], s_scale(ldg(v + i), alpha));
    if (vprev) t = s_sub(t, s_scale(ldg(vprev + i), beta_prev));
    t = s_scale(t, inv_beta);
    w[i] = t;
    x[i] = s_add(x[i], s_scale(t, ycoef));
  }
}

// acc = (acc_init ? s_acc0 xe : acc) + s_acc out, as a separate sweep (the
// sharded SpMV completes `out` only after its halo block)
template <typename T>
__global__ void __launch_bounds__(256) acc_kernel(int64_t n, const T* __restrict__ out, EpiT<T> e) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    acc_update(e, i, ldg(out + i));
}

int blocks_for(int64_t n, int threads, int cap) {
  int64_t b = (n + threads - 1) / threads;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return int(b);
}

void post_launch(const char* what) { cuda_check(cudaGetLastError(), what); }

}  // namespace

// ---------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------
// <<<blocks, 256, 0, st>>> with programmatic stream serialisation (see pdl_wait)
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kernel)(KArgs...), int blocks, int threads, cudaStream_t st,
                       Args&&... args) {
  static const bool on = [] {
    const char* e = std::getenv("PPF_PDL");
    return !(e && e[0] == '0');
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = on ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_check(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "cudaLaunchKernelEx");
}

// SELL launch: KS warps per slice (A->sell_ks), optional second output (ACC)
template <typename T, bool ACC>
static void launch_sell(ppf_mat* A, const T* xt, T* ot, const T* val, const EpiT<T>& et,
                        bool has_x, cudaStream_t st) {
  const int KS = A->sell_ks;
  const int64_t nh = A->C == 32 ? A->sell_heavy : 0;  // one block per heavy slice (sell1 only)
  // threads of a sell1 block: 4 warps (the last blocks drain sooner), 8 when
  // KS = 8 or when heavy slices want 8 warps each (C7: 4 warps cost 8%)
  const int t1 = (KS > 4 || nh > 0) ? 256 : 128;
  const int64_t spb = (t1 / 32) / KS;  // slices per block
  const int blocks = int(nh + (A->nslices - nh + spb - 1) / spb);
  if (blocks == 0) return;
#define PPF_KS(launch) \
  switch (KS) {        \
    case 1: launch(1); break; \
    case 2: launch(2); break; \
    case 4: launch(4); break; \
    default: launch(8); break; \
  }
  if constexpr (sizeof(T) == 8) {
    if (A->C == 64) {
      // 4-warp blocks (8 for KS = 8): half the work per block, so the last
      // blocks drain sooner (C3: 168.1 -> 165.3 ms; C4 unchanged; 2-warp
      // blocks cost C4 1.7%)
      const int bt = KS > 4 ? 256 : 128;
      const int64_t spb2 = (bt / 32) / KS;
      const int b2 = int((A->nslices + spb2 - 1) / spb2);
#define PPF_S2E(K, E)                                                                         \
  launch_pdl(sell2_kernel<K, ACC, E>, b2, bt, st, A->nslices, A->n_local, A->d_ptr, A->d_col,   \
             reinterpret_cast<const double*>(val), xt, ot, et, has_x, A->d_d16, A->d_cb)
#define PPF_S2(K) PPF_S2E(K, false)
#define PPF_S2D(K) PPF_S2E(K, true)
#define PPF_SPX(K, CTB, SCB)                                                                   \
  launch_pdl(sellp_kernel<K, ACC, CTB, SCB>, bp, tp, st, A->nslices, A->n_local, A->d_ptr,     \
             A->d_code8, A->d_tab_off, A->d_tab_val, A->ntab, xt, ot, et, has_x, ct, sch)
#define PPF_SP(K)                           \
  if (A->code_scaled) PPF_SPX(K, false, true); \
  else PPF_SPX(K, false, false)
#define PPF_SPC(K)                          \
  if (A->code_scaled) PPF_SPX(K, true, true); \
  else PPF_SPX(K, true, false)
      if (A->d_code8) {
        PairTab32 ct{};
        // (offsets kept as byte offsets in int32: |col - row| < 2^28)
        bool small = A->ntab <= 32;
        for (int i = 0; small && i < A->ntab; ++i)
          small = A->h_tab_off[i] > -(1 << 28) && A->h_tab_off[i] < (1 << 28);
        if (small)
          for (int i = 0; i < A->ntab; ++i) {
            ct.p[i].v = A->h_tab_val[i];
            ct.p[i].o8 = 8 * A->h_tab_off[i];
          }
        const char* ctv = std::getenv("PPF_SELLP_CTAB");   // (read per launch: A/B in one process)
        const bool use_ct = small && !(ctv && ctv[0] == '0');
        // 8-warp blocks (measured C4 / C3 deg 20: 4-, 8- and 16-warp blocks
        // within 2%)
        const int tp = 256;
        const int64_t spbp = (tp / 32) / KS;
        const int32_t* sch = KS == 1 ? A->d_sched : nullptr;
        const int bp = sch ? A->sched_blocks : int((A->nslices + spbp - 1) / spbp);
        if (use_ct) {
          PPF_KS(PPF_SPC)
        } else {
          PPF_KS(PPF_SP)
        }
        post_launch("sellp_kernel");
        return;
      } else if (A->d_d16) {
        PPF_KS(PPF_S2D)
      } else {
        PPF_KS(PPF_S2)
      }
#undef PPF_S2
#undef PPF_S2D
#undef PPF_SP
#undef PPF_SPC
#undef PPF_SPX
#undef PPF_S2E
      post_launch("sell2_kernel");
      return;
    }
  }
#define PPF_S1P(K)                                                                                  \
  sell1_kernel<T, K, true, ACC><<<blocks, t1, 0, st>>>(A->nslices, A->n_local, A->d_ptr, A->d_col, \
                                                        val, xt, ot, et, has_x, A->d_perm, nh)
#define PPF_S1(K)                                                                                    \
  sell1_kernel<T, K, false, ACC><<<blocks, t1, 0, st>>>(A->nslices, A->n_local, A->d_ptr, A->d_col, \
                                                         val, xt, ot, et, has_x, nullptr, nh)
#define PPF_S1D(K)                                                                                   \
  sell1_kernel<T, K, false, ACC, true><<<blocks, t1, 0, st>>>(A->nslices, A->n_local, A->d_ptr,     \
                                                              A->d_col, val, xt, ot, et, has_x,      \
                                                              nullptr, nh, A->d_d16, A->d_cb)
  if (A->d_perm) {
    PPF_KS(PPF_S1P)
  } else if (A->d_d16) {
    PPF_KS(PPF_S1D)
  } else {
    PPF_KS(PPF_S1)
  }
#undef PPF_S1D
#undef PPF_S1P
#undef PPF_S1
#undef PPF_KS
  post_launch("sell1_kernel");
}

template <typename T>
static void spmv_t(ppf_mat* A, const void* x, void* out, const Epi& e, cudaStream_t st) {
  const EpiT<T> et = to_epi<T>(e, x);
  const bool has_x = (e.s_x[0] != 0.0 || e.s_x[1] != 0.0);
  const T* xt = static_cast<const T*>(x);
  T* ot = static_cast<T*>(out);
  const T* val = static_cast<const T*>(A->d_val);
  if (e.acc) {
    // forward-Newton-basis chain step: second output acc
    if (A->fmt == PPF_FMT_SELL) {
      launch_sell<T, true>(A, xt, ot, val, et, has_x, st);
    } else {
      const int G = A->csr_group;
      const int blocks = int((A->n_local * G + 255) / 256);
      if (blocks == 0) return;
      switch (G) {
        case 1: csr_kernel<T, 1, true><<<blocks, 256, 0, st>>>(A->n_local, A->d_ptr, A->d_col, val, xt, ot, et, has_x); break;
        case 2: csr_kernel<T, 2, true><<<blocks, 256, 0, st>>>(A->n_local, A->d_ptr, A->d_col, val, xt, ot, et, has_x); break;
        case 4: csr_kernel<T, 4, true><<<blocks, 256, 0, st>>>(A->n_local, A->d_ptr, A->d_col, val, xt, ot, et, has_x); break;
        case 8: csr_kernel<T, 8, true><<<blocks, 256, 0, st>>>(A->n_local, A->d_ptr, A->d_col, val, xt, ot, et, has_x); break;
        case 16: csr_kernel<T, 16, true><<<blocks, 256, 0, st>>>(A->n_local, A->d_ptr, A->d_col, val, xt, ot, et, has_x); break;
        default: csr_kernel<T, 32, true><<<blocks, 256, 0, st>>>(A->n_local, A->d_ptr, A->d_col, val, xt, ot, et, has_x); break;
      }
      post_launch("csr_kernel");
    }
    return;
  }
  if (A->fmt == PPF_FMT_SELL) {
    launch_sell<T, false>(A, xt, ot, val, et, has_x, st);
  } else {
    const int G = A->csr_group;
    const int64_t threads = A->n_local * G;
    const int blocks = int((threads + 255) / 256);
    if (blocks == 0) return;
#define PPF_CSR(GG)                                                                           \
  case GG:                                                                                    \
    csr_kernel<T, GG><<<blocks, 256, 0, st>>>(A->n_local, A->d_ptr, A->d_col, val, xt, ot, et, \
                                              has_x);                                         \
    break;
    switch (G) {
      PPF_CSR(1)
      PPF_CSR(2)
      PPF_CSR(4)
      PPF_CSR(8)
      PPF_CSR(16)
      PPF_CSR(32)
      default:
        fail(PPF_EINVAL, "bad CSR group");
    }
#undef PPF_CSR
    post_launch("csr_kernel");
  }
}

void launch_spmv(ppf_mat* A, const void* x, void* out, const Epi& e, cudaStream_t st) {
  if (A->dtype == PPF_R64)
    spmv_t<double>(A, x, out, e, st);
  else
    spmv_t<cplx>(A, x, out, e, st);
}

void launch_acc(ppf_mat* A, const void* x, const void* out, const Epi& e, cudaStream_t st) {
  const int blocks = blocks_for(A->n_local, 256, 148 * 8);
  if (A->dtype == PPF_R64)
    acc_kernel<double><<<blocks, 256, 0, st>>>(A->n_local, static_cast<const double*>(out),
                                               to_epi<double>(e, x));
  else
    acc_kernel<cplx><<<blocks, 256, 0, st>>>(A->n_local, static_cast<const cplx*>(out),
                                             to_epi<cplx>(e, x));
  post_launch("acc_kernel");
}

void launch_halo_pack(ppf_mat* A, const void* x, cudaStream_t st) {
  if (A->send_total == 0) return;
  const int blocks = int((A->send_total + 255) / 256);
  if (A->dtype == PPF_R64)
    halo_pack_kernel<double><<<blocks, 256, 0, st>>>(A->send_total, A->d_send_idx,
                                                     static_cast<const double*>(x),
                                                     static_cast<double*>(A->d_send));
  else
    halo_pack_kernel<cplx><<<blocks, 256, 0, st>>>(A->send_total, A->d_send_idx,
                                                   static_cast<const cplx*>(x),
                                                   static_cast<cplx*>(A->d_send));
  post_launch("halo_pack_kernel");
}

void launch_halo_apply(ppf_mat* A, void* out, const double* s_ax, cudaStream_t st,
                       const void* recv, const unsigned* recv_sel) {
  if (A->halo_rows == 0) return;
  if (!recv) recv = A->d_recv;
  const int blocks = int((A->halo_rows + 255) / 256);
  if (A->dtype == PPF_R64)
    halo_apply_kernel<double><<<blocks, 256, 0, st>>>(
        A->halo_rows, A->d_halo_rows, A->d_halo_ptr, A->d_halo_col,
        static_cast<const double*>(A->d_halo_val), static_cast<const double*>(recv),
        static_cast<double*>(out), s_ax[0], recv_sel, A->halo_total);
  else
    halo_apply_kernel<cplx><<<blocks, 256, 0, st>>>(
        A->halo_rows, A->d_halo_rows, A->d_halo_ptr, A->d_halo_col,
        static_cast<const cplx*>(A->d_halo_val), static_cast<const cplx*>(recv),
        static_cast<cplx*>(out), cplx{s_ax[0], s_ax[1]}, recv_sel, A->halo_total);
  post_launch("halo_apply_kernel");
}

void launch_scale(ppf_dtype dt, int64_t n, const void* src, void* dst, const double* alpha_dev,
                  double alpha_host, cudaStream_t st) {
  const int blocks = blocks_for(n, 256, 148 * 8);
  if (dt == PPF_R64)
    scale_kernel<double><<<blocks, 256, 0, st>>>(n, static_cast<const double*>(src),
                                                 static_cast<double*>(dst), alpha_dev, alpha_host);
  else
    scale_kernel<cplx><<<blocks, 256, 0, st>>>(n, static_cast<const cplx*>(src),
                                               static_cast<cplx*>(dst), alpha_dev, alpha_host);
  post_launch("scale_kernel");
}

void launch_norm(ppf_dtype dt, int64_t n, const void* v, double* out, RedScratch& rs, int grid,
                 cudaStream_t st) {
  const int blocks = blocks_for(n, 256, grid);
  if (dt == PPF_R64)
    norm_kernel<double><<<blocks, 256, 0, st>>>(n, static_cast<const double*>(v), out,
                                                rs.partials, rs.counter, rs.raw);
  else
    norm_kernel<cplx><<<blocks, 256, 0, st>>>(n, static_cast<const cplx*>(v), out, rs.partials,
                                              rs.counter, rs.raw);
  post_launch("norm_kernel");
}

void launch_finalize(int op, int nv, int nd, const double* raw, void* o0, void* o1, void* o2,
                     const void* ci, cudaStream_t st) {
  finalize_kernel<<<1, 256, 0, st>>>(op, nv, nd, raw, static_cast<double*>(o0),
                                     static_cast<double*>(o1), static_cast<double*>(o2),
                                     static_cast<const double*>(ci));
  post_launch("finalize_kernel");
}

void launch_diffnorm(ppf_dtype dt, int64_t n, const void* a, const void* b, double* out,
                     RedScratch& rs, int grid, cudaStream_t st) {
  const int blocks = blocks_for(n, 256, grid);
  if (dt == PPF_R64)
    diffnorm_kernel<double><<<blocks, 256, 0, st>>>(n, static_cast<const double*>(a),
                                                    static_cast<const double*>(b), out,
                                                    rs.partials, rs.counter, rs.raw);
  else
    diffnorm_kernel<cplx><<<blocks, 256, 0, st>>>(n, static_cast<const cplx*>(a),
                                                  static_cast<const cplx*>(b), out, rs.partials,
                                                  rs.counter, rs.raw);
  post_launch("diffnorm_kernel");
}

void launch_lanczos_regen(ppf_dtype dt, int64_t n, void* w, const void* v, const void* vprev,
                          double alpha, double beta_prev, double inv_beta, double ycoef, void* x,
                          cudaStream_t st) {
  const int blocks = blocks_for(n, 256, 148 * 8);
  if (dt == PPF_R64)
    lanczos_regen_kernel<double><<<blocks, 256, 0, st>>>(
        n, static_cast<double*>(w), static_cast<const double*>(v), static_cast<const double*>(vprev),
        alpha, beta_prev, inv_beta, ycoef, static_cast<double*>(x));
  else
    lanczos_regen_kernel<cplx><<<blocks, 256, 0, st>>>(
        n, static_cast<cplx*>(w), static_cast<const cplx*>(v), static_cast<const cplx*>(vprev), alpha,
        beta_prev, inv_beta, ycoef, static_cast<cplx*>(x));
  post_launch("lanczos_regen_kernel");
}

void launch_combine(ppf_dtype dt, int64_t n, const void* V, int64_t ldv, int ncols, const void* y,
                    void* x, cudaStream_t st) {
  const int blocks = blocks_for(n, 256, 148 * 8);
  const size_t sm = size_t(ncols) * (dt == PPF_R64 ? 8 : 16);
  if (dt == PPF_R64)
    combine_kernel<double><<<blocks, 256, sm, st>>>(n, static_cast<const double*>(V), ldv, ncols,
                                                    static_cast<const double*>(y),
                                                    static_cast<double*>(x));
  else
    combine_kernel<cplx><<<blocks, 256, sm, st>>>(n, static_cast<const cplx*>(V), ldv, ncols,
                                                  static_cast<const cplx*>(y),
                                                  static_cast<cplx*>(x));
  post_launch("combine_kernel");
}

// raw (multi-rank): where this launch's rank-local sums go (tile offset applied)
template <typename T, int NC, int FL>
static void cgs_go(int64_t n, const T* V, int64_t ldv, int nct, T* w, const T* ci, T* co, T* hc,
                   T* hs, double* inv, RedScratch& rs, double* raw, int grid, cudaStream_t st) {
  // the attribute is per device: one bit per device ordinal, per instantiation
  // (setting it twice from racing host threads is harmless)
  static std::atomic<unsigned long long> attr_done{0};
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(attr_done.load(std::memory_order_acquire) & bit)) {
    cuda_check(cudaFuncSetAttribute(cgs_kernel<T, NC, FL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    CGS_SMEM),
               "cudaFuncSetAttribute(cgs_kernel)");
    attr_done.fetch_or(bit, std::memory_order_release);
  }
  const int S = cgs_stages<T>(nct);
  const int RC = cgs_rows<T>() * cgs_rpt<T>(nct);
  const size_t smem = size_t(S) * cgs_stage_elems<T>(nct) * sizeof(T) + 2 * 8 * 16;  // ring + 2 x 16 mbarriers
  const int64_t chunks = (n + RC - 1) / RC;
  int blocks = int(chunks < grid ? chunks : grid);
  if (blocks < 1) blocks = 1;
  cgs_kernel<T, NC, FL><<<blocks, cgs_consumers<T>() + 32, smem, st>>>(
      n, V, ldv, nct, w, ci, co, hc, hs, inv, rs.partials, rs.counter, raw);
  post_launch("cgs_kernel");
}

// ---------------------------------------------------------------------------
// "Flat" CGS2 sweeps for operators whose tiled sweeps are launch- and
// latency-bound (n of a few 10^5 rows or less: a 24-column tile launch then
// covers at most a few chunks per SM, and a step at j ~ 75 issued up to 16
// launches).  ONE launch per sweep over ALL columns: each block walks row
// blocks of FLAT_RB rows (grid-stride); the update (UPD) is one thread per row
// summing over the columns in column order (8 loads in flight, 4 interleaved
// partial sums); the projection (PROJ) is one warp per column (columns
// c = warp, warp + 8, ...), lanes over the row block's rows (coalesced),
// accumulated per block in shared memory; the updated w of the row block is
// shared through shared memory, so UPD+PROJ is one pass (the row block's V
// rows are re-read from L1/L2).  Per-block partials, the last block to arrive
// sums them in block order, one thread per value.
// ---------------------------------------------------------------------------
constexpr int FLAT_THREADS = 256;
constexpr int FLAT_RB = FLAT_THREADS;

// In the last block: sum partials[b * stride + i] over b = 0..nb-1 (nb <=
// 32 * FLAT_NBL) for each i in [0, nv).  Each warp takes FLAT_VPW values at a
// time; every lane first loads its blocks b = lane + 32 k of all of them (all
// loads in flight at once -- a loop of dependent adds would pay one L2
// latency per block), adds them in k order, then the warp tree; fixed order.
constexpr int FLAT_NBL = 10, FLAT_VPW = 4;
template <typename F>
__device__ __forceinline__ void reduce_partials_wide(const double* partials, int nb, int stride,
                                                     int nv, F f) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int i0 = w * FLAT_VPW; i0 < nv; i0 += nw * FLAT_VPW) {
    double t[FLAT_NBL][FLAT_VPW];
#pragma unroll
    for (int kk = 0; kk < FLAT_NBL; ++kk)
#pragma unroll
      for (int v = 0; v < FLAT_VPW; ++v) {
        const int b = lane + 32 * kk;
        t[kk][v] = (b < nb && i0 + v < nv) ? __ldcg(partials + int64_t(b) * stride + i0 + v) : 0.0;
      }
#pragma unroll
    for (int v = 0; v < FLAT_VPW; ++v) {
      double s = 0.0;
#pragma unroll
      for (int kk = 0; kk < FLAT_NBL; ++kk) s += t[kk][v];
      s = warp_sum(s);
      if (lane == 0 && i0 + v < nv) f(i0 + v, s);
    }
  }
}

template <typename T, int FL>
__global__ void __launch_bounds__(FLAT_THREADS) cgs_flat_kernel(
    int64_t n, const T* __restrict__ V, int64_t ldv, int ncols, T* __restrict__ w,
    const T* __restrict__ coef_in, T* __restrict__ coef_out, T* __restrict__ Hcol,
    T* __restrict__ Hsub, double* __restrict__ inv, double* partials, unsigned* counter,
    double* raw) {
  constexpr int ND = n_doubles<T>();
  constexpr bool UPD = FL & F_UPD, PROJ = FL & F_PROJ, NRM = FL & F_NRM;
  constexpr int NW = FLAT_THREADS / 32;
  extern __shared__ __align__(16) unsigned char flat_smem[];
  T* cs = reinterpret_cast<T*>(flat_smem);                      // ncols coefficients (UPD)
  double* bacc = reinterpret_cast<double*>(cs + ncols);          // ncols x ND block sums (PROJ)
  __shared__ T wsh[FLAT_RB];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int c = tid; c < ncols; c += FLAT_THREADS) {
    if (UPD) cs[c] = coef_in[c];
    if (PROJ)
      for (int d = 0; d < ND; ++d) bacc[c * ND + d] = 0.0;
  }
  __syncthreads();
  double nrm = 0.0;
  for (int64_t r0 = int64_t(blockIdx.x) * FLAT_RB; r0 < n; r0 += int64_t(gridDim.x) * FLAT_RB) {
    const int64_t r = r0 + tid;
    const bool valid = r < n;
    T wr = valid ? w[r] : s_zero<T>();
    if (UPD) {
      T s0 = s_zero<T>(), s1 = s_zero<T>(), s2 = s_zero<T>(), s3 = s_zero<T>();
      if (valid) {
        const T* vr = V + r;
        int c = 0;
        for (; c + 8 <= ncols; c += 8) {
          T v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = ldg(vr + int64_t(c + u) * ldv);
          s0 = s_fma(v[0], cs[c], s0);
          s1 = s_fma(v[1], cs[c + 1], s1);
          s2 = s_fma(v[2], cs[c + 2], s2);
          s3 = s_fma(v[3], cs[c + 3], s3);
          s0 = s_fma(v[4], cs[c + 4], s0);
          s1 = s_fma(v[5], cs[c + 5], s1);
          s2 = s_fma(v[6], cs[c + 6], s2);
          s3 = s_fma(v[7], cs[c + 7], s3);
        }
        for (; c < ncols; ++c) s0 = s_fma(ldg(vr + int64_t(c) * ldv), cs[c], s0);
      }
      wr = s_sub(wr, s_add(s_add(s0, s1), s_add(s2, s3)));
      if (valid) w[r] = wr;
      if (NRM) nrm += s_abs2(wr);
    }
    if (PROJ) {
      wsh[tid] = wr;
      __syncthreads();
      // FLAT_CPW columns per warp at a time (c = warp + NW q), all their loads
      // in flight together, then the warp trees interleaved
      constexpr int CPW = 4;
      for (int cb = warp; cb < ncols; cb += NW * CPW) {
        T s[CPW];
#pragma unroll
        for (int q = 0; q < CPW; ++q) s[q] = s_zero<T>();
#pragma unroll
        for (int kk = 0; kk < FLAT_RB / 32; ++kk) {
          const int i = kk * 32 + lane;
          const bool ok = r0 + i < n;
          const T wi = wsh[i];
#pragma unroll
          for (int q = 0; q < CPW; ++q) {
            const int c = cb + q * NW;
            if (ok && c < ncols) s[q] = s_cfma(ldg(V + int64_t(c) * ldv + r0 + i), wi, s[q]);
          }
        }
#pragma unroll
        for (int q = 0; q < CPW; ++q) {
          const int c = cb + q * NW;
          const double* a = reinterpret_cast<const double*>(&s[q]);
#pragma unroll
          for (int d = 0; d < ND; ++d) {
            const double v = warp_sum(a[d]);
            if (lane == 0 && c < ncols) bacc[c * ND + d] += v;
          }
        }
      }
      __syncthreads();
    }
  }
  if (PROJ) {
    for (int q = tid; q < ncols * ND; q += FLAT_THREADS)
      partials[int64_t(blockIdx.x) * ncols * ND + q] = bacc[q];
  }
  if (NRM) {
    __shared__ double smn[32];
    const double v = block_sum(nrm, smn);
    if (tid == 0) partials[blockIdx.x] = v;
  }
  if (last_block(counter)) {
    if (PROJ) {
      reduce_partials_wide(partials, gridDim.x, ncols * ND, ncols * ND, [&](int q, double v) {
        if (raw) {
          raw[q] = v;
          return;
        }
        reinterpret_cast<double*>(coef_out)[q] = v;
        if (Hcol) reinterpret_cast<double*>(Hcol)[q] = reinterpret_cast<const double*>(coef_in)[q] + v;
      });
    }
    if (NRM) {
      reduce_partials_wide(partials, gridDim.x, 1, 1, [&](int, double v) {
        if (raw) {
          raw[0] = v;
          return;
        }
        const double nr = sqrt(v);
        double* hs = reinterpret_cast<double*>(Hsub);
        hs[0] = nr;
        if (ND == 2) hs[1] = 0.0;
        inv[0] = 1.0 / nr;
      });
    }
    __syncthreads();
    if (tid == 0) *counter = 0;
  }
}

// ---------------------------------------------------------------------------
// "Wide" CGS2 sweeps (round 2): ALL columns of V per stage, for bases wider
// than one 24-column tile (C7: m = 114, C2 deg 5: m = 76).  A stage holds a
// chunk of WIDE_R rows (512 B per column segment) of every column, fetched by
// 2-D tensor-map bulk copies (boxes of WIDE_R rows x WIDE_CB columns, rows
// past n and columns past ncols zero-filled by the copy engine) plus one 1-D
// bulk copy of w; a producer warp keeps the ring full.  Consumers (8 warps):
//   UPD   one thread per (row, quarter of the columns): lanes on consecutive
//         rows of one column (conflict-free), the quarters added in order;
//         the updated w goes back to the stage and to global memory;
//   PROJ  one thread per column, accumulating over the whole sweep in a
//         register; row order skewed by lane (row (i + lane) mod WIDE_R) so
//         the 32 lanes of a warp hit distinct banks.
// So every sweep is ONE launch reading V once, whatever the column count (the
// tiled sweeps issue one launch per 24-column tile and the UPD+PROJ sweep two
// passes); per-CTA partials, the last CTA sums them in CTA order.
// ---------------------------------------------------------------------------
constexpr int WIDE_CB = 32;                    // columns per tensor box
constexpr int WIDE_THREADS = 256;              // consumer threads
constexpr int WIDE_MAX_COLS = 192;
// rows per chunk: SEG bytes per column segment (512 B or 1 KB -- longer
// segments keep the DRAM row buffers busier; 1 KB when three stages still fit)
template <typename T, int SEG> __host__ __device__ constexpr int wide_rows() { return SEG / int(sizeof(T)); }
template <typename T, int SEG> __host__ __device__ inline int wide_stage_bytes(int ncols) {
  const int ncp = (ncols + WIDE_CB - 1) / WIDE_CB * WIDE_CB;
  return (ncp + 1) * SEG;
}
template <typename T, int SEG> __host__ __device__ inline int wide_stages(int ncols) {
  int S = (CGS_SMEM - 32 * 8) / wide_stage_bytes<T, SEG>(ncols);
  return S > 8 ? 8 : S;
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void* tmap, int c0, int c1,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(WIDE_THREADS) : "memory");
}

template <typename T, int FL, int SEG>
__global__ void __launch_bounds__(WIDE_THREADS + 32, 1) cgs_wide_kernel(
    const __grid_constant__ CUtensorMap tmV, int64_t n, int ncols, T* __restrict__ w,
    const T* __restrict__ coef_in, T* __restrict__ coef_out, T* __restrict__ Hcol,
    T* __restrict__ Hsub, double* __restrict__ inv, double* partials, unsigned* counter,
    double* raw) {
  constexpr int ND = n_doubles<T>();
  constexpr int R = wide_rows<T, SEG>();
  constexpr int DPE = int(sizeof(T)) / 8;   // doubles per element (tensor inner unit)
  constexpr bool UPD = FL & F_UPD, PROJ = FL & F_PROJ, NRM = FL & F_NRM;
  constexpr int NW = WIDE_THREADS / 32;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ T cin[WIDE_MAX_COLS];
  __shared__ T part[WIDE_THREADS / R][R];
  __shared__ double red[NW + 1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int S = wide_stages<T, SEG>(ncols);
  const int ncp = (ncols + WIDE_CB - 1) / WIDE_CB * WIDE_CB;
  const int nbox = ncp / WIDE_CB;
  const uint32_t stage_bytes = uint32_t(wide_stage_bytes<T, SEG>(ncols));
  const uint32_t ring = smem_u32(smem);
  const uint32_t full0 = ring + uint32_t(S) * stage_bytes;
  const uint32_t empty0 = full0 + 8 * 8;
  const int64_t nchunks = (n + R - 1) / R;
  const int64_t nloc = blockIdx.x < nchunks ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (UPD)
    for (int c = tid; c < ncols; c += blockDim.x) cin[c] = coef_in[c];
  __syncthreads();
  T acc = s_zero<T>();
  double nrm = 0.0;
  // projection threads per column: 8, 4, 2 or 1 (a power of two dividing R)
  const int PG = ncols * 8 <= WIDE_THREADS ? 8 : ncols * 4 <= WIDE_THREADS ? 4
                 : ncols * 2 <= WIDE_THREADS ? 2 : 1;
  if (warp == NW) {
    // ---- producer ----
    if (lane == 0) {
      for (int64_t i = 0; i < nloc; ++i) {
        const int s = int(i % S);
        if (i >= S) mbar_wait(empty0 + 8 * s, uint32_t(((i / S) - 1) & 1));
        const int64_t r0 = (int64_t(blockIdx.x) + i * gridDim.x) * R;
        const uint32_t st = ring + uint32_t(s) * stage_bytes;
        const int64_t rows = n - r0 < R ? n - r0 : R;
        const uint32_t wbytes = uint32_t((rows * int64_t(sizeof(T)) + 15) & ~int64_t(15));
        mbar_expect_tx(full0 + 8 * s, uint32_t(nbox) * uint32_t(WIDE_CB * R * sizeof(T)) + wbytes);
        for (int bx = 0; bx < nbox; ++bx)
          tma_load_2d(st + uint32_t(bx * WIDE_CB * R * sizeof(T)), &tmV, int(r0 * DPE),
                      bx * WIDE_CB, full0 + 8 * s);
        bulk_g2s(st + uint32_t(ncp * R * sizeof(T)), w + r0, wbytes, full0 + 8 * s);
      }
    }
  } else {
    // ---- consumers ----
    const int lr = tid % R, p = tid / R;                  // UPD: row, quarter (fp64: 4 x 64)
    constexpr int PARTS = WIDE_THREADS / R;               // 4 (fp64) or 8 (complex)
    for (int64_t i = 0; i < nloc; ++i) {
      const int s = int(i % S);
      mbar_wait(full0 + 8 * s, uint32_t((i / S) & 1));
      const uint32_t st = ring + uint32_t(s) * stage_bytes;
      const uint32_t wseg = st + uint32_t(ncp * R * sizeof(T));
      const int64_t r0 = (int64_t(blockIdx.x) + i * gridDim.x) * R;
      if (UPD) {
        // four chains over this thread's columns c = p, p + PARTS, ...
        T s4[4] = {s_zero<T>(), s_zero<T>(), s_zero<T>(), s_zero<T>()};
        int c = p;
        for (; c + 3 * PARTS < ncols; c += 4 * PARTS) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int cu = c + u * PARTS;
            s4[u] = s_fma(lds_s<T>(st + uint32_t((cu * R + lr) * sizeof(T))), cin[cu], s4[u]);
          }
        }
        for (; c < ncols; c += PARTS)
          s4[0] = s_fma(lds_s<T>(st + uint32_t((c * R + lr) * sizeof(T))), cin[c], s4[0]);
        part[p][lr] = s_add(s_add(s4[0], s4[1]), s_add(s4[2], s4[3]));
        consumers_sync();
        if (p == 0) {
          T sum = part[0][lr];
#pragma unroll
          for (int q2 = 1; q2 < PARTS; ++q2) sum = s_add(sum, part[q2][lr]);
          const bool valid = r0 + lr < n;
          const T wr = valid ? s_sub(lds_s<T>(wseg + uint32_t(lr * sizeof(T))), sum) : s_zero<T>();
          if (valid) w[r0 + lr] = wr;
          if (NRM) nrm += s_abs2(wr);
          if (PROJ) {   // the updated w back into the stage for the projection
            if constexpr (ND == 1) {
              asm volatile("st.shared.f64 [%0], %1;" ::"r"(wseg + uint32_t(lr * 8)), "d"(wr) : "memory");
            } else {
              const cplx z = reinterpret_cast<const cplx&>(wr);
              asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(wseg + uint32_t(lr * 16)), "d"(z.re),
                           "d"(z.im) : "memory");
            }
          }
        }
        if (PROJ) consumers_sync();
      }
      if (PROJ && tid < ncols * PG) {
        // G = PG threads per column (c = tid / PG) take the rows r = g mod PG
        // (g = tid % PG), visited from row (tid * ... ) on: rr = (i PG + tid)
        // mod R keeps each thread's residue class and gives the lanes of a
        // half-warp distinct banks
        const int c = tid / PG;
        const uint32_t col = st + uint32_t(c * R * sizeof(T));
        const int64_t rem = n - r0;
        const int nit = R / PG;               // 8 .. 64, a multiple of 4 for PG <= 16
        // four independent chains (the single FMA chain through shared-memory
        // loads was latency-bound), combined in a fixed order
        T a4[4] = {s_zero<T>(), s_zero<T>(), s_zero<T>(), s_zero<T>()};
        if (rem >= R) {
          for (int i = 0; i < nit; i += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int rr = ((i + u) * PG + tid) & (R - 1);
              a4[u] = s_cfma(lds_s<T>(col + uint32_t(rr * sizeof(T))),
                             lds_s<T>(wseg + uint32_t(rr * sizeof(T))), a4[u]);
            }
          }
        } else {
          for (int i = 0; i < nit; i += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int rr = ((i + u) * PG + tid) & (R - 1);
              if (rr < rem)
                a4[u] = s_cfma(lds_s<T>(col + uint32_t(rr * sizeof(T))),
                               lds_s<T>(wseg + uint32_t(rr * sizeof(T))), a4[u]);
            }
          }
        }
        acc = s_add(acc, s_add(s_add(a4[0], a4[1]), s_add(a4[2], a4[3])));
      }
      consumers_sync();   // the stage (and part[]) are free again
      if (lane == 0) mbar_arrive(empty0 + 8 * s);
    }
  }
  // per-CTA partials: the PG partial sums of a column added in group order
  if (PROJ) {
    T* gsum = &part[0][0];   // WIDE_THREADS entries, free after the loop
    __syncthreads();
    if (warp < NW) gsum[tid] = acc;
    __syncthreads();
    for (int c = tid; c < ncols; c += blockDim.x) {
      T s = gsum[c * PG];
      for (int g = 1; g < PG; ++g) s = s_add(s, gsum[c * PG + g]);
      const double* a = reinterpret_cast<const double*>(&s);
      for (int d = 0; d < ND; ++d) partials[(int64_t(blockIdx.x) * ncols + c) * ND + d] = a[d];
    }
  }
  if (NRM) {
    const double v = block_sum(nrm, red);
    if (tid == 0) partials[blockIdx.x] = v;
  }
  if (last_block(counter)) {
    if (PROJ) {
      reduce_partials_wide(partials, gridDim.x, ncols * ND, ncols * ND, [&](int q, double v) {
        if (raw) {
          raw[q] = v;
          return;
        }
        reinterpret_cast<double*>(coef_out)[q] = v;
        if (Hcol) reinterpret_cast<double*>(Hcol)[q] = reinterpret_cast<const double*>(coef_in)[q] + v;
      });
    }
    if (NRM) {
      reduce_partials_wide(partials, gridDim.x, 1, 1, [&](int, double v) {
        if (raw) {
          raw[0] = v;
          return;
        }
        const double nr = sqrt(v);
        double* hs = reinterpret_cast<double*>(Hsub);
        hs[0] = nr;
        if (ND == 2) hs[1] = 0.0;
        inv[0] = 1.0 / nr;
      });
    }
    __syncthreads();
    if (tid == 0) *counter = 0;
  }
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                 const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiled encode_tiled() {
  static EncodeTiled fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiled>(p);
  }();
  return fn;
}

// wide sweeps: ncols beyond one tile, up to WIDE_MAX_COLS (two stages fit)
static bool cgs_use_wide(int ncols, int tile) {
  const char* e = std::getenv("PPF_CGS_WIDE");
  if (e && e[0] == '0') return false;
  return ncols > tile && ncols <= WIDE_MAX_COLS && encode_tiled() != nullptr;
}

template <typename T, int SEG>
static int cgs_wide_seg(int mode, int64_t n, const T* V, int64_t ldv, int ncols, T* w, const T* ci,
                        T* co, T* hc, T* hs, double* inv, RedScratch& rs, int grid, cudaStream_t st) {
  constexpr int R = wide_rows<T, SEG>();
  constexpr int DPE = int(sizeof(T)) / 8;
  CUtensorMap tm;
  const cuuint64_t dims[2] = {cuuint64_t(n) * DPE, cuuint64_t(ncols)};
  const cuuint64_t strides[1] = {cuuint64_t(ldv) * sizeof(T)};
  const cuuint32_t box[2] = {cuuint32_t(R * DPE), cuuint32_t(WIDE_CB)};
  const cuuint32_t estr[2] = {1, 1};
  if (encode_tiled()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<T*>(V), dims, strides, box,
                     estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    fail(PPF_ECUDA, "cuTensorMapEncodeTiled failed");
  const int S = wide_stages<T, SEG>(ncols);
  const size_t smem = size_t(S) * size_t(wide_stage_bytes<T, SEG>(ncols)) + 2 * 8 * 8;
  const int64_t chunks = (n + R - 1) / R;
  int blocks = int(chunks < grid ? chunks : grid);
  if (blocks < 1) blocks = 1;
  auto go = [&](auto kfn, const T* cin, T* cout, T* hcol, T* hsub, double* iv) {
    // the attribute is per kernel and per device (the three sweep kernels
    // share one function-pointer type, so the key is the pointer itself)
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    {
      std::lock_guard<std::mutex> lk(mu);
      if (done.insert({reinterpret_cast<const void*>(kfn), dev}).second)
        cuda_check(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, CGS_SMEM),
                   "cudaFuncSetAttribute(cgs_wide_kernel)");
    }
    kfn<<<blocks, WIDE_THREADS + 32, smem, st>>>(tm, n, ncols, w, cin, cout, hcol, hsub, iv,
                                                 rs.partials, rs.counter, rs.raw);
    const cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess) {
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, kfn);
      fail(PPF_ECUDA, std::string("cgs_wide_kernel: ") + cudaGetErrorString(le) + " (blocks " +
                          std::to_string(blocks) + ", smem " + std::to_string(smem) + ", ncols " +
                          std::to_string(ncols) + ", maxdyn " + std::to_string(fa.maxDynamicSharedSizeBytes) +
                          ", static " + std::to_string(fa.sharedSizeBytes) + ", regs " +
                          std::to_string(fa.numRegs) + ", maxthr " + std::to_string(fa.maxThreadsPerBlock) + ")");
    }
  };
  if (mode == 0)
    go(cgs_wide_kernel<T, F_PROJ, SEG>, nullptr, co, nullptr, nullptr, nullptr);
  else if (mode == 1)
    go(cgs_wide_kernel<T, F_UPD | F_PROJ, SEG>, ci, co, hc, nullptr, nullptr);
  else
    go(cgs_wide_kernel<T, F_UPD | F_NRM, SEG>, ci, nullptr, nullptr, hs, inv);
  return 1;
}

template <typename T>
static int cgs_wide(int mode, int64_t n, const T* V, int64_t ldv, int ncols, T* w, const T* ci,
                    T* co, T* hc, T* hs, double* inv, RedScratch& rs, int grid, cudaStream_t st) {
  const char* e = std::getenv("PPF_CGS_WIDE_SEG");
  const bool big = e ? e[0] == '1' : wide_stages<T, 1024>(ncols) >= 3;
  if (big) return cgs_wide_seg<T, 1024>(mode, n, V, ldv, ncols, w, ci, co, hc, hs, inv, rs, grid, st);
  return cgs_wide_seg<T, 512>(mode, n, V, ldv, ncols, w, ci, co, hc, hs, inv, rs, grid, st);
}

// rows below which the flat sweeps replace the tiled TMA ones (per rank):
// ~2 chunks of a full 24-column tile per SM
static bool cgs_use_flat(int64_t n, int num_sms_cap, int ncols, int tile) {
  // PPF_CGS_FLAT=1 / 0 forces the flat / tiled sweeps (tests; read per call)
  const char* e = std::getenv("PPF_CGS_FLAT");
  const int force = e ? (e[0] == '1' ? 1 : 0) : -1;
  if (force >= 0) return force == 1;
  // (one tile: the tiled sweeps already need only one launch each)
  return ncols > tile && n < int64_t(2) * 512 * (num_sms_cap / 8);
}

template <typename T>
static int cgs_flat(int mode, int64_t n, const T* V, int64_t ldv, int ncols, T* w, const T* ci,
                    T* co, T* hc, T* hs, double* inv, RedScratch& rs, int grid, cudaStream_t st) {
  constexpr int ND = n_doubles<T>();
  // two blocks per SM at most: the per-block partials (ncols x ND each) and
  // the tail sum stay short
  const int blocks = blocks_for(n, FLAT_RB, grid);
  const size_t smem = size_t(ncols) * (sizeof(T) + ND * sizeof(double));
  if (mode == 0)
    cgs_flat_kernel<T, F_PROJ><<<blocks, FLAT_THREADS, smem, st>>>(
        n, V, ldv, ncols, w, nullptr, co, nullptr, nullptr, nullptr, rs.partials, rs.counter, rs.raw);
  else if (mode == 1)
    cgs_flat_kernel<T, F_UPD | F_PROJ><<<blocks, FLAT_THREADS, smem, st>>>(
        n, V, ldv, ncols, w, ci, co, hc, nullptr, nullptr, rs.partials, rs.counter, rs.raw);
  else
    cgs_flat_kernel<T, F_UPD | F_NRM><<<blocks, FLAT_THREADS, smem, st>>>(
        n, V, ldv, ncols, w, ci, nullptr, nullptr, hs, inv, rs.partials, rs.counter, rs.raw);
  post_launch("cgs_flat_kernel");
  return 1;
}

// column tile width per launch: 24 (two stages of 25 x 4 KB column segments
// fit in shared memory, cgs_rpt), fp64 and complex
template <typename T> constexpr int cgs_tile() { return 24; }

template <typename T, int FL>
static void cgs_nc(int64_t n, const T* V, int64_t ldv, int nct, T* w, const T* ci, T* co, T* hc,
                   T* hs, double* inv, RedScratch& rs, int grid, cudaStream_t st, int c0 = 0) {
  constexpr int ND = n_doubles<T>();
  double* raw = rs.raw ? rs.raw + ((FL & F_PROJ) ? c0 * ND : 0) : nullptr;
  if (nct <= 4)
    cgs_go<T, 4, FL>(n, V, ldv, nct, w, ci, co, hc, hs, inv, rs, raw, grid, st);
  else if (nct <= 8)
    cgs_go<T, 8, FL>(n, V, ldv, nct, w, ci, co, hc, hs, inv, rs, raw, grid, st);
  else if (nct <= 16)
    cgs_go<T, 16, FL>(n, V, ldv, nct, w, ci, co, hc, hs, inv, rs, raw, grid, st);
  else if constexpr (cgs_tile<T>() > 16)
    cgs_go<T, 24, FL>(n, V, ldv, nct, w, ci, co, hc, hs, inv, rs, raw, grid, st);
  else
    fail(PPF_EINVAL, "CGS column tile too wide");
}

template <typename T>
static int cgs_dispatch(int mode, int64_t n, const void* Vv, int64_t ldv, int ncols, void* wv,
                        const void* civ, void* cov, void* hcv, void* hsv, double* inv,
                        RedScratch& rs, int grid, cudaStream_t st) {
  constexpr int TILE = cgs_tile<T>();
  auto V = static_cast<const T*>(Vv);
  auto w = static_cast<T*>(wv);
  auto ci = static_cast<const T*>(civ);
  auto co = static_cast<T*>(cov);
  auto hc = static_cast<T*>(hcv);
  auto hs = static_cast<T*>(hsv);
  int launches = 0;
  if (cgs_use_flat(n, rs.max_blocks, ncols, TILE))
    return cgs_flat<T>(mode, n, V, ldv, ncols, w, ci, co, hc, hs, inv, rs, rs.max_blocks / 4, st);
  if (cgs_use_wide(ncols, TILE))
    return cgs_wide<T>(mode, n, V, ldv, ncols, w, ci, co, hc, hs, inv, rs, grid, st);
  if (ncols <= TILE) {
    if (mode == 0)
      cgs_nc<T, F_PROJ>(n, V, ldv, ncols, w, nullptr, co, nullptr, nullptr, nullptr, rs, grid, st);
    else if (mode == 1)
      cgs_nc<T, F_UPD | F_PROJ>(n, V, ldv, ncols, w, ci, co, hc, nullptr, nullptr, rs, grid, st);
    else
      cgs_nc<T, F_UPD | F_NRM>(n, V, ldv, ncols, w, ci, nullptr, nullptr, hs, inv, rs, grid, st);
    return 1;
  }
  // tiled: updates over all tiles first, then projections / norm
  if (mode != 0) {
    for (int c0 = 0; c0 < ncols; c0 += TILE) {
      const int nct = ncols - c0 < TILE ? ncols - c0 : TILE;
      const bool last = c0 + TILE >= ncols;
      if (mode == 2 && last)
        cgs_nc<T, F_UPD | F_NRM>(n, V + int64_t(c0) * ldv, ldv, nct, w, ci + c0, nullptr, nullptr,
                                 hs, inv, rs, grid, st);
      else
        cgs_nc<T, F_UPD>(n, V + int64_t(c0) * ldv, ldv, nct, w, ci + c0, nullptr, nullptr, nullptr,
                         nullptr, rs, grid, st);
      ++launches;
    }
  }
  if (mode != 2) {
    for (int c0 = 0; c0 < ncols; c0 += TILE) {
      const int nct = ncols - c0 < TILE ? ncols - c0 : TILE;
      cgs_nc<T, F_PROJ>(n, V + int64_t(c0) * ldv, ldv, nct, w, mode == 1 ? ci + c0 : nullptr,
                        co + c0, mode == 1 ? hc + c0 : nullptr, nullptr, nullptr, rs, grid, st,
                        c0);
      ++launches;
    }
  }
  return launches;
}

int launch_cgs(ppf_dtype dt, int mode, int64_t n, const void* V, int64_t ldv, int ncols, void* w,
               const void* coef_in, void* coef_out, void* Hcol, void* Hsub, double* inv,
               RedScratch& rs, int grid, cudaStream_t st) {
  if (dt == PPF_R64)
    return cgs_dispatch<double>(mode, n, V, ldv, ncols, w, coef_in, coef_out, Hcol, Hsub, inv, rs,
                                grid, st);
  return cgs_dispatch<cplx>(mode, n, V, ldv, ncols, w, coef_in, coef_out, Hcol, Hsub, inv, rs,
                            grid, st);
}

void launch_lanczos(ppf_dtype dt, int phase, int64_t n, const void* v, const void* vprev,
                    const double* beta_prev, void* w, void* Hdiag, void* Hsub, void* Hsup,
                    double* inv, RedScratch& rs, int grid, cudaStream_t st) {
  const int blocks = blocks_for(n, 256, grid);
#define PPF_LZ(T)                                                                                \
  if (phase == 1)                                                                                \
    lanczos_kernel<T, 1><<<blocks, 256, 0, st>>>(                                                \
        n, static_cast<const T*>(v), static_cast<const T*>(vprev), beta_prev, static_cast<T*>(w), \
        static_cast<T*>(Hdiag), static_cast<T*>(Hsub), static_cast<T*>(Hsup), inv, rs.partials,  \
        rs.counter, rs.raw);                                                                     \
  else                                                                                           \
    lanczos_kernel<T, 2><<<blocks, 256, 0, st>>>(                                                \
        n, static_cast<const T*>(v), static_cast<const T*>(vprev), beta_prev, static_cast<T*>(w), \
        static_cast<T*>(Hdiag), static_cast<T*>(Hsub), static_cast<T*>(Hsup), inv, rs.partials,  \
        rs.counter, rs.raw);
  if (dt == PPF_R64) {
    PPF_LZ(double)
  } else {
    PPF_LZ(cplx)
  }
#undef PPF_LZ
  post_launch("lanczos_kernel");
}

// ---------------------------------------------------------------------------
// Resident step loop (small operators, round 2).  For an
// operator one CTA can hold (n <= RES_MAX_ROWS, SELL-32), launching ~5 kernels
// and synchronising with the host at every step costs far more than the
// arithmetic (C1: 1024 rows, 9 SpMVs of 5k entries per step took ~62 us).  One
// CTA of 1024 threads runs the steps back to back: the plain SpMV v_j -> U,
// the recorded q(A)q(A) chain (U -> W2, the same epilogues as the graph
// replays), the orthogonalisation (Lanczos or CGS2) writing v_{j+1} and the
// H column -- and after each step stores the H column into a mapped host
// block and bumps a step counter (after __threadfence_system).  The host polls
// the counter, evaluates f(H_m) and the estimate as in the launched path, and
// either lets the device run on (at most RES_AHEAD steps past the last step it
// has decided) or raises `stop`; steps run past the stop are discarded.
// Block-scope coherence: every vector is written and read by this one CTA
// (one SM), so plain loads after __syncthreads() see the writes.
// ---------------------------------------------------------------------------
template <typename T> struct ResCallT {
  const T* x;
  T* out;
  EpiT<T> e;
  int has_x;
};

template <typename T>
__device__ void res_spmv(int64_t n, const int64_t* __restrict__ sptr, const int32_t* __restrict__ col,
                         const T* __restrict__ val, const T* x, T* out, const EpiT<T>& e,
                         bool has_x, const uint16_t* __restrict__ d16,
                         const int32_t* __restrict__ cbase) {
  for (int64_t row = threadIdx.x; row < n; row += blockDim.x) {
    const int64_t base = sptr[row >> 5];
    const int w = int((sptr[(row >> 5) + 1] - base) >> 5);
    const int lane = int(row & 31);
    T acc = s_zero<T>();
    if (d16) {   // 16-bit column deltas (plan encoding), clamped
      const int32_t* cbp = cbase + (base >> 5);
      for (int k = 0; k < w; ++k) {
        const int c = min(max(int(row) + __ldg(cbp + k) + int(__ldg(d16 + base + 32 * k + lane)), 0),
                          int(n - 1));
        acc = s_fma(ldg(val + base + 32 * k + lane), x[c], acc);
      }
    } else {
      for (int k = 0; k < w; ++k)
        acc = s_fma(ldg(val + base + 32 * k + lane), x[__ldg(col + base + 32 * k + lane)], acc);
    }
    T r = s_mul(e.s_ax, acc);
    if (has_x) r = s_fma(e.s_x, e.xe[row], r);
    if (e.z) r = s_fma(e.s_z, e.z[row], r);
    if (e.u) r = s_fma(e.s_u, e.u[row], r);
    out[row] = r;
    if (e.acc) {
      const T b0 = e.acc_init ? s_mul(e.s_acc0, e.xe[row]) : e.acc[row];
      e.acc[row] = s_fma(e.s_acc, r, b0);
    }
  }
}

// block-wide sum of a T (one per thread), fixed order; every thread gets it
template <typename T>
__device__ __forceinline__ T res_block_sum(T v, double* sm) {
  constexpr int ND = n_doubles<T>();
  double* a = reinterpret_cast<double*>(&v);
  T out;
  double* o = reinterpret_cast<double*>(&out);
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    o[d] = block_sum(a[d], sm);
    __syncthreads();
    if (threadIdx.x == 0) sm[32] = o[d];
    __syncthreads();
    o[d] = sm[32];
    __syncthreads();
  }
  return out;
}

template <typename T>
__global__ void __launch_bounds__(1024, 1) resident_steps_kernel(
    int64_t n, const int64_t* __restrict__ sptr, const int32_t* __restrict__ col,
    const T* __restrict__ val, T* V, int64_t ldv, T* U, T* W, T* H, int ldh, int m_max,
    int lanczos, const double* beta0_dev, ResCtl* ctl, const ResCallT<T>* calls_host, int ncalls,
    int ahead, const uint16_t* __restrict__ d16, const int32_t* __restrict__ cbase) {
  constexpr int ND = n_doubles<T>();
  extern __shared__ __align__(16) unsigned char res_smem[];
  ResCallT<T>* calls = reinterpret_cast<ResCallT<T>*>(res_smem);
  T* coef = reinterpret_cast<T*>(res_smem + size_t(ncalls) * sizeof(ResCallT<T>));  // 2 (m_max+1)
  __shared__ double sm[33];
  __shared__ int s_go;
  const int tid = threadIdx.x;
  for (int i = tid; i < ncalls * int(sizeof(ResCallT<T>) / 8); i += blockDim.x)
    reinterpret_cast<uint64_t*>(calls)[i] = reinterpret_cast<const volatile uint64_t*>(calls_host)[i];
  if (tid == 0) ctl->beta0 = *beta0_dev;
  __syncthreads();
  const EpiT<T> plain{s_from<T>(1.0, 0.0), s_zero<T>(), s_zero<T>(), s_zero<T>(), nullptr, nullptr,
                      nullptr, nullptr, s_zero<T>(), s_zero<T>(), false};
  T beta_prev = s_zero<T>();
  double* Hmap = ctl->H;
  for (int j = 0; j < m_max; ++j) {
    if (tid == 0) {
      // soft throttle: wait for the host to catch up to RES_AHEAD steps, but
      // never longer than RES_WAIT_NS -- a host that cannot answer (a tool
      // that serialises the launch, e.g. a profiler replaying the kernel)
      // must not stall the device: it then runs on to m_max, bounded work
      int go = 1;
      uint64_t t0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      for (;;) {
        if (*reinterpret_cast<volatile int*>(&ctl->stop)) {
          go = 0;
          break;
        }
        if (j < *reinterpret_cast<volatile int*>(&ctl->acked) + ahead) break;
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > RES_WAIT_NS) break;
        __nanosleep(500);
      }
      s_go = go;
    }
    __syncthreads();
    if (!s_go) break;
    T* vj = V + int64_t(j) * ldv;
    T* vn = V + int64_t(j + 1) * ldv;
    // u = A v_j, then the chain U -> ... -> W
    res_spmv(n, sptr, col, val, vj, U, plain, false, d16, cbase);
    for (int c = 0; c < ncalls; ++c) {
      __syncthreads();
      const ResCallT<T>& cl = calls[c];
      res_spmv(n, sptr, col, val, cl.x, cl.out, cl.e, cl.has_x != 0, d16, cbase);
    }
    __syncthreads();
    if (lanczos) {
      const T* vp = j > 0 ? V + int64_t(j - 1) * ldv : nullptr;
      T part = s_zero<T>();
      for (int64_t i = tid; i < n; i += blockDim.x) {
        T wi = W[i];
        if (vp) wi = s_sub(wi, s_mul(beta_prev, vp[i]));
        W[i] = wi;
        part = s_cfma(vj[i], wi, part);
      }
      const T alpha = res_block_sum(part, sm);
      double nr = 0.0;
      for (int64_t i = tid; i < n; i += blockDim.x) {
        const T wi = s_sub(W[i], s_mul(alpha, vj[i]));
        W[i] = wi;
        nr += s_abs2(wi);
      }
      const double beta = sqrt(res_block_sum<double>(nr, sm));
      __syncthreads();
      const double inv = 1.0 / beta;
      for (int64_t i = tid; i < n; i += blockDim.x) vn[i] = s_scale(W[i], inv);
      if (tid == 0) {
        H[j + size_t(j) * ldh] = alpha;
        H[j + 1 + size_t(j) * ldh] = s_from<T>(beta, 0.0);
        if (j + 1 < m_max + 1) H[j + size_t(j + 1) * ldh] = s_from<T>(beta, 0.0);
      }
      beta_prev = s_from<T>(beta, 0.0);
    } else {
      // CGS2: h = V^H w; w -= V h; g = V^H w; w -= V g; H(0:j, j) = h + g
      const int nc = j + 1, warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
      for (int pass = 0; pass < 2; ++pass) {
        T* cf = coef + pass * (m_max + 1);
        for (int c = warp; c < nc; c += nw) {
          const T* vc = V + int64_t(c) * ldv;
          T s = s_zero<T>();
          for (int64_t i = lane; i < n; i += 32) s = s_cfma(vc[i], W[i], s);
          double* a = reinterpret_cast<double*>(&s);
#pragma unroll
          for (int d = 0; d < ND; ++d) a[d] = warp_sum(a[d]);
          if (lane == 0) cf[c] = s;
        }
        __syncthreads();
        for (int64_t i = tid; i < n; i += blockDim.x) {
          T s = s_zero<T>();
          for (int c = 0; c < nc; ++c) s = s_fma(V[int64_t(c) * ldv + i], cf[c], s);
          W[i] = s_sub(W[i], s);
        }
        __syncthreads();
      }
      double nr = 0.0;
      for (int64_t i = tid; i < n; i += blockDim.x) nr += s_abs2(W[i]);
      const double beta = sqrt(res_block_sum<double>(nr, sm));
      __syncthreads();
      const double inv = 1.0 / beta;
      for (int64_t i = tid; i < n; i += blockDim.x) vn[i] = s_scale(W[i], inv);
      for (int c = tid; c < nc; c += blockDim.x) H[c + size_t(j) * ldh] = s_add(coef[c], coef[m_max + 1 + c]);
      if (tid == 0) H[j + 1 + size_t(j) * ldh] = s_from<T>(beta, 0.0);
    }
    __syncthreads();
    // column j (rows 0..j+1) to the host, then the step count
    for (int r = tid; r <= j + 1; r += blockDim.x) {
      const double* hv = reinterpret_cast<const double*>(&H[r + size_t(j) * ldh]);
#pragma unroll
      for (int d = 0; d < ND; ++d) Hmap[(size_t(r) + size_t(j) * ldh) * ND + d] = hv[d];
    }
    __threadfence_system();
    __syncthreads();
    if (tid == 0) *reinterpret_cast<volatile int*>(&ctl->done) = j + 1;
  }
}

int resident_max_rows() { return RES_MAX_ROWS; }

// eligible layouts: one rank, SELL-32 without sorting
bool resident_fits(const ppf_mat* A) {
  return A->nranks == 1 && A->fmt == PPF_FMT_SELL && A->C == 32 && A->d_perm == nullptr &&
         A->n_local <= RES_MAX_ROWS;
}

size_t resident_call_bytes(ppf_dtype dt) {
  return dt == PPF_R64 ? sizeof(ResCallT<double>) : sizeof(ResCallT<cplx>);
}

// write the recorded chain (x, out, epilogue per SpMV) into `dst` (host)
void resident_pack_calls(ppf_dtype dt, const std::vector<ResCallSpec>& spec, void* dst) {
  for (size_t i = 0; i < spec.size(); ++i) {
    if (dt == PPF_R64) {
      ResCallT<double> c;
      std::memset(&c, 0, sizeof(c));
      c.x = static_cast<const double*>(spec[i].x);
      c.out = static_cast<double*>(spec[i].out);
      c.e = to_epi<double>(spec[i].e, spec[i].x);
      c.has_x = (spec[i].e.s_x[0] != 0.0 || spec[i].e.s_x[1] != 0.0) ? 1 : 0;
      std::memcpy(static_cast<char*>(dst) + i * sizeof(c), &c, sizeof(c));
    } else {
      ResCallT<cplx> c;
      std::memset(&c, 0, sizeof(c));
      c.x = static_cast<const cplx*>(spec[i].x);
      c.out = static_cast<cplx*>(spec[i].out);
      c.e = to_epi<cplx>(spec[i].e, spec[i].x);
      c.has_x = (spec[i].e.s_x[0] != 0.0 || spec[i].e.s_x[1] != 0.0) ? 1 : 0;
      std::memcpy(static_cast<char*>(dst) + i * sizeof(c), &c, sizeof(c));
    }
  }
}

void launch_resident(ppf_mat* A, void* V, int64_t ldv, void* U, void* W, void* H, int ldh,
                     int m_max, int lanczos, const double* beta0_dev, ResCtl* ctl_dev,
                     const void* calls_dev, int ncalls, int ahead, cudaStream_t st) {
  const size_t cb = resident_call_bytes(A->dtype);
  const size_t sc = A->dtype == PPF_R64 ? 8 : 16;
  const size_t smem = size_t(ncalls) * cb + 2 * size_t(m_max + 1) * sc;
#define PPF_RES(T)                                                                              \
  {                                                                                             \
    auto kfn = resident_steps_kernel<T>;                                                        \
    if (smem > 48 * 1024)                                                                       \
      cuda_check(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                      int(smem)), "cudaFuncSetAttribute(resident)");           \
    kfn<<<1, 1024, smem, st>>>(A->n_local, A->d_ptr, A->d_col, static_cast<const T*>(A->d_val), \
                               static_cast<T*>(V), ldv, static_cast<T*>(U), static_cast<T*>(W), \
                               static_cast<T*>(H), ldh, m_max, lanczos, beta0_dev, ctl_dev,     \
                               static_cast<const ResCallT<T>*>(calls_dev), ncalls, ahead,       \
                               A->d_d16, A->d_cb);                                              \
  }
  if (A->dtype == PPF_R64)
    PPF_RES(double)
  else
    PPF_RES(cplx)
#undef PPF_RES
  post_launch("resident_steps_kernel");
}

// a kernel of this translation unit (its module is force-loaded by peer.cu)
const void* kernels_module_symbol() { return reinterpret_cast<const void*>(&finalize_kernel); }

}  // namespace ppf
