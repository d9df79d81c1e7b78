// blr_pad.cu — the fused pad-grid engine for every truncated convolution on
// the hot path (transport.py:206-303, deformation.py:63-72).  No cuFFT and no
// zero-padded grids: a right-hand side is a chain of batched 1-D transforms
// with the data movement fused in,
//
//   k_xinv    band H [kz][kx][ky] -> inverse x FFT (x derivative multiplier,
//             zero padding fused) -> I [f][kz][ky][x]
//   k_yinv    -> inverse y FFT (y / z multipliers, sums of terms fused)
//             -> S [f][kz][x][y]        (only kz = 0..K: Hermitian half)
//   k_lines   per z-line: C2R (two real lines per complex FFT), the RHS
//             pointwise product streamed into per-output accumulators (reading
//             cached real pad fields), R2C back to S (kz = 0..K)
//   k_yfwd    forward y FFT, band ky kept -> I
//   k_xfwd    forward x FFT, band kx kept, post-transform multipliers (flux
//             divergence), 1/P^3, -(v + .) / negation, fused RK4 stage update
//
// Band state lives in the "H layout" [comp][kz 0..K][kx][ky] (Hermitian half);
// node records are converted back to the reference's full blocks.
#pragma once

#include "blr_fft.cuh"
#include "blr_internal.cuh"

#include <cuda.h>  // CUtensorMap (the encoder is reached through the runtime's driver entry point)
#include <cuda_pipeline_primitives.h>

#include <cmath>
#include <array>
#include <map>
#include <mutex>
#include <cstring>
#include <utility>
#include <type_traits>

namespace blr {

// ---------------------------------------------------------------------------
// geometry
// ---------------------------------------------------------------------------
struct PadGeom {
  int P[3], K[3], B[3];
  int Kz1;       // K[2] + 1
  int64_t nh;    // H-layout component size Kz1*B0*B1
  int64_t ns;    // S-layout field size Kz1*P0*P1
  int64_t n1;    // I-layout field size Kz1*B1*P0
  int64_t np;    // real pad field size
};

constexpr int kWarps = 8;  // warps per CTA in the x / y pass kernels
constexpr int kPassMinBlocks = 1;  // occupancy hint for the pass kernels (4 tried: no gain, spills)

__device__ __forceinline__ int bin_to_index(int p, int P, int K, int B) {
  if (p <= K) return p;
  if (p >= P - K) return p - P + B;
  return -1;
}

// the split twiddle table (2 L entries, blr_fft.cuh twiddle()) into shared memory
template <typename T>
__device__ __forceinline__ void load_tw(T* dst, const double* src, int L) {
  for (int i = threadIdx.x; i < 2 * L; i += blockDim.x) dst[i] = (T)src[i];
}
// The same as cp.async copies in the caller's open cp.async group (no register
// round trip; the caller commits and waits): fp64 16-byte copies of the table,
// fp32 8-byte copies of the fp32 table stored after it (blr_pad.cu engine
// set-up).  Threads `first`, `first + stride`, ... issue.  Used before
// griddepcontrol.wait (A/B r02: y-inverse 1.49 -> 1.45 ms per HVP).
#ifndef BLR_TW_ASYNC
#define BLR_TW_ASYNC 1
#endif
template <typename T>
__device__ __forceinline__ void copy_tw_async(T* dst, const double* src, int L, int first, int stride) {
  if constexpr (sizeof(T) == 8) {
    for (int i = first; i < L; i += stride) __pipeline_memcpy_async(dst + 2 * i, src + 2 * i, 16);
  } else {
    const float* f = reinterpret_cast<const float*>(src + 2 * L);
    for (int i = first; i < L; i += stride) __pipeline_memcpy_async(dst + 2 * i, f + 2 * i, 8);
  }
}
template <typename T>
__device__ __forceinline__ bool load_tw_async(T* dst, const double* src, int L) {
  if constexpr (BLR_TW_ASYNC) {
    copy_tw_async<T>(dst, src, L, threadIdx.x, blockDim.x);
    return true;
  } else {
    load_tw<T>(dst, src, L);
    return false;
  }
}

template <typename T>
__device__ __forceinline__ Cx<T> mul_ik(Cx<T> z, T k) { return cx<T>(-(k * z.y), k * z.x); }

// n / d for 0 <= n < 2^23 and a divisor fixed per kernel: a float reciprocal
// estimate (off by at most one) and one correction, instead of the ~20-
// instruction integer division sequence (the persistent passes divide item
// indices several times per item).  BLR_FDIV=0: plain division.
#ifndef BLR_FDIV
#define BLR_FDIV 1
#endif
struct FDiv {
  int d;
  float r;
  __device__ __forceinline__ explicit FDiv(int dd) : d(dd), r(1.0f / (float)dd) {}
  __device__ __forceinline__ int operator()(int n) const {
    if constexpr (!BLR_FDIV) return n / d;
    int q = __float2int_rz((float)n * r);
    const int rem = n - q * d;
    q += (rem >= d) - (rem < 0);
    return q;
  }
};

// ---------------------------------------------------------------------------
// inverse x pass: band H [kz][kx][ky] -> I [xf][kz][ky][x]
// ---------------------------------------------------------------------------
constexpr int kMaxX = 40;
constexpr int kMaxY = 32;

template <typename T>
struct XPassArgs {
  const Cx<T>* src[kMaxX];
  int mulx[kMaxX];
  int nx;
  Cx<T>* out;
  int fidx[kMaxX];  // TMA: field index of src[xf] in the tensor map (set by launch_xinv)
};

template <typename T>
__device__ __forceinline__ void cp_async(Cx<T>* dst, const Cx<T>* src) {
  __pipeline_memcpy_async(dst, src, sizeof(Cx<T>));
}

// --- programmatic dependent launch ------------------------------------------
// Every engine kernel is launched with programmatic stream serialization and
// executes griddepcontrol.wait -- predecessor complete, its memory visible --
// before the first access to dependent global data; constant tables, barriers
// and index set-up run before it.  No kernel triggers early
// (launch_dependents at entry was measured slower: waiting CTAs of the next
// kernel then hold SM resources through the predecessor's tail); the implicit
// trigger at grid exit still removes the launch gap between kernels
// (-1.1 ms per deformation GN HVP, the same as replaying a CUDA graph).
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
#ifndef BLR_XFWD_PF
#define BLR_XFWD_PF 1
#endif
constexpr bool kXfwdPrefetch = BLR_XFWD_PF != 0;
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BLR_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// --- bulk-copy (TMA engine) staging --------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* bar, uint32_t bytes) {  // no arrive
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// one TMA tile load of a rank-4 tensor map into shared memory, completing on bar
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Inverse passes: the twiddle table lands by one cp.async.bulk on an mbarrier,
// requested before griddepcontrol.wait (expect_tx without arrive); after the
// slab's per-element cp.async copies are issued, thread 0 arrives and every
// thread waits on the barrier (table) and its cp.async group (slab).  A/B r02:
// deformation / state / fp32 GN HVP 8.64 / 4.90 / 6.07 -> 8.61 / 4.88 / 6.02
// ms.  (Bulk copies for the slab rows too -- 12 lines x 16 B per row -- made
// the fp64 y-inverse 1.38 -> 1.64 ms.)
#ifndef BLR_INV_BULK
#define BLR_INV_BULK 1
#endif
template <typename T, int L>
constexpr bool inv_bulk_tw() { return BLR_INV_BULK && (2 * L * (int)sizeof(T)) % 16 == 0; }
template <typename T, int L>
__device__ __forceinline__ void inv_bulk_start(uint64_t* bar, T* tw, const double* twg) {
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t nb = 2 * L * sizeof(T);
    mbar_expect_tx_only(bar, nb);
    bulk_g2s(tw, sizeof(T) == 8 ? (const void*)twg : (const void*)(twg + 2 * L), nb, bar);
  }
}

// Double-buffered slab staging for the persistent pass kernels.  fp64 rows are
// whole 16-byte multiples: warp 0 arms the buffer's mbarrier with the byte
// count and issues one cp.async.bulk per row (the copy engine writes the
// padded smem rows; no per-element instructions); every thread then waits on
// the mbarrier parity.  fp32 rows may be 8-byte aligned only: per-element
// cp.async with commit / wait_group and a CTA barrier.
template <typename T, bool BULK = sizeof(T) == 8>
struct Stager {
  static constexpr bool kBulk = BULK;
  uint64_t* bar;  // [2] in shared memory
  uint32_t phase;
  __device__ __forceinline__ void init(uint64_t* b) {
    bar = b;
    phase = 0;
    if (kBulk && threadIdx.x == 0) {
      mbar_init(bar, 1);
      mbar_init(bar + 1, 1);
      fence_mbar_init();
    }
  }
  // start a load into buffer b of `bytes` in total (bulk: arm the mbarrier
  // before warp 0 issues any copy of it)
  __device__ __forceinline__ void begin(int b, uint32_t bytes) {
    if constexpr (kBulk) {
      if (threadIdx.x < 32) {
        if (threadIdx.x == 0) mbar_expect_tx(bar + b, bytes);
        __syncwarp();
      }
    }
  }
  // nrows rows of ncols elements: global row stride gs, shared row stride ss
  __device__ __forceinline__ void rows(Cx<T>* dst, int ss, const Cx<T>* src, int64_t gs, int nrows, int ncols, int b) {
    if constexpr (kBulk) {
      if (threadIdx.x < 32)
        for (int r = threadIdx.x; r < nrows; r += 32)
          bulk_g2s(dst + r * ss, src + r * gs, (uint32_t)(ncols * sizeof(Cx<T>)), bar + b);
    } else {
      for (int i = threadIdx.x; i < nrows * ncols; i += blockDim.x) {
        const int r = i / ncols, c = i - (i / ncols) * ncols;
        cp_async<T>(dst + r * ss + c, src + r * gs + c);
      }
    }
  }
  __device__ __forceinline__ void commit() {
    if constexpr (!kBulk) __pipeline_commit();
  }
  // wait for buffer b (the other buffer's load may stay in flight)
  __device__ __forceinline__ void wait(int b) {
    if constexpr (kBulk) {
      mbar_wait(bar + b, (phase >> b) & 1u);
      phase ^= 1u << b;
    } else {
      __pipeline_wait_prior(1);
      __syncthreads();
    }
  }
};

// Staged pass kernels: inv_pw<T>() warps per CTA; the CTA's whole input slab is
// copied to shared memory with coalesced cp.async first, then every warp runs
// its four-step FFTs from shared memory.
// warps per CTA of the inverse passes: fp64 2, fp32 4 (A/B r02 with TMA-staged
// slabs: fp64 deformation / state 8.45 / 4.73 -> 8.38 / 4.67 ms at 2 warps,
// 8.82 / 4.92 at 8; fp32 5.85 -> 5.88 at 2); BLR_KPW=n forces n
#ifndef BLR_KPW
#define BLR_KPW 0
#endif
template <typename T>
constexpr int inv_pw() { return BLR_KPW ? BLR_KPW : (sizeof(T) == 8 ? 2 : 4); }
constexpr int kPWF = 2;  // forward passes (y, x): measured best at 2 warps per CTA

// Shared-memory strides chosen so the FFT access patterns are free of bank
// conflicts.  Transposed tiles [row][LPC] are read by lanes walking rows, so
// their row stride is made odd.  Line slabs [line][L] are read by step-A lanes
// (line, n2) at line*LS + n2 + const; LS = L + pad with the smallest pad whose
// worst 128-byte phase maps no two lanes onto one bank.
template <int LPC>
constexpr int t_stride() { return LPC | 1; }

template <class S>
constexpr int phase_conflicts(int LS, int words) {
  const int per_phase = 32 / words;  // lanes served per 128-byte wavefront
  int worst = 0;
  for (int p0 = 0; p0 < 32; p0 += per_phase) {
    int cnt[32] = {};
    for (int lane = p0; lane < p0 + per_phase; ++lane) {
      const int line = lane / S::R2, n2 = lane % S::R2;
      if (line >= S::LPW) continue;
      const int w0 = (line * LS + n2) * words;
      for (int w = 0; w < words; ++w) ++cnt[(w0 + w) % 32];
    }
    for (int b = 0; b < 32; ++b) worst = cnt[b] > worst ? cnt[b] : worst;
  }
  return worst;
}

// ALIAS: the slab must also hold the warp's FFT tile over its own lines
// (LS >= TS), which drops the separate per-warp tiles.  A16: rows must start
// 16-byte aligned (bulk copies of fp32 rows).
template <typename T, class S, bool ALIAS = false, bool A16 = false>
constexpr int row_stride() {
  constexpr int words = (int)(sizeof(Cx<T>) / 4);
  const int base = ALIAS && TileG<T, S>::TS > S::L ? TileG<T, S>::TS : S::L;
  int best = -1, bc = 1 << 30;
  for (int p = 0; p < 8; ++p) {
    if (A16 && ((base + p) * (int)sizeof(Cx<T>)) % 16 != 0) continue;
    const int c = phase_conflicts<S>(base + p, words);
    if (c < bc) { bc = c; best = base + p; }
  }
  return best;
}

// forward passes: rows are staged with bulk copies whenever a row is a whole
// number of 16-byte units (always in fp64; fp32 with even L), else per-element
// cp.async (fp32, odd L)
#ifndef BLR_F32_BULK
#define BLR_F32_BULK 1
#endif
template <typename T, class S>
constexpr bool fwd_bulk_rows() {
  return sizeof(T) == 8 || (BLR_F32_BULK && (S::L * (int)sizeof(Cx<T>)) % 16 == 0);
}
template <typename T, class S>
constexpr int fwd_row_stride() { return row_stride<T, S, true, sizeof(T) == 4 && fwd_bulk_rows<T, S>()>(); }

// TMA (as k_yinv): the slab is one tensor-tile load, box 2 LPC x B0 of the H
// fields viewed as [field][kz][kx][2 ky]
template <typename T, class S, bool TMA = false>
__global__ void __launch_bounds__(inv_pw<T>() * 32) k_xinv(XPassArgs<T> a, PadGeom g, const double* __restrict__ twg,
                                                  const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int LPC = inv_pw<T>() * S::LPW;
  const int K0 = g.K[0], B0 = g.B[0], B1 = g.B[1];
  T* tw = (T*)smem_raw;
  constexpr int LPCS = TMA ? LPC : t_stride<LPC>();
  const uint32_t s0 = smem_u32(smem_raw);
  const size_t slab_off = TMA ? (((s0 + 2 * S::L * sizeof(T) + 127) & ~127u) - s0) : 2 * S::L * sizeof(T);
  Cx<T>* slab = (Cx<T>*)(smem_raw + slab_off);   // [B0][LPCS]
  Cx<T>* tile = slab + B0 * LPCS + (threadIdx.x >> 5) * TileG<T, S>::TILE;
  const int nyb = (B1 + LPC - 1) / LPC;
  const int per = g.Kz1 * nyb;
  const int xf = blockIdx.x / per;
  const int r = blockIdx.x - xf * per;
  const int kz = r / nyb;
  const int cky0 = (r - kz * nyb) * LPC;
  const int nlc = min(LPC, B1 - cky0);
  const Cx<T>* src = a.src[xf] + ((int64_t)kz * B0) * B1 + cky0;
  constexpr bool kBulkTw = TMA || inv_bulk_tw<T, S::L>();
  __shared__ uint64_t bar;
  if constexpr (kBulkTw) inv_bulk_start<T, S::L>(&bar, tw, twg);
  else load_tw_async<T>(tw, twg, S::L);  // constant table: overlaps the predecessor's tail
  pdl_wait();
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      mbar_expect_tx(&bar, (uint32_t)(B0 * 2 * LPC * sizeof(T)));
      tma_load_4d(slab, &tmap, 2 * cky0, 0, kz, a.fidx[xf], &bar);
    }
    mbar_wait(&bar, 0);
  } else {
    for (int i = threadIdx.x; i < B0 * LPC; i += blockDim.x) {
      const int ix = i / LPC, l = i - ix * LPC;
      if (l < nlc) cp_async<T>(slab + ix * LPCS + l, src + ix * B1 + l);
      BLR_CHECK(l >= nlc || (int64_t)kz * B0 * B1 + cky0 + ix * B1 + l < g.nh, "xinv src");
    }
    __pipeline_commit();
    if constexpr (kBulkTw) {
      if (threadIdx.x == 0) mbar_arrive(&bar);  // the table's bytes complete the phase
      mbar_wait(&bar, 0);
    }
    __pipeline_wait_prior(0);
    __syncthreads();
  }
  const int wl0 = (threadIdx.x >> 5) * S::LPW;
  const int nl = min(S::LPW, nlc - wl0);
  if (nl <= 0) return;
  const bool mulx = a.mulx[xf] != 0;
  Cx<T>* out = a.out + xf * g.n1 + ((int64_t)kz * B1 + cky0 + wl0) * S::L;
  const Cx<T>* sl = slab + wl0;
  auto store = [&](int line, int x, int, Cx<T> v) {
    BLR_CHECK(((int64_t)kz * B1 + cky0 + wl0 + line) * S::L + x < g.n1, "xinv out");
    out[line * S::L + x] = v;
  };
  // (a per-lane gather table of band offsets / wavenumbers built once per CTA
  // measured neutral, A/B r02)
  if (mulx) {  // uniform per CTA: two gathers instead of a per-element branch
    auto load = [&](int line, int p, int) -> Cx<T> {
      const int ix = bin_to_index(p, S::L, K0, B0);
      const int ixc = ix >= 0 ? ix : 0;
      const Cx<T> z = mul_ik<T>(sl[ixc * LPCS + line], (T)(kTwoPi * (double)freq_of(ixc, K0, B0)));
      return ix >= 0 ? z : cx<T>(0, 0);
    };
    wfft<T, S, true>(tile, tw, nl, load, store);
  } else {
    auto load = [&](int line, int p, int) -> Cx<T> {
      const int ix = bin_to_index(p, S::L, K0, B0);
      const Cx<T> z = sl[(ix >= 0 ? ix : 0) * LPCS + line];
      return ix >= 0 ? z : cx<T>(0, 0);
    };
    wfft<T, S, true>(tile, tw, nl, load, store);
  }
}

// ---------------------------------------------------------------------------
// inverse y pass: I [xf][kz][ky][x] -> S [yf][kz][x][y]
// ---------------------------------------------------------------------------
template <typename T>
struct YPassArgs {
  int xf[kMaxY][3];
  int axis[kMaxY][3];  // pre-multiplier: -1, 1 (i ky), 2 (i kz)
  int nterms[kMaxY];
  int ny;
  const Cx<T>* in;
  Cx<T>* out;
};

// TMA: the slab of every term is one tensor-tile load (box 2 LPC x B1 of the
// I fields viewed as a rank-4 tensor [field][kz][ky][2 x]) on the mbarrier,
// dense rows (stride LPC) at a 128-byte aligned slab; out-of-range lines of
// the last chunk are zero-filled by the copy engine.
template <typename T, class S, bool TMA = false>
__global__ void __launch_bounds__(inv_pw<T>() * 32) k_yinv(YPassArgs<T> a, PadGeom g, const double* __restrict__ twg, int ntmax,
                                                  const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int LPC = inv_pw<T>() * S::LPW;
  const int P0 = g.P[0], K1 = g.K[1], B1 = g.B[1];
  T* tw = (T*)smem_raw;
  constexpr int LPCS = TMA ? LPC : t_stride<LPC>();
  // TMA destinations 128-byte aligned in the shared window (the dynamic
  // segment itself is only guaranteed 16-byte alignment)
  const uint32_t s0 = smem_u32(smem_raw);
  const size_t slab_off = TMA ? (((s0 + 2 * S::L * sizeof(T) + 127) & ~127u) - s0) : 2 * S::L * sizeof(T);
  Cx<T>* slab = (Cx<T>*)(smem_raw + slab_off);   // [ntmax][B1t][LPCS]
  // TMA: each term's slab starts 128-byte aligned (rows padded to B1t)
  constexpr int kRowAlign = TMA ? 128 / cgcd(128, LPC * (int)sizeof(Cx<T>)) : 1;
  const int B1t = ((B1 + kRowAlign - 1) / kRowAlign) * kRowAlign;
  Cx<T>* tile = slab + ntmax * B1t * LPCS + (threadIdx.x >> 5) * TileG<T, S>::TILE;
  const int nxb = (P0 + LPC - 1) / LPC;
  const int per = g.Kz1 * nxb;
  const int yf = blockIdx.x / per;
  const int r = blockIdx.x - yf * per;
  const int kz = r / nxb;
  const int cx0 = (r - kz * nxb) * LPC;
  const int nlc = min(LPC, P0 - cx0);
  const int nt = a.nterms[yf];
  constexpr bool kBulkTw = TMA || inv_bulk_tw<T, S::L>();
  __shared__ uint64_t bar;
  if constexpr (kBulkTw) inv_bulk_start<T, S::L>(&bar, tw, twg);
  else load_tw_async<T>(tw, twg, S::L);  // constant table: overlaps the predecessor's tail
  pdl_wait();
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      mbar_expect_tx(&bar, (uint32_t)(nt * B1 * 2 * LPC * sizeof(T)));
      for (int t = 0; t < nt; ++t) tma_load_4d(slab + t * B1t * LPC, &tmap, 2 * cx0, 0, kz, a.xf[yf][t], &bar);
    }
    mbar_wait(&bar, 0);
  } else {
    for (int t = 0; t < nt; ++t) {
      const Cx<T>* src = a.in + a.xf[yf][t] * g.n1 + (int64_t)kz * B1 * P0 + cx0;
      Cx<T>* dst = slab + t * B1t * LPCS;
      for (int i = threadIdx.x; i < B1 * LPC; i += blockDim.x) {
        const int iy = i / LPC, l = i - iy * LPC;
        if (l < nlc) cp_async<T>(dst + iy * LPCS + l, src + iy * P0 + l);
        BLR_CHECK(l >= nlc || (int64_t)kz * B1 * P0 + cx0 + iy * P0 + l < g.n1, "yinv src");
      }
    }
    __pipeline_commit();
    if constexpr (kBulkTw) {
      if (threadIdx.x == 0) mbar_arrive(&bar);  // the table's bytes complete the phase
      mbar_wait(&bar, 0);
    }
    __pipeline_wait_prior(0);
    __syncthreads();
  }
  const int wl0 = (threadIdx.x >> 5) * S::LPW;
  const int nl = min(S::LPW, nlc - wl0);
  if (nl <= 0) return;
  int ax[3];
  for (int t = 0; t < 3; ++t) ax[t] = t < nt ? a.axis[yf][t] : -2;
  const T kzk = (T)(kTwoPi * (double)kz);
  Cx<T>* out = a.out + yf * g.ns + ((int64_t)kz * P0 + cx0 + wl0) * S::L;
  auto load = [&](int line, int q, int) -> Cx<T> {
    const int iy = bin_to_index(q, S::L, K1, B1);
    const bool ok = iy >= 0;
    const int iyc = ok ? iy : 0;
    const T ky = (T)(kTwoPi * (double)freq_of(iyc, K1, B1));
    Cx<T> acc = cx<T>(0, 0);
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      if (ax[t] < -1) break;
      Cx<T> z = slab[(t * B1t + iyc) * LPCS + wl0 + line];
      if (ax[t] >= 1) z = mul_ik<T>(z, ax[t] == 1 ? ky : kzk);
      acc = cadd(acc, z);
    }
    return ok ? acc : cx<T>(0, 0);
  };
  auto store = [&](int line, int y, int, Cx<T> v) {
    BLR_CHECK(((int64_t)kz * P0 + cx0 + wl0 + line) * S::L + y < g.ns, "yinv out");
    out[line * S::L + y] = v;
  };
  if (nt == 1) {
    // single-term output (the common case): no term loop in the gather
    const int ax0 = ax[0];
    const Cx<T>* sl = slab + wl0;
    auto load1 = [&](int line, int q, int) -> Cx<T> {
      const int iy = bin_to_index(q, S::L, K1, B1);
      const int iyc = iy >= 0 ? iy : 0;
      Cx<T> z = sl[iyc * LPCS + line];
      if (ax0 >= 1) z = mul_ik<T>(z, ax0 == 1 ? (T)(kTwoPi * (double)freq_of(iyc, K1, B1)) : kzk);
      return iy >= 0 ? z : cx<T>(0, 0);
    };
    wfft<T, S, true>(tile, tw, nl, load1, store);
  } else {
    wfft<T, S, true>(tile, tw, nl, load, store);
  }
}

// ---------------------------------------------------------------------------
// z lines: C2R of the spectral inputs (two per complex FFT), streaming
// pointwise products into per-output accumulators, R2C of the outputs
// ---------------------------------------------------------------------------
enum LineOp {
  kOpRealize = 0,   // write realized inputs (wout) only
  kOpMap = 1,       // out_i = sum_j S[ij] V_j                 (+ wout cache of S)
  kOpMapTC = 2,     // out_i = sum_j S[ij] V_j + sum_j Du_ij dV_j   (Du, V, dV real)
  kOpMapTF = 3,     // out = [Du.V | dDu.V + Du.dV]            (Du, dDu spectral)
  kOpInvVol = 4,    // out = [Dw.V | -V.G - J Dv]
  kOpBwdVol = 5,    // out = [Dw.V | dDw.V + Dw.dV | vol | vol tangent]
  kOpOuter = 6,     // out_ij = rho_i V_j
  kOpOuterPair = 7, // out = [rho x V | drho x V + rho x dV]
  kOpContract = 8,  // out_i = sum_n w_n sum_j M_n(ji|ij) rho_n,j   (M real, cached)
};

constexpr int kMaxLineS = 28;
constexpr int kMaxLineR = 16;
constexpr int kMaxLineO = 18;

template <typename T>
struct LineArgs {
  const Cx<T>* sin[kMaxLineS];
  const T* rin[kMaxLineR];
  Cx<T>* sout[kMaxLineO];
  T* wout[kMaxLineS];
  int op;
  int ns, nr, no;
  int d;
  int n_nodes;
  int64_t sin_node_stride;  // complex entries between nodes (per input field)
  int64_t rin_node_stride;  // real entries between nodes
  double w[32];
  int transpose;
  // ACC-op tables (host-built): output index, real-input index and sign per field
  int oi[kMaxLineS], ri[kMaxLineS];  // ri: staged-slot index for ACC ops
  double sg[kMaxLineS];
  int nst;                           // real fields staged in shared memory (ACC ops)
  int st_idx[4];                     // their rin indices
  int mi[3][3];  // contraction: rin index of M(o, j)
};

// Per-op compile-time traits of the z-line kernel.
//   ACC ops: every realized spectral input adds sign * s * R[ri] to output
//            oi (or, for the contraction, d terms); outputs live in registers.
//   REAL ops: realized inputs are kept in shared memory and the outputs are
//            formed on the fly while loading the R2C.
template <int OP> struct ZOp {
  static constexpr bool acc = OP == kOpMap || OP == kOpMapTC || OP == kOpInvVol || OP == kOpContract;
  static constexpr int nomax = OP == kOpInvVol ? 4 : 3;
};

constexpr int kZWarps = 2;
#ifndef BLR_ZOUT_PRED
#define BLR_ZOUT_PRED 1
#endif
#ifndef BLR_ZTW_ASYNC
#define BLR_ZTW_ASYNC 1
#endif
// Occupancy targets (CTAs per SM) of the z-line kernel per op; 0 = registers
// unconstrained.  The outer op is held at 6 CTAs per SM (its shared-memory
// limit with the unrolled outer products).
#ifndef BLR_ZMINB_OUTER
#define BLR_ZMINB_OUTER 6
#endif
#ifndef BLR_ZMINB_MAPTC
#define BLR_ZMINB_MAPTC 0
#endif
constexpr int zline_min_blocks(int op) {
  return op == 6 ? BLR_ZMINB_OUTER : op == 2 ? BLR_ZMINB_MAPTC : 0;
}

// z-line shared buffers, line strides chosen by the bank model (blr_fft.cuh):
//   xbuf [line][LX] complex: step-B stores / step-A loads of the R2C inputs;
//   Vst / Rsm [field][line][LR] real: read at step-B (and, for the unrolled
//   outer op, step-A) positions.  L = 100 fp64: LX = LR = 106 makes both
//   access patterns conflict-free (the dense stride 100 cost 1.5x / 2x);
//   used only with BLR_BANKPAD=1 (see TileG).
template <typename T, class S>
struct ZLineG {
  static constexpr int L = S::L;
  static constexpr int EC = (int)(2 * sizeof(T)), ER = (int)sizeof(T);
  static constexpr int xcost(int lx) {
    int c = 0;
    for (int k2 = 0; k2 < S::R2; ++k2)
      c += wavefronts([&](int l) { return l / S::R1 < S::LPW ? (l / S::R1) * lx + l % S::R1 + S::R1 * k2 : -1; }, EC);
    for (int n1 = 0; n1 < S::R1; ++n1)
      c += wavefronts([&](int l) { return l / S::R2 < S::LPW ? (l / S::R2) * lx + S::R2 * n1 + l % S::R2 : -1; }, EC);
    return c;
  }
  static constexpr int rcost(int lr) {
    int c = 0;
    for (int k2 = 0; k2 < S::R2; ++k2)
      c += wavefronts([&](int l) { return l / S::R1 < S::LPW ? (l / S::R1) * lr + l % S::R1 + S::R1 * k2 : -1; }, ER);
    for (int n1 = 0; n1 < S::R1; ++n1)
      c += wavefronts([&](int l) { return l / S::R2 < S::LPW ? (l / S::R2) * lr + S::R2 * n1 + l % S::R2 : -1; }, ER);
    return c;
  }
  static constexpr int pick(bool real) {
    if (!bank_pad<T>()) return L;
    int best = L, bc = 1 << 30;
    for (int p = 0; p < 8; ++p) {
      const int c = real ? rcost(L + p) : xcost(L + p);
      if (c < bc) { bc = c; best = L + p; }
    }
    return best;
  }
  static constexpr int LX = pick(false);
  static constexpr int LR = pick(true);
};

template <typename T, class S, int OP>
__device__ __forceinline__ T z_output(const LineArgs<T>& a, const T* Rsm, int ldR, int li, int64_t gi, int o) {
  const int d = a.d, dd = d * d;
  auto Rr = [&](int q) { return __ldg(a.rin[q] + gi); };
  auto Sm = [&](int f) { return Rsm[f * ldR + li]; };
  if constexpr (OP == kOpOuter) {
    const int i = o / d, j = o - i * d;
    return Sm(i) * Rr(j);
  } else if constexpr (OP == kOpOuterPair) {
    if (o < dd) {
      const int i = o / d, j = o - i * d;
      return Sm(i) * Rr(j);
    }
    const int q = o - dd, i = q / d, j = q - i * d;
    return Sm(d + i) * Rr(j) + Sm(i) * Rr(d + j);
  } else if constexpr (OP == kOpMapTF) {
    if (o < d) {
      T b = 0;
      for (int j = 0; j < d; ++j) b += Sm(o * d + j) * Rr(j);
      return b;
    }
    const int i = o - d;
    T a1 = 0, a2 = 0;
    for (int j = 0; j < d; ++j) a1 += Sm(dd + i * d + j) * Rr(j);
    for (int j = 0; j < d; ++j) a2 += Sm(i * d + j) * Rr(d + j);
    return a1 + a2;
  } else if constexpr (OP == kOpBwdVol) {
    // S: Dw [0,dd) dDw [dd,2dd) G [2dd,+d) dG [2dd+d,+d) J dJ ; R: V, dV, Dv, dDv
    if (o < d) {
      T b = 0;
      for (int j = 0; j < d; ++j) b += Sm(o * d + j) * Rr(j);
      return b;
    }
    if (o < 2 * d) {
      const int i = o - d;
      T a1 = 0, a2 = 0;
      for (int j = 0; j < d; ++j) a1 += Sm(dd + i * d + j) * Rr(j);
      for (int j = 0; j < d; ++j) a2 += Sm(i * d + j) * Rr(d + j);
      return a1 + a2;
    }
    const int g0 = 2 * dd, dg0 = 2 * dd + d, jj = 2 * dd + 2 * d;
    if (o == 2 * d) {
      T s = 0;
      for (int q = 0; q < d; ++q) s += Rr(q) * Sm(g0 + q);
      return -s - Sm(jj) * Rr(2 * d);
    }
    T s1 = 0, s2 = 0;
    for (int q = 0; q < d; ++q) s1 += Rr(d + q) * Sm(g0 + q);
    for (int q = 0; q < d; ++q) s2 += Rr(q) * Sm(dg0 + q);
    return -s1 - s2 - Sm(jj + 1) * Rr(2 * d) - Sm(jj) * Rr(2 * d + 1);
  }
  return 0;
}

// z lines: per warp LPW lines (x fixed, consecutive y).  Spectral inputs are
// prefetched pair by pair with cp.async (double buffered), C2R'd two per
// complex FFT, combined with the cached real pad fields, R2C'd back.
template <typename T, class S, int OP>
__global__ void __launch_bounds__(kZWarps * 32, zline_min_blocks(OP)) k_zlines(LineArgs<T> a, PadGeom g, const double* __restrict__ twz_g) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using Tr = ZOp<OP>;
  constexpr int L = S::L;
  constexpr int NOM = Tr::nomax;
  const int P0 = g.P[0], P1 = g.P[1], K2 = g.K[2], Kz1 = g.Kz1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int LPC = kZWarps * S::LPW;
  const int nyc = (P1 + LPC - 1) / LPC;
  const int x = blockIdx.x / nyc;
  const int y0 = (blockIdx.x - x * nyc) * LPC + warp * S::LPW;
  const int ns_blk = OP == kOpContract ? a.d : a.ns;
  // real fields kept in shared memory: REAL ops' realized inputs; the
  // contraction's realized rho_n (d fields, refilled per node)
  const int nreal = OP == kOpContract ? a.d : (Tr::acc || OP == kOpRealize) ? 0 : ns_blk;
  // shared layout: tw | per warp { tile | stage[max(2*2*Kz1*LPW, LPW*L)] (xbuf aliases it after the
  //                                 C2R phase) | Vst[nst][LPW*L] | Rsm[nreal][LPW*L] }
  // (one shared zero row after the four field regions serves the out-of-band
  // rows of the Hermitian gather; per-field zero rows cost the outer op a CTA
  // per SM, A/B r02 2.14 -> 2.31 ms)
  const int fstride = Kz1 * S::LPW;  // per-field stage: Kz1 spectra rows
  const int zoff = 4 * fstride;      // the shared zero row
  using ZG = ZLineG<T, S>;
  constexpr int LX = ZG::LX, LR = ZG::LR;
  const int stage_n = max(zoff + S::LPW, S::LPW * LX);  // must match launch_lines
  const int nst = Tr::acc ? a.nst : 0;
  const size_t warp_bytes = sizeof(Cx<T>) * ((size_t)TileG<T, S>::TILE + stage_n) +
                            sizeof(T) * (size_t)(nreal + nst) * S::LPW * LR;
  // fp64: twiddles straight from the engine's global table (L1-resident), which
  // keeps the CTA's shared footprint at 6 CTAs per SM; fp32 converts into smem
  // register-bound ACC ops keep the twiddles in (otherwise unused) shared memory
  // shared twiddles: each warp copies the table into its own shared copy with
  // cp.async before griddepcontrol.wait; the copies join the first prefetch
  // group, so no CTA barrier and no register round trip at kernel start
  constexpr bool kTwG = sizeof(T) == 8 && !(Tr::acc && OP != kOpContract);
  constexpr bool kTwAsync = !kTwG && BLR_ZTW_ASYNC;
  constexpr int kTwN = kTwG ? 0 : (kTwAsync ? kZWarps * L : L);
  T* tw = (T*)smem_raw + (kTwAsync ? warp * 2 * L : 0);
  const T* twp = kTwG ? reinterpret_cast<const T*>(twz_g) : tw;
  unsigned char* wb = smem_raw + sizeof(Cx<T>) * kTwN + warp * warp_bytes;  // kTwN complex = 2 kTwN T
  Cx<T>* tile = (Cx<T>*)wb;
  Cx<T>* stage = tile + TileG<T, S>::TILE;
  Cx<T>* xbuf = stage;
  T* Vst = (T*)(stage + stage_n);
  T* Rsm = Vst + nst * S::LPW * LR;
  const int ldR = S::LPW * LR;
  const int nl = min(S::LPW, P1 - y0);
  if constexpr (kTwAsync) {
    if (nl <= 0) return;
    copy_tw_async<T>(tw, twz_g, L, lane, 32);
  } else if constexpr (!kTwG) {
    load_tw<T>(tw, twz_g, L);
    __syncthreads();
  }
  pdl_wait();
  if (nl <= 0) return;
  const int64_t sline = (int64_t)x * P1 + y0;
  const int64_t kzs = (int64_t)P0 * P1;
  const int64_t rline = ((int64_t)x * P1 + y0) * L;
  // stage the real fields the contributions read (one contiguous L run per line,
  // to line stride LR in shared memory)
  for (int q = 0; q < nst; ++q) {
    constexpr int V = 16 / sizeof(T);  // elements per 16-byte copy
    if constexpr (LR == L) {  // dense rows: one contiguous nl * L run
      const T* src = a.rin[a.st_idx[q]] + rline;
      T* dst = Vst + q * ldR;
      if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
        const int nv = (nl * L) / V;
        for (int i = lane; i < nv; i += 32) __pipeline_memcpy_async(dst + V * i, src + V * i, 16);
        for (int i = nv * V + lane; i < nl * L; i += 32) __pipeline_memcpy_async(dst + i, src + i, sizeof(T));
      } else {
        for (int i = lane; i < nl * L; i += 32) __pipeline_memcpy_async(dst + i, src + i, sizeof(T));
      }
      continue;
    }
    for (int ln = 0; ln < nl; ++ln) {
      const T* src = a.rin[a.st_idx[q]] + rline + ln * L;
      T* dst = Vst + q * ldR + ln * LR;
      if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
        constexpr int nv = L / V;
        for (int i = lane; i < nv; i += 32) __pipeline_memcpy_async(dst + V * i, src + V * i, 16);
        for (int i = nv * V + lane; i < L; i += 32) __pipeline_memcpy_async(dst + i, src + i, sizeof(T));
      } else {
        for (int i = lane; i < L; i += 32) __pipeline_memcpy_async(dst + i, src + i, sizeof(T));
      }
    }
  }
  // step-B ownership: lane (bl, k1) owns z = k1 + R1*k2
  const int bl = lane / S::R1, k1 = lane - (lane / S::R1) * S::R1;
  const bool own = bl < nl && bl < S::LPW;
  T acc[NOM][S::R2];
#pragma unroll
  for (int o = 0; o < NOM; ++o)
#pragma unroll
    for (int k2 = 0; k2 < S::R2; ++k2) acc[o][k2] = 0;
  // per-lane Hermitian gather table for step A (lane n2, rows k = R2*n1 + n2):
  // stage row index and sign s: G = (F1.x - s F2.y, s F1.y + F2.x)
  int hidx[S::R1], hsg[S::R1];
  {
    const int n2 = lane - (lane / S::R2) * S::R2;
#pragma unroll
    for (int n1 = 0; n1 < S::R1; ++n1) {
      const int k = S::R2 * n1 + n2;
      int row = -1, sgn = 1;  // out of band: the zero row
      if (k == 0) { row = 0; sgn = 0; }
      else if (k <= K2) { row = k; sgn = 1; }
      else if (k >= L - K2) { row = L - k; sgn = -1; }
      hidx[n1] = row < 0 ? -1 : row * S::LPW;
      hsg[n1] = sgn;
    }
  }
  // the shared zero row (never overwritten by the prefetch)
  if (lane < S::LPW) stage[zoff + lane] = cx<T>(0, 0);
  const int npair = (ns_blk + 1) / 2;
  const int nloop = OP == kOpContract ? a.n_nodes : 1;
  const int total = nloop * npair;
  // prefetch spectra of pair index q (node-major) into stage buffer q & 1
  // per-lane element offsets of the spectra gather, fixed across fields and
  // pairs: slot j covers stage entry i = lane + 32 j -> (row k, line l), global
  // offset k * kzs + l (32-bit: Kz1 * P0 * P1 < 2^31); -1 marks an empty slot
  // Kz1 = K + 1 <= (L - 1) / 3 + 1 since the pad satisfies L >= 3K + 1
  constexpr int kPfSlots = (S::LPW * ((S::L - 1) / 3 + 1) + 31) / 32;
  int pf_off[kPfSlots];
#pragma unroll
  for (int j = 0; j < kPfSlots; ++j) {
    const int i = lane + 32 * j;
    const int k = i / S::LPW, l = i - (i / S::LPW) * S::LPW;  // compile-time divisor
    pf_off[j] = (i < Kz1 * S::LPW && l < nl) ? k * (int)kzs + l : -1;
  }
  auto prefetch = [&](int q) {
    const int node = OP == kOpContract ? q / npair : 0, p = q - node * npair;  // one node unless contracting
    const int64_t noff = OP == kOpContract ? node * a.sin_node_stride : 0;
    Cx<T>* st = stage + (q & 1) * 2 * fstride;
    for (int ff = 0; ff < 2; ++ff) {
      const int f = 2 * p + ff;
      if (f >= ns_blk) {  // odd field count: the partner reads zeros
        for (int i = lane; i < Kz1 * S::LPW; i += 32) st[ff * fstride + i] = cx<T>(0, 0);
        break;
      }
      const Cx<T>* src = a.sin[f] + noff + sline;
#pragma unroll
      for (int j = 0; j < kPfSlots; ++j) {
        if (pf_off[j] >= 0) __pipeline_memcpy_async(st + ff * fstride + lane + 32 * j, src + pf_off[j], sizeof(Cx<T>));
        BLR_CHECK(pf_off[j] < 0 || ((q & 1) * 2 * fstride + ff * fstride + lane + 32 * j < zoff &&
                                    sline + pf_off[j] < g.ns), "zlines sin");
      }
    }
    __pipeline_commit();
  };
  prefetch(0);  // first spectra in flight while the per-lane register operands load
  // Outer: V_j at this lane's step-A positions (line la, z = R2*n1 + n2), used by every R2C gather
  T vreg[OP == kOpOuter ? 3 : 1][OP == kOpOuter ? S::R1 : 1];
  if constexpr (OP == kOpOuter) {
    const int la = lane / S::R2, n2a = lane - (lane / S::R2) * S::R2;
    const bool oka = la < nl && la < S::LPW;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const T* vj = a.rin[j < a.d ? j : 0] + rline + (oka ? la : 0) * L + n2a;
#pragma unroll
      for (int n1 = 0; n1 < S::R1; ++n1) vreg[j][n1] = oka ? __ldg(vj + S::R2 * n1) : (T)0;
    }
  }
  // MapTC: acc_i += sum_j Du_ij dV_j (rin: Du [0,dd) V [dd,dd+d) dV [dd+d, dd+2d)).
  // The k2 columns are split into five chunks, one per input pair: a chunk's
  // loads are issued before that pair's transform and consumed after it, so
  // the D(u) / dv reads overlap FFT work instead of stalling the kernel start.
  // Absent components (d < 3) read component 0 and are masked.
  constexpr int DCH = (S::R2 + 4) / 5;  // k2 columns per chunk
  constexpr bool kDu = OP == kOpMapTC;
  T dbuf[kDu ? DCH : 1][12];
  auto du_issue = [&](auto cc) {
    constexpr int c = decltype(cc)::value;
    if constexpr (OP == kOpMapTC) {
      const int d = a.d, dd = d * d;
      const int64_t base = rline + (own ? bl : 0) * L + k1;
      BLR_CHECK(base + S::R1 * (S::R2 - 1) < g.np, "zlines du");
#pragma unroll
      for (int u = 0; u < DCH; ++u) {
        const int k2 = c * DCH + u;
        if (k2 >= S::R2) continue;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const int jc = j < d ? j : 0;
          // (masking absent components here would wait for the load before the
          // FFT it is meant to overlap: A/B r02 map_tc 2.72 -> 2.90 ms; the
          // mask stays at the use)
          dbuf[u][j] = __ldg(a.rin[dd + d + jc] + base + S::R1 * k2);
#pragma unroll
          for (int o = 0; o < 3; ++o) dbuf[u][3 + 3 * o + j] = __ldg(a.rin[(o < d ? o : 0) * d + jc] + base + S::R1 * k2);
        }
      }
    }
  };
  auto du_acc = [&](auto cc) {
    constexpr int c = decltype(cc)::value;
    if constexpr (OP == kOpMapTC) {
      const int d = a.d;
#pragma unroll
      for (int u = 0; u < DCH; ++u) {
        const int k2 = c * DCH + u;
        if (k2 >= S::R2) continue;
#pragma unroll
        for (int o = 0; o < NOM; ++o) {
          T sdu = 0;
#pragma unroll
          for (int j = 0; j < 3; ++j) sdu += (j < d ? dbuf[u][3 + 3 * (o < 3 ? o : 0) + j] : (T)0) * dbuf[u][j];
          acc[o][k2] += sdu;
        }
      }
    }
  };
  auto du_chunk = [&](int c, auto f) {
    switch (c) {
      case 0: f(std::integral_constant<int, 0>{}); break;
      case 1: f(std::integral_constant<int, 1>{}); break;
      case 2: f(std::integral_constant<int, 2>{}); break;
      case 3: f(std::integral_constant<int, 3>{}); break;
      case 4: f(std::integral_constant<int, 4>{}); break;
      default: break;
    }
  };
  // one input pair
  auto pair_step = [&](int q) {
    if (q + 1 < total) {
      prefetch(q + 1);
      __pipeline_wait_prior(1);
    } else {
      __pipeline_wait_prior(0);
    }
    __syncwarp();
    const int node = OP == kOpContract ? q / npair : 0, p = q - node * npair;  // one node unless contracting
    const int f = 2 * p;
    const bool two = f + 1 < ns_blk;
    const int st1o = (q & 1) * 2 * fstride, st2o = st1o + fstride;
    // ACC ops: per-pair output coefficients (uniform), applied in the FFT store
    T c1[NOM], c2[NOM];
    const T* V1 = Vst;
    const T* V2 = Vst;
    if constexpr (Tr::acc && OP != kOpContract) {
      const int o1 = a.oi[f], o2 = two ? a.oi[f + 1] : -1;
      const T sg1 = (T)a.sg[f], sg2 = two ? (T)a.sg[f + 1] : (T)0;
#pragma unroll
      for (int o = 0; o < NOM; ++o) {
        c1[o] = o == o1 ? sg1 : (T)0;
        c2[o] = o == o2 ? sg2 : (T)0;
      }
      V1 = Vst + a.ri[f] * ldR;
      V2 = Vst + (two ? a.ri[f + 1] : 0) * ldR;
    }
    auto load = [&](int line, int, int n1) -> Cx<T> {
      // branch-free Hermitian packing of F1 + i F2 (zero rows index the zero pad row)
      const int h = hidx[n1];
      BLR_CHECK((h >= 0 ? st2o + h : zoff) + line < stage_n, "zlines gather");
      const Cx<T> F1 = stage[(h >= 0 ? st1o + h : zoff) + line];
      const Cx<T> F2 = stage[(h >= 0 ? st2o + h : zoff) + line];
      const T sg = (T)hsg[n1];
      return cx<T>(F1.x - sg * F2.y, sg * F1.y + F2.x);
    };
    auto store = [&](int line, int z, int k2, Cx<T> v) {
      const int li = line * LR + z;                // shared (Rsm / Vst)
      const int64_t gi = rline + line * L + z;     // global (pad field)
      BLR_CHECK(gi < g.np && li < ldR, "zlines store");
      BLR_CHECK(Tr::acc || OP == kOpRealize || (f + 1) * ldR <= nreal * ldR, "zlines Rsm");
      if constexpr (OP == kOpRealize) {
        a.wout[f][gi] = v.x;
        if (two) a.wout[f + 1][gi] = v.y;
      } else if constexpr (!Tr::acc || OP == kOpContract) {
        Rsm[f * ldR + li] = v.x;
        if (two) Rsm[(f + 1) * ldR + li] = v.y;
      } else {
        if (OP == kOpMap && a.wout[f]) {
          a.wout[f][gi] = v.x;
          if (two) a.wout[f + 1][gi] = v.y;
        }
        const T p1 = v.x * V1[li];
        const T p2 = v.y * V2[li];
#pragma unroll
        for (int o = 0; o < NOM; ++o) acc[o][k2] += c1[o] * p1 + c2[o] * p2;
      }
    };
    if constexpr (kDu) du_chunk(q, du_issue);
    wfft<T, S, true>(tile, twp, nl, load, store);
    if constexpr (kDu) du_chunk(q, du_acc);
    if constexpr (OP == kOpContract) {
      if (p == npair - 1) {
        // node complete: rho_n is realized in Rsm.  Stream the cached D(phi_n)
        // fields with lane-contiguous (coalesced) loads, two positions x d^2
        // fields issued per batch; lane owns positions li = lane + 32 m.
        __syncwarp();
        const int d = a.d;
        const T wn = (T)a.w[node];
        const T* Mb[3][3];
#pragma unroll
        for (int o = 0; o < 3; ++o)
#pragma unroll
          for (int j = 0; j < 3; ++j)
            Mb[o][j] = a.rin[(o < d && j < d) ? a.mi[o][j] : 0] + rline + node * a.rin_node_stride;
        const int npos = nl * L;
#pragma unroll
        for (int m0 = 0; m0 < S::R2; m0 += 2) {
          T mv[2][3][3];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int li = lane + 32 * (m0 + u);
            const bool ok = m0 + u < S::R2 && li < npos;
#pragma unroll
            for (int o = 0; o < 3; ++o)
#pragma unroll
              for (int j = 0; j < 3; ++j) mv[u][o][j] = (ok && o < d && j < d) ? __ldg(Mb[o][j] + li) : (T)0;
          }
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int li = lane + 32 * (m0 + u);
            if (m0 + u < S::R2 && li < npos) {
              T r[3];
#pragma unroll
              const int lis = (li / L) * LR + li % L;
#pragma unroll
              for (int j = 0; j < 3; ++j) r[j] = j < d ? Rsm[j * ldR + lis] : (T)0;
#pragma unroll
              for (int o = 0; o < NOM; ++o)
                acc[o][m0 + u] += wn * (mv[u][o][0] * r[0] + mv[u][o][1] * r[1] + mv[u][o][2] * r[2]);
            }
          }
        }
        __syncwarp();
      }
    }
  };
  // (unrolling the five 3-D MapTC pairs with compile-time output slots: A/B
  // r02 map_tc 2.82 -> 3.86 ms, code size and spills)
  for (int q = 0; q < total; ++q) pair_step(q);
  if constexpr (kDu) {
    for (int c = total; c < 5; ++c) {  // fewer than five input pairs (d < 3)
      du_chunk(c, du_issue);
      du_chunk(c, du_acc);
    }
  }
  if constexpr (OP == kOpRealize) return;
  const int no = a.no;
  // Outer (3-D): the five output pairs unrolled, so each product's rho / V
  // slots are compile-time constants (rho read from Rsm; holding it in
  // registers spills at 6 CTAs/SM).  A/B (r02): outer z-lines 2.13 -> 1.90 ms,
  // deformation GN HVP 9.52 -> 9.31 ms.
  const bool outer3 = OP == kOpOuter && a.d == 3 && no == 9;
  // One output pair (o, o + 1).  OS >= 0: o is a compile-time constant.
  auto out_step = [&](int o, auto oc) {
    constexpr int OS = decltype(oc)::value;
    const bool two = o + 1 < no;
    if constexpr (OP == kOpContract) {
#pragma unroll
      for (int m = 0; m < S::R2; ++m) {
        const int li = lane + 32 * m;
        T v1 = 0, v2 = 0;
#pragma unroll
        for (int q = 0; q < NOM; ++q) {
          if (q == o) v1 = acc[q][m];
          if (q == o + 1) v2 = acc[q][m];
        }
        if (li < nl * L) xbuf[(li / L) * LX + li % L] = cx<T>(v1, v2);
      }
      __syncwarp();
    } else if constexpr (Tr::acc) {
      if (own) {
#pragma unroll
        for (int k2 = 0; k2 < S::R2; ++k2) {
          T v1 = 0, v2 = 0;
#pragma unroll
          for (int q = 0; q < NOM; ++q) {
            if (q == o) v1 = acc[q][k2];
            if (q == o + 1) v2 = acc[q][k2];
          }
          BLR_CHECK(bl * LX + k1 + S::R1 * k2 < stage_n, "zlines xbuf acc");
          xbuf[bl * LX + k1 + S::R1 * k2] = cx<T>(v1, v2);
        }
      }
      __syncwarp();
    }
    // Outer: output o = (i, j) pairs, index math hoisted out of the gather
    const int oi1 = o / a.d, oj1 = o - oi1 * a.d;
    const int oi2 = two ? (o + 1) / a.d : 0, oj2 = two ? o + 1 - oi2 * a.d : 0;
    const T* R1p = Rsm + oi1 * ldR;
    const T* R2p = Rsm + oi2 * ldR;
    auto load = [&](int line, int z, int n1) -> Cx<T> {
      if constexpr (Tr::acc) {
        return xbuf[line * LX + z];
      } else if constexpr (OP == kOpOuter && OS >= 0) {
        constexpr int I1 = OS / 3, J1 = OS % 3, I2 = (OS + 1) / 3, J2 = (OS + 1) % 3;
        const int li = line * LR + z;
        return cx<T>(Rsm[I1 * ldR + li] * vreg[J1][n1],
                     OS + 1 < 9 ? Rsm[(I2 < 3 ? I2 : 0) * ldR + li] * vreg[J2][n1] : (T)0);
      } else if constexpr (OP == kOpOuter) {
        const int li = line * LR + z;
        const T v1 = oj1 == 0 ? vreg[0][n1] : (oj1 == 1 ? vreg[1][n1] : vreg[2][n1]);
        const T v2 = oj2 == 0 ? vreg[0][n1] : (oj2 == 1 ? vreg[1][n1] : vreg[2][n1]);
        return cx<T>(R1p[li] * v1, two ? R2p[li] * v2 : (T)0);
      } else {
        const int li = line * LR + z;
        const int64_t gi = rline + line * L + z;
        return cx<T>(z_output<T, S, OP>(a, Rsm, ldR, li, gi, o),
                     two ? z_output<T, S, OP>(a, Rsm, ldR, li, gi, o + 1) : (T)0);
      }
    };
    auto store = [&](int line, int k, int, Cx<T> v) {
      BLR_CHECK(line * LX + k < stage_n, "zlines xbuf");
      // only the bins the Hermitian extraction reads: k < Kz1 and L - k for them
      // (fp64 only; A/B r02: deformation 8.48 -> 8.45 ms, fp32 5.85 -> 5.86 ms)
      if (!(BLR_ZOUT_PRED && sizeof(T) == 8) || k < Kz1 || k > L - Kz1) xbuf[line * LX + k] = v;
    };
    wfft<T, S, false>(tile, twp, nl, load, store);
    Cx<T>* O1 = a.sout[o] + sline;
    Cx<T>* O2 = two ? a.sout[o + 1] + sline : nullptr;
    {
      // A/B (r02): the fixed-trip extraction is -1.4% on the deformation GN HVP
      // (9.64 -> 9.51 ms) against a strided idx loop
      // fixed-trip extraction over the prefetch slots (same (k, l) mapping and
      // global offsets): all shared loads of the warp's rows can be in flight
      Cx<T> Zs[kPfSlots], Zms[kPfSlots];
#pragma unroll
      for (int j = 0; j < kPfSlots; ++j) {
        const int idx = lane + 32 * j;
        const int k = idx / S::LPW, l = idx - (idx / S::LPW) * S::LPW;
        const int kk = pf_off[j] >= 0 ? k : 0, ll = pf_off[j] >= 0 ? l : 0;
        Zs[j] = xbuf[ll * LX + kk];
        Zms[j] = xbuf[ll * LX + (kk == 0 ? 0 : L - kk)];
      }
#pragma unroll
      for (int j = 0; j < kPfSlots; ++j) {
        if (pf_off[j] < 0) continue;
        BLR_CHECK(sline + pf_off[j] < g.ns, "zlines out");
        const Cx<T> Z = Zs[j];
        Cx<T> Zm = Zms[j];
        Zm.y = -Zm.y;
        O1[pf_off[j]] = cx<T>((T)0.5 * (Z.x + Zm.x), (T)0.5 * (Z.y + Zm.y));
        if (two) O2[pf_off[j]] = cx<T>((T)0.5 * (Z.y - Zm.y), (T)-0.5 * (Z.x - Zm.x));
      }
    }
    __syncwarp();
  };
  if (outer3) {
    if constexpr (OP == kOpOuter) {
      out_step(0, std::integral_constant<int, 0>{});
      out_step(2, std::integral_constant<int, 2>{});
      out_step(4, std::integral_constant<int, 4>{});
      out_step(6, std::integral_constant<int, 6>{});
      out_step(8, std::integral_constant<int, 8>{});
    }
  } else {
    for (int o = 0; o < no; o += 2) out_step(o, std::integral_constant<int, -1>{});
  }
}

// ---------------------------------------------------------------------------
// forward y pass: S [o][kz][x][y] -> I [o][kz][ky][x] (band ky kept)
// ---------------------------------------------------------------------------
// A forward-y "job" produces one I field: sum_t m_t * Y(S_t), m_t = 1, i k_y
// (after the transform) or i k_z.  Flux divergence folds its y and z terms
// into one job; the x term needs i k_x after the x pass and stays separate.
constexpr int kMaxYF = 24;
// forward passes: twiddles by cp.async in flight with the first slab -- fp32
// only; A/B r02: fp32 x / y forward 1.68 / 1.47 -> 1.61 / 1.43 ms, but fp64
// 1.83 / 1.69 -> 1.89 / 1.85 ms (the synchronous fp64 load stays)
#ifndef BLR_FWD_TW_ASYNC
#define BLR_FWD_TW_ASYNC 1
#endif
template <typename T>
constexpr bool fwd_tw_async() { return BLR_FWD_TW_ASYNC != 0 && sizeof(T) == 4; }
// fp64: the table by one cp.async.bulk on the first slab's mbarrier (no CTA
// barrier at start); A/B r02: x / y forward 1.84 / 1.69 -> 1.78 / 1.61 ms per
// deformation GN HVP (fp32 keeps the cp.async copies: bulk was 1.60 -> 1.69)
#ifndef BLR_FWD_TW_BULK
#define BLR_FWD_TW_BULK 1
#endif
template <typename T>
struct YFwdArgs {
  const Cx<T>* sin[kMaxYF][3];
  int axis[kMaxYF][3];
  int nterms[kMaxYF];
  int nj;
  Cx<T>* out;
};

// Persistent, double-buffered: each CTA walks items blockIdx.x + k*gridDim.x;
// the cp.async slab of the next (item, term) load streams in while the warps
// transform the current one, so HBM stays busy through the FFT phase.
template <typename T, class S>
#ifndef BLR_YFWD_MINB
#define BLR_YFWD_MINB 4
#endif
__global__ void __launch_bounds__(kPWF * 32, BLR_YFWD_MINB) k_yfwd(YFwdArgs<T> a, PadGeom g, const double* __restrict__ twg) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int LPC = kPWF * S::LPW;
  constexpr int LS = fwd_row_stride<T, S>();
  constexpr int LPCS = t_stride<LPC>();
  constexpr int SLAB = LPC * LS;
  const int P0 = g.P[0], K1 = g.K[1], B1 = g.B[1];
  T* tw = (T*)smem_raw;
  Cx<T>* slab = (Cx<T>*)(tw + 2 * S::L);         // [2][LPC][LS]; each warp's FFT tile overlays its lines
  Cx<T>* res = slab + 2 * SLAB;                  // [B1][LPCS] job accumulator
  const int nxb = (P0 + LPC - 1) / LPC;
  const int per = g.Kz1 * nxb;
  const FDiv div_per(per), div_nxb(nxb);
  const int nitems = a.nj * per;
  __shared__ uint64_t bars[2];
  Stager<T, fwd_bulk_rows<T, S>()> stg;
  stg.init(bars);
  __syncthreads();
  auto issue = [&](int it, int t, int b) {
    const int jb = div_per(it);
    const int r = it - jb * per;
    const int kz = div_nxb(r);
    const int cx0 = (r - kz * nxb) * LPC;
    const int nlc = min(LPC, P0 - cx0);
    const Cx<T>* src = a.sin[jb][t] + ((int64_t)kz * P0 + cx0) * S::L;  // nlc contiguous rows
    stg.begin(b, (uint32_t)(nlc * S::L * sizeof(Cx<T>)));
    stg.rows(slab + b * SLAB, LS, src, S::L, nlc, S::L, b);
  };
  // twiddles by cp.async in their own group, in flight with the first slab
  constexpr bool kTwBulk = BLR_FWD_TW_BULK && sizeof(T) == 8 && decltype(stg)::kBulk &&
                           (2 * S::L * sizeof(T)) % 16 == 0;
  if constexpr (kTwBulk) {  // on the first slab's mbarrier: its first wait covers the table
    if (threadIdx.x == 0) {
      const uint32_t nb = 2 * S::L * sizeof(T);
      mbar_expect_tx_only(bars, nb);
      bulk_g2s(tw, sizeof(T) == 8 ? (const void*)twg : (const void*)(twg + 2 * S::L), nb, bars);
    }
  } else if constexpr (fwd_tw_async<T>()) {
    copy_tw_async<T>(tw, twg, S::L, threadIdx.x, blockDim.x);
    __pipeline_commit();
  } else {
    load_tw<T>(tw, twg, S::L);
  }
  int it = blockIdx.x, t = 0, b = 0;
  pdl_trigger();  // persistent grid: every CTA is already resident
  pdl_wait();
  if (it < nitems) issue(it, 0, 0);
  stg.commit();
  const int wl0 = (threadIdx.x >> 5) * S::LPW;
  if constexpr (!kTwBulk && fwd_tw_async<T>()) __pipeline_wait_prior(decltype(stg)::kBulk ? 0 : 1);
  if constexpr (!kTwBulk) __syncthreads();  // twiddles
  while (it < nitems) {
    const int jb = div_per(it);
    const int nt = a.nterms[jb];
    int nit = it, ntt = t + 1;
    if (ntt >= nt) { nit = it + gridDim.x; ntt = 0; }
    if (nit < nitems) issue(nit, ntt, b ^ 1);
    stg.commit();
    stg.wait(b);
    const int r = it - jb * per;
    const int kz = div_nxb(r);
    const int cx0 = (r - kz * nxb) * LPC;
    const int nl = min(S::LPW, min(LPC, P0 - cx0) - wl0);
    if (nl > 0) {
      const int ax = a.axis[jb][t];
      const T kzk = (T)(kTwoPi * (double)kz);
      const Cx<T>* sl = slab + b * SLAB + wl0 * LS;
      auto load = [&](int line, int y, int) -> Cx<T> { return sl[line * LS + y]; };
      auto store = [&](int line, int q, int, Cx<T> v) {
        const int iy = bin_to_index(q, S::L, K1, B1);
        if (iy < 0) return;
        if (ax == 1) v = mul_ik<T>(v, (T)(kTwoPi * (double)freq_of(iy, K1, B1)));
        else if (ax == 2) v = mul_ik<T>(v, kzk);
        Cx<T>* rp = res + iy * LPCS + wl0 + line;  // owned by this lane for every term
        BLR_CHECK(iy * LPCS + wl0 + line < B1 * LPCS, "yfwd res");
        *rp = t == 0 ? v : cadd(*rp, v);
      };
      wfft<T, S, false, true>(slab + b * SLAB + wl0 * LS, tw, nl, load, store);
    }
    if (t == nt - 1) {
      const int nlc = min(LPC, P0 - cx0);
      Cx<T>* dst = a.out + jb * g.n1 + (int64_t)kz * B1 * P0 + cx0;
      __syncthreads();
      for (int i = threadIdx.x; i < B1 * LPC; i += blockDim.x) {
        const int iy = i / LPC, l = i - (i / LPC) * LPC;  // compile-time divisor
        BLR_CHECK(l >= nlc || jb * g.n1 + (int64_t)kz * B1 * P0 + cx0 + iy * P0 + l < a.nj * g.n1, "yfwd out");
        if (l < nlc) dst[iy * P0 + l] = res[iy * LPCS + l];
      }
    }
    __syncthreads();
    it = nit;
    t = ntt;
    b ^= 1;
  }
}

// ---------------------------------------------------------------------------
// forward x pass + epilogue: I [..][kz][ky][x] -> band, multipliers, 1/P^3,
// -(v + .) / negation, fused RK4 stage update (kz = 0 symmetrized in-item)
// ---------------------------------------------------------------------------
constexpr int kMaxFwd = 18;
enum FwdMode { kEpiPlain = 0, kEpiNeg = 1, kEpiNegAdd = 2 };

template <typename T>
struct FwdOut {
  int f[3];         // I-layout input fields
  int axis[3];      // post-transform derivative 3-axis or -1
  int nterms;
  int mode;
  const Cx<T>* vt;  // H-layout component for kEpiNegAdd
};

template <typename T>
struct FwdArgs {
  FwdOut<T> o[kMaxFwd];
  int no;
  const Cx<T>* in;  // I layout
  T scale;
  Cx<T>* kout;      // H layout [no][nh] or nullptr
  int rk_s;         // 0: no RK4 update
  T cs, h6;
  Cx<T>* cur;
  Cx<T>* acc;
  Cx<T>* stage;
};

// Cooperative epilogue of one (output, kz, ky-chunk) block from the result
// tile res[ix][LPCS]: consecutive threads take consecutive ky (coalesced), and
// each thread issues the operand loads of U elements before any store, so the
// RK4 read-modify-write costs one memory latency per U elements, not one each.
// elem(ix, l, e, r) -> false for an empty slot, else the element's flat
// H-layout index e and its (scaled) result r.
template <typename T, int LPC, class Elem>
__device__ __forceinline__ void epilogue_block(const FwdArgs<T>& a, const FwdOut<T>& O, int o, const PadGeom& g,
                                               Elem elem) {
#ifndef BLR_EPI_U
#define BLR_EPI_U 4
#endif
  constexpr int U = BLR_EPI_U;
  const int B0 = g.B[0];
  const int n = B0 * LPC;
  const int s = a.rk_s;
  for (int i0 = threadIdx.x; i0 < n; i0 += U * blockDim.x) {
    Cx<T> r[U], v[U], cc[U], ac[U];
    int64_t e[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * blockDim.x;
      const int ix = i / LPC, l = i - (i / LPC) * LPC;  // compile-time divisor
      ok[u] = i < n && elem(ix, l, e[u], r[u]);
      if (!ok[u]) continue;
      const int64_t h = (int64_t)o * g.nh + e[u];
      BLR_CHECK(e[u] >= 0 && e[u] < g.nh, "epilogue index");
      if (O.mode == kEpiNegAdd) v[u] = O.vt[e[u]];
      if (s) cc[u] = a.cur[h];
      if (s > 1) ac[u] = a.acc[h];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!ok[u]) continue;
      const int64_t h = (int64_t)o * g.nh + e[u];
      Cx<T> k;
      if (O.mode == kEpiNegAdd) k = cx<T>(-(v[u].x + r[u].x), -(v[u].y + r[u].y));
      else if (O.mode == kEpiNeg) k = cx<T>(-r[u].x, -r[u].y);
      else k = r[u];
      if (a.kout) a.kout[h] = k;
      if (s) {
        Cx<T> acv;
        if (s == 1) {
          acv = k;
        } else {
          const T m = s < 4 ? (T)2 : (T)1;
          acv = cx<T>(ac[u].x + m * k.x, ac[u].y + m * k.y);
        }
        if (s < 4) {
          a.acc[h] = acv;
          a.stage[h] = cx<T>(cc[u].x + a.cs * k.x, cc[u].y + a.cs * k.y);
        } else {
          a.cur[h] = cx<T>(cc[u].x + a.h6 * acv.x, cc[u].y + a.h6 * acv.y);
        }
      }
    }
  }
}

// kz > 0 items: LPC consecutive ky lines.  kz = 0 items pair every ky line
// with its mirror -ky (warp 0: units p0.., warp 1: their mirrors), so the
// Hermitian symmetrization of the kz = 0 plane (the reference's symmetrize)
// happens inside the item: no separate fix-up kernel.
#ifndef BLR_XFWD_MINB
#define BLR_XFWD_MINB 3
#endif
// (deferring the epilogue to a streaming kernel: 156 instead of 226 registers
// here, but A/B r02 x-forward 1.92 -> 2.04 ms per HVP)
template <typename T, class S>
__global__ void __launch_bounds__(kPWF * 32, BLR_XFWD_MINB) k_xfwd(FwdArgs<T> a, PadGeom g, const double* __restrict__ twg) {
  static_assert(kPWF == 2, "kz = 0 mirror items use one warp per half");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int LPW = S::LPW;
  constexpr int LPC = kPWF * LPW;
  constexpr int LS = fwd_row_stride<T, S>();
  constexpr int LPCS = t_stride<LPC>();
  constexpr int SLAB = LPC * LS;
  const int K0 = g.K[0], B0 = g.B[0], B1 = g.B[1], K1 = g.K[1];
  T* tw = (T*)smem_raw;
  Cx<T>* slab = (Cx<T>*)(tw + 2 * S::L);         // [2][LPC][LS] (persistent, as k_yfwd)
  Cx<T>* res = slab + 2 * SLAB;                  // [B0][LPCS] finished block
  const int nyb = (B1 + LPC - 1) / LPC;
  const int n0 = (K1 + 1 + LPW - 1) / LPW;      // kz = 0 items (LPW mirror units each)
  const int per = n0 + (g.Kz1 - 1) * nyb;
  const FDiv div_per(per), div_nyb(nyb);
  const int nitems = a.no * per;
  // item r of an output -> kz, first ky (kz > 0) or first unit p0 and the two half sizes (kz = 0)
  struct Item { int kz, cky0, p0, c1, c2; };
  auto decode = [&](int r) -> Item {
    Item m;
    if (r < n0) {
      m.kz = 0;
      m.cky0 = 0;
      m.p0 = r * LPW;
      m.c1 = min(LPW, K1 + 1 - m.p0);
      m.c2 = m.p0 == 0 ? m.c1 - 1 : m.c1;  // unit 0 (ky = 0) is its own mirror
    } else {
      const int q = r - n0;
      const int qk = div_nyb(q);
      m.kz = 1 + qk;
      m.cky0 = (q - qk * nyb) * LPC;
      m.p0 = -1;
      m.c1 = min(LPC, B1 - m.cky0);
      m.c2 = 0;
    }
    return m;
  };
  // kz = 0: ky index of slot s, and the slot holding its mirror
  auto slot_iy = [&](const Item& m, int s) -> int {
    if (s < LPW) return m.p0 + s;
    return B1 - (m.p0 + (s - LPW) + (m.p0 == 0 ? 1 : 0));
  };
  auto mirror_slot = [&](const Item& m, int s) -> int {
    const int z = m.p0 == 0 ? 1 : 0;
    if (s < LPW) return (m.p0 + s == 0) ? 0 : LPW + s - z;
    return s - LPW + z;
  };
  __shared__ uint64_t bars[2];
  Stager<T, fwd_bulk_rows<T, S>()> stg;
  stg.init(bars);
  __syncthreads();
  auto issue = [&](int it, int t, int b) {
    const int o = div_per(it);
    const Item m = decode(it - o * per);
    const Cx<T>* base = a.in + a.o[o].f[t] * g.n1 + (int64_t)m.kz * B1 * S::L;
    Cx<T>* dst = slab + b * SLAB;
    if (m.kz > 0) {
      stg.begin(b, (uint32_t)(m.c1 * S::L * sizeof(Cx<T>)));
      stg.rows(dst, LS, base + (int64_t)m.cky0 * S::L, S::L, m.c1, S::L, b);
    } else {
      stg.begin(b, (uint32_t)((m.c1 + m.c2) * S::L * sizeof(Cx<T>)));
      stg.rows(dst, LS, base + (int64_t)m.p0 * S::L, S::L, m.c1, S::L, b);
      if (m.c2 > 0)  // mirrors, descending ky
        stg.rows(dst + LPW * LS, LS, base + (int64_t)slot_iy(m, LPW) * S::L, -(int64_t)S::L, m.c2, S::L, b);
    }
  };
  // L1 prefetch of a kz > 0 item's epilogue operand rows (RK4 cur / acc and the
  // kEpiNegAdd addend): each (kz, kx) row is c1 <= LPC consecutive ky, at most
  // two 128-byte lines, so two prefetches per row and operand.  Issued when the
  // item's first term starts, the lines land during its transforms instead of
  // stalling the epilogue.  Rows are read only by this item (no staleness).
  auto prefetch_epi = [&](int it_) {
    if constexpr (kXfwdPrefetch) {
      const int o = div_per(it_);
      const Item m = decode(it_ - o * per);
      if (m.kz == 0) return;  // mirror items: scattered rows
      const FwdOut<T>& O = a.o[o];
      const int s = a.rk_s;
      if (!s && O.mode != kEpiNegAdd) return;
      for (int r = threadIdx.x; r < 2 * B0; r += blockDim.x) {
        const int ix = r >> 1;
        const int64_t e = ((int64_t)m.kz * B0 + ix) * B1 + m.cky0 + ((r & 1) ? m.c1 - 1 : 0);
        const int64_t h = (int64_t)o * g.nh + e;
        if (O.mode == kEpiNegAdd) prefetch_l1(O.vt + e);
        if (s) prefetch_l1(a.cur + h);
        if (s > 1) prefetch_l1(a.acc + h);
      }
    }
  };
  constexpr bool kTwBulk = BLR_FWD_TW_BULK && sizeof(T) == 8 && decltype(stg)::kBulk &&
                           (2 * S::L * sizeof(T)) % 16 == 0;
  if constexpr (kTwBulk) {  // on the first slab's mbarrier: its first wait covers the table
    if (threadIdx.x == 0) {
      const uint32_t nb = 2 * S::L * sizeof(T);
      mbar_expect_tx_only(bars, nb);
      bulk_g2s(tw, sizeof(T) == 8 ? (const void*)twg : (const void*)(twg + 2 * S::L), nb, bars);
    }
  } else if constexpr (fwd_tw_async<T>()) {  // as k_yfwd
    copy_tw_async<T>(tw, twg, S::L, threadIdx.x, blockDim.x);
    __pipeline_commit();
  } else {
    load_tw<T>(tw, twg, S::L);
  }
  int it = blockIdx.x, t = 0, b = 0;
  pdl_trigger();  // persistent grid: every CTA is already resident
  pdl_wait();
  if (it < nitems) issue(it, 0, 0);
  stg.commit();
  const int warp = threadIdx.x >> 5;
  const int wl0 = warp * LPW;
  if constexpr (!kTwBulk && fwd_tw_async<T>()) __pipeline_wait_prior(decltype(stg)::kBulk ? 0 : 1);
  if constexpr (!kTwBulk) __syncthreads();  // twiddles
  while (it < nitems) {
    const int o = div_per(it);
    const FwdOut<T>& O = a.o[o];
    const int nt = O.nterms;
    int nit = it, ntt = t + 1;
    if (ntt >= nt) { nit = it + gridDim.x; ntt = 0; }
    if (nit < nitems) issue(nit, ntt, b ^ 1);
    stg.commit();
    if (t == 0) prefetch_epi(it);
    stg.wait(b);
    const Item m = decode(it - o * per);
    const int kz = m.kz;
    const int nl = kz > 0 ? min(LPW, m.c1 - wl0) : (warp == 0 ? m.c1 : m.c2);
    if (nl > 0) {
      const T kzk = (T)(kTwoPi * (double)kz);
      const Cx<T>* sl = slab + b * SLAB + wl0 * LS;
      const int ax = O.axis[t];
      auto load = [&](int line, int x, int) -> Cx<T> { return sl[line * LS + x]; };
      auto store = [&](int line, int q, int, Cx<T> v) {
        const int ix = bin_to_index(q, S::L, K0, B0);
        if (ix < 0) return;
        if (ax == 0) {
          v = mul_ik<T>(v, (T)(kTwoPi * (double)freq_of(ix, K0, B0)));
        } else if (ax == 1) {
          const int iy = kz > 0 ? m.cky0 + wl0 + line : slot_iy(m, wl0 + line);
          v = mul_ik<T>(v, (T)(kTwoPi * (double)freq_of(iy, K1, B1)));
        } else if (ax == 2) {
          v = mul_ik<T>(v, kzk);
        }
        Cx<T>* rp = res + ix * LPCS + wl0 + line;  // owned by this lane for every term
        BLR_CHECK(ix * LPCS + wl0 + line < B0 * LPCS, "xfwd res");
        *rp = t == 0 ? v : cadd(*rp, v);
      };
      wfft<T, S, false, true>(slab + b * SLAB + wl0 * LS, tw, nl, load, store);
    }
    if (t == nt - 1) {
      __syncthreads();
      const Cx<T>* src = res;
      T sc = a.scale;
      if (kz == 0) {
        // symmetrize (kx, ky) with (-kx, -ky) inside the item into the consumed
        // slab, then the common epilogue
        Cx<T>* sym = slab + b * SLAB;
        for (int i = threadIdx.x; i < B0 * LPC; i += blockDim.x) {
          const int ix = i / LPC, sl = i - (i / LPC) * LPC;
          if (sl < LPW ? sl >= m.c1 : sl - LPW >= m.c2) continue;
          const int mix = ix == 0 ? 0 : B0 - ix;
          const Cx<T> p = res[ix * LPCS + sl], q = res[mix * LPCS + mirror_slot(m, sl)];
          sym[ix * LPCS + sl] = cx<T>((T)0.5 * a.scale * (p.x + q.x), (T)0.5 * a.scale * (p.y - q.y));
        }
        __syncthreads();
        src = sym;
        sc = (T)1;
      }
      auto elem = [&](int ix, int l, int64_t& e, Cx<T>& r) {
        int iy;
        if (kz > 0) {
          if (l >= m.c1) return false;
          iy = m.cky0 + l;
        } else {
          if (l < LPW ? l >= m.c1 : l - LPW >= m.c2) return false;
          iy = slot_iy(m, l);
        }
        e = ((int64_t)kz * B0 + ix) * B1 + iy;
        r = cscale(src[ix * LPCS + l], sc);
        return true;
      };
      epilogue_block<T, LPC>(a, O, o, g, elem);
    }
    __syncthreads();
    it = nit;
    t = ntt;
    b ^= 1;
  }
}

// ---------------------------------------------------------------------------
// layout conversion: full block [comp][kx][ky][kz] <-> H layout [comp][kz][kx][ky]
// ---------------------------------------------------------------------------
// Tiled conversions: one CTA per (component, kx) slice; the H rows of the
// slice (and, for the negative kz half, of its mirror slice -kx) go through
// shared memory so both the H-layout and the full-block side are row-coalesced.
template <typename T>
__global__ void __launch_bounds__(256) k_h_to_full_t(const Cx<T>* __restrict__ H, int ncomp, PadGeom g,
                                                     Cx<T>* __restrict__ full) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  pdl_wait();
  const int B0 = g.B[0], B1 = g.B[1], B2 = g.B[2], Kz1 = g.Kz1;
  const int c = blockIdx.x / B0, ix = blockIdx.x - (blockIdx.x / B0) * B0;
  const int mx = ix == 0 ? 0 : B0 - ix;
  Cx<T>* T1 = (Cx<T>*)smem_raw;  // [Kz1][B1] slice ix
  Cx<T>* T2 = T1 + Kz1 * B1;     // [Kz1][B1] slice -kx
  const Cx<T>* Hc = H + c * g.nh;
  for (int i = threadIdx.x; i < Kz1 * B1; i += blockDim.x) {
    const int kz = i / B1, iy = i - (i / B1) * B1;
    T1[i] = Hc[((int64_t)kz * B0 + ix) * B1 + iy];
    T2[i] = Hc[((int64_t)kz * B0 + mx) * B1 + iy];
  }
  __syncthreads();
  Cx<T>* out = full + ((int64_t)c * B0 + ix) * B1 * B2;
  for (int i = threadIdx.x; i < B1 * B2; i += blockDim.x) {
    const int iy = i / B2, iz = i - (i / B2) * B2;
    if (iz < Kz1) {
      out[i] = T1[iz * B1 + iy];
    } else {
      const int my = iy == 0 ? 0 : B1 - iy;
      out[i] = cconj(T2[(B2 - iz) * B1 + my]);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_full_to_h_t(const Cx<T>* __restrict__ full, int ncomp, PadGeom g,
                                                     Cx<T>* __restrict__ H) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  pdl_wait();
  const int B0 = g.B[0], B1 = g.B[1], B2 = g.B[2], Kz1 = g.Kz1;
  const int c = blockIdx.x / B0, ix = blockIdx.x - (blockIdx.x / B0) * B0;
  Cx<T>* Tt = (Cx<T>*)smem_raw;  // [Kz1][B1]
  const Cx<T>* in = full + ((int64_t)c * B0 + ix) * B1 * B2;
  for (int i = threadIdx.x; i < B1 * Kz1; i += blockDim.x) {
    const int iy = i / Kz1, kz = i - (i / Kz1) * Kz1;
    Tt[kz * B1 + iy] = in[(int64_t)iy * B2 + kz];
  }
  __syncthreads();
  Cx<T>* Hc = H + c * g.nh;
  for (int i = threadIdx.x; i < Kz1 * B1; i += blockDim.x) {
    const int kz = i / B1, iy = i - (i / B1) * B1;
    Hc[((int64_t)kz * B0 + ix) * B1 + iy] = Tt[i];
  }
}

template <typename T>
__global__ void k_full_to_h(const Cx<T>* __restrict__ full, int ncomp, PadGeom g, Cx<T>* __restrict__ H) {
  pdl_wait();
  const int64_t total = g.nh * ncomp;
  const int B0 = g.B[0], B1 = g.B[1], B2 = g.B[2];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / g.nh);
    int64_t r = i - c * g.nh;
    const int iy = (int)(r % B1);
    r /= B1;
    const int ix = (int)(r % B0);
    const int kz = (int)(r / B0);
    H[i] = full[(int64_t)c * B0 * B1 * B2 + ((int64_t)ix * B1 + iy) * B2 + kz];
  }
}

template <typename T>
__global__ void k_h_to_full(const Cx<T>* __restrict__ H, int ncomp, PadGeom g, Cx<T>* __restrict__ full) {
  pdl_wait();
  const int B0 = g.B[0], B1 = g.B[1], B2 = g.B[2];
  const int64_t nb = (int64_t)B0 * B1 * B2;
  const int64_t total = nb * ncomp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / nb);
    int64_t r = i - c * nb;
    const int iz = (int)(r % B2);
    r /= B2;
    const int iy = (int)(r % B1);
    const int ix = (int)(r / B1);
    const Cx<T>* Hc = H + c * g.nh;
    if (iz <= g.K[2]) {
      full[i] = Hc[((int64_t)iz * B0 + ix) * B1 + iy];
    } else {
      const int kz = B2 - iz;
      const int mx = ix == 0 ? 0 : B0 - ix, my = iy == 0 ? 0 : B1 - iy;
      full[i] = cconj(Hc[((int64_t)kz * B0 + mx) * B1 + my]);
    }
  }
}


struct PadEngine {
  bool ok = false;
  bool tried = false;
  PadGeom g{};
  double* tw[3] = {nullptr, nullptr, nullptr};  // split twiddle tables (2 L doubles per axis)
  int line_smem_max = 0;
  void* buf[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t buf_bytes[4] = {0, 0, 0, 0};
};


// Per-kernel launch facts, computed once per (kernel, shared bytes): kernels
// of one signature share a function-pointer type, so these are keyed by the
// kernel's address, not by template statics; the mutex makes the first use
// safe when several host threads launch concurrently.
struct KernelFacts {
  std::mutex mu;
  std::map<std::pair<const void*, size_t>, int> occupancy;  // CTAs per SM
  std::map<const void*, bool> smem_raised;
  int nsm = 0;
};
inline KernelFacts& kernel_facts() {
  static KernelFacts f;
  return f;
}

// forward-pass persistent grids: at most per_sm * nsm / BLR_FWD_GRID_DIV CTAs
#ifndef BLR_FWD_GRID_DIV
#define BLR_FWD_GRID_DIV 1
#endif
template <class K>
static int persistent_grid(K kernel, int threads, size_t smem, int nitems, int div = 1) {
  KernelFacts& f = kernel_facts();
  std::lock_guard<std::mutex> lk(f.mu);
  if (!f.nsm) {
    int dev;
    BLR_CUDA(cudaGetDevice(&dev));
    BLR_CUDA(cudaDeviceGetAttribute(&f.nsm, cudaDevAttrMultiProcessorCount, dev));
  }
  const auto key = std::make_pair((const void*)kernel, smem);
  auto it = f.occupancy.find(key);
  if (it == f.occupancy.end()) {
    int per_sm = 0;
    BLR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
    it = f.occupancy.emplace(key, std::max(per_sm, 1)).first;
  }
  return std::max(1, std::min(nitems, it->second * f.nsm / div));
}

// raise the kernel's dynamic shared-memory limit to the device maximum once
// (not per launch) when it needs more than the default 48 KB
template <typename K>
static void ensure_smem(K kernel, size_t bytes) {
  if (bytes <= 48 * 1024) return;
  KernelFacts& f = kernel_facts();
  std::lock_guard<std::mutex> lk(f.mu);
  if (f.smem_raised[(const void*)kernel]) return;
  int dev, maxsm;
  BLR_CUDA(cudaGetDevice(&dev));
  BLR_CUDA(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  cudaFuncAttributes fa;
  BLR_CUDA(cudaFuncGetAttributes(&fa, kernel));
  maxsm -= (int)fa.sharedSizeBytes;  // static shared memory (mbarriers) counts against the opt-in limit
  BLR_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
  f.smem_raised[(const void*)kernel] = true;
}

// TMA tensor maps (y-inverse slabs): the encoder comes from the driver through
// the runtime's entry-point query, so the library needs no -lcuda
#ifndef BLR_YINV_TMA
#define BLR_YINV_TMA 1
#endif
// x-inverse TMA: opt-in (build flag); A/B r02: 128^3 x-inverse 0.99 -> 0.98 ms
// (deformation 8.50 -> 8.48 ms) but 256^3 (L = 196, 128-byte box rows) 7.45 ->
// 8.21 ms per HVP
#ifndef BLR_XINV_TMA
#define BLR_XINV_TMA 0
#endif
using TmapEncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
inline TmapEncodeFn tmap_encoder() {
  static const TmapEncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return (TmapEncodeFn)p;
  }();
  return fn;
}
// rank-4 map of nf fields [field][kz][ky][x0] (x0 in T units, innermost),
// box {bx, B1, 1, 1}; false when the layout does not meet the TMA rules
template <typename T>
bool inv_tma_map(CUtensorMap& map, const void* base, int64_t x0, int B1, int Kz1, int nf, int64_t field, int bx) {
  const TmapEncodeFn enc = tmap_encoder();
  const size_t es = sizeof(T);
  if (!enc || (x0 * es) % 16 || (bx * es) % 16 || bx > 256 || B1 > 256 || (reinterpret_cast<uintptr_t>(base) & 15))
    return false;
  const cuuint64_t dims[4] = {(cuuint64_t)x0, (cuuint64_t)B1, (cuuint64_t)Kz1, (cuuint64_t)nf};
  const cuuint64_t strides[3] = {(cuuint64_t)(x0 * es), (cuuint64_t)(x0 * B1 * es), (cuuint64_t)(2 * field * es)};
  const cuuint32_t box[4] = {(cuuint32_t)bx, (cuuint32_t)B1, 1, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(&map, es == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
             const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename T, class S>
void launch_xinv(blr_ctx* c, PadEngine* e, const XPassArgs<T>& a0) {
  const PadGeom& g = e->g;
  constexpr int LPC = inv_pw<T>() * S::LPW;
  const int nyb = (g.B[1] + LPC - 1) / LPC;
  XPassArgs<T> a = a0;
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  // TMA when every source is base + k * nh (one rank-4 map over the fields)
  bool tma = BLR_XINV_TMA && (2 * S::L * sizeof(T)) % 16 == 0 && a.nx > 0;
  const Cx<T>* base = a.src[0];
  for (int i = 0; i < a.nx && tma; ++i) base = std::min(base, a.src[i]);
  int nf = 1;
  for (int i = 0; i < a.nx && tma; ++i) {
    const int64_t d = a.src[i] - base;
    tma = d % g.nh == 0 && d / g.nh < (1 << 20);
    a.fidx[i] = tma ? (int)(d / g.nh) : 0;
    nf = std::max(nf, a.fidx[i] + 1);
  }
  if (tma && inv_tma_map<T>(map, base, 2 * (int64_t)g.B[1], g.B[0], g.Kz1, nf, g.nh, 2 * LPC)) {
    const size_t sm = 2 * S::L * sizeof(T) + 128 + sizeof(Cx<T>) * ((size_t)g.B[0] * LPC + inv_pw<T>() * TileG<T, S>::TILE);
    ensure_smem(k_xinv<T, S, true>, sm);
    launch_pdl(k_xinv<T, S, true>, a.nx * g.Kz1 * nyb, inv_pw<T>() * 32, sm, c->stream, a, g, (const double*)e->tw[0], map);
    BLR_LAUNCHED();
    return;
  }
  const size_t sm = sizeof(Cx<T>) * (S::L + (size_t)g.B[0] * t_stride<LPC>() + inv_pw<T>() * TileG<T, S>::TILE);
  ensure_smem(k_xinv<T, S>, sm);
  launch_pdl(k_xinv<T, S>, a.nx * g.Kz1 * nyb, inv_pw<T>() * 32, sm, c->stream, a, g, (const double*)e->tw[0], map);
  BLR_LAUNCHED();
}
template <typename T, class S>
void launch_yinv(blr_ctx* c, PadEngine* e, const YPassArgs<T>& a) {
  const PadGeom& g = e->g;
  constexpr int LPC = inv_pw<T>() * S::LPW;
  int ntmax = 1, nf = 1;
  for (int i = 0; i < a.ny; ++i) {
    ntmax = std::max(ntmax, a.nterms[i]);
    for (int t = 0; t < a.nterms[i]; ++t) nf = std::max(nf, a.xf[i][t] + 1);
  }
  const int nxb = (g.P[0] + LPC - 1) / LPC;
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  if (BLR_YINV_TMA && (2 * S::L * sizeof(T)) % 16 == 0 &&
      inv_tma_map<T>(map, a.in, 2 * (int64_t)g.P[0], g.B[1], g.Kz1, nf, g.n1, 2 * LPC)) {
    constexpr int ra = 128 / cgcd(128, LPC * (int)sizeof(Cx<T>));
    const size_t b1t = ((g.B[1] + ra - 1) / ra) * ra;
    const size_t sm = 2 * S::L * sizeof(T) + 128 +  // + alignment slack of the slab
                      sizeof(Cx<T>) * ((size_t)ntmax * b1t * LPC + inv_pw<T>() * TileG<T, S>::TILE);
    ensure_smem(k_yinv<T, S, true>, sm);
    launch_pdl(k_yinv<T, S, true>, a.ny * g.Kz1 * nxb, inv_pw<T>() * 32, sm, c->stream, a, g, (const double*)e->tw[1], ntmax,
               map);
    BLR_LAUNCHED();
    return;
  }
  const size_t sm = sizeof(Cx<T>) * (S::L + (size_t)ntmax * g.B[1] * t_stride<LPC>() + inv_pw<T>() * TileG<T, S>::TILE);
  ensure_smem(k_yinv<T, S>, sm);
  launch_pdl(k_yinv<T, S>, a.ny * g.Kz1 * nxb, inv_pw<T>() * 32, sm, c->stream, a, g, (const double*)e->tw[1], ntmax, map);
  BLR_LAUNCHED();
}
template <typename T, class S, int OP>
void launch_lines(blr_ctx* c, PadEngine* e, const LineArgs<T>& a) {
  const PadGeom& g = e->g;
  const int ns_blk = OP == kOpContract ? a.d : a.ns;
  const int nreal = OP == kOpContract ? a.d : (ZOp<OP>::acc || OP == kOpRealize) ? 0 : ns_blk;
  const int nst = ZOp<OP>::acc ? a.nst : 0;
  const size_t stage_n = std::max<size_t>(4 * (size_t)g.Kz1 * S::LPW + S::LPW,
                                          (size_t)S::LPW * ZLineG<T, S>::LX);
  const size_t warp_bytes = sizeof(Cx<T>) * ((size_t)TileG<T, S>::TILE + stage_n) +
                            sizeof(T) * (size_t)(nreal + nst) * S::LPW * ZLineG<T, S>::LR;
  const bool twg = sizeof(T) == 8 && !(ZOp<OP>::acc && OP != kOpContract);  // as kTwG in the kernel
  const bool twa = !twg && BLR_ZTW_ASYNC;  // as kTwAsync: a table per warp
  const size_t sm = (twg ? 0 : (twa ? kZWarps : 1) * S::L * sizeof(Cx<T>)) + kZWarps * warp_bytes;
  if (sm > (size_t)e->line_smem_max) throw Error(1, "z-line kernel shared memory exceeds the device limit");
  ensure_smem(k_zlines<T, S, OP>, sm);
  constexpr int LPC = kZWarps * S::LPW;
  const int nyc = (g.P[1] + LPC - 1) / LPC;
  launch_pdl(k_zlines<T, S, OP>, g.P[0] * nyc, kZWarps * 32, sm, c->stream, a, g, (const double*)e->tw[2]);
  BLR_LAUNCHED();
}
// (a lean one-shot y-forward shaped like the inverse passes tied this
// persistent kernel, A/B r02 1.77 vs 1.76 ms per HVP)
template <typename T, class S>
void launch_yfwd(blr_ctx* c, PadEngine* e, const YFwdArgs<T>& a) {
  const PadGeom& g = e->g;
  constexpr int LPC = kPWF * S::LPW;
  const size_t sm = sizeof(Cx<T>) * (S::L + 2 * (size_t)LPC * fwd_row_stride<T, S>() +
                                     (size_t)g.B[1] * t_stride<LPC>());
  ensure_smem(k_yfwd<T, S>, sm);
  const int nxb = (g.P[0] + LPC - 1) / LPC;
  const int grid = persistent_grid(k_yfwd<T, S>, kPWF * 32, sm, a.nj * g.Kz1 * nxb, BLR_FWD_GRID_DIV);
  launch_pdl(k_yfwd<T, S>, grid, kPWF * 32, sm, c->stream, a, g, (const double*)e->tw[1]);
  BLR_LAUNCHED();
}

template <typename T, class S>
void launch_xfwd(blr_ctx* c, PadEngine* e, const FwdArgs<T>& a) {
  const PadGeom& g = e->g;
  constexpr int LPC = kPWF * S::LPW;
  const size_t sm = sizeof(Cx<T>) * (S::L + 2 * (size_t)LPC * fwd_row_stride<T, S>() +
                                     (size_t)g.B[0] * t_stride<LPC>());
  const int nyb = (g.B[1] + LPC - 1) / LPC;
  const int n0 = (g.K[1] + 1 + S::LPW - 1) / S::LPW;
  const int items = a.no * (n0 + (g.Kz1 - 1) * nyb);
  ensure_smem(k_xfwd<T, S>, sm);
  const int grid = persistent_grid(k_xfwd<T, S>, kPWF * 32, sm, items, BLR_FWD_GRID_DIV);
  launch_pdl(k_xfwd<T, S>, grid, kPWF * 32, sm, c->stream, a, g, (const double*)e->tw[0]);
  BLR_LAUNCHED();
}


}  // namespace blr

#include "blr_fwd2.cuh"
