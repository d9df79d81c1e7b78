// blr_fwd2.cuh — fused forward projection: y pass + x pass + epilogue in one
// kernel per (output, kz plane), one thread-block cluster per plane.
//
// The unfused path (k_yfwd -> I layout in global memory -> k_xfwd) spends two
// latency-bound kernels per projection with only ~2 items per CTA.  Here a
// cluster of kF2Cl CTAs owns one (output o, kz) plane of S:
//
//   phase 1  CTA r takes x rows [r*XL, (r+1)*XL): bulk-copies each term's rows,
//            forward y FFTs (band ky kept, i ky / i kz pre-multipliers, terms of
//            a job summed) into its slice I_j[ky][x - r*XL] of shared memory;
//   cluster barrier (the whole I plane now lives in the cluster's smem);
//   phase 2  CTA r takes ky lines [r*KYL, ...): x FFTs whose inputs are read
//            from the owning CTAs' slices through distributed shared memory
//            (ld.shared::cluster), band kx kept, i kx post-multiplier, jobs
//            summed; kz = 0 planes exchange mirror values through DSMEM for the
//            Hermitian symmetrization; then the epilogue of k_xfwd (1/P^3,
//            -(v + .) / negation, fused RK4 stage update).
//
// Arithmetic is the unfused path's, operation for operation (same transforms,
// multipliers and summation order), so results are bit-identical; the I layout
// never touches global memory and one launch replaces two.
#pragma once

#include <cooperative_groups.h>

namespace blr {

namespace cg = cooperative_groups;

constexpr int kF2Cl = 4;  // CTAs per cluster (one (o, kz) plane)
constexpr int kF2W = 4;   // warps per CTA
constexpr int kF2MaxJobs = 2;

template <typename T>
struct Fwd2Job {
  const Cx<T>* s[3];  // S-layout term fields
  int yax[3];         // pre-y multiplier per term: -1 none, 1 i ky, 2 i kz
  int nt;             // terms
  int xax;            // 0: i kx after the x pass, -1 none
};

template <typename T>
struct Fwd2Args {
  Fwd2Job<T> job[kMaxFwd][kF2MaxJobs];
  int nj[kMaxFwd];
  FwdArgs<T> e;  // epilogue: o[].mode / o[].vt, scale, kout, RK4 (o[].f / in unused)
};

// epilogue_block with a runtime chunk width (ky lines of this CTA)
template <typename T, class Elem>
__device__ __forceinline__ void epilogue_rt(const FwdArgs<T>& a, const FwdOut<T>& O, int o, const PadGeom& g,
                                            int nky, Elem elem) {
  constexpr int U = BLR_EPI_U;
  const int n = g.B[0] * nky;
  const int s = a.rk_s;
  for (int i0 = threadIdx.x; i0 < n; i0 += U * blockDim.x) {
    Cx<T> r[U], v[U], cc[U], ac[U];
    int64_t e[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * blockDim.x;
      const int ix = i / nky, l = i - (i / nky) * nky;
      ok[u] = i < n && elem(ix, l, e[u], r[u]);
      if (!ok[u]) continue;
      const int64_t h = (int64_t)o * g.nh + e[u];
      BLR_CHECK(e[u] >= 0 && e[u] < g.nh, "fwd2 epilogue");
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

// shared layout (complex entries unless noted):
//   tw [2L] T | slab [2][ROWS][LS] (phase 1: double-buffered rows, warp tiles
//   overlay their rows; phase 2: x-FFT tiles + res [B0][KYLP] overlay it) |
//   I [KYL][XP]: this CTA's ky lines over every x, written by the whole cluster
template <typename T, class S>
struct Fwd2Geom {
  static constexpr int ROWS = kF2W * S::LPW;             // rows per phase-1 step
  static constexpr int LS = row_stride<T, S, true>();    // slab row stride (>= tile stride)
  static constexpr int SLAB = ROWS * LS;
  static_assert(SLAB >= kF2W * TileG<T, S>::TILE, "tiles overlay the slab");
  __host__ __device__ static int xl(int P) { return (P + kF2Cl - 1) / kF2Cl; }
  __host__ __device__ static int xp(int P) { return P | 1; }
  __host__ __device__ static int kyl(int B1) { return (B1 + kF2Cl - 1) / kF2Cl; }
  __host__ __device__ static int kylp(int B1) { return kyl(B1) | 1; }
  static size_t smem(const PadGeom& g, int) {
    return sizeof(T) * 2 * S::L + sizeof(Cx<T>) * (2 * (size_t)SLAB + (size_t)kyl(g.B[1]) * xp(g.P[0]));
  }
};

// One launch per projection of single-job outputs (every output's x pass sums
// one I field; the flux divergence's two-job outputs keep the two-kernel path).
template <typename T, class S>
__global__ void __launch_bounds__(kF2W * 32) k_fwd2(Fwd2Args<T> a, PadGeom g, int njmax,
                                                    const double* __restrict__ twg) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using G = Fwd2Geom<T, S>;
  constexpr int L = S::L, LPW = S::LPW, LS = G::LS;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int unit = blockIdx.x / kF2Cl;
  const int o = unit / g.Kz1, kz = unit - (unit / g.Kz1) * g.Kz1;
  const int P = g.P[0], B0 = g.B[0], B1 = g.B[1], K0 = g.K[0], K1 = g.K[1];
  const int XL = G::xl(P), XP = G::xp(P), KYL = G::kyl(B1), KYLP = G::kylp(B1);
  T* tw = (T*)smem_raw;
  Cx<T>* slab = (Cx<T>*)(tw + 2 * L);  // [2][SLAB]
  Cx<T>* Iown = slab + 2 * G::SLAB;    // [KYL][XP]
  const int warp = threadIdx.x >> 5;
  const int wl0 = warp * LPW;
  __shared__ uint64_t bars[2];
  Stager<T> stg;
  stg.init(bars);
  load_tw<T>(tw, twg, L);
  const FwdOut<T>& O = a.e.o[o];
  const Fwd2Job<T>& J = a.job[o][0];
  const T kzk = (T)(kTwoPi * (double)kz);
  const int ky0 = rank * KYL, nky = max(0, min(KYL, B1 - ky0));
  if (kXfwdPrefetch && nky > 0 && (a.e.rk_s || O.mode == kEpiNegAdd)) {
    for (int r = threadIdx.x; r < 2 * B0; r += blockDim.x) {
      const int ix = r >> 1;
      const int64_t e = ((int64_t)kz * B0 + ix) * B1 + ky0 + ((r & 1) ? nky - 1 : 0);
      const int64_t h = (int64_t)o * g.nh + e;
      if (O.mode == kEpiNegAdd) prefetch_l1(O.vt + e);
      if (a.e.rk_s) prefetch_l1(a.e.cur + h);
      if (a.e.rk_s > 1) prefetch_l1(a.e.acc + h);
    }
  }
  Cx<T>* rem[kF2Cl];
#pragma unroll
  for (int q = 0; q < kF2Cl; ++q) rem[q] = cluster.map_shared_rank(Iown, q);
  __syncthreads();  // mbarrier init + twiddles
  pdl_wait();

  // ---- phase 1: forward y FFTs of this CTA's x rows, pushed to the owners ----
  // steps (round r0, term t), double-buffered: step k+1's rows stream in while
  // step k is transformed; each lane keeps its outputs of one round in
  // registers across the terms and stores them once, to the CTA that owns the
  // ky line (st.shared::cluster: no load latency on the critical path)
  const int x0 = rank * XL, nx = max(0, min(XL, P - x0));
  const int nt = J.nt;
  const int nsteps = ((nx + G::ROWS - 1) / G::ROWS) * nt;
  auto issue = [&](int k, int b) {
    const int r0 = (k / nt) * G::ROWS, t = k - (k / nt) * nt;
    const int nr = min(G::ROWS, nx - r0);
    const Cx<T>* src = J.s[t] + ((int64_t)kz * P + x0 + r0) * L;  // nr contiguous rows
    stg.begin(b, (uint32_t)(nr * L * sizeof(Cx<T>)));
    stg.rows(slab + b * G::SLAB, LS, src, L, nr, L, b);
  };
  if (nsteps > 0) issue(0, 0);
  stg.commit();
  Cx<T> yacc[S::R2];
  for (int k = 0; k < nsteps; ++k) {
    const int b = k & 1;
    if (k + 1 < nsteps) issue(k + 1, b ^ 1);
    stg.commit();
    stg.wait(b);
    const int r0 = (k / nt) * G::ROWS, t = k - (k / nt) * nt;
    const int nr = min(G::ROWS, nx - r0);
    const int nl = min(LPW, nr - wl0);
    if (nl > 0) {
      const int ax = J.yax[t];
      const Cx<T>* sl = slab + b * G::SLAB + wl0 * LS;
      auto load = [&](int line, int y, int) -> Cx<T> { return sl[line * LS + y]; };
      auto store = [&](int line, int q, int k2, Cx<T> v) {
        const int iy = bin_to_index(q, L, K1, B1);
        if (iy >= 0) {
          if (ax == 1) v = mul_ik<T>(v, (T)(kTwoPi * (double)freq_of(iy, K1, B1)));
          else if (ax == 2) v = mul_ik<T>(v, kzk);
        }
        yacc[k2] = t == 0 ? v : cadd(yacc[k2], v);
        if (t == nt - 1 && iy >= 0) {  // this round's sum is complete: push it to the owner
          const int qo = iy / KYL, l = iy - (iy / KYL) * KYL;
          BLR_CHECK(qo < kF2Cl && x0 + r0 + wl0 + line < P, "fwd2 push");
          rem[qo][(size_t)l * XP + x0 + r0 + wl0 + line] = yacc[k2];
        }
      };
      wfft<T, S, false, true>(slab + b * G::SLAB + wl0 * LS, tw, nl, load, store);
    }
    __syncthreads();  // buffer b is refilled by step k + 2
  }
  cluster.sync();  // every CTA's pushes complete and visible

  // ---- phase 2: forward x FFTs of this CTA's ky lines (local I) ----
  Cx<T>* tile = slab + warp * TileG<T, S>::TILE;
  Cx<T>* res = slab + kF2W * TileG<T, S>::TILE;  // [B0][KYLP]
  const int xax = J.xax;
  for (int l0 = 0; l0 < nky; l0 += kF2W * LPW) {
    const int nl = min(LPW, nky - l0 - wl0);
    if (nl > 0) {
      auto load = [&](int line, int x, int) -> Cx<T> { return Iown[(size_t)(l0 + wl0 + line) * XP + x]; };
      auto store = [&](int line, int qb, int, Cx<T> v) {
        const int ix = bin_to_index(qb, L, K0, B0);
        if (ix < 0) return;
        if (xax == 0) v = mul_ik<T>(v, (T)(kTwoPi * (double)freq_of(ix, K0, B0)));
        BLR_CHECK(l0 + wl0 + line < KYL, "fwd2 res");
        res[(size_t)ix * KYLP + l0 + wl0 + line] = v;
      };
      wfft<T, S, false>(tile, tw, nl, load, store);
    }
  }
  __syncthreads();
  if (kz == 0) {
    // Hermitian symmetrization of the kz = 0 plane (reference symmetrize):
    // h(kx, ky) <- (h(kx, ky) + conj(h(-kx, -ky))) / 2; the mirror ky line may
    // belong to another CTA of the cluster (its res, read over DSMEM)
    cluster.sync();
    Cx<T>* rres[kF2Cl];
#pragma unroll
    for (int q = 0; q < kF2Cl; ++q) rres[q] = cluster.map_shared_rank(res, q);
    Cx<T>* sym = Iown;  // [B0][KYLP] (I is consumed; B0 * KYLP <= KYL * XP)
    for (int i = threadIdx.x; i < B0 * nky; i += blockDim.x) {
      const int ix = i / nky, l = i - (i / nky) * nky;
      const int iy = ky0 + l;
      const int mix = ix == 0 ? 0 : B0 - ix, miy = iy == 0 ? 0 : B1 - iy;
      const int mq = miy / KYL, ml = miy - (miy / KYL) * KYL;
      BLR_CHECK(mq < kF2Cl, "fwd2 mirror");
      const Cx<T> p = res[(size_t)ix * KYLP + l], m = rres[mq][(size_t)mix * KYLP + ml];
      sym[(size_t)ix * KYLP + l] = cx<T>((T)0.5 * a.e.scale * (p.x + m.x), (T)0.5 * a.e.scale * (p.y - m.y));
    }
    cluster.sync();  // mirror reads done before any CTA moves on (res stays live)
    epilogue_rt<T>(a.e, O, o, g, nky, [&](int ix, int l, int64_t& e, Cx<T>& r) {
      e = ((int64_t)kz * B0 + ix) * B1 + ky0 + l;
      r = sym[(size_t)ix * KYLP + l];
      return true;
    });
  } else {
    const T sc = a.e.scale;
    epilogue_rt<T>(a.e, O, o, g, nky, [&](int ix, int l, int64_t& e, Cx<T>& r) {
      e = ((int64_t)kz * B0 + ix) * B1 + ky0 + l;
      r = cscale(res[(size_t)ix * KYLP + l], sc);
      return true;
    });
  }
}

template <typename T, class S>
bool fwd2_fits(const PadGeom& g) {
  using G = Fwd2Geom<T, S>;
  return 2 * (size_t)G::SLAB >= (size_t)kF2W * TileG<T, S>::TILE + (size_t)g.B[0] * G::kylp(g.B[1]) &&
         (size_t)G::kyl(g.B[1]) * G::xp(g.P[0]) >= (size_t)g.B[0] * G::kylp(g.B[1]);
}

template <typename T, class S>
void launch_fwd2(blr_ctx* c, PadEngine* e, const Fwd2Args<T>& a, int no, int njmax) {
  const PadGeom& g = e->g;
  const size_t sm = Fwd2Geom<T, S>::smem(g, njmax);
  if (sm > (size_t)e->line_smem_max) throw Error(1, "fused forward pass: shared memory exceeds the device limit");
  ensure_smem(k_fwd2<T, S>, sm);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(no * g.Kz1 * kF2Cl);
  cfg.blockDim = dim3(kF2W * 32);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kF2Cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  BLR_CUDA(cudaLaunchKernelEx(&cfg, k_fwd2<T, S>, a, g, njmax, (const double*)e->tw[0]));
  BLR_LAUNCHED();
}

}  // namespace blr
