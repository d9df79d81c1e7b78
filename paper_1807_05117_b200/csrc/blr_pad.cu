// blr_pad.cu — the fused pad-grid engine (v2) for every truncated
// convolution on the hot path (transport.py:206-303, deformation.py:63-72).
//
// A right-hand side is three kernels, no cuFFT, no full-grid zero padding:
//
//   k_inv2d   one CTA per (field, kz) plane: gathers the band plane with the
//             derivative multiplier (i 2 pi k_j) fused, inverse Stockham FFT
//             along x then along y in shared memory, writes the plane of the
//             "S layout" [field][kz][x][y] (kz = 0..K only: Hermitian half).
//   k_lines   one CTA per (x, y-chunk): per z-line, two-for-one C2R of the
//             spectral inputs, the pointwise product of the RHS (reading the
//             cached real pad fields: D(u) stages, v, dv), two-for-one R2C of
//             the outputs back to the S layout (kz = 0..K).
//   k_fwd2d   one CTA per (output, kz) plane: forward FFT along y then x,
//             keeps the band, applies post-transform derivative multipliers
//             (flux divergence), 1/P^3, symmetrizes the kz = 0 plane, the RHS
//             epilogue (-(v + .), negation) and the RK4 stage update.
//
// Band state lives in the "H layout" [comp][kz 0..K][kx][ky] (Hermitian half);
// node records are converted back to the reference's full blocks.
#include "blr_fft.cuh"
#include "blr_internal.cuh"

#include <cmath>
#include <cstring>

namespace blr {

// ---------------------------------------------------------------------------
// geometry
// ---------------------------------------------------------------------------
struct PadGeom {
  int P[3], K[3], B[3];
  int Kz1;       // K[2] + 1
  int64_t nh;    // H-layout component size Kz1*B0*B1
  int64_t ns;    // S-layout field size Kz1*P0*P1
  int64_t np;    // real pad field size
  FftSpec fx, fy, fz;
  int G;         // line group for the 2-D kernels
  int Yt;        // lines per CTA in k_lines (set per launch)
};

__device__ __forceinline__ int bin_to_index(int p, int P, int K, int B) {
  if (p <= K) return p;
  if (p >= P - K) return p - P + B;
  return -1;
}

template <typename T>
__device__ __forceinline__ void load_tw(Cx<T>* dst, const double2* src, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = cx<T>((T)src[i].x, (T)src[i].y);
}

// ---------------------------------------------------------------------------
// k_inv2d
// ---------------------------------------------------------------------------
constexpr int kMaxInv = 32;

template <typename T>
struct InvField {
  const Cx<T>* src[3];  // H-layout component bases
  int axis[3];          // derivative 3-axis or -1
  int nterms;
};

template <typename T>
struct InvArgs {
  InvField<T> f[kMaxInv];
  int nf;
};

template <typename T>
__global__ void __launch_bounds__(256) k_inv2d(InvArgs<T> a, PadGeom g, const double2* __restrict__ twx_g,
                                               const double2* __restrict__ twy_g, Cx<T>* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int P0 = g.P[0], P1 = g.P[1], B0 = g.B[0], B1 = g.B[1];
  const int Pm = P0 > P1 ? P0 : P1;
  Cx<T>* twx = (Cx<T>*)smem_raw;
  Cx<T>* twy = twx + P0;
  Cx<T>* Tb = twy + P1;            // [B1][P0]
  Cx<T>* w0 = Tb + B1 * P0;        // [G][Pm]
  Cx<T>* w1 = w0 + g.G * Pm;
  const int f = blockIdx.x / g.Kz1;
  const int kz = blockIdx.x - f * g.Kz1;
  const InvField<T> F = a.f[f];
  load_tw<T>(twx, twx_g, P0);
  load_tw<T>(twy, twy_g, P1);
  const int64_t plane = (int64_t)kz * B0 * B1;
  const T kz_ang = (T)(kTwoPi * (double)kz);
  __syncthreads();
  // x-pass over the B1 band columns
  for (int c0 = 0; c0 < B1; c0 += g.G) {
    const int ng = min(g.G, B1 - c0);
    for (int idx = threadIdx.x; idx < ng * P0; idx += blockDim.x) {
      const int gl = idx / P0, p = idx - gl * P0;
      const int ix = bin_to_index(p, P0, g.K[0], B0);
      Cx<T> val = cx<T>(0, 0);
      if (ix >= 0) {
        const int iy = c0 + gl;
        const int64_t off = plane + (int64_t)ix * B1 + iy;
        for (int t = 0; t < F.nterms; ++t) {
          Cx<T> z = F.src[t][off];
          const int ax = F.axis[t];
          if (ax >= 0) {
            T k;
            if (ax == 0) k = (T)(kTwoPi * (double)freq_of(ix, g.K[0], B0));
            else if (ax == 1) k = (T)(kTwoPi * (double)freq_of(iy, g.K[1], B1));
            else k = kz_ang;
            z = cx<T>(-(k * z.y), k * z.x);
          }
          val = cadd(val, z);
        }
      }
      w0[gl * P0 + p] = val;
    }
    __syncthreads();
    Cx<T>* r = fft_lines<T, true>(w0, w1, ng, g.fx, twx);
    for (int idx = threadIdx.x; idx < ng * P0; idx += blockDim.x) Tb[c0 * P0 + idx] = r[idx];
    __syncthreads();
  }
  // y-pass over the P0 rows, straight to global
  Cx<T>* outp = out + (int64_t)f * g.ns + (int64_t)kz * P0 * P1;
  for (int x0 = 0; x0 < P0; x0 += g.G) {
    const int ng = min(g.G, P0 - x0);
    for (int idx = threadIdx.x; idx < ng * P1; idx += blockDim.x) {
      const int gl = idx / P1, q = idx - gl * P1;
      const int iy = bin_to_index(q, P1, g.K[1], B1);
      w0[gl * P1 + q] = iy >= 0 ? Tb[iy * P0 + x0 + gl] : cx<T>(0, 0);
    }
    __syncthreads();
    Cx<T>* r = fft_lines<T, true>(w0, w1, ng, g.fy, twy);
    for (int idx = threadIdx.x; idx < ng * P1; idx += blockDim.x) outp[(int64_t)x0 * P1 + idx] = r[idx];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// k_lines
// ---------------------------------------------------------------------------
enum LineOp {
  kOpRealize = 0,   // write realized inputs (wout) only
  kOpMap = 1,       // out_i = sum_j S[ij] R[j]
  kOpMapTC = 2,     // out_i = sum_j S[ij] V_j + sum_j Du_ij dV_j   (Du, V, dV real)
  kOpMapTF = 3,     // out = [Du.V | dDu.V + Du.dV]                 (Du, dDu spectral)
  kOpInvVol = 4,    // out = [Dw.V | -V.G - J Dv]
  kOpBwdVol = 5,    // out = [Dw.V | dDw.V + Dw.dV | vol | vol tangent]
  kOpOuter = 6,     // out_ij = rho_i V_j
  kOpOuterPair = 7, // out = [rho x V | drho x V + rho x dV]
  kOpContract = 8,  // out_i = sum_n w_n sum_j M_n(ji or ij) rho_n,j  (M real, cached)
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
  int ns, nr, no;
  int d;
  // contract
  int n_nodes;
  int64_t sin_node_stride;  // complex entries between nodes (per input field)
  int64_t rin_node_stride;  // real entries between nodes
  double w[32];
  int transpose;
};

template <typename T, int OP>
__device__ __forceinline__ void line_point(const LineArgs<T>& a, const T* Rs, int ldR, int li,
                                           int64_t gi, T* out, int ldO) {
  const int d = a.d;
  auto S = [&](int f) { return Rs[f * ldR + li]; };
  auto Rg = [&](int f) { return a.rin[f][gi]; };
  if constexpr (OP == kOpMap) {
    for (int i = 0; i < d; ++i) {
      T acc = 0;
      for (int j = 0; j < d; ++j) acc += S(i * d + j) * Rg(j);
      out[i * ldO + li] = acc;
    }
  } else if constexpr (OP == kOpMapTC) {
    const int dd = d * d;
    for (int i = 0; i < d; ++i) {
      T a1 = 0, a2 = 0;
      for (int j = 0; j < d; ++j) a1 += S(i * d + j) * Rg(dd + j);
      for (int j = 0; j < d; ++j) a2 += Rg(i * d + j) * Rg(dd + d + j);
      out[i * ldO + li] = a1 + a2;
    }
  } else if constexpr (OP == kOpMapTF) {
    const int dd = d * d;
    for (int i = 0; i < d; ++i) {
      T b = 0, a1 = 0, a2 = 0;
      for (int j = 0; j < d; ++j) b += S(i * d + j) * Rg(j);
      for (int j = 0; j < d; ++j) a1 += S(dd + i * d + j) * Rg(j);
      for (int j = 0; j < d; ++j) a2 += S(i * d + j) * Rg(d + j);
      out[i * ldO + li] = b;
      out[(d + i) * ldO + li] = a1 + a2;
    }
  } else if constexpr (OP == kOpInvVol) {
    const int dd = d * d;
    for (int i = 0; i < d; ++i) {
      T b = 0;
      for (int j = 0; j < d; ++j) b += S(i * d + j) * Rg(j);
      out[i * ldO + li] = b;
    }
    T s = 0;
    for (int q = 0; q < d; ++q) s += Rg(q) * S(dd + q);
    out[d * ldO + li] = -s - S(dd + d) * Rg(d);
  } else if constexpr (OP == kOpBwdVol) {
    const int dd = d * d;
    // S: Dw [0,dd) dDw [dd,2dd) G [2dd,2dd+d) dG [2dd+d, 2dd+2d) J, dJ
    // R: V [0,d) dV [d,2d) Dv 2d dDv 2d+1
    for (int i = 0; i < d; ++i) {
      T b = 0, a1 = 0, a2 = 0;
      for (int j = 0; j < d; ++j) b += S(i * d + j) * Rg(j);
      for (int j = 0; j < d; ++j) a1 += S(dd + i * d + j) * Rg(j);
      for (int j = 0; j < d; ++j) a2 += S(i * d + j) * Rg(d + j);
      out[i * ldO + li] = b;
      out[(d + i) * ldO + li] = a1 + a2;
    }
    const int g0 = 2 * dd, dg0 = 2 * dd + d, jj = 2 * dd + 2 * d;
    T s = 0, s1 = 0, s2 = 0;
    for (int q = 0; q < d; ++q) s += Rg(q) * S(g0 + q);
    out[2 * d * ldO + li] = -s - S(jj) * Rg(2 * d);
    for (int q = 0; q < d; ++q) s1 += Rg(d + q) * S(g0 + q);
    for (int q = 0; q < d; ++q) s2 += Rg(q) * S(dg0 + q);
    out[(2 * d + 1) * ldO + li] = -s1 - s2 - S(jj + 1) * Rg(2 * d) - S(jj) * Rg(2 * d + 1);
  } else if constexpr (OP == kOpOuter) {
    for (int i = 0; i < d; ++i) {
      T r = S(i);
      for (int j = 0; j < d; ++j) out[(i * d + j) * ldO + li] = r * Rg(j);
    }
  } else if constexpr (OP == kOpOuterPair) {
    const int dd = d * d;
    for (int i = 0; i < d; ++i) {
      T r = S(i), dr = S(d + i);
      for (int j = 0; j < d; ++j) {
        out[(i * d + j) * ldO + li] = r * Rg(j);
        out[(dd + i * d + j) * ldO + li] = dr * Rg(j) + r * Rg(d + j);
      }
    }
  }
}

template <typename T, int OP>
__global__ void __launch_bounds__(256) k_lines(LineArgs<T> a, PadGeom g, const double2* __restrict__ twz_g) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int P0 = g.P[0], P1 = g.P[1], P2 = g.P[2], K2 = g.K[2];
  const int Yt = g.Yt;
  const int nyc = (P1 + Yt - 1) / Yt;
  const int x = blockIdx.x / nyc;
  const int y0 = (blockIdx.x - x * nyc) * Yt;
  const int nl = min(Yt, P1 - y0);
  const int ns_blk = OP == kOpContract ? a.d : a.ns;
  const int no_blk = OP == kOpRealize ? 0 : a.no;
  Cx<T>* twz = (Cx<T>*)smem_raw;
  Cx<T>* w0 = twz + P2;
  Cx<T>* w1 = w0 + Yt * P2;
  T* Rs = (T*)(w1 + Yt * P2);        // [ns_blk][Yt*P2]
  T* Ro = Rs + ns_blk * Yt * P2;     // [no][Yt*P2]
  const int ldR = Yt * P2;
  load_tw<T>(twz, twz_g, P2);
  const int64_t sline = (int64_t)x * P1 + y0;          // S-layout offset of line 0 at kz = 0
  const int64_t kzs = (int64_t)P0 * P1;                 // S-layout kz stride
  const int64_t rline = ((int64_t)x * P1 + y0) * P2;    // R-layout offset of line 0
  if (OP == kOpContract)
    for (int i = threadIdx.x; i < no_blk * ldR; i += blockDim.x) Ro[i] = 0;
  __syncthreads();

  const int nloop = OP == kOpContract ? a.n_nodes : 1;
  for (int node = 0; node < nloop; ++node) {
    // ---- realize spectral inputs, two per complex FFT ----
    for (int f = 0; f < ns_blk; f += 2) {
      const bool two = f + 1 < ns_blk;
      const int64_t noff = OP == kOpContract ? node * a.sin_node_stride : 0;
      const Cx<T>* S1 = a.sin[f] + noff + sline;
      const Cx<T>* S2 = two ? a.sin[f + 1] + noff + sline : nullptr;
      for (int idx = threadIdx.x; idx < nl * P2; idx += blockDim.x) {
        const int l = idx % nl, k = idx / nl;
        Cx<T> G = cx<T>(0, 0);
        if (k == 0) {
          G.x = S1[l].x;
          G.y = two ? S2[l].x : (T)0;
        } else if (k <= K2) {
          Cx<T> F1 = S1[k * kzs + l];
          Cx<T> F2 = two ? S2[k * kzs + l] : cx<T>(0, 0);
          G = cx<T>(F1.x - F2.y, F1.y + F2.x);
        } else if (k >= P2 - K2) {
          const int kk = P2 - k;
          Cx<T> F1 = S1[kk * kzs + l];
          Cx<T> F2 = two ? S2[kk * kzs + l] : cx<T>(0, 0);
          G = cx<T>(F1.x + F2.y, F2.x - F1.y);
        }
        w0[l * P2 + k] = G;
      }
      __syncthreads();
      Cx<T>* r = fft_lines<T, true>(w0, w1, nl, g.fz, twz);
      T* W1 = (OP != kOpContract) ? a.wout[f] : nullptr;
      T* W2 = (OP != kOpContract && two) ? a.wout[f + 1] : nullptr;
      for (int idx = threadIdx.x; idx < nl * P2; idx += blockDim.x) {
        Cx<T> v = r[idx];
        Rs[f * ldR + idx] = v.x;
        if (two) Rs[(f + 1) * ldR + idx] = v.y;
        if (W1) W1[rline + idx] = v.x;
        if (W2) W2[rline + idx] = v.y;
      }
      __syncthreads();
    }
    if (OP == kOpRealize) return;
    // ---- pointwise products ----
    for (int idx = threadIdx.x; idx < nl * P2; idx += blockDim.x) {
      const int64_t gi = rline + idx;
      if constexpr (OP == kOpContract) {
        const int d = a.d;
        const int64_t roff = node * a.rin_node_stride + gi;
        const T wn = (T)a.w[node];
        for (int i = 0; i < d; ++i) {
          T acc = 0;
          for (int j = 0; j < d; ++j) {
            const int mi = a.transpose ? (j * d + i) : (i * d + j);
            acc += a.rin[mi][roff] * Rs[j * ldR + idx];
          }
          Ro[i * ldR + idx] += wn * acc;
        }
      } else {
        line_point<T, OP>(a, Rs, ldR, idx, gi, Ro, ldR);
      }
    }
    __syncthreads();
  }
  // ---- R2C of the outputs, two per complex FFT ----
  for (int o = 0; o < no_blk; o += 2) {
    const bool two = o + 1 < no_blk;
    for (int idx = threadIdx.x; idx < nl * P2; idx += blockDim.x)
      w0[idx] = cx<T>(Ro[o * ldR + idx], two ? Ro[(o + 1) * ldR + idx] : (T)0);
    __syncthreads();
    Cx<T>* r = fft_lines<T, false>(w0, w1, nl, g.fz, twz);
    Cx<T>* O1 = a.sout[o] + sline;
    Cx<T>* O2 = two ? a.sout[o + 1] + sline : nullptr;
    for (int idx = threadIdx.x; idx < nl * (K2 + 1); idx += blockDim.x) {
      const int l = idx % nl, k = idx / nl;
      Cx<T> Z = r[l * P2 + k];
      Cx<T> Zm = r[l * P2 + (k == 0 ? 0 : P2 - k)];
      Zm.y = -Zm.y;
      O1[k * kzs + l] = cx<T>((T)0.5 * (Z.x + Zm.x), (T)0.5 * (Z.y + Zm.y));
      if (two) O2[k * kzs + l] = cx<T>((T)0.5 * (Z.y - Zm.y), (T)-0.5 * (Z.x - Zm.x));
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// k_fwd2d
// ---------------------------------------------------------------------------
constexpr int kMaxFwd = 18;
enum FwdMode { kEpiPlain = 0, kEpiNeg = 1, kEpiNegAdd = 2 };

template <typename T>
struct FwdOut {
  const Cx<T>* sin[3];  // S-layout term fields
  int axis[3];          // post-transform derivative 3-axis or -1
  int nterms;
  int mode;
  const Cx<T>* vt;      // H-layout component for kEpiNegAdd
};

template <typename T>
struct FwdArgs {
  FwdOut<T> o[kMaxFwd];
  int no;
  T scale;
  Cx<T>* kout;          // H-layout [no][nh] or nullptr
  int rk_s;             // 0: no RK4 update
  T cs, h6;
  Cx<T>* cur;
  Cx<T>* acc;
  Cx<T>* stage;
};

template <typename T>
__global__ void __launch_bounds__(256) k_fwd2d(FwdArgs<T> a, PadGeom g, const double2* __restrict__ twx_g,
                                               const double2* __restrict__ twy_g) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int P0 = g.P[0], P1 = g.P[1], B0 = g.B[0], B1 = g.B[1];
  const int Pm = P0 > P1 ? P0 : P1;
  Cx<T>* twx = (Cx<T>*)smem_raw;
  Cx<T>* twy = twx + P0;
  Cx<T>* Tb = twy + P1;            // [B1][P0]
  Cx<T>* Rb = Tb + B1 * P0;        // [B0][B1] result
  Cx<T>* w0 = Rb + B0 * B1;        // [G][Pm]
  Cx<T>* w1 = w0 + g.G * Pm;
  const int o = blockIdx.x / g.Kz1;
  const int kz = blockIdx.x - o * g.Kz1;
  const FwdOut<T> O = a.o[o];
  load_tw<T>(twx, twx_g, P0);
  load_tw<T>(twy, twy_g, P1);
  for (int i = threadIdx.x; i < B0 * B1; i += blockDim.x) Rb[i] = cx<T>(0, 0);
  __syncthreads();
  for (int t = 0; t < O.nterms; ++t) {
    const Cx<T>* src = O.sin[t] + (int64_t)kz * P0 * P1;
    // y-pass over rows x, keep band ky
    for (int x0 = 0; x0 < P0; x0 += g.G) {
      const int ng = min(g.G, P0 - x0);
      for (int idx = threadIdx.x; idx < ng * P1; idx += blockDim.x) w0[idx] = src[(int64_t)x0 * P1 + idx];
      __syncthreads();
      Cx<T>* r = fft_lines<T, false>(w0, w1, ng, g.fy, twy);
      for (int idx = threadIdx.x; idx < ng * B1; idx += blockDim.x) {
        const int gl = idx / B1, iy = idx - gl * B1;
        const int q = pmod(freq_of(iy, g.K[1], B1), P1);
        Tb[iy * P0 + x0 + gl] = r[gl * P1 + q];
      }
      __syncthreads();
    }
    // x-pass over the band columns, keep band kx, accumulate with multiplier
    const int ax = O.axis[t];
    for (int c0 = 0; c0 < B1; c0 += g.G) {
      const int ng = min(g.G, B1 - c0);
      for (int idx = threadIdx.x; idx < ng * P0; idx += blockDim.x) w0[idx] = Tb[c0 * P0 + idx];
      __syncthreads();
      Cx<T>* r = fft_lines<T, false>(w0, w1, ng, g.fx, twx);
      for (int idx = threadIdx.x; idx < ng * B0; idx += blockDim.x) {
        const int gl = idx / B0, ix = idx - gl * B0;
        const int iy = c0 + gl;
        const int p = pmod(freq_of(ix, g.K[0], B0), P0);
        Cx<T> z = r[gl * P0 + p];
        if (ax >= 0) {
          T k;
          if (ax == 0) k = (T)(kTwoPi * (double)freq_of(ix, g.K[0], B0));
          else if (ax == 1) k = (T)(kTwoPi * (double)freq_of(iy, g.K[1], B1));
          else k = (T)(kTwoPi * (double)kz);
          z = cx<T>(-(k * z.y), k * z.x);
        }
        Rb[ix * B1 + iy] = cadd(Rb[ix * B1 + iy], z);
      }
      __syncthreads();
    }
  }
  // scale + symmetrize the kz = 0 plane (pairs handled by one thread)
  const T sc = a.scale;
  for (int e = threadIdx.x; e < B0 * B1; e += blockDim.x) {
    const int ix = e / B1, iy = e - ix * B1;
    if (kz == 0) {
      const int mx = ix == 0 ? 0 : B0 - ix, my = iy == 0 ? 0 : B1 - iy;
      const int e2 = mx * B1 + my;
      if (e2 < e) continue;
      Cx<T> p = cscale(Rb[e], sc), q = cscale(Rb[e2], sc);
      Rb[e] = cx<T>((T)0.5 * (p.x + q.x), (T)0.5 * (p.y - q.y));
      if (e2 != e) Rb[e2] = cx<T>((T)0.5 * (q.x + p.x), (T)0.5 * (q.y - p.y));
    } else {
      Rb[e] = cscale(Rb[e], sc);
    }
  }
  __syncthreads();
  // epilogue + fused RK4 stage update
  const int64_t base = (int64_t)o * g.nh + (int64_t)kz * B0 * B1;
  for (int e = threadIdx.x; e < B0 * B1; e += blockDim.x) {
    Cx<T> r = Rb[e];
    Cx<T> k;
    if (O.mode == kEpiNegAdd) {
      Cx<T> v = O.vt[(int64_t)kz * B0 * B1 + e];
      k = cx<T>(-(v.x + r.x), -(v.y + r.y));
    } else if (O.mode == kEpiNeg) {
      k = cx<T>(-r.x, -r.y);
    } else {
      k = r;
    }
    const int64_t h = base + e;
    if (a.kout) a.kout[h] = k;
    if (a.rk_s) {
      Cx<T> cc = a.cur[h], ac;
      const int s = a.rk_s;
      if (s == 1) {
        ac = k;
      } else {
        ac = a.acc[h];
        const T m = s < 4 ? (T)2 : (T)1;
        ac = cx<T>(ac.x + m * k.x, ac.y + m * k.y);
      }
      if (s < 4) {
        a.acc[h] = ac;
        a.stage[h] = cx<T>(cc.x + a.cs * k.x, cc.y + a.cs * k.y);
      } else {
        a.cur[h] = cx<T>(cc.x + a.h6 * ac.x, cc.y + a.h6 * ac.y);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// layout conversion: full block [comp][kx][ky][kz] <-> H layout [comp][kz][kx][ky]
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_full_to_h(const Cx<T>* __restrict__ full, int ncomp, PadGeom g, Cx<T>* __restrict__ H) {
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
      const int kz = B2 - iz;  // -(iz - B2)
      const int mx = ix == 0 ? 0 : B0 - ix, my = iy == 0 ? 0 : B1 - iy;
      full[i] = cconj(Hc[((int64_t)kz * B0 + mx) * B1 + my]);
    }
  }
}

// ---------------------------------------------------------------------------
// host side: engine setup and launch helpers
// ---------------------------------------------------------------------------
struct PadEngine {
  bool ok = false;
  bool tried = false;
  PadGeom g{};
  double2* tw[3] = {nullptr, nullptr, nullptr};
  size_t smem_inv = 0, smem_fwd = 0;
  int line_smem_budget = 0;
};

static std::map<blr_ctx*, PadEngine>& engines() {
  static std::map<blr_ctx*, PadEngine> m;
  return m;
}

void pad_engine_release(blr_ctx* c) {
  auto it = engines().find(c);
  if (it == engines().end()) return;
  for (auto* p : it->second.tw)
    if (p) cudaFree(p);
  engines().erase(it);
}

template <typename T>
static size_t inv_smem(const PadGeom& g) {
  const int Pm = std::max(g.P[0], g.P[1]);
  return sizeof(Cx<T>) * ((size_t)g.P[0] + g.P[1] + (size_t)g.B[1] * g.P[0] + 2 * (size_t)g.G * Pm);
}
template <typename T>
static size_t fwd_smem(const PadGeom& g) {
  return inv_smem<T>(g) + sizeof(Cx<T>) * (size_t)g.B[0] * g.B[1];
}
template <typename T>
static size_t line_smem(const PadGeom& g, int Yt, int ns_blk, int no) {
  return sizeof(Cx<T>) * ((size_t)g.P[2] + 2 * (size_t)Yt * g.P[2]) +
         sizeof(T) * (size_t)(ns_blk + no) * Yt * g.P[2];
}

static int g_pad_disabled = -1;

template <typename T>
static PadEngine* engine(blr_ctx* c) {
  PadEngine& e = engines()[c];
  if (e.tried) return e.ok ? &e : nullptr;
  e.tried = true;
  if (g_pad_disabled < 0) {
    const char* env = getenv("BLR_PAD_ENGINE");
    g_pad_disabled = (env && env[0] == '0') ? 1 : 0;
  }
  if (g_pad_disabled) return nullptr;
  const Geom& gg = c->g;
  PadGeom& g = e.g;
  bool ok0, ok1, ok2;
  for (int a = 0; a < 3; ++a) { g.P[a] = gg.P[a]; g.K[a] = gg.K[a]; g.B[a] = gg.B[a]; }
  g.fx = make_fft(g.P[0], &ok0);
  g.fy = make_fft(g.P[1], &ok1);
  g.fz = make_fft(g.P[2], &ok2);
  if (!(ok0 && ok1 && ok2)) return nullptr;
  g.Kz1 = g.K[2] + 1;
  g.nh = (int64_t)g.Kz1 * g.B[0] * g.B[1];
  g.ns = (int64_t)g.Kz1 * g.P[0] * g.P[1];
  g.np = (int64_t)g.P[0] * g.P[1] * g.P[2];
  int dev;
  BLR_CUDA(cudaGetDevice(&dev));
  int maxsm = 0;
  BLR_CUDA(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  g.G = 16;
  while (g.G > 1 && fwd_smem<T>(g) > (size_t)maxsm) g.G /= 2;
  if (fwd_smem<T>(g) > (size_t)maxsm) return nullptr;
  e.smem_inv = inv_smem<T>(g);
  e.smem_fwd = fwd_smem<T>(g);
  e.line_smem_budget = std::min(maxsm, 110 * 1024);
  for (int a = 0; a < 3; ++a) {
    const int L = g.P[a];
    std::vector<double2> tw(L);
    for (int m = 0; m < L; ++m) {
      double s, co;
      sincospi(-2.0 * m / L, &s, &co);
      tw[m] = make_double2(co, s);
    }
    BLR_CUDA(cudaMalloc(&e.tw[a], L * sizeof(double2)));
    BLR_CUDA(cudaMemcpy(e.tw[a], tw.data(), L * sizeof(double2), cudaMemcpyHostToDevice));
  }
  BLR_CUDA(cudaFuncSetAttribute(k_inv2d<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem_inv));
  BLR_CUDA(cudaFuncSetAttribute(k_fwd2d<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)e.smem_fwd));
  e.ok = true;
  return &e;
}

template <typename T>
bool pad_engine_ok(blr_ctx* c) { return engine<T>(c) != nullptr; }

// --- inverse 2-D ---------------------------------------------------------------
template <typename T>
struct InvSpec {
  const Cx<T>* src[3];
  int axis[3];
  int nterms;
};

template <typename T>
static InvSpec<T> inv1(const Cx<T>* src, int axis) {
  InvSpec<T> s;
  s.src[0] = src; s.axis[0] = axis; s.nterms = 1;
  s.src[1] = s.src[2] = nullptr; s.axis[1] = s.axis[2] = -1;
  return s;
}

template <typename T>
static void inv2d(blr_ctx* c, PadEngine* e, const std::vector<InvSpec<T>>& f, Cx<T>* S) {
  for (size_t off = 0; off < f.size(); off += kMaxInv) {
    InvArgs<T> a;
    std::memset(&a, 0, sizeof(a));
    a.nf = (int)std::min<size_t>(kMaxInv, f.size() - off);
    for (int i = 0; i < a.nf; ++i) {
      const InvSpec<T>& s = f[off + i];
      for (int t = 0; t < 3; ++t) { a.f[i].src[t] = s.src[t]; a.f[i].axis[t] = s.axis[t]; }
      a.f[i].nterms = s.nterms;
    }
    ProfScope ps(c, "pad_inv2d", (double)a.nf * (e->g.nh + e->g.ns) * sizeof(Cx<T>));
    k_inv2d<T><<<a.nf * e->g.Kz1, 256, e->smem_inv, c->stream>>>(a, e->g, e->tw[0], e->tw[1],
                                                                   S + (int64_t)off * e->g.ns);
    BLR_LAUNCHED();
  }
}

// --- lines -------------------------------------------------------------------------
template <typename T, int OP>
static void lines(blr_ctx* c, PadEngine* e, LineArgs<T>& a, double bytes) {
  PadGeom g = e->g;
  const int ns_blk = OP == kOpContract ? a.d : a.ns;
  const int no = OP == kOpRealize ? 0 : a.no;
  int Yt = 16;
  while (Yt > 1 && line_smem<T>(g, Yt, ns_blk, no) > (size_t)e->line_smem_budget) --Yt;
  g.Yt = Yt;
  const size_t smem = line_smem<T>(g, Yt, ns_blk, no);
  static bool attr_set[2][16] = {};
  bool& done = attr_set[sizeof(T) == 8 ? 0 : 1][OP];
  if (!done) {
    int dev, maxsm;
    BLR_CUDA(cudaGetDevice(&dev));
    BLR_CUDA(cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    BLR_CUDA(cudaFuncSetAttribute(k_lines<T, OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm));
    done = true;
  }
  const int nyc = (g.P[1] + Yt - 1) / Yt;
  ProfScope ps(c, "pad_lines", bytes);
  k_lines<T, OP><<<g.P[0] * nyc, 256, smem, c->stream>>>(a, g, e->tw[2]);
  BLR_LAUNCHED();
}

// --- forward 2-D ---------------------------------------------------------------------
template <typename T>
struct FwdSpec {
  const Cx<T>* sin[3];
  int axis[3];
  int nterms;
  int mode;
  const Cx<T>* vt;
};

template <typename T>
static FwdSpec<T> fwd1(const Cx<T>* s, int mode, const Cx<T>* vt = nullptr) {
  FwdSpec<T> f;
  f.sin[0] = s; f.axis[0] = -1; f.nterms = 1;
  f.sin[1] = f.sin[2] = nullptr; f.axis[1] = f.axis[2] = -1;
  f.mode = mode;
  f.vt = vt;
  return f;
}

struct Rk {
  int s = 0;
  double cs = 0, h6 = 0;
  void* cur = nullptr;
  void* acc = nullptr;
  void* stage = nullptr;
};

template <typename T>
static void fwd2d(blr_ctx* c, PadEngine* e, const std::vector<FwdSpec<T>>& outs, Cx<T>* kout, const Rk& rk) {
  // chunks must keep the state/kout component index = output index
  for (size_t off = 0; off < outs.size(); off += kMaxFwd) {
    FwdArgs<T> a;
    std::memset(&a, 0, sizeof(a));
    a.no = (int)std::min<size_t>(kMaxFwd, outs.size() - off);
    int nterm = 0;
    for (int i = 0; i < a.no; ++i) {
      const FwdSpec<T>& s = outs[off + i];
      for (int t = 0; t < 3; ++t) { a.o[i].sin[t] = s.sin[t]; a.o[i].axis[t] = s.axis[t]; }
      a.o[i].nterms = s.nterms;
      a.o[i].mode = s.mode;
      a.o[i].vt = s.vt;
      nterm += s.nterms;
    }
    a.scale = (T)(1.0 / (double)e->g.np);
    const int64_t shift = (int64_t)off * e->g.nh;
    a.kout = kout ? kout + shift : nullptr;
    a.rk_s = rk.s;
    a.cs = (T)rk.cs;
    a.h6 = (T)rk.h6;
    a.cur = rk.cur ? (Cx<T>*)rk.cur + shift : nullptr;
    a.acc = rk.acc ? (Cx<T>*)rk.acc + shift : nullptr;
    a.stage = rk.stage ? (Cx<T>*)rk.stage + shift : nullptr;
    ProfScope ps(c, "pad_fwd2d",
                 ((double)nterm * e->g.ns + a.no * e->g.nh * (rk.s ? 4 : 2)) * sizeof(Cx<T>));
    k_fwd2d<T><<<a.no * e->g.Kz1, 256, e->smem_fwd, c->stream>>>(a, e->g, e->tw[0], e->tw[1]);
    BLR_LAUNCHED();
  }
}

template <typename T>
static void full_to_h(blr_ctx* c, PadEngine* e, const Cx<T>* full, int ncomp, Cx<T>* H) {
  k_full_to_h<T><<<grid_blocks(e->g.nh * ncomp, 256), 256, 0, c->stream>>>(full, ncomp, e->g, H);
  BLR_LAUNCHED();
}

template <typename T>
static void h_to_full(blr_ctx* c, PadEngine* e, const Cx<T>* H, int ncomp, Cx<T>* full) {
  k_h_to_full<T><<<grid_blocks(c->g.nb() * ncomp, 256), 256, 0, c->stream>>>(H, ncomp, e->g, full);
  BLR_LAUNCHED();
}

// ---------------------------------------------------------------------------
// stream-ordered temporaries
// ---------------------------------------------------------------------------
struct Tmp2 {
  blr_ctx* c;
  std::vector<void*> ptrs;
  explicit Tmp2(blr_ctx* ctx) : c(ctx) {}
  template <typename X>
  X* get(int64_t n) {
    void* p = nullptr;
    BLR_CUDA(cudaMallocAsync(&p, (size_t)std::max<int64_t>(n, 1) * sizeof(X), c->stream));
    ptrs.push_back(p);
    return (X*)p;
  }
  ~Tmp2() {
    for (void* p : ptrs) cudaFreeAsync(p, c->stream);
  }
};

// ---------------------------------------------------------------------------
// velocity samples (H layout + real pad realization [+ divergence])
// ---------------------------------------------------------------------------
template <typename T>
struct VelBank2 {
  blr_ctx* c;
  PadEngine* e;
  FlowRef f;
  bool with_div;
  int nreal;
  struct Entry {
    double t;
    bool valid;
    Cx<T>* H;      // [d][nh]
    T* real;       // [d (+1)][np]
    int64_t age;
  } en[3];
  Cx<T>* lerp = nullptr;
  Cx<T>* S = nullptr;
  int64_t clock = 0;

  VelBank2(blr_ctx* ctx, PadEngine* eng, FlowRef flow, bool div, Tmp2& tmp)
      : c(ctx), e(eng), f(flow), with_div(div) {
    const Geom& g = c->g;
    nreal = g.d + (div ? 1 : 0);
    const int ne = f.stationary() ? 1 : 3;
    for (auto& x : en) { x.valid = false; x.H = nullptr; x.real = nullptr; x.age = 0; }
    for (int i = 0; i < ne; ++i) {
      en[i].H = tmp.get<Cx<T>>(g.d * e->g.nh);
      en[i].real = tmp.get<T>(nreal * e->g.np);
    }
    if (!f.stationary()) lerp = tmp.get<Cx<T>>(g.d * g.nb());
    S = tmp.get<Cx<T>>(nreal * e->g.ns);
    if (f.stationary()) fill(en[0], (const Cx<T>*)f.v, 0.0);
  }

  void fill(Entry& x, const Cx<T>* full, double t) {
    const Geom& g = c->g;
    full_to_h<T>(c, e, full, g.d, x.H);
    std::vector<InvSpec<T>> fs;
    for (int a = 0; a < g.d; ++a) fs.push_back(inv1<T>(x.H + a * e->g.nh, -1));
    if (with_div) {
      InvSpec<T> s;
      s.nterms = g.d;
      for (int t = 0; t < 3; ++t) { s.src[t] = nullptr; s.axis[t] = -1; }
      for (int a = 0; a < g.d; ++a) { s.src[a] = x.H + a * e->g.nh; s.axis[a] = g.axis_of(a); }
      fs.push_back(s);
    }
    inv2d<T>(c, e, fs, S);
    LineArgs<T> la;
    std::memset(&la, 0, sizeof(la));
    la.ns = nreal;
    la.d = g.d;
    for (int i = 0; i < nreal; ++i) {
      la.sin[i] = S + i * e->g.ns;
      la.wout[i] = x.real + i * e->g.np;
    }
    lines<T, kOpRealize>(c, e, la, (double)nreal * (e->g.ns * sizeof(Cx<T>) + e->g.np * sizeof(T)));
    x.t = t;
    x.valid = true;
  }

  const Entry& at(double t) {
    if (f.stationary()) return en[0];
    ++clock;
    for (auto& x : en)
      if (x.valid && x.t == t) { x.age = clock; return x; }
    Entry* victim = &en[0];
    for (auto& x : en)
      if (!x.valid || x.age < victim->age) victim = &x;
    const Geom& g = c->g;
    const int n = f.n_steps;
    double s = std::min(std::max(t, 0.0), 1.0) * n;
    int i = std::min((int)std::floor(s), n - 1);
    double w = s - i;
    const Cx<T>* base = (const Cx<T>*)f.v;
    const int64_t L = g.d * g.nb();
    const Cx<T>* band = base + i * L;
    if (w != 0.0) {
      band_lerp<T>(c, base + i * L, base + (i + 1) * L, w, lerp, L);
      band = lerp;
    }
    fill(*victim, band, t);
    victim->age = clock;
    return *victim;
  }
};

// ---------------------------------------------------------------------------
// RK4 driver with the stage update fused into k_fwd2d
// ---------------------------------------------------------------------------
struct Rec2 {
  int comp0;   // first H component
  int ncomp;
  void* dst;   // full blocks [n_steps+1][ncomp][nb]
};

template <typename T, typename Rhs>
static void rk4_v2(blr_ctx* c, PadEngine* e, int n_steps, int substeps, bool forward, Cx<T>* cur, int ncomp,
                   const std::vector<Rec2>& rec, Tmp2& tmp, Rhs rhs) {
  const int64_t L = ncomp * e->g.nh;
  Cx<T>* acc = tmp.get<Cx<T>>(L);
  Cx<T>* stage = tmp.get<Cx<T>>(L);
  const int n = n_steps;
  const double dt = (forward ? 1.0 : -1.0) / n;
  const double h = dt / substeps;
  const int64_t nb = c->g.nb();
  auto record = [&](int node) {
    for (const auto& r : rec)
      if (r.dst)
        h_to_full<T>(c, e, cur + r.comp0 * e->g.nh, r.ncomp, (Cx<T>*)r.dst + (int64_t)node * r.ncomp * nb);
  };
  record(forward ? 0 : n);
  int si = 0;
  for (int step = 0; step < n; ++step) {
    const int node = forward ? step : n - step;
    const double t0 = (double)node / n;
    for (int ks = 0; ks < substeps; ++ks) {
      const double t = t0 + ks * h;
      Rk rk;
      rk.cur = cur;
      rk.acc = acc;
      rk.stage = stage;
      rk.h6 = h / 6.0;
      rk.s = 1; rk.cs = 0.5 * h;
      rhs(si + 0, t, (const Cx<T>*)cur, rk);
      rk.s = 2; rk.cs = 0.5 * h;
      rhs(si + 1, t + 0.5 * h, (const Cx<T>*)stage, rk);
      rk.s = 3; rk.cs = h;
      rhs(si + 2, t + 0.5 * h, (const Cx<T>*)stage, rk);
      rk.s = 4; rk.cs = h;
      rhs(si + 3, t + h, (const Cx<T>*)stage, rk);
      si += 4;
    }
    record(forward ? node + 1 : node - 1);
  }
}

template <typename T>
static void push_jac(const Geom& g, const PadGeom& pg, const Cx<T>* uH, std::vector<InvSpec<T>>& f) {
  for (int i = 0; i < g.d; ++i)
    for (int j = 0; j < g.d; ++j) f.push_back(inv1<T>(uH + i * pg.nh, g.axis_of(j)));
}

template <typename T>
static void push_grad(const Geom& g, const Cx<T>* sH, std::vector<InvSpec<T>>& f) {
  for (int a = 0; a < g.d; ++a) f.push_back(inv1<T>(sH, g.axis_of(a)));
}

template <typename T>
static void set_unit(blr_ctx* c, Cx<T>* H0) {
  Cx<T> one;
  one.x = (T)1;
  one.y = (T)0;
  BLR_CUDA(cudaMemcpyAsync(H0, &one, sizeof(one), cudaMemcpyHostToDevice, c->stream));
}

static double sbytes(const PadGeom& g, int ns, int nr, int no, int nw, size_t T_size) {
  return (double)(ns + no) * g.ns * 2 * T_size + (double)(nr + nw) * g.np * T_size;
}

// ---------------------------------------------------------------------------
// integrators (v2)
// ---------------------------------------------------------------------------
template <typename T>
bool forward_map_v2(blr_ctx* c, FlowRef v, int substeps, Cx<T>* phi, T* du_cache) {
  PadEngine* e = engine<T>(c);
  if (!e) return false;
  const Geom& g = c->g;
  const PadGeom& pg = e->g;
  const int d = g.d, dd = d * d;
  Tmp2 tmp(c);
  VelBank2<T> V(c, e, v, false, tmp);
  Cx<T>* cur = tmp.get<Cx<T>>(d * pg.nh);
  BLR_CUDA(cudaMemsetAsync(cur, 0, d * pg.nh * sizeof(Cx<T>), c->stream));
  Cx<T>* S = tmp.get<Cx<T>>(dd * pg.ns);
  Cx<T>* So = tmp.get<Cx<T>>(d * pg.ns);
  rk4_v2<T>(c, e, v.n_steps, substeps, true, cur, d, {{0, d, phi}}, tmp,
            [&](int si, double t, const Cx<T>* s, const Rk& rk) {
              const auto& vt = V.at(t);
              std::vector<InvSpec<T>> f;
              push_jac<T>(g, pg, s, f);
              inv2d<T>(c, e, f, S);
              LineArgs<T> la;
              std::memset(&la, 0, sizeof(la));
              la.ns = dd; la.nr = d; la.no = d; la.d = d;
              for (int i = 0; i < dd; ++i) {
                la.sin[i] = S + i * pg.ns;
                la.wout[i] = du_cache ? du_cache + ((int64_t)si * dd + i) * pg.np : nullptr;
              }
              for (int j = 0; j < d; ++j) la.rin[j] = vt.real + j * pg.np;
              for (int i = 0; i < d; ++i) la.sout[i] = So + i * pg.ns;
              lines<T, kOpMap>(c, e, la, sbytes(pg, dd, d, d, du_cache ? dd : 0, sizeof(T)));
              std::vector<FwdSpec<T>> outs;
              for (int i = 0; i < d; ++i) outs.push_back(fwd1<T>(So + i * pg.ns, kEpiNegAdd, vt.H + i * pg.nh));
              fwd2d<T>(c, e, outs, nullptr, rk);
            });
  return true;
}

template <typename T>
bool inverse_map_and_volume_v2(blr_ctx* c, FlowRef v, int substeps, Cx<T>* psi, Cx<T>* vol) {
  PadEngine* e = engine<T>(c);
  if (!e) return false;
  const Geom& g = c->g;
  const PadGeom& pg = e->g;
  const int d = g.d, dd = d * d;
  Tmp2 tmp(c);
  VelBank2<T> V(c, e, v, true, tmp);
  const int ncomp = d + 1;
  Cx<T>* cur = tmp.get<Cx<T>>(ncomp * pg.nh);
  BLR_CUDA(cudaMemsetAsync(cur, 0, ncomp * pg.nh * sizeof(Cx<T>), c->stream));
  set_unit<T>(c, cur + d * pg.nh);
  const int nsi = dd + d + 1;
  Cx<T>* S = tmp.get<Cx<T>>(nsi * pg.ns);
  Cx<T>* So = tmp.get<Cx<T>>(ncomp * pg.ns);
  rk4_v2<T>(c, e, v.n_steps, substeps, false, cur, ncomp, {{0, d, psi}, {d, 1, vol}}, tmp,
            [&](int, double t, const Cx<T>* s, const Rk& rk) {
              const auto& vt = V.at(t);
              std::vector<InvSpec<T>> f;
              push_jac<T>(g, pg, s, f);
              push_grad<T>(g, s + d * pg.nh, f);
              f.push_back(inv1<T>(s + d * pg.nh, -1));
              inv2d<T>(c, e, f, S);
              LineArgs<T> la;
              std::memset(&la, 0, sizeof(la));
              la.ns = nsi; la.nr = d + 1; la.no = ncomp; la.d = d;
              for (int i = 0; i < nsi; ++i) la.sin[i] = S + i * pg.ns;
              for (int j = 0; j <= d; ++j) la.rin[j] = vt.real + j * pg.np;
              for (int i = 0; i < ncomp; ++i) la.sout[i] = So + i * pg.ns;
              lines<T, kOpInvVol>(c, e, la, sbytes(pg, nsi, d + 1, ncomp, 0, sizeof(T)));
              std::vector<FwdSpec<T>> outs;
              for (int i = 0; i < d; ++i) outs.push_back(fwd1<T>(So + i * pg.ns, kEpiNegAdd, vt.H + i * pg.nh));
              outs.push_back(fwd1<T>(So + d * pg.ns, kEpiPlain));
              fwd2d<T>(c, e, outs, nullptr, rk);
            });
  return true;
}

template <typename T>
bool state_tangents_v2(blr_ctx* c, FlowRef v, FlowRef dv, int substeps, int flags, const T* du_cache,
                       Cx<T>* dphi, Cx<T>* dpsi, Cx<T>* dvol) {
  PadEngine* e = engine<T>(c);
  if (!e) return false;
  const Geom& g = c->g;
  const PadGeom& pg = e->g;
  const int d = g.d, dd = d * d;
  const bool want_fwd = flags & 1, want_bwd = flags & 2, want_vol = (flags & 4) && want_bwd;
  if (want_bwd && !want_vol) return false;  // (w, dw) without volume: v1 path
  Tmp2 tmp(c);
  if (want_fwd) {
    VelBank2<T> V(c, e, v, false, tmp);
    VelBank2<T> dV(c, e, dv, false, tmp);
    const bool cached = du_cache != nullptr;
    const int ncomp = cached ? d : 2 * d;
    Cx<T>* cur = tmp.get<Cx<T>>(ncomp * pg.nh);
    BLR_CUDA(cudaMemsetAsync(cur, 0, ncomp * pg.nh * sizeof(Cx<T>), c->stream));
    const int nsi = cached ? dd : 2 * dd;
    Cx<T>* S = tmp.get<Cx<T>>(nsi * pg.ns);
    Cx<T>* So = tmp.get<Cx<T>>(2 * d * pg.ns);
    const int du0 = cached ? 0 : d;
    rk4_v2<T>(c, e, v.n_steps, substeps, true, cur, ncomp, {{du0, d, dphi}}, tmp,
              [&](int si, double t, const Cx<T>* s, const Rk& rk) {
                const auto& vt = V.at(t);
                const auto& dvt = dV.at(t);
                std::vector<InvSpec<T>> f;
                push_jac<T>(g, pg, s, f);
                if (!cached) push_jac<T>(g, pg, s + d * pg.nh, f);
                inv2d<T>(c, e, f, S);
                LineArgs<T> la;
                std::memset(&la, 0, sizeof(la));
                la.d = d;
                for (int i = 0; i < nsi; ++i) la.sin[i] = S + i * pg.ns;
                std::vector<FwdSpec<T>> outs;
                if (cached) {
                  la.ns = dd; la.nr = dd + 2 * d; la.no = d;
                  const T* Du = du_cache + (int64_t)si * dd * pg.np;
                  for (int i = 0; i < dd; ++i) la.rin[i] = Du + i * pg.np;
                  for (int j = 0; j < d; ++j) {
                    la.rin[dd + j] = vt.real + j * pg.np;
                    la.rin[dd + d + j] = dvt.real + j * pg.np;
                  }
                  for (int i = 0; i < d; ++i) la.sout[i] = So + i * pg.ns;
                  lines<T, kOpMapTC>(c, e, la, sbytes(pg, dd, dd + 2 * d, d, 0, sizeof(T)));
                  for (int i = 0; i < d; ++i)
                    outs.push_back(fwd1<T>(So + i * pg.ns, kEpiNegAdd, dvt.H + i * pg.nh));
                } else {
                  la.ns = 2 * dd; la.nr = 2 * d; la.no = 2 * d;
                  for (int j = 0; j < d; ++j) {
                    la.rin[j] = vt.real + j * pg.np;
                    la.rin[d + j] = dvt.real + j * pg.np;
                  }
                  for (int i = 0; i < 2 * d; ++i) la.sout[i] = So + i * pg.ns;
                  lines<T, kOpMapTF>(c, e, la, sbytes(pg, 2 * dd, 2 * d, 2 * d, 0, sizeof(T)));
                  for (int i = 0; i < d; ++i)
                    outs.push_back(fwd1<T>(So + i * pg.ns, kEpiNegAdd, vt.H + i * pg.nh));
                  for (int i = 0; i < d; ++i)
                    outs.push_back(fwd1<T>(So + (d + i) * pg.ns, kEpiNegAdd, dvt.H + i * pg.nh));
                }
                fwd2d<T>(c, e, outs, nullptr, rk);
              });
  }
  if (want_bwd) {
    VelBank2<T> V(c, e, v, true, tmp);
    VelBank2<T> dV(c, e, dv, true, tmp);
    const int ncomp = 2 * d + 2;  // [w | dw | J | dJ]
    Cx<T>* cur = tmp.get<Cx<T>>(ncomp * pg.nh);
    BLR_CUDA(cudaMemsetAsync(cur, 0, ncomp * pg.nh * sizeof(Cx<T>), c->stream));
    set_unit<T>(c, cur + 2 * d * pg.nh);
    const int nsi = 2 * dd + 2 * d + 2;
    Cx<T>* S = tmp.get<Cx<T>>(nsi * pg.ns);
    Cx<T>* So = tmp.get<Cx<T>>(ncomp * pg.ns);
    rk4_v2<T>(c, e, v.n_steps, substeps, false, cur, ncomp, {{d, d, dpsi}, {2 * d + 1, 1, dvol}}, tmp,
              [&](int, double t, const Cx<T>* s, const Rk& rk) {
                const auto& vt = V.at(t);
                const auto& dvt = dV.at(t);
                const Cx<T>* JH = s + 2 * d * pg.nh;
                const Cx<T>* dJH = s + (2 * d + 1) * pg.nh;
                std::vector<InvSpec<T>> f;
                push_jac<T>(g, pg, s, f);
                push_jac<T>(g, pg, s + d * pg.nh, f);
                push_grad<T>(g, JH, f);
                push_grad<T>(g, dJH, f);
                f.push_back(inv1<T>(JH, -1));
                f.push_back(inv1<T>(dJH, -1));
                inv2d<T>(c, e, f, S);
                LineArgs<T> la;
                std::memset(&la, 0, sizeof(la));
                la.d = d; la.ns = nsi; la.nr = 2 * d + 2; la.no = ncomp;
                for (int i = 0; i < nsi; ++i) la.sin[i] = S + i * pg.ns;
                for (int j = 0; j < d; ++j) {
                  la.rin[j] = vt.real + j * pg.np;
                  la.rin[d + j] = dvt.real + j * pg.np;
                }
                la.rin[2 * d] = vt.real + d * pg.np;
                la.rin[2 * d + 1] = dvt.real + d * pg.np;
                for (int i = 0; i < ncomp; ++i) la.sout[i] = So + i * pg.ns;
                lines<T, kOpBwdVol>(c, e, la, sbytes(pg, nsi, 2 * d + 2, ncomp, 0, sizeof(T)));
                std::vector<FwdSpec<T>> outs;
                for (int i = 0; i < d; ++i) outs.push_back(fwd1<T>(So + i * pg.ns, kEpiNegAdd, vt.H + i * pg.nh));
                for (int i = 0; i < d; ++i)
                  outs.push_back(fwd1<T>(So + (d + i) * pg.ns, kEpiNegAdd, dvt.H + i * pg.nh));
                outs.push_back(fwd1<T>(So + 2 * d * pg.ns, kEpiPlain));
                outs.push_back(fwd1<T>(So + (2 * d + 1) * pg.ns, kEpiPlain));
                fwd2d<T>(c, e, outs, nullptr, rk);
              });
  }
  return true;
}

// flux divergence outputs: out_i = -(sum_j i k_j F_ij)
template <typename T>
static void push_flux(const Geom& g, const PadGeom& pg, const Cx<T>* So, std::vector<FwdSpec<T>>& outs) {
  const int d = g.d;
  for (int i = 0; i < d; ++i) {
    FwdSpec<T> f;
    f.nterms = d;
    for (int t = 0; t < 3; ++t) { f.sin[t] = nullptr; f.axis[t] = -1; }
    for (int j = 0; j < d; ++j) {
      f.sin[j] = So + (i * d + j) * pg.ns;
      f.axis[j] = g.axis_of(j);
    }
    f.mode = kEpiNeg;
    f.vt = nullptr;
    outs.push_back(f);
  }
}

template <typename T>
bool momentum_v2(blr_ctx* c, FlowRef v, int substeps, const Cx<T>* rho_end, Cx<T>* rho) {
  PadEngine* e = engine<T>(c);
  if (!e) return false;
  const Geom& g = c->g;
  const PadGeom& pg = e->g;
  const int d = g.d, dd = d * d;
  Tmp2 tmp(c);
  VelBank2<T> V(c, e, v, false, tmp);
  Cx<T>* cur = tmp.get<Cx<T>>(d * pg.nh);
  full_to_h<T>(c, e, rho_end, d, cur);
  Cx<T>* S = tmp.get<Cx<T>>(d * pg.ns);
  Cx<T>* So = tmp.get<Cx<T>>(dd * pg.ns);
  rk4_v2<T>(c, e, v.n_steps, substeps, false, cur, d, {{0, d, rho}}, tmp,
            [&](int, double t, const Cx<T>* s, const Rk& rk) {
              const auto& vt = V.at(t);
              std::vector<InvSpec<T>> f;
              for (int a = 0; a < d; ++a) f.push_back(inv1<T>(s + a * pg.nh, -1));
              inv2d<T>(c, e, f, S);
              LineArgs<T> la;
              std::memset(&la, 0, sizeof(la));
              la.d = d; la.ns = d; la.nr = d; la.no = dd;
              for (int i = 0; i < d; ++i) la.sin[i] = S + i * pg.ns;
              for (int j = 0; j < d; ++j) la.rin[j] = vt.real + j * pg.np;
              for (int i = 0; i < dd; ++i) la.sout[i] = So + i * pg.ns;
              lines<T, kOpOuter>(c, e, la, sbytes(pg, d, d, dd, 0, sizeof(T)));
              std::vector<FwdSpec<T>> outs;
              push_flux<T>(g, pg, So, outs);
              fwd2d<T>(c, e, outs, nullptr, rk);
            });
  return true;
}

template <typename T>
bool momentum_pair_v2(blr_ctx* c, FlowRef v, FlowRef dv, int substeps, const Cx<T>* rho_end,
                      const Cx<T>* drho_end, Cx<T>* rho, Cx<T>* drho) {
  PadEngine* e = engine<T>(c);
  if (!e) return false;
  const Geom& g = c->g;
  const PadGeom& pg = e->g;
  const int d = g.d, dd = d * d;
  Tmp2 tmp(c);
  VelBank2<T> V(c, e, v, false, tmp);
  VelBank2<T> dV(c, e, dv, false, tmp);
  Cx<T>* cur = tmp.get<Cx<T>>(2 * d * pg.nh);
  full_to_h<T>(c, e, rho_end, d, cur);
  full_to_h<T>(c, e, drho_end, d, cur + d * pg.nh);
  Cx<T>* S = tmp.get<Cx<T>>(2 * d * pg.ns);
  Cx<T>* So = tmp.get<Cx<T>>(2 * dd * pg.ns);
  rk4_v2<T>(c, e, v.n_steps, substeps, false, cur, 2 * d, {{0, d, rho}, {d, d, drho}}, tmp,
            [&](int, double t, const Cx<T>* s, const Rk& rk) {
              const auto& vt = V.at(t);
              const auto& dvt = dV.at(t);
              std::vector<InvSpec<T>> f;
              for (int a = 0; a < 2 * d; ++a) f.push_back(inv1<T>(s + a * pg.nh, -1));
              inv2d<T>(c, e, f, S);
              LineArgs<T> la;
              std::memset(&la, 0, sizeof(la));
              la.d = d; la.ns = 2 * d; la.nr = 2 * d; la.no = 2 * dd;
              for (int i = 0; i < 2 * d; ++i) la.sin[i] = S + i * pg.ns;
              for (int j = 0; j < d; ++j) {
                la.rin[j] = vt.real + j * pg.np;
                la.rin[d + j] = dvt.real + j * pg.np;
              }
              for (int i = 0; i < 2 * dd; ++i) la.sout[i] = So + i * pg.ns;
              lines<T, kOpOuterPair>(c, e, la, sbytes(pg, 2 * d, 2 * d, 2 * dd, 0, sizeof(T)));
              std::vector<FwdSpec<T>> outs;
              push_flux<T>(g, pg, So, outs);
              push_flux<T>(g, pg, So + dd * pg.ns, outs);
              fwd2d<T>(c, e, outs, nullptr, rk);
            });
  return true;
}

// contract: out = sum_i w_i (rho_i + pi(D(phi_i)^T rho_i)) or per node
template <typename T>
bool contract_v2(blr_ctx* c, const Cx<T>* phi, const Cx<T>* rho, int n_nodes, const double* weights,
                 bool transpose, T* dphi_cache, int cache_mode, Cx<T>* out) {
  PadEngine* e = engine<T>(c);
  if (!e) return false;
  if (n_nodes > 32) return false;
  const Geom& g = c->g;
  const PadGeom& pg = e->g;
  const int d = g.d, dd = d * d;
  const int64_t nb = g.nb(), L = d * nb;
  Tmp2 tmp(c);
  // D(phi_i) realizations (cache fill or temporary)
  T* M = dphi_cache;
  if (cache_mode == 0) M = tmp.get<T>((int64_t)n_nodes * dd * pg.np);
  if (cache_mode != 2) {
    Cx<T>* H = tmp.get<Cx<T>>(d * pg.nh);
    Cx<T>* S = tmp.get<Cx<T>>(dd * pg.ns);
    for (int i = 0; i < n_nodes; ++i) {
      full_to_h<T>(c, e, phi + i * L, d, H);
      std::vector<InvSpec<T>> f;
      push_jac<T>(g, pg, H, f);
      inv2d<T>(c, e, f, S);
      LineArgs<T> la;
      std::memset(&la, 0, sizeof(la));
      la.ns = dd; la.d = d;
      for (int k = 0; k < dd; ++k) {
        la.sin[k] = S + k * pg.ns;
        la.wout[k] = M + ((int64_t)i * dd + k) * pg.np;
      }
      lines<T, kOpRealize>(c, e, la, sbytes(pg, dd, 0, 0, dd, sizeof(T)));
    }
  }
  // rho nodes -> S layout (all nodes)
  Cx<T>* RH = tmp.get<Cx<T>>(d * pg.nh);
  Cx<T>* RS = tmp.get<Cx<T>>((int64_t)n_nodes * d * pg.ns);
  for (int i = 0; i < n_nodes; ++i) {
    full_to_h<T>(c, e, rho + i * L, d, RH);
    std::vector<InvSpec<T>> f;
    for (int a = 0; a < d; ++a) f.push_back(inv1<T>(RH + a * pg.nh, -1));
    inv2d<T>(c, e, f, RS + (int64_t)i * d * pg.ns);
  }
  Cx<T>* So = tmp.get<Cx<T>>(d * pg.ns);
  Cx<T>* Kh = tmp.get<Cx<T>>(d * pg.nh);
  Cx<T>* Kf = tmp.get<Cx<T>>(L);
  const bool summed = weights != nullptr;
  const int nrun = summed ? 1 : n_nodes;
  if (summed) BLR_CUDA(cudaMemsetAsync(out, 0, L * sizeof(Cx<T>), c->stream));
  for (int run = 0; run < nrun; ++run) {
    LineArgs<T> la;
    std::memset(&la, 0, sizeof(la));
    la.d = d; la.no = d; la.transpose = transpose ? 1 : 0;
    la.n_nodes = summed ? n_nodes : 1;
    const int node0 = summed ? 0 : run;
    la.sin_node_stride = (int64_t)d * pg.ns;
    la.rin_node_stride = (int64_t)dd * pg.np;
    for (int a = 0; a < d; ++a) la.sin[a] = RS + ((int64_t)node0 * d + a) * pg.ns;
    for (int k = 0; k < dd; ++k) la.rin[k] = M + ((int64_t)node0 * dd + k) * pg.np;
    for (int i = 0; i < la.n_nodes; ++i) la.w[i] = summed ? weights[i] : 1.0;
    for (int i = 0; i < d; ++i) la.sout[i] = So + i * pg.ns;
    lines<T, kOpContract>(c, e, la,
                          (double)la.n_nodes * (d * pg.ns * sizeof(Cx<T>) + dd * pg.np * sizeof(T)) +
                              d * pg.ns * sizeof(Cx<T>));
    std::vector<FwdSpec<T>> outs;
    for (int i = 0; i < d; ++i) outs.push_back(fwd1<T>(So + i * pg.ns, kEpiPlain));
    fwd2d<T>(c, e, outs, Kh, Rk());
    h_to_full<T>(c, e, Kh, d, Kf);
    Cx<T>* o = summed ? out : out + run * L;
    if (summed) {
      for (int i = 0; i < n_nodes; ++i) band_axpby<T>(c, weights[i], rho + i * L, 1.0, o, L);
      band_axpby<T>(c, 1.0, Kf, 1.0, o, L);
    } else {
      BLR_CUDA(cudaMemcpyAsync(o, rho + run * L, L * sizeof(Cx<T>), cudaMemcpyDeviceToDevice, c->stream));
      band_axpby<T>(c, 1.0, Kf, 1.0, o, L);
    }
  }
  return true;
}

#define BLR_PINST(T)                                                                                   \
  template bool pad_engine_ok<T>(blr_ctx*);                                                            \
  template bool forward_map_v2<T>(blr_ctx*, FlowRef, int, Cx<T>*, T*);                                 \
  template bool inverse_map_and_volume_v2<T>(blr_ctx*, FlowRef, int, Cx<T>*, Cx<T>*);                  \
  template bool state_tangents_v2<T>(blr_ctx*, FlowRef, FlowRef, int, int, const T*, Cx<T>*, Cx<T>*,   \
                                     Cx<T>*);                                                          \
  template bool momentum_v2<T>(blr_ctx*, FlowRef, int, const Cx<T>*, Cx<T>*);                          \
  template bool momentum_pair_v2<T>(blr_ctx*, FlowRef, FlowRef, int, const Cx<T>*, const Cx<T>*,       \
                                    Cx<T>*, Cx<T>*);                                                   \
  template bool contract_v2<T>(blr_ctx*, const Cx<T>*, const Cx<T>*, int, const double*, bool, T*, int, \
                               Cx<T>*);
BLR_PINST(double)
BLR_PINST(float)

}  // namespace blr
