// blr_fft.cuh — batched mixed-radix (2, 3, 4, 5, 7) Stockham FFTs in shared
// memory, used by the fused pad-grid kernels (blr_pad.cu).
//
// A CTA transforms `nlines` independent lines of length L stored contiguously
// ([line][L]) in shared memory, ping-ponging between two buffers; every thread
// of the CTA takes butterflies in a strided loop.  Twiddles come from a
// shared table tw[m] = exp(-2 pi i m / L) (double-accurate, cast to T).
// Stockham autosort: pass with radix R after Ns = prod(previous radices):
//   v[r] = x[j + r*L/R] * w^(k r), k = j mod Ns, w = exp(-2 pi i / (Ns R))
//   y[(j/Ns)*Ns*R + k + r*Ns] = DFT_R(v)[r]
#pragma once

#include "blr_common.cuh"

namespace blr {

struct FftSpec {
  int L;
  int nfac;
  int fac[12];
};

// host: factor L into radices (4 first, then 2, 3, 5, 7); ok=false if not 7-smooth
inline FftSpec make_fft(int L, bool* ok) {
  FftSpec s;
  s.L = L;
  s.nfac = 0;
  int r = L;
  const int rad[5] = {4, 2, 3, 5, 7};
  for (int q : rad)
    while (r % q == 0 && s.nfac < 12) {
      s.fac[s.nfac++] = q;
      r /= q;
    }
  *ok = (r == 1);
  return s;
}

template <typename T>
__device__ __forceinline__ Cx<T> cx(T re, T im) {
  Cx<T> z;
  z.x = re;
  z.y = im;
  return z;
}
#define BLR_CX_OPS(C, R)                                                                     \
  __device__ __forceinline__ C cadd(C a, C b) { C z; z.x = a.x + b.x; z.y = a.y + b.y; return z; } \
  __device__ __forceinline__ C csub(C a, C b) { C z; z.x = a.x - b.x; z.y = a.y - b.y; return z; } \
  __device__ __forceinline__ C cmul(C a, C b) {                                              \
    C z; z.x = a.x * b.x - a.y * b.y; z.y = a.x * b.y + a.y * b.x; return z;                 \
  }                                                                                          \
  __device__ __forceinline__ C cconj(C a) { a.y = -a.y; return a; }                          \
  __device__ __forceinline__ C cmul_i(C a) { C z; z.x = -a.y; z.y = a.x; return z; }         \
  __device__ __forceinline__ C cscale(C a, R s) { a.x *= s; a.y *= s; return a; }
BLR_CX_OPS(double2, double)
BLR_CX_OPS(float2, float)
#undef BLR_CX_OPS

// cos / sin (2 pi q / R) for the odd radices (q = m*r mod R); constant-folded
__device__ __forceinline__ constexpr double rad_cos(int R, int q) {
  switch (R * 8 + q) {
    case 24: return 1.0;
    case 25: return -0.4999999999999998;
    case 26: return -0.5000000000000004;
    case 40: return 1.0;
    case 41: return 0.30901699437494745;
    case 42: return -0.8090169943749473;
    case 43: return -0.8090169943749476;
    case 44: return 0.30901699437494723;
    case 56: return 1.0;
    case 57: return 0.6234898018587336;
    case 58: return -0.22252093395631434;
    case 59: return -0.900968867902419;
    case 60: return -0.9009688679024191;
    case 61: return -0.2225209339563146;
    case 62: return 0.6234898018587334;
  }
  return 0.0;
}
__device__ __forceinline__ constexpr double rad_sin(int R, int q) {
  switch (R * 8 + q) {
    case 24: return 0.0;
    case 25: return 0.8660254037844387;
    case 26: return -0.8660254037844384;
    case 40: return 0.0;
    case 41: return 0.9510565162951535;
    case 42: return 0.5877852522924732;
    case 43: return -0.587785252292473;
    case 44: return -0.9510565162951536;
    case 56: return 0.0;
    case 57: return 0.7818314824680298;
    case 58: return 0.9749279121818236;
    case 59: return 0.43388373911755823;
    case 60: return -0.433883739117558;
    case 61: return -0.9749279121818236;
    case 62: return -0.7818314824680299;
  }
  return 0.0;
}

// in-register radix-R DFT; INV selects exp(+2 pi i m r / R)
template <typename T, int R, bool INV>
__device__ __forceinline__ void dft(Cx<T>* v) {
  if constexpr (R == 2) {
    Cx<T> a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (R == 4) {
    Cx<T> t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
    Cx<T> t2 = cadd(v[1], v[3]), t3 = csub(v[1], v[3]);
    Cx<T> it3 = cmul_i(t3);
    v[0] = cadd(t0, t2);
    v[2] = csub(t0, t2);
    if (INV) {
      v[1] = cadd(t1, it3);
      v[3] = csub(t1, it3);
    } else {
      v[1] = csub(t1, it3);
      v[3] = cadd(t1, it3);
    }
  } else {
    constexpr int H = (R - 1) / 2;
    Cx<T> a[H], b[H];
    Cx<T> y0 = v[0];
#pragma unroll
    for (int r = 1; r <= H; ++r) {
      a[r - 1] = cadd(v[r], v[R - r]);
      b[r - 1] = csub(v[r], v[R - r]);
      y0 = cadd(y0, a[r - 1]);
    }
    Cx<T> out[R];
    out[0] = y0;
#pragma unroll
    for (int m = 1; m <= H; ++m) {
      Cx<T> A = v[0], Bs = cx<T>(0, 0);
#pragma unroll
      for (int r = 1; r <= H; ++r) {
        const T c = (T)rad_cos(R, (m * r) % R);
        const T s = (T)rad_sin(R, (m * r) % R);
        A = cadd(A, cscale(a[r - 1], c));
        Bs = cadd(Bs, cscale(b[r - 1], s));
      }
      Cx<T> iB = cmul_i(Bs);
      if (INV) {
        out[m] = cadd(A, iB);
        out[R - m] = csub(A, iB);
      } else {
        out[m] = csub(A, iB);
        out[R - m] = cadd(A, iB);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = out[r];
  }
}

template <typename T, int R, bool INV>
__device__ __forceinline__ void stockham_pass(const Cx<T>* __restrict__ x, Cx<T>* __restrict__ y,
                                              int nlines, int L, int Ns, const Cx<T>* tw) {
  const int nbf = L / R;
  const int twstep = L / (Ns * R);
  const int total = nlines * nbf;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int line = idx / nbf;
    const int j = idx - line * nbf;
    const int k = j % Ns;
    const Cx<T>* xl = x + line * L;
    Cx<T> v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = xl[j + r * nbf];
    if (Ns > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) {
        Cx<T> w = tw[(k * r * twstep) % L];
        if (INV) w.y = -w.y;
        v[r] = cmul(v[r], w);
      }
    }
    dft<T, R, INV>(v);
    Cx<T>* yl = y + line * L + (j / Ns) * Ns * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) yl[r * Ns] = v[r];
  }
}

// Transform nlines lines in `a` (ping-pong with `b`); returns the buffer
// holding the result.  Synchronizes the CTA between passes and at the end.
template <typename T, bool INV>
__device__ Cx<T>* fft_lines(Cx<T>* a, Cx<T>* b, int nlines, const FftSpec& s, const Cx<T>* tw) {
  int Ns = 1;
  for (int p = 0; p < s.nfac; ++p) {
    const int R = s.fac[p];
    switch (R) {
      case 2: stockham_pass<T, 2, INV>(a, b, nlines, s.L, Ns, tw); break;
      case 3: stockham_pass<T, 3, INV>(a, b, nlines, s.L, Ns, tw); break;
      case 4: stockham_pass<T, 4, INV>(a, b, nlines, s.L, Ns, tw); break;
      case 5: stockham_pass<T, 5, INV>(a, b, nlines, s.L, Ns, tw); break;
      default: stockham_pass<T, 7, INV>(a, b, nlines, s.L, Ns, tw); break;
    }
    __syncthreads();
    Cx<T>* t = a;
    a = b;
    b = t;
    Ns *= R;
  }
  return a;
}

}  // namespace blr
