// blr_fft.cuh — warp-synchronous FFTs for the fused pad-grid kernels.
//
// Line length L = R1 * R2 (R1, R2 <= 16, 7-smooth).  Four-step across lanes:
//   x[n], n = R2*n1 + n2;   X[k], k = k1 + R1*k2;
//   step A, lane (line, n2): DFT_R1 over n1 in registers, times W_L^(n2 k1),
//                            written to a per-warp shared tile [line][k1][n2];
//   __syncwarp();
//   step B, lane (line, k1): DFT_R2 over n2 in registers -> X[k1 + R1 k2].
// Every warp transforms its own LPW = 32 / max(R1, R2) lines: no CTA-wide
// barriers, the whole butterfly network of a pass lives in registers.
// Composite register DFTs (6, 8, 9, 10, 12, 14, 15, 16) recurse into the
// radix-2/3/4/5/7 kernels with compile-time twiddles.
#pragma once

#include "blr_common.cuh"

namespace blr {

template <typename T>
__device__ __forceinline__ Cx<T> cx(T re, T im) {
  Cx<T> z;
  z.x = re;
  z.y = im;
  return z;
}
#define BLR_CX_OPS(C, R)                                                                           \
  __device__ __forceinline__ C cadd(C a, C b) { C z; z.x = a.x + b.x; z.y = a.y + b.y; return z; } \
  __device__ __forceinline__ C csub(C a, C b) { C z; z.x = a.x - b.x; z.y = a.y - b.y; return z; } \
  __device__ __forceinline__ C cmul(C a, C b) {                                                    \
    C z; z.x = a.x * b.x - a.y * b.y; z.y = a.x * b.y + a.y * b.x; return z;                       \
  }                                                                                                \
  __device__ __forceinline__ C cconj(C a) { a.y = -a.y; return a; }                                \
  __device__ __forceinline__ C cmul_i(C a) { C z; z.x = -a.y; z.y = a.x; return z; }               \
  __device__ __forceinline__ C cscale(C a, R s) { a.x *= s; a.y *= s; return a; }
BLR_CX_OPS(double2, double)
BLR_CX_OPS(float2, float)
#undef BLR_CX_OPS

// cos / sin (2 pi m / N); constant-folded after unrolling
__host__ __device__ __forceinline__ constexpr double tw_cos(int N, int m) {
  switch (N * 32 + m) {
    case 96: return 1.0;
    case 97: return -0.4999999999999998;
    case 98: return -0.5000000000000004;
    case 160: return 1.0;
    case 161: return 0.30901699437494745;
    case 162: return -0.8090169943749473;
    case 163: return -0.8090169943749476;
    case 164: return 0.30901699437494723;
    case 192: return 1.0;
    case 193: return 0.5000000000000001;
    case 194: return -0.4999999999999998;
    case 195: return -1.0;
    case 196: return -0.5000000000000004;
    case 197: return 0.5000000000000001;
    case 224: return 1.0;
    case 225: return 0.6234898018587336;
    case 226: return -0.22252093395631434;
    case 227: return -0.900968867902419;
    case 228: return -0.9009688679024191;
    case 229: return -0.2225209339563146;
    case 230: return 0.6234898018587334;
    case 256: return 1.0;
    case 257: return 0.7071067811865476;
    case 258: return 6.123233995736766e-17;
    case 259: return -0.7071067811865475;
    case 260: return -1.0;
    case 261: return -0.7071067811865477;
    case 262: return -1.8369701987210297e-16;
    case 263: return 0.7071067811865474;
    case 288: return 1.0;
    case 289: return 0.766044443118978;
    case 290: return 0.17364817766693041;
    case 291: return -0.4999999999999998;
    case 292: return -0.9396926207859083;
    case 293: return -0.9396926207859084;
    case 294: return -0.5000000000000004;
    case 295: return 0.17364817766692997;
    case 296: return 0.7660444431189778;
    case 320: return 1.0;
    case 321: return 0.8090169943749475;
    case 322: return 0.30901699437494745;
    case 323: return -0.30901699437494734;
    case 324: return -0.8090169943749473;
    case 325: return -1.0;
    case 326: return -0.8090169943749476;
    case 327: return -0.30901699437494756;
    case 328: return 0.30901699437494723;
    case 329: return 0.8090169943749473;
    case 384: return 1.0;
    case 385: return 0.8660254037844387;
    case 386: return 0.5000000000000001;
    case 387: return 6.123233995736766e-17;
    case 388: return -0.4999999999999998;
    case 389: return -0.8660254037844387;
    case 390: return -1.0;
    case 391: return -0.8660254037844388;
    case 392: return -0.5000000000000004;
    case 393: return -1.8369701987210297e-16;
    case 394: return 0.5000000000000001;
    case 395: return 0.8660254037844384;
    case 448: return 1.0;
    case 449: return 0.9009688679024191;
    case 450: return 0.6234898018587336;
    case 451: return 0.22252093395631445;
    case 452: return -0.22252093395631434;
    case 453: return -0.6234898018587335;
    case 454: return -0.900968867902419;
    case 455: return -1.0;
    case 456: return -0.9009688679024191;
    case 457: return -0.6234898018587337;
    case 458: return -0.2225209339563146;
    case 459: return 0.22252093395631334;
    case 460: return 0.6234898018587334;
    case 461: return 0.9009688679024194;
    case 480: return 1.0;
    case 481: return 0.9135454576426009;
    case 482: return 0.6691306063588582;
    case 483: return 0.30901699437494745;
    case 484: return -0.10452846326765333;
    case 485: return -0.4999999999999998;
    case 486: return -0.8090169943749473;
    case 487: return -0.9781476007338057;
    case 488: return -0.9781476007338057;
    case 489: return -0.8090169943749476;
    case 490: return -0.5000000000000004;
    case 491: return -0.10452846326765423;
    case 492: return 0.30901699437494723;
    case 493: return 0.6691306063588585;
    case 494: return 0.913545457642601;
    case 512: return 1.0;
    case 513: return 0.9238795325112867;
    case 514: return 0.7071067811865476;
    case 515: return 0.38268343236508984;
    case 516: return 6.123233995736766e-17;
    case 517: return -0.3826834323650897;
    case 518: return -0.7071067811865475;
    case 519: return -0.9238795325112867;
    case 520: return -1.0;
    case 521: return -0.9238795325112868;
    case 522: return -0.7071067811865477;
    case 523: return -0.38268343236509034;
    case 524: return -1.8369701987210297e-16;
    case 525: return 0.38268343236509;
    case 526: return 0.7071067811865474;
    case 527: return 0.9238795325112865;
  }
  return 1.0;
}
__host__ __device__ __forceinline__ constexpr double tw_sin(int N, int m) {
  switch (N * 32 + m) {
    case 96: return 0.0;
    case 97: return 0.8660254037844387;
    case 98: return -0.8660254037844384;
    case 160: return 0.0;
    case 161: return 0.9510565162951535;
    case 162: return 0.5877852522924732;
    case 163: return -0.587785252292473;
    case 164: return -0.9510565162951536;
    case 192: return 0.0;
    case 193: return 0.8660254037844386;
    case 194: return 0.8660254037844387;
    case 195: return 1.2246467991473532e-16;
    case 196: return -0.8660254037844384;
    case 197: return -0.8660254037844386;
    case 224: return 0.0;
    case 225: return 0.7818314824680298;
    case 226: return 0.9749279121818236;
    case 227: return 0.43388373911755823;
    case 228: return -0.433883739117558;
    case 229: return -0.9749279121818236;
    case 230: return -0.7818314824680299;
    case 256: return 0.0;
    case 257: return 0.7071067811865475;
    case 258: return 1.0;
    case 259: return 0.7071067811865476;
    case 260: return 1.2246467991473532e-16;
    case 261: return -0.7071067811865475;
    case 262: return -1.0;
    case 263: return -0.7071067811865477;
    case 288: return 0.0;
    case 289: return 0.6427876096865393;
    case 290: return 0.984807753012208;
    case 291: return 0.8660254037844387;
    case 292: return 0.3420201433256689;
    case 293: return -0.34202014332566866;
    case 294: return -0.8660254037844384;
    case 295: return -0.9848077530122081;
    case 296: return -0.6427876096865396;
    case 320: return 0.0;
    case 321: return 0.5877852522924731;
    case 322: return 0.9510565162951535;
    case 323: return 0.9510565162951536;
    case 324: return 0.5877852522924732;
    case 325: return 1.2246467991473532e-16;
    case 326: return -0.587785252292473;
    case 327: return -0.9510565162951535;
    case 328: return -0.9510565162951536;
    case 329: return -0.5877852522924734;
    case 384: return 0.0;
    case 385: return 0.49999999999999994;
    case 386: return 0.8660254037844386;
    case 387: return 1.0;
    case 388: return 0.8660254037844387;
    case 389: return 0.49999999999999994;
    case 390: return 1.2246467991473532e-16;
    case 391: return -0.4999999999999997;
    case 392: return -0.8660254037844384;
    case 393: return -1.0;
    case 394: return -0.8660254037844386;
    case 395: return -0.5000000000000004;
    case 448: return 0.0;
    case 449: return 0.4338837391175581;
    case 450: return 0.7818314824680298;
    case 451: return 0.9749279121818236;
    case 452: return 0.9749279121818236;
    case 453: return 0.7818314824680299;
    case 454: return 0.43388373911755823;
    case 455: return 1.2246467991473532e-16;
    case 456: return -0.433883739117558;
    case 457: return -0.7818314824680297;
    case 458: return -0.9749279121818236;
    case 459: return -0.9749279121818238;
    case 460: return -0.7818314824680299;
    case 461: return -0.4338837391175575;
    case 480: return 0.0;
    case 481: return 0.40673664307580015;
    case 482: return 0.7431448254773941;
    case 483: return 0.9510565162951535;
    case 484: return 0.9945218953682734;
    case 485: return 0.8660254037844387;
    case 486: return 0.5877852522924732;
    case 487: return 0.20791169081775931;
    case 488: return -0.20791169081775907;
    case 489: return -0.587785252292473;
    case 490: return -0.8660254037844384;
    case 491: return -0.9945218953682733;
    case 492: return -0.9510565162951536;
    case 493: return -0.743144825477394;
    case 494: return -0.40673664307580015;
    case 512: return 0.0;
    case 513: return 0.3826834323650898;
    case 514: return 0.7071067811865475;
    case 515: return 0.9238795325112867;
    case 516: return 1.0;
    case 517: return 0.9238795325112867;
    case 518: return 0.7071067811865476;
    case 519: return 0.3826834323650899;
    case 520: return 1.2246467991473532e-16;
    case 521: return -0.38268343236508967;
    case 522: return -0.7071067811865475;
    case 523: return -0.9238795325112865;
    case 524: return -1.0;
    case 525: return -0.9238795325112866;
    case 526: return -0.7071067811865477;
    case 527: return -0.3826834323650904;
  }
  return 0.0;
}

constexpr int first_factor(int N) {
  return N % 4 == 0 ? 4 : N % 2 == 0 ? 2 : N % 3 == 0 ? 3 : N % 5 == 0 ? 5 : N % 7 == 0 ? 7 : N;
}

constexpr int cgcd(int a, int b) { return b == 0 ? a : cgcd(b, a % b); }
constexpr int inv_mod(int a, int m) {  // a^-1 mod m (gcd(a, m) = 1)
  int r = 1;
  while ((a * r) % m != 1 % m) ++r;
  return r % m;
}
#ifndef BLR_PFA
#define BLR_PFA 1
#endif
constexpr bool kPfa = BLR_PFA != 0;

// in-register DFT of size N; INV selects exp(+2 pi i m r / N)
template <typename T, int N, bool INV>
__device__ __forceinline__ void dft(Cx<T>* v) {
  if constexpr (N == 1) {
    return;
  } else if constexpr (N == 2) {
    Cx<T> a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (N == 4) {
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
  } else if constexpr (N == 3 || N == 5 || N == 7) {
    constexpr int H = (N - 1) / 2;
    Cx<T> a[H], b[H];
    Cx<T> y0 = v[0];
#pragma unroll
    for (int r = 1; r <= H; ++r) {
      a[r - 1] = cadd(v[r], v[N - r]);
      b[r - 1] = csub(v[r], v[N - r]);
      y0 = cadd(y0, a[r - 1]);
    }
    Cx<T> out[N];
    out[0] = y0;
#pragma unroll
    for (int m = 1; m <= H; ++m) {
      Cx<T> A = v[0], Bs = cx<T>(0, 0);
#pragma unroll
      for (int r = 1; r <= H; ++r) {
        const T c = (T)tw_cos(N, (m * r) % N);
        const T s = (T)tw_sin(N, (m * r) % N);
        A = cadd(A, cscale(a[r - 1], c));
        Bs = cadd(Bs, cscale(b[r - 1], s));
      }
      Cx<T> iB = cmul_i(Bs);
      if (INV) {
        out[m] = cadd(A, iB);
        out[N - m] = csub(A, iB);
      } else {
        out[m] = csub(A, iB);
        out[N - m] = cadd(A, iB);
      }
    }
#pragma unroll
    for (int r = 0; r < N; ++r) v[r] = out[r];
  } else if constexpr (kPfa && cgcd(first_factor(N), N / first_factor(N)) == 1) {
    // composite with coprime factors (10 = 2 x 5, 14 = 2 x 7, 20, 28): Good-Thomas
    // prime-factor mapping, n = (B*n1 + A*n2) mod N, k = (k1*B*Binv + k2*A*Ainv) mod N.
    // No twiddle multiplies between the sub-transforms; the index maps are
    // compile-time (fully unrolled register indices), so they cost nothing.
    constexpr int A = first_factor(N);
    constexpr int B = N / A;
    constexpr int Binv = inv_mod(B, A), Ainv = inv_mod(A, B);
    Cx<T> t[N];
#pragma unroll
    for (int n2 = 0; n2 < B; ++n2) {
      Cx<T> s[A];
#pragma unroll
      for (int n1 = 0; n1 < A; ++n1) s[n1] = v[(B * n1 + A * n2) % N];
      dft<T, A, INV>(s);
#pragma unroll
      for (int k1 = 0; k1 < A; ++k1) t[k1 * B + n2] = s[k1];
    }
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) {
      Cx<T> s[B];
#pragma unroll
      for (int n2 = 0; n2 < B; ++n2) s[n2] = t[k1 * B + n2];
      dft<T, B, INV>(s);
#pragma unroll
      for (int k2 = 0; k2 < B; ++k2) v[(k1 * B * Binv + k2 * A * Ainv) % N] = s[k2];
    }
  } else {
    // composite: four-step in registers, n = B*n1 + n2, k = k1 + A*k2
    constexpr int A = first_factor(N);
    constexpr int B = N / A;
    Cx<T> t[N];
#pragma unroll
    for (int n2 = 0; n2 < B; ++n2) {
      Cx<T> s[A];
#pragma unroll
      for (int n1 = 0; n1 < A; ++n1) s[n1] = v[B * n1 + n2];
      dft<T, A, INV>(s);
#pragma unroll
      for (int k1 = 0; k1 < A; ++k1) {
        if (n2 * k1 != 0) {
          const T c = (T)tw_cos(N, (n2 * k1) % N);
          const T sn = (T)(INV ? tw_sin(N, (n2 * k1) % N) : -tw_sin(N, (n2 * k1) % N));
          s[k1] = cmul(s[k1], cx<T>(c, sn));
        }
        t[k1 * B + n2] = s[k1];
      }
    }
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) {
      Cx<T> s[B];
#pragma unroll
      for (int n2 = 0; n2 < B; ++n2) s[n2] = t[k1 * B + n2];
      dft<T, B, INV>(s);
#pragma unroll
      for (int k2 = 0; k2 < B; ++k2) v[k1 + A * k2] = s[k2];
    }
  }
}

// Warp four-step transform of a line length L = R1 * R2.
template <int R1_, int R2_>
struct WShape {
  static constexpr int R1 = R1_;
  static constexpr int R2 = R2_;
  static constexpr int L = R1 * R2;
  static constexpr int RM = R1 > R2 ? R1 : R2;
  static constexpr int LPW = 32 / RM;               // lines per warp
};

// --- shared-memory bank model ----------------------------------------------
// A warp request of E-byte accesses is served in phases of 128/E lanes; a
// phase costs the largest number of distinct 4-byte words any one bank must
// deliver (same word = broadcast).  ncu's "L1 Wavefronts Shared" match this
// model on the r02 captures (tile stores 1.50x ideal, twiddle loads 2.5x).
// addr(lane) < 0: inactive lane.
template <class F>
constexpr int wavefronts(F addr, int E) {
  const int per = 128 / E, words = E / 4;
  int tot = 0;
  for (int p0 = 0; p0 < 32; p0 += per) {
    int uniq[32] = {}, nu = 0;  // distinct element addresses of the phase
    for (int lane = p0; lane < p0 + per; ++lane) {
      const int a = addr(lane);
      bool dup = a < 0;
      for (int q = 0; q < nu && !dup; ++q) dup = uniq[q] == a;
      if (!dup) uniq[nu++] = a;
    }
    int cnt[32] = {};
    for (int q = 0; q < nu; ++q)
      for (int w = 0; w < words; ++w) ++cnt[(uniq[q] * words + w) % 32];
    int worst = 0;
    for (int b = 0; b < 32; ++b) worst = cnt[b] > worst ? cnt[b] : worst;
    tot += worst;
  }
  return tot;
}

// Per-warp FFT tile [line][k1][n2] at line * TS + k1 * KS + n2, strides chosen
// by the bank model for the step-A stores and step-B loads (fp64: 80
// wavefronts per L=100 transform instead of 100 with the dense R2+1 stride).
template <class S>
constexpr int tile_cost(int TS, int KS, int E) {
  int c = 0;
  for (int k1 = 0; k1 < S::R1; ++k1)
    c += wavefronts([&](int l) { return l / S::R2 < S::LPW ? (l / S::R2) * TS + k1 * KS + l % S::R2 : -1; }, E);
  for (int n2 = 0; n2 < S::R2; ++n2)
    c += wavefronts([&](int l) { return l / S::R1 < S::LPW ? (l / S::R1) * TS + (l % S::R1) * KS + n2 : -1; }, E);
  return c;
}
// Bank-model strides: always for fp32, for fp64 only with BLR_BANKPAD=1.  A/B
// on the B200 (r02): in fp64 the conflict-free layout cut the z-line kernels'
// shared wavefronts by 30-45% but not their time (latency-bound at 8-12 warps
// per SM) and its larger footprint cost the outer op a CTA per SM (deformation
// GN HVP 10.25 vs 10.0 ms); in fp32 it is a win (7.08 vs 7.56 ms).
#ifndef BLR_BANKPAD
#define BLR_BANKPAD 0
#endif
template <typename T>
constexpr bool bank_pad() { return BLR_BANKPAD || sizeof(T) == 4; }
template <typename T, class S>
struct TileG {
  static constexpr int E = (int)(2 * sizeof(T));
  static constexpr int best() {  // KS * 256 + TS
    if (!bank_pad<T>()) return (S::R2 + 1) * 256 + S::R1 * (S::R2 + 1);
    int bc = 1 << 30, bv = 0;
    for (int ks = S::R2; ks < S::R2 + 8; ++ks) {
      const int base = (S::R1 - 1) * ks + S::R2;
      for (int ts = base; ts < base + 8; ++ts) {
        const int c = tile_cost<S>(ts, ks, E);
        if (c < bc) { bc = c; bv = ks * 256 + ts; }
      }
    }
    return bv;
  }
  static constexpr int KS = best() / 256;
  static constexpr int TS = best() % 256;          // shared tile entries per line
  static constexpr int TILE = S::LPW * TS;         // shared tile entries per warp
};

// Step-A twiddles W_L^(k1 n2) are read from a split table of T: real parts at
// twr[k1 * R2 + n2], imaginary parts at twr[L + k1 * R2 + n2].  Lanes of a
// request differ in n2 only, so the two 8-byte (fp64) loads are conflict-free
// (the packed table tw[k1 * n2] cost 2.4x the ideal wavefronts).
#ifndef BLR_TW_SYM
#define BLR_TW_SYM 2
#endif
template <typename T, class S>
__device__ __forceinline__ Cx<T> twiddle(const T* twr, int k1, int n2) {
  return cx<T>(twr[k1 * S::R2 + n2], twr[S::L + k1 * S::R2 + n2]);
}

// step A: lanes (line, n2) gather x[R2*n1 + n2] with load(line, n, n1), DFT_R1,
// twiddle W_L^(n2 k1), store to the tile.
// ALIAS: the tile overlays the warp's own input lines in shared memory, so all
// lanes finish loading before any lane stores.
template <typename T, class S, bool INV, bool ALIAS = false, class Load>
__device__ __forceinline__ void wfft_a(Cx<T>* tile, const T* twr, int nl, Load& load) {
  using G = TileG<T, S>;
  const int lane = threadIdx.x & 31;
  const int line = lane / S::R2, n2 = lane - (lane / S::R2) * S::R2;
  const bool act = line < nl && line < S::LPW;
  Cx<T> v[S::R1];
  if (act) {
#pragma unroll
    for (int n1 = 0; n1 < S::R1; ++n1) v[n1] = load(line, S::R2 * n1 + n2, n1);
  }
  if (ALIAS) __syncwarp();
  if (act) {
    dft<T, S::R1, INV>(v);
    Cx<T>* t = tile + line * G::TS + n2;
    BLR_CHECK(line * G::TS + (S::R1 - 1) * G::KS + n2 < G::TILE, "wfft_a tile");
    if constexpr (BLR_TW_SYM && S::R1 >= 4) {
      // half the table loads: W^(k1 n2) for k1 <= M from the table, W^(R1 n2)
      // from their products, and W^(k1 n2) = W^(R1 n2) conj(W^((R1 - k1) n2))
      // for k1 > M (shared-memory / L1 loads traded for fp64 multiplies)
      constexpr int M = (S::R1 + 1) / 2;
      // BLR_TW_SYM >= 2: only k1 <= 5 - BLR_TW_SYM from the table, the rest of
      // k1 <= M as products of two lower powers
      constexpr int NLmax = BLR_TW_SYM >= 2 ? 5 - BLR_TW_SYM : M;
      constexpr int NL = M > NLmax ? NLmax : M;
      Cx<T> w[S::R1];
#pragma unroll
      for (int k1 = 1; k1 <= NL; ++k1) w[k1] = twiddle<T, S>(twr, k1, n2);
#pragma unroll
      for (int k1 = NL + 1; k1 <= M; ++k1) w[k1] = cmul(w[k1 / 2], w[k1 - k1 / 2]);
      const Cx<T> wr = S::R1 % 2 == 0 ? cmul(w[S::R1 / 2], w[S::R1 / 2]) : cmul(w[M - 1], w[M]);
#pragma unroll
      for (int k1 = M + 1; k1 < S::R1; ++k1) {
        Cx<T> c = w[S::R1 - k1];
        c.y = -c.y;
        w[k1] = cmul(wr, c);
      }
#pragma unroll
      for (int k1 = 0; k1 < S::R1; ++k1) {
        Cx<T> z = v[k1];
        if (k1 * n2 != 0) {
          Cx<T> ww = w[k1 > 0 ? k1 : 1];
          if (INV) ww.y = -ww.y;
          z = cmul(z, ww);
        }
        t[k1 * G::KS] = z;
      }
    } else {
#pragma unroll
      for (int k1 = 0; k1 < S::R1; ++k1) {
        Cx<T> z = v[k1];
        if (k1 * n2 != 0) {
          Cx<T> w = twiddle<T, S>(twr, k1, n2);
          if (INV) w.y = -w.y;
          z = cmul(z, w);
        }
        t[k1 * G::KS] = z;
      }
    }
  }
  __syncwarp();
}

// step B: lanes (line, k1) read the tile, DFT_R2, hand X[k1 + R1 k2] to
// store(line, k, value) (k2 ascending).
template <typename T, class S, bool INV, class Store>
__device__ __forceinline__ void wfft_b(const Cx<T>* tile, int nl, Store& store) {
  using G = TileG<T, S>;
  const int lane = threadIdx.x & 31;
  const int line = lane / S::R1, k1 = lane - (lane / S::R1) * S::R1;
  if (line < nl && line < S::LPW) {
    Cx<T> u[S::R2];
    const Cx<T>* t = tile + line * G::TS + k1 * G::KS;
    BLR_CHECK(line * G::TS + k1 * G::KS + S::R2 - 1 < G::TILE, "wfft_b tile");
#pragma unroll
    for (int n2 = 0; n2 < S::R2; ++n2) u[n2] = t[n2];
    dft<T, S::R2, INV>(u);
#pragma unroll
    for (int k2 = 0; k2 < S::R2; ++k2) store(line, k1 + S::R1 * k2, k2, u[k2]);
  }
  __syncwarp();
}

template <typename T, class S, bool INV, bool ALIAS = false, class Load, class Store>
__device__ __forceinline__ void wfft(Cx<T>* tile, const T* twr, int nl, Load load, Store store) {
  wfft_a<T, S, INV, ALIAS>(tile, twr, nl, load);
  wfft_b<T, S, INV>(tile, nl, store);
}

// supported line lengths -> (R1, R2); dispatch helper
#define BLR_FOR_EACH_L(X) \
  X(1, 1, 1)              \
  X(10, 5, 2)             \
  X(14, 7, 2)             \
  X(16, 4, 4)             \
  X(20, 5, 4)             \
  X(25, 5, 5)             \
  X(28, 7, 4)             \
  X(32, 8, 4)             \
  X(40, 8, 5)             \
  X(49, 7, 7)             \
  X(50, 10, 5)            \
  X(64, 8, 8)             \
  X(100, 10, 10)          \
  X(196, 14, 14)

// lengths of the z axis (always a real axis: no L = 1)
#define BLR_FOR_EACH_LZ(X) \
  X(10, 5, 2)              \
  X(14, 7, 2)              \
  X(16, 4, 4)              \
  X(20, 5, 4)              \
  X(25, 5, 5)              \
  X(28, 7, 4)              \
  X(32, 8, 4)              \
  X(40, 8, 5)              \
  X(49, 7, 7)              \
  X(50, 10, 5)             \
  X(64, 8, 8)              \
  X(100, 10, 10)           \
  X(196, 14, 14)

inline int shape_r2(int L) {
#define BLR_CASE(LL, A, B) if (L == LL) return B;
  BLR_FOR_EACH_L(BLR_CASE)
#undef BLR_CASE
  return 1;
}

inline bool supported_len(int L) {
#define BLR_CASE(LL, A, B) if (L == LL) return true;
  BLR_FOR_EACH_L(BLR_CASE)
#undef BLR_CASE
  return false;
}

}  // namespace blr
