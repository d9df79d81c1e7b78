// blr_common.cuh — shared types, geometry and launch helpers for the
// blreg_b200 sm_100a library.
//
// Geometry convention: every domain is embedded in 3 axes with the real axes
// trailing (2-D (N0,N1) -> (1,N0,N1), bandwidth (0,K0,K1)).  A dummy axis has
// N = B = P = 1 and K = 0, so it contributes only the zero frequency.  Vector
// component c (0..d-1) lives on 3-axis a = 3 - d + c.
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>
#include <stdint.h>

#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace blr {

constexpr double kTwoPi = 6.283185307179586;  // 2*pi rounded to double (== numpy 2.0*np.pi)

template <typename T> struct CxT;
template <> struct CxT<double> { using type = double2; };
template <> struct CxT<float> { using type = float2; };
template <typename T> using Cx = typename CxT<T>::type;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void check_cuda(cudaError_t e, const char* what);
void check_fft(cufftResult r, const char* what);
void count_launch(int n = 1);

#define BLR_CUDA(x) ::blr::check_cuda((x), #x)

// Bounds-checked builds (BLR_CHECKED=1, e.g. BLR_DEFINES="BLR_CHECKED=1" with
// BLR_OUT_DIR for a variant library): every BLR_CHECK asserts an index range
// on the device and traps with the check's tag on violation.  This replaces
// compute-sanitizer, which the GPU pool does not allow.  Compiled out by default.
#ifndef BLR_CHECKED
#define BLR_CHECKED 0
#endif
#if BLR_CHECKED
#include <cstdio>
#define BLR_CHECK(cond, tag)                                                                          \
  do {                                                                                                \
    if (!(cond)) {                                                                                    \
      printf("BLR_CHECK failed: %s (%s:%d) block %d thread %d\n", tag, __FILE__, __LINE__,            \
             (int)blockIdx.x, (int)threadIdx.x);                                                      \
      asm volatile("trap;");                                                                          \
    }                                                                                                 \
  } while (0)
#else
#define BLR_CHECK(cond, tag) do { } while (0)
#endif
#define BLR_FFT(x) ::blr::check_fft((x), #x)
#define BLR_LAUNCHED() do { ::blr::check_cuda(cudaGetLastError(), "kernel launch"); ::blr::count_launch(); } while (0)

// A periodic grid that band blocks are realized on (the full image grid or the
// pad grid), with the band geometry needed to map frequencies to bins.
struct GridDesc {
  int G[3];   // grid points per axis
  int Gh;     // G[2]/2 + 1 (Hermitian half of the last axis)
  int K[3];   // bandwidth per axis
  int B[3];   // 2K+1
  __host__ __device__ int64_t real_size() const { return (int64_t)G[0] * G[1] * G[2]; }
  __host__ __device__ int64_t half_size() const { return (int64_t)G[0] * G[1] * Gh; }
};

struct Geom {
  int d;
  int N[3], K[3], B[3], P[3];
  double alpha;
  int order;
  int64_t nb() const { return (int64_t)B[0] * B[1] * B[2]; }
  int64_t np() const { return (int64_t)P[0] * P[1] * P[2]; }
  int64_t nn() const { return (int64_t)N[0] * N[1] * N[2]; }
  int axis_of(int comp) const { return 3 - d + comp; }
  GridDesc grid(bool pad) const {
    GridDesc g;
    for (int a = 0; a < 3; ++a) {
      g.G[a] = pad ? P[a] : N[a];
      g.K[a] = K[a];
      g.B[a] = B[a];
    }
    g.Gh = g.G[2] / 2 + 1;
    return g;
  }
};

// Block-index -> integer frequency (FFT wrap order, domain.py:93-97).
__host__ __device__ inline int freq_of(int i, int K, int B) { return i <= K ? i : i - B; }
__host__ __device__ inline int pmod(int a, int m) { int r = a % m; return r < 0 ? r + m : r; }

inline int grid_blocks(int64_t n, int threads, int max_blocks = 148 * 16) {
  int64_t b = (n + threads - 1) / threads;
  if (b > max_blocks) b = max_blocks;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace blr

// ---------------------------------------------------------------------------
// the context (opaque in the C ABI)
// ---------------------------------------------------------------------------
struct blr_ctx {
  int dtype = 0;  // 0 f64, 1 f32
  int device = 0;
  cudaStream_t stream = nullptr;
  blr::Geom g{};
  double* d_sym = nullptr;   // per-axis alpha-free symbol terms, 3 segments of B[a]
  std::vector<double> h_sym;  // same, host copy

  // cuFFT plans keyed by (pad?, batch, forward?)
  std::map<int64_t, cufftHandle> plans;
  void* fft_work = nullptr;
  size_t fft_work_size = 0;

  // scratch (bytes), grown on demand
  void* real_buf = nullptr; size_t real_bytes = 0;
  void* half_buf = nullptr; size_t half_bytes = 0;
  void* band_buf = nullptr; size_t band_bytes = 0;
  void* full_buf = nullptr; size_t full_bytes = 0;
  double* d_red = nullptr;   // reduction partials
  double* h_red = nullptr;   // pinned host result
  int red_cap = 0;

  size_t elem() const { return dtype == 0 ? 8 : 4; }
};

namespace blr {
cufftHandle get_plan(blr_ctx* c, bool pad, int batch, bool forward);
void* scratch(blr_ctx* c, void*& buf, size_t& cap, size_t need);
}  // namespace blr
