// blr_grid.cu — full-grid operations on sm_100a (gridops.py, objectives/*.py).
//
// Periodic warps (nearest / trilinear / cubic B-spline with an exact FFT
// prefilter), central and spectral gradients, the Jacobian determinant, and
// the fused per-voxel data terms of the two objectives.
#include "blr_internal.cuh"

#include <cmath>

namespace blr {

struct FullDesc {
  int N[3];
  int d;
  int64_t nn;
};

static FullDesc full_desc(const Geom& g) {
  FullDesc f;
  for (int a = 0; a < 3; ++a) f.N[a] = g.N[a];
  f.d = g.d;
  f.nn = g.nn();
  return f;
}

__device__ inline void unravel(const FullDesc& fd, int64_t i, int* x) {
  if (fd.nn <= 0x7fffffff) {  // 32-bit divisions (the 64-bit ones cost ~5x)
    int j = (int)i;
    x[2] = j % fd.N[2];
    j /= fd.N[2];
    x[1] = j % fd.N[1];
    x[0] = j / fd.N[1];
    return;
  }
  x[2] = (int)(i % fd.N[2]);
  i /= fd.N[2];
  x[1] = (int)(i % fd.N[1]);
  x[0] = (int)(i / fd.N[1]);
}

__device__ inline int64_t ravel(const FullDesc& fd, int x0, int x1, int x2) {
  return ((int64_t)x0 * fd.N[1] + x1) * fd.N[2] + x2;
}

// Index-space sample coordinate of id + u on every real axis
// (gridops.py:21-29: coords = i + u * N, computed in float64).
template <typename T>
__device__ inline void sample_coords(const FullDesc& fd, const T* disp, int64_t i, const int* x,
                                     double* c) {
  // static axis loop (no dynamically indexed local arrays): axis a carries
  // displacement component a - (3 - d) when that is >= 0
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int comp = a - (3 - fd.d);
    c[a] = comp >= 0 ? (double)x[a] + (double)disp[comp * fd.nn + i] * (double)fd.N[a] : 0.0;
  }
}

// cubic B-spline weights for fractional t at taps -1, 0, 1, 2
__device__ inline void bspline3(double t, double* w) {
  double t2 = t * t, t3 = t2 * t, u = 1.0 - t;
  w[0] = u * u * u / 6.0;
  w[1] = (3.0 * t3 - 6.0 * t2 + 4.0) / 6.0;
  w[2] = (-3.0 * t3 + 3.0 * t2 + 3.0 * t + 1.0) / 6.0;
  w[3] = t3 / 6.0;
}

template <typename T>
__device__ inline double interp_at(const T* __restrict__ f, const FullDesc& fd, const double* c,
                                   int interp) {
  if (interp == 0) {  // nearest: floor(x + 0.5), wrapped
    int ix[3];
    for (int a = 0; a < 3; ++a) ix[a] = pmod((int)floor(c[a] + 0.5), fd.N[a]);
    return (double)f[ravel(fd, ix[0], ix[1], ix[2])];
  }
  if (interp == 1) {
    int i0[3], i1[3];
    double t[3];
    for (int a = 0; a < 3; ++a) {
      double fl = floor(c[a]);
      t[a] = c[a] - fl;
      i0[a] = pmod((int)fl, fd.N[a]);
      i1[a] = i0[a] + 1 == fd.N[a] ? 0 : i0[a] + 1;
    }
    double acc = 0.0;
#pragma unroll
    for (int p = 0; p < 2; ++p) {
      double w0 = p ? t[0] : 1.0 - t[0];
      int x0 = p ? i1[0] : i0[0];
      if (w0 == 0.0 && fd.N[0] == 1 && p) continue;
      double a1 = 0.0;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        double w1 = q ? t[1] : 1.0 - t[1];
        int x1 = q ? i1[1] : i0[1];
        double a2 = 0.0;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          double w2 = s ? t[2] : 1.0 - t[2];
          int x2 = s ? i1[2] : i0[2];
          a2 += w2 * (double)f[ravel(fd, x0, x1, x2)];
        }
        a1 += w1 * a2;
      }
      acc += w0 * a1;
    }
    return acc;
  }
  // cubic on prefiltered coefficients
  int ib[3];
  double w[3][4];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double fl = floor(c[a]);
    ib[a] = (int)fl - 1;
    if (fd.N[a] == 1) {
      w[a][0] = 0.0; w[a][1] = 1.0; w[a][2] = 0.0; w[a][3] = 0.0;
    } else {
      bspline3(c[a] - fl, w[a]);
    }
  }
  double acc = 0.0;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    if (w[0][p] == 0.0) continue;
    int x0 = pmod(ib[0] + p, fd.N[0]);
    double a1 = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (w[1][q] == 0.0) continue;
      int x1 = pmod(ib[1] + q, fd.N[1]);
      double a2 = 0.0;
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        int x2 = pmod(ib[2] + s, fd.N[2]);
        a2 += w[2][s] * (double)f[ravel(fd, x0, x1, x2)];
      }
      a1 += w[1][q] * a2;
    }
    acc += w[0][p] * a1;
  }
  return acc;
}

// out[k][j] = f[j](x + u_k(x)); nimg images, n_disp displacements
template <typename T>
__global__ void __launch_bounds__(256) k_warp(const T* __restrict__ f, int nimg,
                                              const T* __restrict__ disp, int n_disp, int interp,
                                              FullDesc fd, T* __restrict__ out) {
  const int64_t total = fd.nn * n_disp;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int k = (int)(idx / fd.nn);
    int64_t i = idx - k * fd.nn;
    int x[3];
    unravel(fd, i, x);
    double c[3];
    sample_coords<T>(fd, disp + (int64_t)k * fd.d * fd.nn, i, x, c);
    for (int j = 0; j < nimg; ++j)
      out[((int64_t)k * nimg + j) * fd.nn + i] = (T)interp_at<T>(f + j * fd.nn, fd, c, interp);
  }
}

// cubic prefilter in the Fourier domain: divide by prod_a (4 + 2 cos(2 pi k/N))/6
template <typename T>
__global__ void k_bspline_div(Cx<T>* H, int nf, GridDesc gd, T scale) {
  const int64_t hs = gd.half_size();
  const int64_t total = hs * nf;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = idx % hs;
    int b2 = (int)(r % gd.Gh);
    r /= gd.Gh;
    int b1 = (int)(r % gd.G[1]);
    int b0 = (int)(r / gd.G[1]);
    double s = ((4.0 + 2.0 * cos(kTwoPi * b0 / gd.G[0])) / 6.0) *
               ((4.0 + 2.0 * cos(kTwoPi * b1 / gd.G[1])) / 6.0) *
               ((4.0 + 2.0 * cos(kTwoPi * b2 / gd.G[2])) / 6.0);
    double m = (double)scale / s;
    Cx<T> z = H[idx];
    z.x = (T)(z.x * m);
    z.y = (T)(z.y * m);
    H[idx] = z;
  }
}

template <typename T>
static void bspline_prefilter(blr_ctx* c, const T* f, int nf, T* coef) {
  GridDesc gd = c->g.grid(false);
  const int64_t hs = gd.half_size(), rs = gd.real_size();
  for (int off = 0; off < nf;) {
    int n = std::min(kMaxScatter, nf - off);
    T* in = (T*)scratch(c, c->full_buf, c->full_bytes, (size_t)n * rs * sizeof(T));
    BLR_CUDA(cudaMemcpyAsync(in, f + (int64_t)off * rs, (size_t)n * rs * sizeof(T),
                             cudaMemcpyDeviceToDevice, c->stream));
    Cx<T>* H = (Cx<T>*)scratch(c, c->half_buf, c->half_bytes, (size_t)n * hs * sizeof(Cx<T>));
    exec_r2c<T>(c, false, n, in, H);
    k_bspline_div<T><<<grid_blocks(hs * n, 256), 256, 0, c->stream>>>(H, n, gd, (T)(1.0 / rs));
    BLR_LAUNCHED();
    exec_c2r<T>(c, false, n, H, coef + (int64_t)off * rs);
    off += n;
  }
}

template <typename T>
void warp(blr_ctx* c, const T* f, int nimg, const T* disp, int n_disp, int interp, T* out) {
  FullDesc fd = full_desc(c->g);
  const T* src = f;
  T* coef = nullptr;
  if (interp == 3) {
    BLR_CUDA(cudaMallocAsync((void**)&coef, (size_t)nimg * fd.nn * sizeof(T), c->stream));
    bspline_prefilter<T>(c, f, nimg, coef);
    src = coef;
  }
  ProfScope ps(c, "warp", (double)fd.nn * n_disp * (fd.d + 2 * nimg) * sizeof(T));
  k_warp<T><<<grid_blocks(fd.nn * n_disp, 256), 256, 0, c->stream>>>(src, nimg, disp, n_disp, interp,
                                                                      fd, out);
  BLR_LAUNCHED();
  if (coef) BLR_CUDA(cudaFreeAsync(coef, c->stream));
}

// ---------------------------------------------------------------------------
// gradients
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_central_grad(const T* __restrict__ f, int nf, FullDesc fd, T* __restrict__ out) {
  const int64_t total = fd.nn * nf;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int j = (int)(idx / fd.nn);
    int64_t i = idx - j * fd.nn;
    int x[3];
    unravel(fd, i, x);
    const T* fj = f + j * fd.nn;
    for (int comp = 0; comp < fd.d; ++comp) {
      int a = 3 - fd.d + comp;
      int xp[3] = {x[0], x[1], x[2]}, xm[3] = {x[0], x[1], x[2]};
      xp[a] = x[a] + 1 == fd.N[a] ? 0 : x[a] + 1;
      xm[a] = x[a] == 0 ? fd.N[a] - 1 : x[a] - 1;
      T denom = (T)(2.0 * (1.0 / fd.N[a]));  // 2h, gridops.py:86-89
      out[((int64_t)j * fd.d + comp) * fd.nn + i] =
          (fj[ravel(fd, xp[0], xp[1], xp[2])] - fj[ravel(fd, xm[0], xm[1], xm[2])]) / denom;
    }
  }
}

// multiply a half spectrum by i*2*pi*k_axis (Nyquist zeroed), gridops.py:90-99
template <typename T>
__global__ void k_spec_deriv(const Cx<T>* H, GridDesc gd, int axis, T scale, Cx<T>* out) {
  const int64_t hs = gd.half_size();
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < hs;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = idx;
    int b[3];
    b[2] = (int)(r % gd.Gh);
    r /= gd.Gh;
    b[1] = (int)(r % gd.G[1]);
    b[0] = (int)(r / gd.G[1]);
    int n = gd.G[axis];
    int k = b[axis] <= (n - 1) / 2 ? b[axis] : b[axis] - n;
    if (n % 2 == 0 && b[axis] == n / 2) k = 0;
    T m = (T)(kTwoPi * (double)k);
    Cx<T> z = H[idx], o;
    o.x = -(m * z.y) * scale;
    o.y = (m * z.x) * scale;
    out[idx] = o;
  }
}

template <typename T>
void grid_gradient(blr_ctx* c, const T* f, int nf, int mode, T* out) {
  FullDesc fd = full_desc(c->g);
  if (mode == 0) {
    k_central_grad<T><<<grid_blocks(fd.nn * nf, 256), 256, 0, c->stream>>>(f, nf, fd, out);
    BLR_LAUNCHED();
    return;
  }
  GridDesc gd = c->g.grid(false);
  const int64_t hs = gd.half_size(), rs = gd.real_size();
  const int d = c->g.d;
  Cx<T>* H = nullptr;
  Cx<T>* D = nullptr;
  T* in = nullptr;
  BLR_CUDA(cudaMallocAsync((void**)&H, hs * sizeof(Cx<T>), c->stream));
  BLR_CUDA(cudaMallocAsync((void**)&D, hs * sizeof(Cx<T>), c->stream));
  BLR_CUDA(cudaMallocAsync((void**)&in, rs * sizeof(T), c->stream));
  for (int j = 0; j < nf; ++j) {
    BLR_CUDA(cudaMemcpyAsync(in, f + j * rs, rs * sizeof(T), cudaMemcpyDeviceToDevice, c->stream));
    exec_r2c<T>(c, false, 1, in, H);
    for (int comp = 0; comp < d; ++comp) {
      k_spec_deriv<T><<<grid_blocks(hs, 256), 256, 0, c->stream>>>(H, gd, c->g.axis_of(comp),
                                                                   (T)(1.0 / rs), D);
      BLR_LAUNCHED();
      exec_c2r<T>(c, false, 1, D, out + ((int64_t)j * d + comp) * rs);
    }
  }
  BLR_CUDA(cudaFreeAsync(H, c->stream));
  BLR_CUDA(cudaFreeAsync(D, c->stream));
  BLR_CUDA(cudaFreeAsync(in, c->stream));
}

// det(I + Du) with central differences (gridops.py:103-131)
template <typename T>
__global__ void k_jdet(const T* __restrict__ u, FullDesc fd, T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < fd.nn;
       i += (int64_t)gridDim.x * blockDim.x) {
    int x[3];
    unravel(fd, i, x);
    T J[3][3];
    const int d = fd.d;
    for (int r = 0; r < d; ++r)
      for (int comp = 0; comp < d; ++comp) {
        int a = 3 - d + comp;
        int xp[3] = {x[0], x[1], x[2]}, xm[3] = {x[0], x[1], x[2]};
        xp[a] = x[a] + 1 == fd.N[a] ? 0 : x[a] + 1;
        xm[a] = x[a] == 0 ? fd.N[a] - 1 : x[a] - 1;
        T denom = (T)(2.0 * (1.0 / fd.N[a]));
        const T* ur = u + r * fd.nn;
        T g = (ur[ravel(fd, xp[0], xp[1], xp[2])] - ur[ravel(fd, xm[0], xm[1], xm[2])]) / denom;
        J[r][comp] = g + (r == comp ? (T)1 : (T)0);
      }
    T det;
    if (d == 1) det = J[0][0];
    else if (d == 2) det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    else
      det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
            J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
            J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    out[i] = det;
  }
}

template <typename T>
void jacobian_det(blr_ctx* c, const T* u, T* out) {
  FullDesc fd = full_desc(c->g);
  k_jdet<T><<<grid_blocks(fd.nn, 256), 256, 0, c->stream>>>(u, fd, out);
  BLR_LAUNCHED();
}

// ---------------------------------------------------------------------------
// fused objective data terms
// ---------------------------------------------------------------------------
// acc[a] = sum_i w_i * (vol_i * dlam(x + psi_i)) * gm_i[a]   (state.py:125-137)
// node weights travel as a kernel parameter (no host->device copy per call)
constexpr int kMaxNodeW = 64;
struct NodeW {
  double w[kMaxNodeW];
};

#ifndef BLR_SGN_MINB
#define BLR_SGN_MINB 4
#endif
#ifndef BLR_SGN_UNROLL
#define BLR_SGN_UNROLL 4
#endif
constexpr int kSgnUnroll = BLR_SGN_UNROLL;
template <typename T>
__global__ void __launch_bounds__(256, BLR_SGN_MINB) k_state_gn(const T* __restrict__ dlam, const T* __restrict__ vol,
                                                  const T* __restrict__ psi, const T* __restrict__ gm,
                                                  int n_nodes, NodeW w, int interp,
                                                  FullDesc fd, int add, T* __restrict__ acc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < fd.nn;
       i += (int64_t)gridDim.x * blockDim.x) {
    int x[3];
    unravel(fd, i, x);
    T s[3] = {0, 0, 0};
#pragma unroll kSgnUnroll
    for (int k = 0; k < n_nodes; ++k) {
      double c[3];
      sample_coords<T>(fd, psi + (int64_t)k * fd.d * fd.nn, i, x, c);
      T val = (T)interp_at<T>(dlam, fd, c, interp);
      T lam = vol[(int64_t)k * fd.nn + i] * val;
      T wk = (T)w.w[k];
#pragma unroll
      for (int a = 0; a < 3; ++a)
        if (a < fd.d) s[a] += wk * (lam * gm[((int64_t)k * fd.d + a) * fd.nn + i]);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
      if (a < fd.d) acc[a * fd.nn + i] = add ? acc[a * fd.nn + i] + s[a] : s[a];
  }
}

template <typename T>
void state_gn_accumulate(blr_ctx* c, const T* dlam, const T* vol, const T* psi, const T* gm,
                         int n_nodes, const double* weights, int interp, T* acc) {
  FullDesc fd = full_desc(c->g);
  const T* src = dlam;
  T* coef = nullptr;
  if (interp == 3) {
    BLR_CUDA(cudaMallocAsync((void**)&coef, fd.nn * sizeof(T), c->stream));
    bspline_prefilter<T>(c, dlam, 1, coef);
    src = coef;
  }
  ProfScope ps(c, "state_gn_accumulate", (double)fd.nn * (n_nodes * (1 + 2 * fd.d) + 1 + fd.d) * sizeof(T));
  for (int k0 = 0; k0 < n_nodes; k0 += kMaxNodeW) {  // node chunks: weights ride in the parameters
    const int nk = std::min(kMaxNodeW, n_nodes - k0);
    NodeW dw;
    for (int k = 0; k < nk; ++k) dw.w[k] = weights[k0 + k];
    k_state_gn<T><<<grid_blocks(fd.nn, 256), 256, 0, c->stream>>>(
        src, vol + (int64_t)k0 * fd.nn, psi + (int64_t)k0 * fd.d * fd.nn, gm + (int64_t)k0 * fd.d * fd.nn, nk, dw,
        interp, fd, k0 > 0 ? 1 : 0, acc);
    BLR_LAUNCHED();
  }
  if (coef) BLR_CUDA(cudaFreeAsync(coef, c->stream));
}

// out = c * sum_a g[a] u[a]
template <typename T>
__global__ void k_dot_fields(const T* g, const T* u, T cc, FullDesc fd, T* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < fd.nn;
       i += (int64_t)gridDim.x * blockDim.x) {
    T s = 0;
    for (int a = 0; a < fd.d; ++a) s += g[a * fd.nn + i] * u[a * fd.nn + i];
    out[i] = cc * s;
  }
}

template <typename T>
__global__ void k_scale_fields(const T* s, const T* g, FullDesc fd, T* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < fd.nn;
       i += (int64_t)gridDim.x * blockDim.x) {
    T sv = s[i];
    for (int a = 0; a < fd.d; ++a) out[a * fd.nn + i] = sv * g[a * fd.nn + i];
  }
}

template <typename T>
__global__ void k_scaled_diff(const T* a, const T* b, T cc, int64_t n, T* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = cc * (a[i] - b[i]);
}

template <typename T>
__global__ void k_mul(const T* a, const T* b, int64_t n, T* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[i] * b[i];
}

// state gradient data: sum_i w_i (vol_i lamw_i) gm_i  or per node
template <typename T>
__global__ void k_state_data(const T* vol, const T* lamw, const T* gm, int n_nodes, const double* w,
                             FullDesc fd, T* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < fd.nn;
       i += (int64_t)gridDim.x * blockDim.x) {
    T s[3] = {0, 0, 0};
    for (int k = 0; k < n_nodes; ++k) {
      T lam = vol[(int64_t)k * fd.nn + i] * lamw[(int64_t)k * fd.nn + i];
      for (int a = 0; a < fd.d; ++a) {
        T term = lam * gm[((int64_t)k * fd.d + a) * fd.nn + i];
        if (w) s[a] += (T)w[k] * term;
        else out[((int64_t)k * fd.d + a) * fd.nn + i] = term;
      }
    }
    if (w)
      for (int a = 0; a < fd.d; ++a) out[a * fd.nn + i] = s[a];
  }
}

template <typename T>
void dot_fields(blr_ctx* c, const T* g, const T* u, double cc, T* out) {
  FullDesc fd = full_desc(c->g);
  k_dot_fields<T><<<grid_blocks(fd.nn, 256), 256, 0, c->stream>>>(g, u, (T)cc, fd, out);
  BLR_LAUNCHED();
}
template <typename T>
void scale_fields(blr_ctx* c, const T* s, const T* g, T* out) {
  FullDesc fd = full_desc(c->g);
  k_scale_fields<T><<<grid_blocks(fd.nn, 256), 256, 0, c->stream>>>(s, g, fd, out);
  BLR_LAUNCHED();
}
template <typename T>
void scaled_diff(blr_ctx* c, const T* a, const T* b, double cc, T* out) {
  int64_t n = c->g.nn();
  k_scaled_diff<T><<<grid_blocks(n, 256), 256, 0, c->stream>>>(a, b, (T)cc, n, out);
  BLR_LAUNCHED();
}
template <typename T>
void mul(blr_ctx* c, const T* a, const T* b, int64_t n, T* out) {
  k_mul<T><<<grid_blocks(n, 256), 256, 0, c->stream>>>(a, b, n, out);
  BLR_LAUNCHED();
}
template <typename T>
void state_data(blr_ctx* c, const T* vol, const T* lamw, const T* gm, int n_nodes, const double* weights,
                T* out) {
  FullDesc fd = full_desc(c->g);
  double* dw = nullptr;
  if (weights) {
    BLR_CUDA(cudaMallocAsync((void**)&dw, n_nodes * sizeof(double), c->stream));
    BLR_CUDA(cudaMemcpyAsync(dw, weights, n_nodes * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  }
  ProfScope ps(c, "state_data", (double)fd.nn * (n_nodes * (2 + fd.d) + fd.d) * sizeof(T));
  k_state_data<T><<<grid_blocks(fd.nn, 256), 256, 0, c->stream>>>(vol, lamw, gm, n_nodes, dw, fd, out);
  BLR_LAUNCHED();
  if (dw) BLR_CUDA(cudaFreeAsync(dw, c->stream));
}


// ---------------------------------------------------------------------------
// full-Newton data terms (no torch-eager node loops)
// ---------------------------------------------------------------------------
// dm[k] = sum_a g[k][a] u[k][a] for n_nodes nodes (state.py:143: dm = sgw . dphi)
template <typename T>
__global__ void k_dot_nodes(const T* __restrict__ g, const T* __restrict__ u, int n_nodes, FullDesc fd,
                            T* __restrict__ out) {
  const int64_t total = fd.nn * n_nodes;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(idx / fd.nn);
    const int64_t i = idx - k * fd.nn, od = (int64_t)k * fd.d * fd.nn + i;
    T s = 0;
    for (int a = 0; a < fd.d; ++a) s += g[od + a * fd.nn] * u[od + a * fd.nn];
    out[idx] = s;
  }
}

// Full-Newton state data term at node k (state.py:138-154):
//   dlam_k = dvol_k aew_k + vol_k (agw_k . dpsi_k) + vol_k dl_k,   dl_k = dlam1 o (id + psi_k)
//   term_k = dlam_k wg_k + (vol_k aew_k) grad(dm_k)
// summed with weights w_k (stationary; one projection afterwards) or written per node.
// grad(dm_k): central differences of dm (gridops.py:84-89) or the precomputed gdm.
template <typename T>
__global__ void __launch_bounds__(256) k_state_newton(
    const T* __restrict__ dlam, const T* __restrict__ dl, int interp, const T* __restrict__ vol,
    const T* __restrict__ aew, const T* __restrict__ dvol, const T* __restrict__ agw,
    const T* __restrict__ dpsi, const T* __restrict__ psi, const T* __restrict__ wg,
    const T* __restrict__ dm, const T* __restrict__ gdm, int n_nodes, NodeW w, int use_w, FullDesc fd,
    int add, T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < fd.nn;
       i += (int64_t)gridDim.x * blockDim.x) {
    int x[3];
    unravel(fd, i, x);
    T s[3] = {0, 0, 0};
    for (int k = 0; k < n_nodes; ++k) {
      const int64_t o1 = (int64_t)k * fd.nn + i, od = (int64_t)k * fd.d * fd.nn + i;
      T dlk;
      if (dl) {
        dlk = dl[o1];
      } else {
        double c[3];
        sample_coords<T>(fd, psi + (int64_t)k * fd.d * fd.nn, i, x, c);
        dlk = (T)interp_at<T>(dlam, fd, c, interp);
      }
      const T vk = vol[o1], ak = aew[o1];
      T ad = 0;
#pragma unroll
      for (int b = 0; b < 3; ++b)
        if (b < fd.d) ad += agw[od + b * fd.nn] * dpsi[od + b * fd.nn];
      const T q = dvol[o1] * ak + vk * ad + vk * dlk;
      const T lam = vk * ak;
      const T* dmk = dm + (int64_t)k * fd.nn;
#pragma unroll
      for (int comp = 0; comp < 3; ++comp) {
        if (comp >= fd.d) continue;
        T G;
        if (gdm) {
          G = gdm[od + comp * fd.nn];
        } else {
          const int ax = 3 - fd.d + comp;
          int xp[3] = {x[0], x[1], x[2]}, xm[3] = {x[0], x[1], x[2]};
          xp[ax] = x[ax] + 1 == fd.N[ax] ? 0 : x[ax] + 1;
          xm[ax] = x[ax] == 0 ? fd.N[ax] - 1 : x[ax] - 1;
          const T denom = (T)(2.0 * (1.0 / fd.N[ax]));
          G = (dmk[ravel(fd, xp[0], xp[1], xp[2])] - dmk[ravel(fd, xm[0], xm[1], xm[2])]) / denom;
        }
        const T term = q * wg[od + comp * fd.nn] + lam * G;
        if (use_w) s[comp] += (T)w.w[k] * term;
        else out[od + comp * fd.nn] = term;
      }
    }
    if (use_w) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
        if (a < fd.d) out[a * fd.nn + i] = add ? out[a * fd.nn + i] + s[a] : s[a];
    }
  }
}

template <typename T>
void state_newton(blr_ctx* c, const T* dlam, const T* dl, int interp, const T* vol, const T* aew, const T* dvol,
                  const T* agw, const T* dpsi, const T* psi, const T* wg, const T* sgw, const T* dphi,
                  int n_nodes, const double* weights, int grad_mode, T* out) {
  FullDesc fd = full_desc(c->g);
  T *dm = nullptr, *gdm = nullptr, *coef = nullptr;
  BLR_CUDA(cudaMallocAsync((void**)&dm, (size_t)n_nodes * fd.nn * sizeof(T), c->stream));
  k_dot_nodes<T><<<grid_blocks(fd.nn * n_nodes, 256), 256, 0, c->stream>>>(sgw, dphi, n_nodes, fd, dm);
  BLR_LAUNCHED();
  if (grad_mode != 0) {
    BLR_CUDA(cudaMallocAsync((void**)&gdm, (size_t)n_nodes * fd.d * fd.nn * sizeof(T), c->stream));
    grid_gradient<T>(c, dm, n_nodes, grad_mode, gdm);
  }
  const T* src = dlam;
  if (!dl && interp == 3) {
    BLR_CUDA(cudaMallocAsync((void**)&coef, fd.nn * sizeof(T), c->stream));
    bspline_prefilter<T>(c, dlam, 1, coef);
    src = coef;
  }
  ProfScope ps(c, "state_newton", (double)fd.nn * n_nodes * (6 + 5 * fd.d) * sizeof(T));
  const int64_t nd = (int64_t)fd.d * fd.nn;
  if (!weights) {
    NodeW dw{};
    k_state_newton<T><<<grid_blocks(fd.nn, 256), 256, 0, c->stream>>>(
        src, dl, interp, vol, aew, dvol, agw, dpsi, psi, wg, dm, gdm, n_nodes, dw, 0, fd, 0, out);
    BLR_LAUNCHED();
  } else {
    for (int k0 = 0; k0 < n_nodes; k0 += kMaxNodeW) {  // node chunks: weights ride in the parameters
      const int nk = std::min(kMaxNodeW, n_nodes - k0);
      NodeW dw;
      for (int k = 0; k < nk; ++k) dw.w[k] = weights[k0 + k];
      k_state_newton<T><<<grid_blocks(fd.nn, 256), 256, 0, c->stream>>>(
          src, dl ? dl + k0 * fd.nn : nullptr, interp, vol + k0 * fd.nn, aew + k0 * fd.nn, dvol + k0 * fd.nn,
          agw + k0 * nd, dpsi + k0 * nd, psi + k0 * nd, wg + k0 * nd, dm + k0 * fd.nn,
          gdm ? gdm + k0 * nd : nullptr, nk, dw, 1, fd, k0 > 0 ? 1 : 0, out);
      BLR_LAUNCHED();
    }
  }
  BLR_CUDA(cudaFreeAsync(dm, c->stream));
  if (gdm) BLR_CUDA(cudaFreeAsync(gdm, c->stream));
  if (coef) BLR_CUDA(cudaFreeAsync(coef, c->stream));
}

// out[a] += s * sum_b H[a][b] u[b]   (deformation.py:141-145, transposed Newton endpoint term)
// or, H == nullptr, out[a] += s * u[a]   (direct: lam * grad(dm1))
template <typename T>
__global__ void k_lam_matvec_add(const T* __restrict__ s, const T* __restrict__ H, const T* __restrict__ u,
                                 FullDesc fd, T* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < fd.nn;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T sv = s[i];
    for (int a = 0; a < fd.d; ++a) {
      T m;
      if (H) {
        m = 0;
        for (int b = 0; b < fd.d; ++b) m += H[(a * fd.d + b) * fd.nn + i] * u[b * fd.nn + i];
      } else {
        m = u[a * fd.nn + i];
      }
      out[a * fd.nn + i] += sv * m;
    }
  }
}

template <typename T>
void lam_matvec_add(blr_ctx* c, const T* s, const T* H, const T* u, T* out) {
  FullDesc fd = full_desc(c->g);
  k_lam_matvec_add<T><<<grid_blocks(fd.nn, 256), 256, 0, c->stream>>>(s, H, u, fd, out);
  BLR_LAUNCHED();
}

#define BLR_GINST(T)                                                                             \
  template void warp<T>(blr_ctx*, const T*, int, const T*, int, int, T*);                        \
  template void grid_gradient<T>(blr_ctx*, const T*, int, int, T*);                              \
  template void jacobian_det<T>(blr_ctx*, const T*, T*);                                         \
  template void state_gn_accumulate<T>(blr_ctx*, const T*, const T*, const T*, const T*, int,    \
                                       const double*, int, T*);                                  \
  template void dot_fields<T>(blr_ctx*, const T*, const T*, double, T*);                         \
  template void scale_fields<T>(blr_ctx*, const T*, const T*, T*);                               \
  template void scaled_diff<T>(blr_ctx*, const T*, const T*, double, T*);                        \
  template void mul<T>(blr_ctx*, const T*, const T*, int64_t, T*);                               \
  template void state_data<T>(blr_ctx*, const T*, const T*, const T*, int, const double*, T*);   \
  template void state_newton<T>(blr_ctx*, const T*, const T*, int, const T*, const T*, const T*,  \
                                const T*, const T*, const T*, const T*, const T*, const T*, int,  \
                                const double*, int, T*);                                          \
  template void lam_matvec_add<T>(blr_ctx*, const T*, const T*, const T*, T*);
BLR_GINST(double)
BLR_GINST(float)

}  // namespace blr
