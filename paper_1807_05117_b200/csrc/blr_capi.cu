// blr_capi.cu — the extern "C" boundary (include/blreg_b200.h).
//
// Each entry point validates its arguments, dispatches on the context's
// precision and translates C++ exceptions into status codes plus a
// thread-local message.
#include "../../include/blreg_b200.h"
#include "blr_internal.cuh"

#include <cstdio>
#include <cstring>

using namespace blr;

static thread_local std::string g_err;

template <typename F>
static int guarded(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

static void need(bool ok, const char* msg) {
  if (!ok) throw Error(1, msg);
}

// Makes the context's device current for the duration of one entry point and
// restores the caller's device afterwards (a Domain on device k works without
// the caller having called cudaSetDevice(k)).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) BLR_CUDA(cudaSetDevice(dev));
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

#define DISPATCH(ctx, ...)                  \
  do {                                      \
    DeviceGuard dev_guard_((ctx)->device);  \
    if ((ctx)->dtype == 0) {                \
      using T = double;                     \
      __VA_ARGS__;                          \
    } else {                                \
      using T = float;                      \
      __VA_ARGS__;                          \
    }                                       \
  } while (0)

extern "C" {

const char* blr_last_error(void) { return g_err.c_str(); }
int64_t blr_launch_count(void) { return launch_count(); }
int blr_version(void) { return 1; }

int blr_set_fused_forward(int on) {
  return guarded([&] { set_fused_forward(on); });
}

int blr_profile_enable(int on) {
  return guarded([&] { profile_enable(on != 0); });
}

int blr_profile_report(char* buf, int64_t len) {
  return guarded([&] {
    need(buf && len > 0, "bad arguments");
    std::string r = profile_report();
    if ((int64_t)r.size() + 1 > len) throw Error(1, "buffer too small for profile report");
    std::memcpy(buf, r.c_str(), r.size() + 1);
  });
}

int blr_ctx_create(blr_ctx** out, int ndim, const int* shape, const int* bandwidth, const int* pad,
                   double alpha, int order, const double* symbol_tab, int dtype, int device) {
  return guarded([&] {
    need(out && shape && bandwidth && pad && symbol_tab, "null argument");
    need(ndim >= 1 && ndim <= 3, "ndim must be 1, 2 or 3");
    need(dtype == 0 || dtype == 1, "dtype must be 0 (f64) or 1 (f32)");
    need(order >= 1, "order must be >= 1");
    auto* c = new blr_ctx();
    c->dtype = dtype;
    c->device = device;
    Geom& g = c->g;
    g.d = ndim;
    g.alpha = alpha;
    g.order = order;
    for (int a = 0; a < 3; ++a) { g.N[a] = 1; g.K[a] = 0; g.B[a] = 1; g.P[a] = 1; }
    for (int i = 0; i < ndim; ++i) {
      int a = 3 - ndim + i;
      g.N[a] = shape[i];
      g.K[a] = bandwidth[i];
      g.B[a] = 2 * bandwidth[i] + 1;
      g.P[a] = pad[i];
      if (!(shape[i] >= 2 && bandwidth[i] >= 1 && 2 * bandwidth[i] <= shape[i]) ||
          pad[i] < 3 * bandwidth[i] + 1) {
        delete c;
        throw Error(1, "invalid shape/bandwidth/pad (need 1 <= K <= N/2 and pad >= 3K+1)");
      }
    }
    // symbol tables, 3-axis layout (dummy axes: one zero entry)
    int nsym = g.B[0] + g.B[1] + g.B[2];
    c->h_sym.assign(nsym, 0.0);
    int src = 0, dst = 0;
    for (int a = 0; a < 3; ++a) {
      if (a >= 3 - ndim) {
        for (int i = 0; i < g.B[a]; ++i) c->h_sym[dst + i] = symbol_tab[src + i];
        src += g.B[a];
      }
      dst += g.B[a];
    }
    DeviceGuard dev_guard(device);
    BLR_CUDA(cudaMalloc(&c->d_sym, nsym * sizeof(double)));
    BLR_CUDA(cudaMemcpy(c->d_sym, c->h_sym.data(), nsym * sizeof(double), cudaMemcpyHostToDevice));
    // keep stream-ordered temporaries cached across calls
    cudaMemPool_t pool;
    BLR_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    BLR_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    *out = c;
  });
}

int blr_ctx_destroy(blr_ctx* c) {
  return guarded([&] {
    if (!c) return;
    DeviceGuard dev_guard(c->device);
    cudaStreamSynchronize(c->stream);
    pad_engine_release(c);
    for (auto& kv : c->plans) cufftDestroy(kv.second);
    for (void* p : {(void*)c->d_sym, c->fft_work, c->real_buf, c->half_buf, c->band_buf, c->full_buf,
                    (void*)c->d_red})
      if (p) cudaFree(p);
    if (c->h_red) cudaFreeHost(c->h_red);
    delete c;
  });
}

int blr_set_stream(blr_ctx* c, void* s) {
  return guarded([&] {
    need(c, "null context");
    c->stream = (cudaStream_t)s;
  });
}

// ---- spectral ----------------------------------------------------------------
int blr_include(blr_ctx* c, int grid, const void* blocks, int nfields, const int* deriv, void* out) {
  return guarded([&] {
    need(c && blocks && out && nfields >= 0, "bad arguments");
    need(grid == 0 || grid == 1, "grid must be 0 (full) or 1 (pad)");
    if (nfields == 0) return;
    DISPATCH(c, {
      std::vector<ScatterField<T>> f;
      for (int i = 0; i < nfields; ++i) {
        int ax = -1;
        if (deriv && deriv[i] >= 0) {
          need(deriv[i] < c->g.d, "derivative axis out of range");
          ax = c->g.axis_of(deriv[i]);
        }
        f.push_back(fld<T>((const Cx<T>*)blocks + i * c->g.nb(), ax));
      }
      realize<T>(c, grid == 1, f, (T*)out);
    });
  });
}

int blr_project(blr_ctx* c, int grid, const void* fields, int nfields, void* out) {
  return guarded([&] {
    need(c && fields && out && nfields >= 0, "bad arguments");
    need(grid == 0 || grid == 1, "grid must be 0 (full) or 1 (pad)");
    if (nfields == 0) return;
    DISPATCH(c, {
      // R2C must not clobber the caller's input: stage through scratch
      int64_t rs = c->g.grid(grid == 1).real_size();
      T* tmp = nullptr;
      BLR_CUDA(cudaMallocAsync((void**)&tmp, (size_t)nfields * rs * sizeof(T), c->stream));
      BLR_CUDA(cudaMemcpyAsync(tmp, fields, (size_t)nfields * rs * sizeof(T), cudaMemcpyDeviceToDevice,
                               c->stream));
      project<T>(c, grid == 1, tmp, nfields, (Cx<T>*)out);
      BLR_CUDA(cudaFreeAsync(tmp, c->stream));
    });
  });
}

int blr_helmholtz(blr_ctx* c, const void* in, int nblocks, int inverse, void* out) {
  return guarded([&] {
    need(c && in && out, "bad arguments");
    DISPATCH(c, band_helmholtz<T>(c, (const Cx<T>*)in, nblocks, inverse, (Cx<T>*)out));
  });
}

int blr_leray(blr_ctx* c, const void* in, int nvec, void* out) {
  return guarded([&] {
    need(c && in && out, "bad arguments");
    DISPATCH(c, band_leray<T>(c, (const Cx<T>*)in, nvec, (Cx<T>*)out));
  });
}

int blr_divergence(blr_ctx* c, const void* in, int nvec, void* out) {
  return guarded([&] {
    need(c && in && out, "bad arguments");
    DISPATCH(c, band_divergence<T>(c, (const Cx<T>*)in, nvec, (Cx<T>*)out));
  });
}

int blr_symmetrize(blr_ctx* c, const void* in, int nblocks, void* out) {
  return guarded([&] {
    need(c && in && out && in != out, "bad arguments (in-place not supported)");
    DISPATCH(c, band_symmetrize<T>(c, (const Cx<T>*)in, nblocks, (Cx<T>*)out));
  });
}

// ---- linear algebra ----------------------------------------------------------
int blr_inner(blr_ctx* c, const void* a, const void* b, int64_t n, double* result) {
  return guarded([&] {
    need(c && a && b && result, "bad arguments");
    DISPATCH(c, *result = reduce_host<T, 0>(c, a, b, n));
  });
}

int blr_inner_nodes(blr_ctx* c, const void* a, const void* b, int n_nodes, int64_t n,
                    const double* weights, double* result) {
  return guarded([&] {
    need(c && a && b && result && weights, "bad arguments");
    double total = 0.0;
    DISPATCH(c, {
      for (int i = 0; i < n_nodes; ++i)
        total += weights[i] * reduce_host<T, 0>(c, (const Cx<T>*)a + i * n, (const Cx<T>*)b + i * n, n);
    });
    *result = total;
  });
}

int blr_axpby(blr_ctx* c, double a, const void* x, double b, void* y, int64_t n) {
  return guarded([&] {
    need(c && x && y, "bad arguments");
    DISPATCH(c, band_axpby<T>(c, a, (const Cx<T>*)x, b, (Cx<T>*)y, n));
  });
}

int blr_pcg_update(blr_ctx* c, double a, const void* p, const void* hp, void* x, void* r, int64_t n) {
  return guarded([&] {
    need(c && p && hp && x && r, "bad arguments");
    DISPATCH(c, band_pcg_update<T>(c, a, (const Cx<T>*)p, (const Cx<T>*)hp, (Cx<T>*)x, (Cx<T>*)r, n));
  });
}

int blr_max_abs(blr_ctx* c, const void* f, int64_t n, double* result) {
  return guarded([&] {
    need(c && f && result, "bad arguments");
    DISPATCH(c, *result = reduce_host<T, 1>(c, f, nullptr, n));
  });
}

int blr_sq_dist(blr_ctx* c, const void* a, const void* b, int64_t n, double* result) {
  return guarded([&] {
    need(c && a && result, "bad arguments");
    DISPATCH(c, *result = reduce_host<T, 2>(c, a, b, n));
  });
}

int blr_all_finite(blr_ctx* c, const void* f, int64_t n, int* result) {
  return guarded([&] {
    need(c && f && result, "bad arguments");
    double bad = 0;
    DISPATCH(c, bad = reduce_host<T, 3>(c, f, nullptr, n));
    *result = bad == 0.0 ? 1 : 0;
  });
}

// ---- transport ---------------------------------------------------------------
static FlowRef flow(const void* v, int n_stored, int n_steps) {
  need(v != nullptr, "null flow");
  need(n_steps >= 1, "n_steps must be >= 1");
  need(n_stored == 1 || n_stored == n_steps + 1, "n_stored must be 1 or n_steps+1");
  return FlowRef{v, n_stored, n_steps};
}

int blr_forward_map(blr_ctx* c, const void* v, int n_stored, int n_steps, int substeps, void* phi,
                    void* du_cache) {
  return guarded([&] {
    need(c && substeps >= 1, "bad arguments");
    FlowRef f = flow(v, n_stored, n_steps);
    DISPATCH(c, forward_map<T>(c, f, substeps, (Cx<T>*)phi, (T*)du_cache));
  });
}

int blr_inverse_map_and_volume(blr_ctx* c, const void* v, int n_stored, int n_steps, int substeps,
                               void* psi, void* vol) {
  return guarded([&] {
    need(c && substeps >= 1, "bad arguments");
    FlowRef f = flow(v, n_stored, n_steps);
    DISPATCH(c, inverse_map_and_volume<T>(c, f, substeps, (Cx<T>*)psi, (Cx<T>*)vol));
  });
}

int blr_state_tangents(blr_ctx* c, const void* v, const void* dv, int n_stored, int n_steps,
                       int substeps, int flags, const void* du_cache, void* dphi, void* dpsi,
                       void* dvol) {
  return guarded([&] {
    need(c && substeps >= 1, "bad arguments");
    FlowRef f = flow(v, n_stored, n_steps), df = flow(dv, n_stored, n_steps);
    DISPATCH(c, state_tangents<T>(c, f, df, substeps, flags, (const T*)du_cache, (Cx<T>*)dphi,
                                  (Cx<T>*)dpsi, (Cx<T>*)dvol));
  });
}

int blr_momentum(blr_ctx* c, const void* v, int n_stored, int n_steps, int substeps,
                 const void* rho_end, void* rho) {
  return guarded([&] {
    need(c && rho_end && rho && substeps >= 1, "bad arguments");
    FlowRef f = flow(v, n_stored, n_steps);
    DISPATCH(c, momentum<T>(c, f, substeps, (const Cx<T>*)rho_end, (Cx<T>*)rho));
  });
}

int blr_momentum_tangent(blr_ctx* c, const void* v, const void* dv, int n_stored, int n_steps,
                         int substeps, const void* rho_end, const void* drho_end, int gauss_newton,
                         void* rho, void* drho) {
  return guarded([&] {
    need(c && rho_end && drho_end && drho && substeps >= 1, "bad arguments");
    need(gauss_newton || rho, "rho output required in Newton mode");
    FlowRef f = flow(v, n_stored, n_steps), df = flow(dv, n_stored, n_steps);
    DISPATCH(c, momentum_tangent<T>(c, f, df, substeps, (const Cx<T>*)rho_end, (const Cx<T>*)drho_end,
                                    gauss_newton != 0, (Cx<T>*)rho, (Cx<T>*)drho));
  });
}

int blr_contract(blr_ctx* c, const void* phi, const void* rho, int n_nodes, const double* weights,
                 int transpose, void* dphi_cache, int cache_mode, void* out) {
  return guarded([&] {
    need(c && rho && out && n_nodes >= 1, "bad arguments");
    need(cache_mode >= 0 && cache_mode <= 2, "bad cache_mode");
    need(cache_mode == 0 || dphi_cache, "cache_mode needs a cache buffer");
    need(cache_mode == 2 || phi, "phi nodes required");
    DISPATCH(c, contract<T>(c, (const Cx<T>*)phi, (const Cx<T>*)rho, n_nodes, weights, transpose != 0,
                            (T*)dphi_cache, cache_mode, (Cx<T>*)out));
  });
}

int blr_momentum_contract(blr_ctx* c, const void* v, int n_stored, int n_steps, int substeps,
                          const void* rho_end, const void* phi, const double* weights, int transpose,
                          void* dphi_cache, int cache_mode, void* out) {
  return guarded([&] {
    need(c && v && rho_end && out && weights && substeps >= 1, "bad arguments");
    need(cache_mode >= 0 && cache_mode <= 2, "bad cache_mode");
    need(cache_mode == 0 || dphi_cache, "cache_mode needs a cache buffer");
    need(cache_mode == 2 || phi, "phi nodes required");
    FlowRef f = flow(v, n_stored, n_steps);
    DISPATCH(c, momentum_contract<T>(c, f, substeps, (const Cx<T>*)rho_end, (const Cx<T>*)phi, weights,
                                     transpose != 0, (T*)dphi_cache, cache_mode, (Cx<T>*)out));
  });
}

int blr_conv_matvec(blr_ctx* c, const void* M, const void* x, int transpose, void* out) {
  return guarded([&] {
    need(c && M && x && out, "bad arguments");
    DISPATCH(c, conv_matvec<T>(c, (const Cx<T>*)M, (const Cx<T>*)x, transpose != 0, (Cx<T>*)out));
  });
}

// ---- full grid ---------------------------------------------------------------
int blr_warp(blr_ctx* c, const void* f, int nimg, const void* disp, int n_disp, int interp, void* out) {
  return guarded([&] {
    need(c && f && disp && out && nimg >= 1 && n_disp >= 1, "bad arguments");
    need(interp == 0 || interp == 1 || interp == 3, "interp must be 0, 1 or 3");
    need(n_disp == 1 || nimg == 1, "several displacements need a single image");
    DISPATCH(c, warp<T>(c, (const T*)f, nimg, (const T*)disp, n_disp, interp, (T*)out));
  });
}

int blr_grid_gradient(blr_ctx* c, const void* f, int nf, int mode, void* out) {
  return guarded([&] {
    need(c && f && out && (mode == 0 || mode == 1), "bad arguments");
    DISPATCH(c, grid_gradient<T>(c, (const T*)f, nf, mode, (T*)out));
  });
}

int blr_jacobian_det(blr_ctx* c, const void* disp, void* out) {
  return guarded([&] {
    need(c && disp && out, "bad arguments");
    DISPATCH(c, jacobian_det<T>(c, (const T*)disp, (T*)out));
  });
}

int blr_state_gn_accumulate(blr_ctx* c, const void* dlam, const void* vol, const void* psi,
                            const void* gm, int n_nodes, const double* weights, int interp, void* acc) {
  return guarded([&] {
    need(c && dlam && vol && psi && gm && weights && acc, "bad arguments");
    need(interp == 0 || interp == 1 || interp == 3, "interp must be 0, 1 or 3");
    DISPATCH(c, state_gn_accumulate<T>(c, (const T*)dlam, (const T*)vol, (const T*)psi, (const T*)gm,
                                       n_nodes, weights, interp, (T*)acc));
  });
}

int blr_dot_fields(blr_ctx* c, const void* g, const void* u, double cc, void* out) {
  return guarded([&] {
    need(c && g && u && out, "bad arguments");
    DISPATCH(c, dot_fields<T>(c, (const T*)g, (const T*)u, cc, (T*)out));
  });
}

int blr_scale_fields(blr_ctx* c, const void* s, const void* g, void* out) {
  return guarded([&] {
    need(c && s && g && out, "bad arguments");
    DISPATCH(c, scale_fields<T>(c, (const T*)s, (const T*)g, (T*)out));
  });
}

int blr_scaled_diff(blr_ctx* c, const void* a, const void* b, double cc, void* out) {
  return guarded([&] {
    need(c && a && b && out, "bad arguments");
    DISPATCH(c, scaled_diff<T>(c, (const T*)a, (const T*)b, cc, (T*)out));
  });
}

int blr_mul(blr_ctx* c, const void* a, const void* b, int64_t n, void* out) {
  return guarded([&] {
    need(c && a && b && out, "bad arguments");
    DISPATCH(c, mul<T>(c, (const T*)a, (const T*)b, n, (T*)out));
  });
}

int blr_state_data(blr_ctx* c, const void* vol, const void* lamw, const void* gm, int n_nodes,
                   const double* weights, void* out) {
  return guarded([&] {
    need(c && vol && lamw && gm && out, "bad arguments");
    DISPATCH(c, state_data<T>(c, (const T*)vol, (const T*)lamw, (const T*)gm, n_nodes, weights, (T*)out));
  });
}


int blr_state_newton(blr_ctx* c, const void* dlam, const void* dl, int interp, const void* vol,
                     const void* aew, const void* dvol, const void* agw, const void* dpsi, const void* psi,
                     const void* wg, const void* sgw, const void* dphi, int n_nodes, const double* weights,
                     int grad_mode, void* out) {
  return guarded([&] {
    need(c && vol && aew && dvol && agw && dpsi && wg && sgw && dphi && out && n_nodes >= 1, "bad arguments");
    need(dl || (dlam && psi && interp >= 0 && interp <= 3), "need dl, or dlam + psi with a grid interp");
    need(grad_mode == 0 || grad_mode == 1, "grad_mode must be 0 (central) or 1 (spectral)");
    DISPATCH(c, state_newton<T>(c, (const T*)dlam, (const T*)dl, interp, (const T*)vol, (const T*)aew,
                                (const T*)dvol, (const T*)agw, (const T*)dpsi, (const T*)psi, (const T*)wg,
                                (const T*)sgw, (const T*)dphi, n_nodes, weights, grad_mode, (T*)out));
  });
}

int blr_lam_matvec_add(blr_ctx* c, const void* s, const void* H, const void* u, void* out) {
  return guarded([&] {
    need(c && s && u && out, "bad arguments");
    DISPATCH(c, lam_matvec_add<T>(c, (const T*)s, (const T*)H, (const T*)u, (T*)out));
  });
}
}  // extern "C"
