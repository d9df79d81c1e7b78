// blr_internal.cuh — internal (non-ABI) declarations shared by the .cu files.
#pragma once

#include <algorithm>
#include <atomic>

#include "blr_common.cuh"

namespace blr {

constexpr int kMaxScatter = 24;

// One realized field: sum over nterms of coef_t * (i*2*pi*k_axis_t)^[axis_t>=0] * src_t.
template <typename T>
struct ScatterField {
  const Cx<T>* src[3];
  int axis[3];  // 3-axis index or -1
  T coef[3];
  int nterms;
};

template <typename T>
struct ScatterArgs {
  ScatterField<T> f[kMaxScatter];
  int nf;
};

int64_t launch_count();

// Per-kernel-category CUDA-event profiler (off by default).  When enabled,
// each instrumented launch records start/stop events on the launching stream
// plus the kernel's algorithmic bytes; blr_profile_report() aggregates them.
bool profiling();
struct ProfScope {
  int slot = -1;
  cudaStream_t stream = nullptr;
  ProfScope(blr_ctx* c, const char* name, double bytes, cudaStream_t s = nullptr);
  ~ProfScope();
};
void profile_enable(bool on);
std::string profile_report();

template <typename T> void realize(blr_ctx* c, bool pad, const std::vector<ScatterField<T>>& fields, T* out);
template <typename T> void project(blr_ctx* c, bool pad, T* in, int nf, Cx<T>* out);
template <typename T> ScatterField<T> fld(const Cx<T>* src, int axis);
template <typename T> ScatterField<T> fld_div(const Geom& g, const Cx<T>* vec);
template <typename T> void exec_c2r(blr_ctx* c, bool pad, int batch, Cx<T>* in, T* out);
template <typename T> void exec_r2c(blr_ctx* c, bool pad, int batch, T* in, Cx<T>* out);

template <typename T> void band_flux_div(blr_ctx* c, const Cx<T>* F, int nsets, Cx<T>* out);
template <typename T> void band_helmholtz(blr_ctx* c, const Cx<T>* in, int nblocks, int inverse, Cx<T>* out);
template <typename T> void band_leray(blr_ctx* c, const Cx<T>* in, int nvec, Cx<T>* out);
template <typename T> void band_divergence(blr_ctx* c, const Cx<T>* in, int nvec, Cx<T>* out);
template <typename T> void band_symmetrize(blr_ctx* c, const Cx<T>* in, int nblocks, Cx<T>* out);
template <typename T> void band_neg_add(blr_ctx* c, const Cx<T>* a, const Cx<T>* b, Cx<T>* out, int64_t n);
template <typename T> void band_rk4(blr_ctx* c, int s, const Cx<T>* k, Cx<T>* cur, Cx<T>* acc, Cx<T>* stage,
                                    double cs, double h6, int64_t n);
template <typename T> void band_lerp(blr_ctx* c, const Cx<T>* a, const Cx<T>* b, double w, Cx<T>* out, int64_t n);
template <typename T> void band_axpby(blr_ctx* c, double a, const Cx<T>* x, double b, Cx<T>* y, int64_t n);
template <typename T> void band_pcg_update(blr_ctx* c, double a, const Cx<T>* p, const Cx<T>* hp, Cx<T>* x,
                                           Cx<T>* r, int64_t n);
template <typename T, int MODE> double reduce_host(blr_ctx* c, const void* a, const void* b, int64_t n);

// transport (blr_transport.cu)
struct FlowRef {
  const void* v;  // [n_stored][d][nb]
  int n_stored;
  int n_steps;
  bool stationary() const { return n_stored == 1; }
};

template <typename T> void forward_map(blr_ctx* c, FlowRef v, int substeps, Cx<T>* phi, T* du_cache);
template <typename T> void inverse_map_and_volume(blr_ctx* c, FlowRef v, int substeps, Cx<T>* psi, Cx<T>* vol);
template <typename T> void state_tangents(blr_ctx* c, FlowRef v, FlowRef dv, int substeps, int flags,
                                          const T* du_cache, Cx<T>* dphi, Cx<T>* dpsi, Cx<T>* dvol);
template <typename T> void momentum(blr_ctx* c, FlowRef v, int substeps, const Cx<T>* rho_end, Cx<T>* rho);
template <typename T> void momentum_tangent(blr_ctx* c, FlowRef v, FlowRef dv, int substeps, const Cx<T>* rho_end,
                                            const Cx<T>* drho_end, bool gn, Cx<T>* rho, Cx<T>* drho);
template <typename T> void contract(blr_ctx* c, const Cx<T>* phi, const Cx<T>* rho, int n_nodes,
                                    const double* weights, bool transpose, T* dphi_cache, int cache_mode,
                                    Cx<T>* out);
template <typename T> void momentum_contract(blr_ctx* c, FlowRef v, int substeps, const Cx<T>* rho_end,
                                             const Cx<T>* phi, const double* weights, bool transpose,
                                             T* dphi_cache, int cache_mode, Cx<T>* out);
template <typename T> void conv_matvec(blr_ctx* c, const Cx<T>* M, const Cx<T>* x, bool transpose, Cx<T>* out);


// fused pad engine (blr_pad.cu); each returns false when unavailable (v1 fallback)
template <typename T> bool pad_engine_ok(blr_ctx* c);
void pad_engine_release(blr_ctx* c);
void set_fused_forward(int on);
template <typename T> bool forward_map_v2(blr_ctx* c, FlowRef v, int substeps, Cx<T>* phi, T* du_cache);
template <typename T> bool inverse_map_and_volume_v2(blr_ctx* c, FlowRef v, int substeps, Cx<T>* psi, Cx<T>* vol);
template <typename T> bool state_tangents_v2(blr_ctx* c, FlowRef v, FlowRef dv, int substeps, int flags,
                                             const T* du_cache, Cx<T>* dphi, Cx<T>* dpsi, Cx<T>* dvol);
template <typename T> bool momentum_v2(blr_ctx* c, FlowRef v, int substeps, const Cx<T>* rho_end, Cx<T>* rho);
template <typename T> bool momentum_pair_v2(blr_ctx* c, FlowRef v, FlowRef dv, int substeps, const Cx<T>* rho_end,
                                            const Cx<T>* drho_end, Cx<T>* rho, Cx<T>* drho);
template <typename T> bool contract_v2(blr_ctx* c, const Cx<T>* phi, const Cx<T>* rho, int n_nodes,
                                       const double* weights, bool transpose, T* dphi_cache, int cache_mode,
                                       Cx<T>* out);
template <typename T> bool momentum_contract_v2(blr_ctx* c, FlowRef v, int substeps, const Cx<T>* rho_end,
                                                const Cx<T>* phi, const double* weights, bool transpose,
                                                T* dphi_cache, int cache_mode, Cx<T>* out);

// full grid (blr_grid.cu)
template <typename T> void warp(blr_ctx* c, const T* f, int nimg, const T* disp, int n_disp, int interp, T* out);
template <typename T> void grid_gradient(blr_ctx* c, const T* f, int nf, int mode, T* out);
template <typename T> void jacobian_det(blr_ctx* c, const T* u, T* out);
template <typename T> void state_gn_accumulate(blr_ctx* c, const T* dlam, const T* vol, const T* psi,
                                               const T* gm, int n_nodes, const double* weights, int interp,
                                               T* acc);
template <typename T> void dot_fields(blr_ctx* c, const T* g, const T* u, double cc, T* out);
template <typename T> void scale_fields(blr_ctx* c, const T* s, const T* g, T* out);
template <typename T> void scaled_diff(blr_ctx* c, const T* a, const T* b, double cc, T* out);
template <typename T> void mul(blr_ctx* c, const T* a, const T* b, int64_t n, T* out);
template <typename T> void state_data(blr_ctx* c, const T* vol, const T* lamw, const T* gm, int n_nodes,
                                      const double* weights, T* out);
template <typename T> void state_newton(blr_ctx* c, const T* dlam, const T* dl, int interp, const T* vol,
                                        const T* aew, const T* dvol, const T* agw, const T* dpsi, const T* psi,
                                        const T* wg, const T* sgw, const T* dphi, int n_nodes,
                                        const double* weights, int grad_mode, T* out);
template <typename T> void lam_matvec_add(blr_ctx* c, const T* s, const T* H, const T* u, T* out);

}  // namespace blr
