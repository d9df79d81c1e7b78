/*
 * blreg_b200 — C ABI of the B200 (sm_100a) band-limited LDDMM hot path.
 *
 * Plain pointers and sizes only.  Every array pointer is DEVICE memory on the
 * context's device, contiguous, in the precision chosen at context creation
 * (dtype 0: float64 / complex128, dtype 1: float32 / complex64).  Complex
 * arrays are interleaved (re, im).  All work is enqueued on the stream set
 * with blr_set_stream (default: the legacy default stream); functions return
 * without synchronising unless they return a host scalar.
 *
 * Layouts (the reference's, objectives/base.py + transport.py:36-126):
 *   band block      [B0][B1][B2]       complex, FFT wrap order, B = 2K+1
 *   vector block    [d][B0][B1][B2]
 *   node trajectory [n_nodes][comp][B0][B1][B2]   (ascending time)
 *   grid field      [N0][N1][N2]       real, C order
 * Lower-dimensional domains use the trailing axes (2-D: [N0][N1] etc.).
 *
 * The reference ("blreg", /root/reference/pkg/src/blreg) has no FFI; its
 * boundary is the Python objective protocol.  Each entry point below cites
 * the reference function it replaces.  The Python host package
 * paper_1807_05117_b200 binds this ABI with ctypes.
 *
 * Return value: 0 on success, nonzero on error; blr_last_error() gives the
 * message (thread-local).  Error codes: 1 invalid argument, 2 CUDA error,
 * 3 cuFFT error, 4 CFL / numerical condition.
 */
#ifndef BLREG_B200_H
#define BLREG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct blr_ctx blr_ctx;

/* ---- context ------------------------------------------------------------ */

/* Domain + pad grid + metric.  Replaces Domain (domain.py:19-97) and the pad
 * choice _pad_shape (spectral.py:142-145; any pad >= 3K+1 is exact).
 * symbol_tab: per axis, B_a doubles of alpha-free symbol terms s_a(k)
 * (spectral.py:242-257: 2 N^2 (1 - cos(2 pi k / N)) or (2 pi k)^2),
 * concatenated over the d axes. */
int blr_ctx_create(blr_ctx** out, int ndim, const int* shape, const int* bandwidth,
                   const int* pad, double alpha, int order, const double* symbol_tab,
                   int dtype, int device);
int blr_ctx_destroy(blr_ctx* ctx);
int blr_set_stream(blr_ctx* ctx, void* cuda_stream);
const char* blr_last_error(void);
/* number of kernels this library launched since load (all contexts) */
int64_t blr_launch_count(void);
int blr_version(void);
/* CUDA-event profiler over kernel categories (scatter, gather, cuFFT, products,
 * RK4 updates, warps, ...).  Off by default; when on, every instrumented launch
 * records events on its stream.  report: JSON {"name": [launches, total_ms,
 * algorithmic_bytes], ...} of everything recorded since the last report. */
/* engine option: 1 fused y+x forward projection (one thread-block cluster
 * per (output, kz) plane), 0 (default) the two-kernel path; both give
 * bit-identical results (tests/test_gpu_fused.py) */
int blr_set_fused_forward(int on);
int blr_profile_enable(int on);
int blr_profile_report(char* buf, int64_t len);

/* ---- spectral algebra (spectral.py) -------------------------------------- */

/* include: band blocks -> real grid fields (spectral.py:89-119).
 * grid 0 = full image grid, 1 = pad grid.  deriv[f] in {-1, 0..d-1}: realize
 * i*2*pi*k_axis * block (spectral_gradient / spectral_jacobian fused), or NULL. */
int blr_include(blr_ctx* ctx, int grid, const void* blocks, int nfields, const int* deriv,
                void* out);
/* project: real grid fields -> band blocks (forward DFT / prod, truncate,
 * symmetrize; spectral.py:122-135). */
int blr_project(blr_ctx* ctx, int grid, const void* fields, int nfields, void* out);
/* out = in * A(k)^power, power in {+order, -order} via sign (spectral.py:260-272) */
int blr_helmholtz(blr_ctx* ctx, const void* in, int nblocks, int inverse, void* out);
/* Leray projection of vector blocks (spectral.py:312-328) */
int blr_leray(blr_ctx* ctx, const void* in, int nvec, void* out);
/* spectral divergence of vector blocks (spectral.py:284-289), per vector */
int blr_divergence(blr_ctx* ctx, const void* in, int nvec, void* out);
/* out = symmetrize(in) (spectral.py:45-47) */
int blr_symmetrize(blr_ctx* ctx, const void* in, int nblocks, void* out);

/* ---- linear algebra on flows (solver.py:88-126, transport.py:147-153) ----- */

/* host result: Re sum a * conj(b) over n complex entries (spectral.inner) */
int blr_inner(blr_ctx* ctx, const void* a, const void* b, int64_t n, double* result);
/* host result: time-weighted sum_i w_i Re<a_i, b_i> over n_nodes nodes of n each */
int blr_inner_nodes(blr_ctx* ctx, const void* a, const void* b, int n_nodes, int64_t n,
                    const double* weights, double* result);
/* y = a*x + b*y (complex arrays of n entries, real scalars) */
int blr_axpby(blr_ctx* ctx, double a, const void* x, double b, void* y, int64_t n);
/* out = x + a*p  and  r2 = r - a*hp in one pass (PCG update, solver.py:115-117) */
int blr_pcg_update(blr_ctx* ctx, double a, const void* p, const void* hp, void* x, void* r,
                   int64_t n);
/* host result: max |f| over n real entries */
int blr_max_abs(blr_ctx* ctx, const void* f, int64_t n, double* result);
/* host result: sum (a-b)^2 over n real entries (b may be NULL) */
int blr_sq_dist(blr_ctx* ctx, const void* a, const void* b, int64_t n, double* result);
/* host result: 1 if all n real entries are finite */
int blr_all_finite(blr_ctx* ctx, const void* f, int64_t n, int* result);

/* ---- transport (transport.py:206-465) ------------------------------------ */
/* v / dv: flow nodes [n_stored][d][B^3]; stationary iff n_stored == 1.
 * Node outputs are [n_steps+1][...] ascending in time; NULL skips recording. */

/* forward map phi~ (transport.py:351-363).  du_cache (nullable): receives the
 * pad-grid realizations of D(u) at every RK4 stage ([4*n_steps*substeps][d*d][P^3]
 * reals), reused by blr_state_tangents to skip the base re-integration. */
int blr_forward_map(blr_ctx* ctx, const void* v, int n_stored, int n_steps, int substeps,
                    void* phi_nodes, void* du_cache);
/* inverse map psi~ and volume J~ (transport.py:366-383) */
int blr_inverse_map_and_volume(blr_ctx* ctx, const void* v, int n_stored, int n_steps,
                               int substeps, void* psi_nodes, void* vol_nodes);
/* tangents (transport.py:386-432).  flags: bit0 = forward pair (dphi),
 * bit1 = backward pair (dpsi), bit2 = volume pair (dvol, needs bit1),
 * bit3 = record only the final forward node (dphi_nodes holds one node).
 * du_cache (nullable) from blr_forward_map with the same v and substeps. */
int blr_state_tangents(blr_ctx* ctx, const void* v, const void* dv, int n_stored, int n_steps,
                       int substeps, int flags, const void* du_cache, void* dphi_nodes,
                       void* dpsi_nodes, void* dvol_nodes);
/* backward conservative momentum transport (transport.py:435-445) */
int blr_momentum(blr_ctx* ctx, const void* v, int n_stored, int n_steps, int substeps,
                 const void* rho_end, void* rho_nodes);
/* momentum + tangent (transport.py:448-465); gauss_newton drops the rho x dv
 * source, in which case rho_nodes may be NULL and the base is not integrated. */
int blr_momentum_tangent(blr_ctx* ctx, const void* v, const void* dv, int n_stored, int n_steps,
                         int substeps, const void* rho_end, const void* drho_end,
                         int gauss_newton, void* rho_nodes, void* drho_nodes);
/* Jacobian contraction (deformation.py:63-72) summed over nodes:
 *   out[i] = rho_i + pi(D(phi_i)^T rho_i)  (transpose=1) or D(phi_i) rho_i.
 * weights == NULL: per-node outputs out[n_nodes][d][B^3]; otherwise the
 * weighted sum sum_i w_i out_i into out[d][B^3].
 * dphi_cache (nullable): [n_nodes][d*d][P^3] realizations of D(phi_i);
 * cache_mode 0 = ignore, 1 = fill it, 2 = read it (phi_nodes unused). */
int blr_contract(blr_ctx* ctx, const void* phi_nodes, const void* rho_nodes, int n_nodes,
                 const double* weights, int transpose, void* dphi_cache, int cache_mode,
                 void* out);
/* backward momentum transport fused with the summed contraction:
 * out = sum_n w_n (rho_n + project(D(phi_n)^(T|.) rho_n)), rho_n the momentum
 * nodes of blr_momentum(v, rho_end).  Equals blr_momentum followed by
 * blr_contract(weights != NULL) without materializing the rho node records
 * (the Gauss-Newton deformation HVP data term, deformation.py:140-153 +
 * transport.py:435-445).  weights: n_steps + 1 doubles (host). */
int blr_momentum_contract(blr_ctx* ctx, const void* v, int n_stored, int n_steps, int substeps,
                          const void* rho_end, const void* phi_nodes, const double* weights,
                          int transpose, void* dphi_cache, int cache_mode, void* out);
/* generic truncated product pi(iota(M) . iota(x)) with optional transpose
 * (spectral.conv_matvec, spectral.py:194-200) for one (d x d, d) pair. */
int blr_conv_matvec(blr_ctx* ctx, const void* M, const void* x, int transpose, void* out);

/* ---- full-grid operations (gridops.py) ----------------------------------- */
/* warp: out[j] = f[j](x + u(x)) periodic; interp 0 nearest, 1 linear, 3 cubic
 * (gridops.py:21-48; cubic = periodic B-spline with exact prefilter).
 * nimg images share one displacement [d][N^3]; n_disp displacements
 * (stride d*N^3) map to n_disp*nimg outputs when n_disp > 1 (nimg must be 1). */
int blr_warp(blr_ctx* ctx, const void* f, int nimg, const void* disp, int n_disp, int interp,
             void* out);
/* central (mode 0) or spectral (mode 1) gradient of nf scalar fields
 * (gridops.py:78-100); out [nf][d][N^3] */
int blr_grid_gradient(blr_ctx* ctx, const void* f, int nf, int mode, void* out);
/* det(I + D u) by central differences (gridops.py:103-131) */
int blr_jacobian_det(blr_ctx* ctx, const void* disp, void* out);
/* fused Gauss-Newton state data term (state.py:125-137 + base.py:165-168):
 *   acc[a](x) = sum_i w_i * vol_i(x) * dlam(x + psi_i(x)) * gm_i[a](x)
 * vol [n_nodes][N^3], psi [n_nodes][d][N^3], gm [n_nodes][d][N^3] */
int blr_state_gn_accumulate(blr_ctx* ctx, const void* dlam, const void* vol, const void* psi,
                            const void* gm, int n_nodes, const double* weights, int interp,
                            void* acc);
/* pointwise: out = c * sum_a g[a] * u[a]   (dlam1 = -(2/sigma2) grad(I0)o phi . dphi) */
int blr_dot_fields(blr_ctx* ctx, const void* g, const void* u, double c, void* out);
/* pointwise: out[a] = s * g[a]  (a < d) */
int blr_scale_fields(blr_ctx* ctx, const void* s, const void* g, void* out);
/* pointwise: out = c * (a - b) */
int blr_scaled_diff(blr_ctx* ctx, const void* a, const void* b, double c, void* out);
/* pointwise: out = a * b */
int blr_mul(blr_ctx* ctx, const void* a, const void* b, int64_t n, void* out);
/* state gradient data term: acc[a] = sum_i w_i vol_i * lamw_i * gm_i[a];
 * weights NULL -> per-node outputs [n_nodes][d][N^3] */
int blr_state_data(blr_ctx* ctx, const void* vol, const void* lamw, const void* gm,
                   int n_nodes, const double* weights, void* out);
/* full-Newton state data term (state.py:138-154), one pass over the nodes:
 *   dm_k = sgw_k . dphi_k,  dl_k = dlam o (id + psi_k)  (or the given dl [n][N^3]),
 *   dlam_k = dvol_k aew_k + vol_k (agw_k . dpsi_k) + vol_k dl_k,
 *   term_k = dlam_k wg_k + vol_k aew_k grad(dm_k)   (grad_mode 0 central, 1 spectral)
 * out = sum_k w_k term_k [d][N^3], or weights NULL -> per node [n][d][N^3].
 * scalars [n][N^3]: vol, aew, dvol; vectors [n][d][N^3]: agw, dpsi, psi, wg, sgw, dphi */
int blr_state_newton(blr_ctx* ctx, const void* dlam, const void* dl, int interp, const void* vol,
                     const void* aew, const void* dvol, const void* agw, const void* dpsi,
                     const void* psi, const void* wg, const void* sgw, const void* dphi, int n_nodes,
                     const double* weights, int grad_mode, void* out);
/* out[a] += s * sum_b H[a][b] u[b]  (deformation.py:141-145, transposed Newton endpoint
 * term, H [d][d][N^3]); H NULL -> out[a] += s * u[a] */
int blr_lam_matvec_add(blr_ctx* ctx, const void* s, const void* H, const void* u, void* out);

#ifdef __cplusplus
}
#endif

#endif /* BLREG_B200_H */
