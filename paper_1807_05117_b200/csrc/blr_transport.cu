// blr_transport.cu — RK4 spectral transport on sm_100a (transport.py:206-465).
//
// Every right-hand side is a truncated convolution: realize band blocks on
// the pad grid (fused scatter + C2R), form the pointwise products in one
// streaming kernel, project back (R2C + fused gather/symmetrize), then apply
// the band epilogue (-(v + .), flux divergence).  RK4 state is one contiguous
// complex array per sweep so each stage update is a single launch.
//
// Redundant work the reference performs and this path skips (outputs are
// identical):
//   * D(u) is realized once per stage and shared by the base and tangent RHS;
//   * a stationary v / dv (and div v) is realized once per sweep;
//   * blr_forward_map can record D(u) at every stage so blr_state_tangents
//     does not re-integrate the base map;
//   * in Gauss-Newton mode the base momentum is not integrated (its output
//     is unused, transport.py:460-462).
#include "blr_internal.cuh"

#include <cmath>
#include <cstring>

namespace blr {

// ---------------------------------------------------------------------------
// pad-grid pointwise products
// ---------------------------------------------------------------------------
enum ProdOp {
  kMatVec = 0,     // out_i = sum_j M_ij x_j  (+ sum_j M2_ij x2_j)
  kMatVecT = 1,    // out_i = sum_j M_ji x_j
  kVolume = 2,     // out = -sum_a V_a G_a - J * Dv
  kVolumeT = 3,    // out = -sum dV.G - sum V.dG - dJ*Dv - J*dDv
  kOuter = 4,      // out_ij = a_i b_j (+ a2_i b2_j)
  kMatVecAcc = 5,  // out_i += w * sum_j M_(ij|ji) x_j
};

template <typename T>
struct ProdArgs {
  const T* M;   // [d*d][np]
  const T* x;   // [d][np]
  const T* M2;
  const T* x2;
  const T* a;   // volume: V [d]; outer: a [d]
  const T* b;   // volume: G [d]; outer: b [d]
  const T* a2;  // volume tangent: dV ; outer: a2
  const T* b2;  // volume tangent: dG ; outer: b2
  const T* J;
  const T* Dv;
  const T* dJ;
  const T* dDv;
  T* out;
  T w;
  int transpose;
  int64_t np;
  int d;
};

template <typename T, int OP>
__global__ void __launch_bounds__(256) k_prod(ProdArgs<T> p) {
  const int64_t np = p.np;
  const int d = p.d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (OP == kMatVec || OP == kMatVecT || OP == kMatVecAcc) {
      T xv[3], x2v[3];
      for (int j = 0; j < d; ++j) {
        xv[j] = p.x[j * np + i];
        if (p.M2) x2v[j] = p.x2[j * np + i];
      }
      for (int r = 0; r < d; ++r) {
        T acc = 0;
        for (int j = 0; j < d; ++j) {
          int mi = (OP == kMatVecT || (OP == kMatVecAcc && p.transpose)) ? (j * d + r) : (r * d + j);
          acc += p.M[(int64_t)mi * np + i] * xv[j];
        }
        if (OP == kMatVec && p.M2) {
          T acc2 = 0;
          for (int j = 0; j < d; ++j) acc2 += p.M2[(int64_t)(r * d + j) * np + i] * x2v[j];
          acc = acc + acc2;
        }
        if (OP == kMatVecAcc) p.out[r * np + i] += p.w * acc;
        else p.out[r * np + i] = acc;
      }
    } else if (OP == kVolume) {
      T s = 0;
      for (int a = 0; a < d; ++a) s += p.a[a * np + i] * p.b[a * np + i];
      p.out[i] = -s - p.J[i] * p.Dv[i];
    } else if (OP == kVolumeT) {
      T s1 = 0, s2 = 0;
      for (int a = 0; a < d; ++a) s1 += p.a2[a * np + i] * p.b[a * np + i];
      for (int a = 0; a < d; ++a) s2 += p.a[a * np + i] * p.b2[a * np + i];
      p.out[i] = -s1 - s2 - p.dJ[i] * p.Dv[i] - p.J[i] * p.dDv[i];
    } else if (OP == kOuter) {
      for (int r = 0; r < d; ++r) {
        T ar = p.a[r * np + i];
        T a2r = p.a2 ? p.a2[r * np + i] : (T)0;
        for (int j = 0; j < d; ++j) {
          T v = ar * p.b[j * np + i];
          if (p.a2) v = v + a2r * p.b2[j * np + i];
          p.out[(int64_t)(r * d + j) * np + i] = v;
        }
      }
    }
  }
}

template <typename T, int OP>
static void prod(blr_ctx* c, ProdArgs<T> p) {
  p.np = c->g.np();
  p.d = c->g.d;
  const int d = p.d;
  double fields = 0;
  if (OP == kMatVec) fields = (p.M2 ? 2 : 1) * (d * d + d) + d;
  if (OP == kMatVecT) fields = d * d + 2 * d;
  if (OP == kMatVecAcc) fields = d * d + 3 * d;
  if (OP == kVolume) fields = 2 * d + 3;
  if (OP == kVolumeT) fields = 4 * d + 5;
  if (OP == kOuter) fields = (p.a2 ? 4 * d : 2 * d) + d * d;
  ProfScope ps(c, "pad_product", fields * p.np * sizeof(T));
  k_prod<T, OP><<<grid_blocks(p.np, 256), 256, 0, c->stream>>>(p);
  BLR_LAUNCHED();
}

template <typename T>
static ProdArgs<T> pargs() {
  ProdArgs<T> p;
  std::memset(&p, 0, sizeof(p));
  p.w = (T)1;
  return p;
}

// ---------------------------------------------------------------------------
// stream-ordered temporaries
// ---------------------------------------------------------------------------
struct Tmp {
  blr_ctx* c;
  std::vector<void*> ptrs;
  explicit Tmp(blr_ctx* ctx) : c(ctx) {}
  template <typename X>
  X* get(int64_t n) {
    void* p = nullptr;
    BLR_CUDA(cudaMallocAsync(&p, (size_t)std::max<int64_t>(n, 1) * sizeof(X), c->stream));
    ptrs.push_back(p);
    return (X*)p;
  }
  ~Tmp() {
    for (void* p : ptrs) cudaFreeAsync(p, c->stream);
  }
};

// ---------------------------------------------------------------------------
// velocity samples: band block + pad realization (+ divergence) at time t
// ---------------------------------------------------------------------------
template <typename T>
struct VelBank {
  blr_ctx* c;
  FlowRef f;
  bool with_div;
  int nfields;  // d (+1)
  struct Entry {
    double t;
    bool valid;
    const Cx<T>* band;
    Cx<T>* own;
    T* real;
    int64_t age;
  } e[3];
  int64_t clock = 0;

  VelBank(blr_ctx* ctx, FlowRef flow, bool div, Tmp& tmp) : c(ctx), f(flow), with_div(div) {
    const Geom& g = c->g;
    nfields = g.d + (div ? 1 : 0);
    int ne = f.stationary() ? 1 : 3;
    for (int i = 0; i < 3; ++i) {
      e[i].valid = false;
      e[i].own = nullptr;
      e[i].real = nullptr;
      e[i].band = nullptr;
      e[i].age = 0;
    }
    for (int i = 0; i < ne; ++i) {
      e[i].real = tmp.get<T>(nfields * g.np());
      if (!f.stationary()) e[i].own = tmp.get<Cx<T>>(g.d * g.nb());
    }
    if (f.stationary()) fill(e[0], (const Cx<T>*)f.v, 0.0);
  }

  void fill(Entry& en, const Cx<T>* band, double t) {
    const Geom& g = c->g;
    std::vector<ScatterField<T>> fl;
    for (int a = 0; a < g.d; ++a) fl.push_back(fld<T>(band + a * g.nb(), -1));
    if (with_div) fl.push_back(fld_div<T>(g, band));
    realize<T>(c, true, fl, en.real);
    en.band = band;
    en.t = t;
    en.valid = true;
  }

  const Entry& at(double t) {
    if (f.stationary()) return e[0];
    ++clock;
    for (auto& en : e)
      if (en.valid && en.t == t) {
        en.age = clock;
        return en;
      }
    Entry* victim = &e[0];
    for (auto& en : e)
      if (!en.valid || en.age < victim->age) victim = &en;
    // TimeFlow.sample (transport.py:77-86)
    const Geom& g = c->g;
    const int n = f.n_steps;
    double s = std::min(std::max(t, 0.0), 1.0) * n;
    int i = std::min((int)std::floor(s), n - 1);
    double w = s - i;
    const Cx<T>* base = (const Cx<T>*)f.v;
    const int64_t L = g.d * g.nb();
    const Cx<T>* band;
    if (w == 0.0) {
      band = base + i * L;
    } else {
      band_lerp<T>(c, base + i * L, base + (i + 1) * L, w, victim->own, L);
      band = victim->own;
    }
    fill(*victim, band, t);
    victim->age = clock;
    return *victim;
  }
};

// ---------------------------------------------------------------------------
// RK4 driver (transport.py:310-344)
// ---------------------------------------------------------------------------
struct Recorder {
  int64_t offset;  // within the state (complex entries)
  int64_t len;
  void* dst;       // [n_steps+1][len] or nullptr
};

template <typename T, typename Rhs>
static void rk4(blr_ctx* c, int n_steps, int substeps, bool forward, Cx<T>* cur, int64_t L,
                const std::vector<Recorder>& rec, Tmp& tmp, Rhs rhs) {
  Cx<T>* k = tmp.get<Cx<T>>(L);
  Cx<T>* acc = tmp.get<Cx<T>>(L);
  Cx<T>* stage = tmp.get<Cx<T>>(L);
  const int n = n_steps;
  const double dt = (forward ? 1.0 : -1.0) / n;
  const double h = dt / substeps;
  auto record = [&](int node) {
    for (const auto& r : rec)
      if (r.dst)
        BLR_CUDA(cudaMemcpyAsync((Cx<T>*)r.dst + (int64_t)node * r.len, cur + r.offset,
                                 r.len * sizeof(Cx<T>), cudaMemcpyDeviceToDevice, c->stream));
  };
  record(forward ? 0 : n);
  int stage_idx = 0;
  for (int step = 0; step < n; ++step) {
    int node = forward ? step : n - step;
    double t0 = (double)node / n;
    for (int ks = 0; ks < substeps; ++ks) {
      double t = t0 + ks * h;
      rhs(stage_idx + 0, t, (const Cx<T>*)cur, k);
      band_rk4<T>(c, 1, k, cur, acc, stage, 0.5 * h, h / 6.0, L);
      rhs(stage_idx + 1, t + 0.5 * h, (const Cx<T>*)stage, k);
      band_rk4<T>(c, 2, k, cur, acc, stage, 0.5 * h, h / 6.0, L);
      rhs(stage_idx + 2, t + 0.5 * h, (const Cx<T>*)stage, k);
      band_rk4<T>(c, 3, k, cur, acc, stage, h, h / 6.0, L);
      rhs(stage_idx + 3, t + h, (const Cx<T>*)stage, k);
      band_rk4<T>(c, 4, k, cur, acc, stage, h, h / 6.0, L);
      stage_idx += 4;
    }
    record(forward ? node + 1 : node - 1);
  }
}

template <typename T>
static void set_unit_scalar(blr_ctx* c, Cx<T>* blk) {
  Cx<T> one;
  one.x = (T)1;
  one.y = (T)0;
  BLR_CUDA(cudaMemcpyAsync(blk, &one, sizeof(one), cudaMemcpyHostToDevice, c->stream));
}

// D(u) fields, out[i*d+j] = d_j u_i  (spectral_jacobian, spectral.py:292-300)
template <typename T>
static void push_jac(const Geom& g, const Cx<T>* u, std::vector<ScatterField<T>>& f) {
  for (int i = 0; i < g.d; ++i)
    for (int j = 0; j < g.d; ++j) f.push_back(fld<T>(u + i * g.nb(), g.axis_of(j)));
}

template <typename T>
static void push_grad(const Geom& g, const Cx<T>* s, std::vector<ScatterField<T>>& f) {
  for (int a = 0; a < g.d; ++a) f.push_back(fld<T>(s, g.axis_of(a)));
}

// ---------------------------------------------------------------------------
// integrators
// ---------------------------------------------------------------------------
template <typename T>
void forward_map(blr_ctx* c, FlowRef v, int substeps, Cx<T>* phi, T* du_cache) {
  if (forward_map_v2<T>(c, v, substeps, phi, du_cache)) return;
  const Geom& g = c->g;
  const int d = g.d;
  const int64_t nb = g.nb(), np = g.np(), L = d * nb;
  Tmp tmp(c);
  VelBank<T> V(c, v, false, tmp);
  Cx<T>* cur = tmp.get<Cx<T>>(L);
  BLR_CUDA(cudaMemsetAsync(cur, 0, L * sizeof(Cx<T>), c->stream));
  T* Jslots = du_cache ? nullptr : tmp.get<T>(d * d * np);
  T* P = tmp.get<T>(d * np);
  rk4<T>(c, v.n_steps, substeps, true, cur, L, {{0, L, phi}}, tmp,
         [&](int si, double t, const Cx<T>* s, Cx<T>* k) {
           const auto& vt = V.at(t);
           T* J = du_cache ? du_cache + (int64_t)si * d * d * np : Jslots;
           std::vector<ScatterField<T>> f;
           push_jac<T>(g, s, f);
           realize<T>(c, true, f, J);
           ProdArgs<T> p = pargs<T>();
           p.M = J;
           p.x = vt.real;
           p.out = P;
           prod<T, kMatVec>(c, p);
           project<T>(c, true, P, d, k);
           band_neg_add<T>(c, vt.band, k, k, L);  // -(v + Du*v)   (transport.py:206-213)
         });
}

template <typename T>
void inverse_map_and_volume(blr_ctx* c, FlowRef v, int substeps, Cx<T>* psi, Cx<T>* vol) {
  if (inverse_map_and_volume_v2<T>(c, v, substeps, psi, vol)) return;
  const Geom& g = c->g;
  const int d = g.d;
  const int64_t nb = g.nb(), np = g.np(), L = (d + 1) * nb;
  Tmp tmp(c);
  VelBank<T> V(c, v, true, tmp);
  Cx<T>* cur = tmp.get<Cx<T>>(L);
  BLR_CUDA(cudaMemsetAsync(cur, 0, L * sizeof(Cx<T>), c->stream));
  set_unit_scalar<T>(c, cur + d * nb);
  T* R = tmp.get<T>((d * d + d + 1) * np);  // [Dw (d*d) | grad J (d) | J]
  T* P = tmp.get<T>((d + 1) * np);
  rk4<T>(c, v.n_steps, substeps, false, cur, L, {{0, d * nb, psi}, {d * nb, nb, vol}}, tmp,
         [&](int, double t, const Cx<T>* s, Cx<T>* k) {
           const auto& vt = V.at(t);
           std::vector<ScatterField<T>> f;
           push_jac<T>(g, s, f);
           push_grad<T>(g, s + d * nb, f);
           f.push_back(fld<T>(s + d * nb, -1));
           realize<T>(c, true, f, R);
           ProdArgs<T> p = pargs<T>();
           p.M = R;
           p.x = vt.real;
           p.out = P;
           prod<T, kMatVec>(c, p);
           ProdArgs<T> q = pargs<T>();
           q.a = vt.real;
           q.b = R + d * d * np;
           q.J = R + (d * d + d) * np;
           q.Dv = vt.real + d * np;
           q.out = P + d * np;
           prod<T, kVolume>(c, q);  // transport.py:231-241
           project<T>(c, true, P, d + 1, k);
           band_neg_add<T>(c, vt.band, k, k, d * nb);
         });
}

template <typename T>
void state_tangents(blr_ctx* c, FlowRef v, FlowRef dv, int substeps, int flags, const T* du_cache,
                    Cx<T>* dphi, Cx<T>* dpsi, Cx<T>* dvol) {
  if (state_tangents_v2<T>(c, v, dv, substeps, flags, du_cache, dphi, dpsi, dvol)) return;
  if ((flags & 8) && dphi && (flags & 1)) {
    // final forward node only: run the recording path into a temporary and keep the last node
    const int64_t node = (int64_t)c->g.d * c->g.nb();
    Cx<T>* all = nullptr;
    BLR_CUDA(cudaMallocAsync((void**)&all, (size_t)(v.n_steps + 1) * node * sizeof(Cx<T>), c->stream));
    state_tangents<T>(c, v, dv, substeps, flags & ~8, du_cache, all, dpsi, dvol);
    BLR_CUDA(cudaMemcpyAsync(dphi, all + (int64_t)v.n_steps * node, node * sizeof(Cx<T>),
                             cudaMemcpyDeviceToDevice, c->stream));
    BLR_CUDA(cudaFreeAsync(all, c->stream));
    return;
  }
  const Geom& g = c->g;
  const int d = g.d;
  const int64_t nb = g.nb(), np = g.np();
  Tmp tmp(c);
  const bool want_fwd = flags & 1, want_bwd = flags & 2, want_vol = (flags & 4) && want_bwd;
  if (want_fwd) {
    VelBank<T> V(c, v, false, tmp);
    VelBank<T> dV(c, dv, false, tmp);
    const bool cached = du_cache != nullptr;
    const int64_t L = (cached ? 1 : 2) * d * nb;  // [u | du] or [du]
    Cx<T>* cur = tmp.get<Cx<T>>(L);
    BLR_CUDA(cudaMemsetAsync(cur, 0, L * sizeof(Cx<T>), c->stream));
    T* R = tmp.get<T>((cached ? 1 : 2) * d * d * np);  // [J | dJ] or [dJ]
    T* P = tmp.get<T>(2 * d * np);
    const int64_t du_off = cached ? 0 : d * nb;
    rk4<T>(c, v.n_steps, substeps, true, cur, L, {{du_off, d * nb, dphi}}, tmp,
           [&](int si, double t, const Cx<T>* s, Cx<T>* k) {
             const auto& vt = V.at(t);
             const auto& dvt = dV.at(t);
             std::vector<ScatterField<T>> f;
             const T* J;
             T* dJ;
             if (cached) {
               J = du_cache + (int64_t)si * d * d * np;
               dJ = R;
               push_jac<T>(g, s, f);
             } else {
               J = R;
               dJ = R + d * d * np;
               push_jac<T>(g, s, f);
               push_jac<T>(g, s + d * nb, f);
             }
             realize<T>(c, true, f, cached ? dJ : R);
             T* Pq = cached ? P : P + d * np;
             if (!cached) {
               ProdArgs<T> p = pargs<T>();
               p.M = J;
               p.x = vt.real;
               p.out = P;
               prod<T, kMatVec>(c, p);
             }
             ProdArgs<T> q = pargs<T>();  // dDu v + Du dv  (transport.py:216-228)
             q.M = dJ;
             q.x = vt.real;
             q.M2 = J;
             q.x2 = dvt.real;
             q.out = Pq;
             prod<T, kMatVec>(c, q);
             project<T>(c, true, P, cached ? d : 2 * d, k);
             if (!cached) band_neg_add<T>(c, vt.band, k, k, d * nb);
             band_neg_add<T>(c, dvt.band, k + du_off, k + du_off, d * nb);
           });
  }
  if (want_bwd) {
    VelBank<T> V(c, v, want_vol, tmp);
    VelBank<T> dV(c, dv, want_vol, tmp);
    // state [w | dw | J | dJ]
    const int64_t L = (2 * d + (want_vol ? 2 : 0)) * nb;
    Cx<T>* cur = tmp.get<Cx<T>>(L);
    BLR_CUDA(cudaMemsetAsync(cur, 0, L * sizeof(Cx<T>), c->stream));
    if (want_vol) set_unit_scalar<T>(c, cur + 2 * d * nb);
    const int nr = 2 * d * d + (want_vol ? 2 * d + 2 : 0);
    T* R = tmp.get<T>(nr * np);
    T* P = tmp.get<T>((2 * d + 2) * np);
    std::vector<Recorder> rec = {{d * nb, d * nb, dpsi}};
    if (want_vol) rec.push_back({(2 * d + 1) * nb, nb, dvol});
    rk4<T>(c, v.n_steps, substeps, false, cur, L, rec, tmp,
           [&](int, double t, const Cx<T>* s, Cx<T>* k) {
             const auto& vt = V.at(t);
             const auto& dvt = dV.at(t);
             std::vector<ScatterField<T>> f;
             push_jac<T>(g, s, f);           // J  [0, d*d)
             push_jac<T>(g, s + d * nb, f);  // dJ [d*d, 2d*d)
             if (want_vol) {
               const Cx<T>* Jb = s + 2 * d * nb;
               const Cx<T>* dJb = s + (2 * d + 1) * nb;
               push_grad<T>(g, Jb, f);   // G
               push_grad<T>(g, dJb, f);  // dG
               f.push_back(fld<T>(Jb, -1));
               f.push_back(fld<T>(dJb, -1));
             }
             realize<T>(c, true, f, R);
             ProdArgs<T> p = pargs<T>();
             p.M = R;
             p.x = vt.real;
             p.out = P;
             prod<T, kMatVec>(c, p);
             ProdArgs<T> q = pargs<T>();
             q.M = R + d * d * np;
             q.x = vt.real;
             q.M2 = R;
             q.x2 = dvt.real;
             q.out = P + d * np;
             prod<T, kMatVec>(c, q);
             int np_out = 2 * d;
             if (want_vol) {
               const T* G = R + 2 * d * d * np;
               const T* dG = G + d * np;
               const T* Jr = dG + d * np;
               const T* dJr = Jr + np;
               ProdArgs<T> r = pargs<T>();
               r.a = vt.real;
               r.b = G;
               r.J = Jr;
               r.Dv = vt.real + d * np;
               r.out = P + 2 * d * np;
               prod<T, kVolume>(c, r);
               ProdArgs<T> s2 = pargs<T>();  // transport.py:244-261
               s2.a = vt.real;
               s2.a2 = dvt.real;
               s2.b = G;
               s2.b2 = dG;
               s2.J = Jr;
               s2.dJ = dJr;
               s2.Dv = vt.real + d * np;
               s2.dDv = dvt.real + d * np;
               s2.out = P + (2 * d + 1) * np;
               prod<T, kVolumeT>(c, s2);
               np_out += 2;
             }
             project<T>(c, true, P, np_out, k);
             band_neg_add<T>(c, vt.band, k, k, d * nb);
             band_neg_add<T>(c, dvt.band, k + d * nb, k + d * nb, d * nb);
           });
  }
}

template <typename T>
void momentum(blr_ctx* c, FlowRef v, int substeps, const Cx<T>* rho_end, Cx<T>* rho) {
  if (momentum_v2<T>(c, v, substeps, rho_end, rho)) return;
  const Geom& g = c->g;
  const int d = g.d;
  const int64_t nb = g.nb(), np = g.np(), L = d * nb;
  Tmp tmp(c);
  VelBank<T> V(c, v, false, tmp);
  Cx<T>* cur = tmp.get<Cx<T>>(L);
  BLR_CUDA(cudaMemcpyAsync(cur, rho_end, L * sizeof(Cx<T>), cudaMemcpyDeviceToDevice, c->stream));
  T* R = tmp.get<T>(d * np);
  T* F = tmp.get<T>(d * d * np);
  Cx<T>* Fh = tmp.get<Cx<T>>(d * d * nb);
  rk4<T>(c, v.n_steps, substeps, false, cur, L, {{0, L, rho}}, tmp,
         [&](int, double t, const Cx<T>* s, Cx<T>* k) {
           const auto& vt = V.at(t);
           std::vector<ScatterField<T>> f;
           for (int a = 0; a < d; ++a) f.push_back(fld<T>(s + a * nb, -1));
           realize<T>(c, true, f, R);
           ProdArgs<T> p = pargs<T>();  // rho (x) v  (transport.py:277-281)
           p.a = R;
           p.b = vt.real;
           p.out = F;
           prod<T, kOuter>(c, p);
           project<T>(c, true, F, d * d, Fh);
           band_flux_div<T>(c, Fh, 1, k);
         });
}

template <typename T>
void momentum_tangent(blr_ctx* c, FlowRef v, FlowRef dv, int substeps, const Cx<T>* rho_end,
                      const Cx<T>* drho_end, bool gn, Cx<T>* rho, Cx<T>* drho) {
  if (gn) {
    // Gauss-Newton: the tangent is the homogeneous transport of drho
    // (transport.py:284-303 with dvt None); the base only if asked for.
    if (rho) momentum<T>(c, v, substeps, rho_end, rho);
    momentum<T>(c, v, substeps, drho_end, drho);
    return;
  }
  if (momentum_pair_v2<T>(c, v, dv, substeps, rho_end, drho_end, rho, drho)) return;
  const Geom& g = c->g;
  const int d = g.d;
  const int64_t nb = g.nb(), np = g.np(), L = 2 * d * nb;
  Tmp tmp(c);
  VelBank<T> V(c, v, false, tmp);
  VelBank<T> dV(c, dv, false, tmp);
  Cx<T>* cur = tmp.get<Cx<T>>(L);
  BLR_CUDA(cudaMemcpyAsync(cur, rho_end, d * nb * sizeof(Cx<T>), cudaMemcpyDeviceToDevice, c->stream));
  BLR_CUDA(cudaMemcpyAsync(cur + d * nb, drho_end, d * nb * sizeof(Cx<T>), cudaMemcpyDeviceToDevice,
                           c->stream));
  T* R = tmp.get<T>(2 * d * np);
  T* F = tmp.get<T>(2 * d * d * np);
  Cx<T>* Fh = tmp.get<Cx<T>>(2 * d * d * nb);
  rk4<T>(c, v.n_steps, substeps, false, cur, L, {{0, d * nb, rho}, {d * nb, d * nb, drho}}, tmp,
         [&](int, double t, const Cx<T>* s, Cx<T>* k) {
           const auto& vt = V.at(t);
           const auto& dvt = dV.at(t);
           std::vector<ScatterField<T>> f;
           for (int a = 0; a < 2 * d; ++a) f.push_back(fld<T>(s + a * nb, -1));
           realize<T>(c, true, f, R);
           ProdArgs<T> p = pargs<T>();
           p.a = R;
           p.b = vt.real;
           p.out = F;
           prod<T, kOuter>(c, p);
           ProdArgs<T> q = pargs<T>();  // drho (x) v + rho (x) dv
           q.a = R + d * np;
           q.b = vt.real;
           q.a2 = R;
           q.b2 = dvt.real;
           q.out = F + d * d * np;
           prod<T, kOuter>(c, q);
           project<T>(c, true, F, 2 * d * d, Fh);
           band_flux_div<T>(c, Fh, 2, k);
         });
}

// ---------------------------------------------------------------------------
// Jacobian contraction (deformation.py:63-72) and generic conv_matvec
// ---------------------------------------------------------------------------
// backward momentum + summed contraction (the GN deformation HVP data term)
template <typename T>
void momentum_contract(blr_ctx* c, FlowRef v, int substeps, const Cx<T>* rho_end, const Cx<T>* phi,
                       const double* weights, bool transpose, T* dphi_cache, int cache_mode, Cx<T>* out) {
  if (momentum_contract_v2<T>(c, v, substeps, rho_end, phi, weights, transpose, dphi_cache, cache_mode, out))
    return;
  const int64_t node = (int64_t)c->g.d * c->g.nb();
  const int n_nodes = v.n_steps + 1;
  Cx<T>* rho = nullptr;
  BLR_CUDA(cudaMallocAsync((void**)&rho, (size_t)n_nodes * node * sizeof(Cx<T>), c->stream));
  momentum<T>(c, v, substeps, rho_end, rho);
  contract<T>(c, phi, rho, n_nodes, weights, transpose, dphi_cache, cache_mode, out);
  BLR_CUDA(cudaFreeAsync(rho, c->stream));
}

template <typename T>
void contract(blr_ctx* c, const Cx<T>* phi, const Cx<T>* rho, int n_nodes, const double* weights,
              bool transpose, T* dphi_cache, int cache_mode, Cx<T>* out) {
  if (contract_v2<T>(c, phi, rho, n_nodes, weights, transpose, dphi_cache, cache_mode, out)) return;
  const Geom& g = c->g;
  const int d = g.d;
  const int64_t nb = g.nb(), np = g.np(), L = d * nb;
  Tmp tmp(c);
  T* Jslot = cache_mode == 0 ? tmp.get<T>(d * d * np) : nullptr;
  T* R = tmp.get<T>(d * np);
  T* P = tmp.get<T>(d * np);
  Cx<T>* Ph = tmp.get<Cx<T>>(L);
  const bool summed = weights != nullptr;
  if (summed) {
    BLR_CUDA(cudaMemsetAsync(P, 0, d * np * sizeof(T), c->stream));
    BLR_CUDA(cudaMemsetAsync(out, 0, L * sizeof(Cx<T>), c->stream));
  }
  for (int i = 0; i < n_nodes; ++i) {
    T* J = cache_mode == 0 ? Jslot : dphi_cache + (int64_t)i * d * d * np;
    std::vector<ScatterField<T>> f;
    if (cache_mode != 2) push_jac<T>(g, phi + i * L, f);
    for (int a = 0; a < d; ++a) f.push_back(fld<T>(rho + i * L + a * nb, -1));
    if (cache_mode != 2) {
      realize<T>(c, true, std::vector<ScatterField<T>>(f.begin(), f.begin() + d * d), J);
    }
    realize<T>(c, true, std::vector<ScatterField<T>>(f.end() - d, f.end()), R);
    ProdArgs<T> p = pargs<T>();
    p.M = J;
    p.x = R;
    p.transpose = transpose ? 1 : 0;
    if (summed) {
      p.out = P;
      p.w = (T)weights[i];
      prod<T, kMatVecAcc>(c, p);
      band_axpby<T>(c, weights[i], rho + i * L, 1.0, out, L);
    } else {
      p.out = P;
      if (transpose) prod<T, kMatVecT>(c, p);
      else prod<T, kMatVec>(c, p);
      project<T>(c, true, P, d, Ph);
      // out_i = rho_i + pi(.)
      BLR_CUDA(cudaMemcpyAsync(out + i * L, rho + i * L, L * sizeof(Cx<T>), cudaMemcpyDeviceToDevice,
                               c->stream));
      band_axpby<T>(c, 1.0, Ph, 1.0, out + i * L, L);
    }
  }
  if (summed) {
    project<T>(c, true, P, d, Ph);
    band_axpby<T>(c, 1.0, Ph, 1.0, out, L);
  }
}

template <typename T>
void conv_matvec(blr_ctx* c, const Cx<T>* M, const Cx<T>* x, bool transpose, Cx<T>* out) {
  const Geom& g = c->g;
  const int d = g.d;
  const int64_t nb = g.nb(), np = g.np();
  Tmp tmp(c);
  T* R = tmp.get<T>((d * d + d) * np);
  T* P = tmp.get<T>(d * np);
  std::vector<ScatterField<T>> f;
  for (int a = 0; a < d * d; ++a) f.push_back(fld<T>(M + a * nb, -1));
  for (int a = 0; a < d; ++a) f.push_back(fld<T>(x + a * nb, -1));
  realize<T>(c, true, f, R);
  ProdArgs<T> p = pargs<T>();
  p.M = R;
  p.x = R + d * d * np;
  p.out = P;
  if (transpose) prod<T, kMatVecT>(c, p);
  else prod<T, kMatVec>(c, p);
  project<T>(c, true, P, d, out);
}

#define BLR_TINST(T)                                                                           \
  template void forward_map<T>(blr_ctx*, FlowRef, int, Cx<T>*, T*);                            \
  template void inverse_map_and_volume<T>(blr_ctx*, FlowRef, int, Cx<T>*, Cx<T>*);             \
  template void state_tangents<T>(blr_ctx*, FlowRef, FlowRef, int, int, const T*, Cx<T>*,      \
                                  Cx<T>*, Cx<T>*);                                             \
  template void momentum<T>(blr_ctx*, FlowRef, int, const Cx<T>*, Cx<T>*);                     \
  template void momentum_tangent<T>(blr_ctx*, FlowRef, FlowRef, int, const Cx<T>*,             \
                                    const Cx<T>*, bool, Cx<T>*, Cx<T>*);                       \
  template void contract<T>(blr_ctx*, const Cx<T>*, const Cx<T>*, int, const double*, bool, T*, \
                            int, Cx<T>*);                                                      \
  template void momentum_contract<T>(blr_ctx*, FlowRef, int, const Cx<T>*, const Cx<T>*,         \
                                     const double*, bool, T*, int, Cx<T>*);                      \
  template void conv_matvec<T>(blr_ctx*, const Cx<T>*, const Cx<T>*, bool, Cx<T>*);
BLR_TINST(double)
BLR_TINST(float)

}  // namespace blr
