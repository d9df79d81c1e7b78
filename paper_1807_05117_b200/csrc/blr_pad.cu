// blr_pad.cu — host orchestration of the fused pad-grid engine: engine setup,
// length dispatch, realization / projection helpers and the RK4 integrators
// (kernels: blr_pad_kernels.cuh, instantiated per length in blr_pad_L*.cu).
#include "blr_pad_kernels.cuh"

#include <atomic>

#include <array>
#include <cmath>
#include <cstring>
#include <mutex>

namespace blr {

// launchers are instantiated per line length in blr_pad_L*.cu (parallel build)
#define BLR_EXTERN_L(LL, A, B)                                                                         \
  extern template void launch_xinv<double, WShape<A, B>>(blr_ctx*, PadEngine*, const XPassArgs<double>&); \
  extern template void launch_xinv<float, WShape<A, B>>(blr_ctx*, PadEngine*, const XPassArgs<float>&);   \
  extern template void launch_yinv<double, WShape<A, B>>(blr_ctx*, PadEngine*, const YPassArgs<double>&); \
  extern template void launch_yinv<float, WShape<A, B>>(blr_ctx*, PadEngine*, const YPassArgs<float>&);   \
  extern template void launch_yfwd<double, WShape<A, B>>(blr_ctx*, PadEngine*, const YFwdArgs<double>&); \
  extern template void launch_yfwd<float, WShape<A, B>>(blr_ctx*, PadEngine*, const YFwdArgs<float>&);   \
  extern template void launch_xfwd<double, WShape<A, B>>(blr_ctx*, PadEngine*, const FwdArgs<double>&);   \
  extern template void launch_xfwd<float, WShape<A, B>>(blr_ctx*, PadEngine*, const FwdArgs<float>&);
BLR_FOR_EACH_L(BLR_EXTERN_L)
#undef BLR_EXTERN_L
#define BLR_EXTERN_F2(LL, A, B)                                                                        \
  extern template void launch_fwd2<double, WShape<A, B>>(blr_ctx*, PadEngine*, const Fwd2Args<double>&, int, \
                                                         int);                                         \
  extern template void launch_fwd2<float, WShape<A, B>>(blr_ctx*, PadEngine*, const Fwd2Args<float>&, int,   \
                                                        int);                                          \
  extern template bool fwd2_fits<double, WShape<A, B>>(const PadGeom&);                                \
  extern template bool fwd2_fits<float, WShape<A, B>>(const PadGeom&);
BLR_FOR_EACH_LZ(BLR_EXTERN_F2)
#undef BLR_EXTERN_F2
#define BLR_EXTERN_LZ(LL, A, B, OP)                                                                     \
  extern template void launch_lines<double, WShape<A, B>, OP>(blr_ctx*, PadEngine*, const LineArgs<double>&); \
  extern template void launch_lines<float, WShape<A, B>, OP>(blr_ctx*, PadEngine*, const LineArgs<float>&);
#define BLR_EXTERN_L_ALLOPS(LL, A, B) \
  BLR_EXTERN_LZ(LL, A, B, 0) BLR_EXTERN_LZ(LL, A, B, 1) BLR_EXTERN_LZ(LL, A, B, 2) BLR_EXTERN_LZ(LL, A, B, 3) \
  BLR_EXTERN_LZ(LL, A, B, 4) BLR_EXTERN_LZ(LL, A, B, 5) BLR_EXTERN_LZ(LL, A, B, 6) BLR_EXTERN_LZ(LL, A, B, 7) \
  BLR_EXTERN_LZ(LL, A, B, 8)
BLR_FOR_EACH_LZ(BLR_EXTERN_L_ALLOPS)
#undef BLR_EXTERN_L_ALLOPS
#undef BLR_EXTERN_LZ
// ---------------------------------------------------------------------------
// host side: engine setup and launch helpers
// ---------------------------------------------------------------------------

// Engine registry, one entry per context.  Entries are node-stable (std::map),
// so a returned PadEngine* stays valid while other threads insert; the mutex
// guards the map itself and each engine's one-time set-up.  Each context is
// used by a single (thread, stream) pair (domain.py Context), so an engine's
// scratch is never shared across threads or streams.
static std::mutex g_engines_mu;
static std::map<blr_ctx*, PadEngine>& engines() {
  static std::map<blr_ctx*, PadEngine> m;
  return m;
}

void pad_engine_release(blr_ctx* c) {
  std::lock_guard<std::mutex> lk(g_engines_mu);
  auto it = engines().find(c);
  if (it == engines().end()) return;
  for (auto* p : it->second.tw)
    if (p) cudaFree(p);
  for (auto* p : it->second.buf)
    if (p) cudaFree(p);
  engines().erase(it);
}

static int g_pad_disabled = -1;

template <typename T>
static PadEngine* engine(blr_ctx* c) {
  std::lock_guard<std::mutex> lk(g_engines_mu);
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
  for (int a = 0; a < 3; ++a) {
    g.P[a] = gg.P[a]; g.K[a] = gg.K[a]; g.B[a] = gg.B[a];
    if (!supported_len(g.P[a])) return nullptr;
  }
  g.Kz1 = g.K[2] + 1;
  g.nh = (int64_t)g.Kz1 * g.B[0] * g.B[1];
  g.ns = (int64_t)g.Kz1 * g.P[0] * g.P[1];
  g.n1 = (int64_t)g.Kz1 * g.B[1] * g.P[0];
  g.np = (int64_t)g.P[0] * g.P[1] * g.P[2];
  int dev;
  BLR_CUDA(cudaGetDevice(&dev));
  BLR_CUDA(cudaDeviceGetAttribute(&e.line_smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  // split twiddle tables per axis (blr_fft.cuh twiddle()): W_L^(k1 n2) for
  // k1 < R1, n2 < R2, real parts then imaginary parts
  for (int a = 0; a < 3; ++a) {
    const int L = g.P[a], R2 = shape_r2(L), R1 = L / R2;
    std::vector<double> tw(2 * (size_t)L);
    for (int k1 = 0; k1 < R1; ++k1)
      for (int n2 = 0; n2 < R2; ++n2) {
        double s, co;
        sincospi(-2.0 * (k1 * n2) / L, &s, &co);
        tw[k1 * R2 + n2] = co;
        tw[L + k1 * R2 + n2] = s;
      }
    // followed by the same table rounded to fp32 (2 L floats), so fp32 kernels
    // can stage it with cp.async instead of converting element by element
    std::vector<float> twf(2 * (size_t)L);
    for (size_t i = 0; i < twf.size(); ++i) twf[i] = (float)tw[i];
    const size_t nb = 2 * (size_t)L * sizeof(double);
    BLR_CUDA(cudaMalloc(&e.tw[a], nb + 2 * (size_t)L * sizeof(float)));
    BLR_CUDA(cudaMemcpy(e.tw[a], tw.data(), nb, cudaMemcpyHostToDevice));
    BLR_CUDA(cudaMemcpy((char*)e.tw[a] + nb, twf.data(), twf.size() * sizeof(float), cudaMemcpyHostToDevice));
  }
  e.ok = true;
  return &e;
}

template <typename T>
bool pad_engine_ok(blr_ctx* c) { return engine<T>(c) != nullptr; }

// persistent, grow-only per-engine scratch buffers (stream-ordered users only)
static void* e_scratch(blr_ctx* c, PadEngine* e, int slot, size_t bytes) {
  return scratch(c, e->buf[slot], e->buf_bytes[slot], bytes);
}

template <typename T>
static void dispatch_xinv(blr_ctx* c, PadEngine* e, const XPassArgs<T>& a) {
  switch (e->g.P[0]) {
#define X(LL, A, B) case LL: launch_xinv<T, WShape<A, B>>(c, e, a); break;
    BLR_FOR_EACH_L(X)
#undef X
    default: throw Error(1, "unsupported pad length");
  }
}
template <typename T>
static void dispatch_yinv(blr_ctx* c, PadEngine* e, const YPassArgs<T>& a) {
  switch (e->g.P[1]) {
#define X(LL, A, B) case LL: launch_yinv<T, WShape<A, B>>(c, e, a); break;
    BLR_FOR_EACH_L(X)
#undef X
    default: throw Error(1, "unsupported pad length");
  }
}
template <typename T, int OP>
static void dispatch_lines(blr_ctx* c, PadEngine* e, const LineArgs<T>& a) {
  switch (e->g.P[2]) {
#define X(LL, A, B) case LL: launch_lines<T, WShape<A, B>, OP>(c, e, a); break;
    BLR_FOR_EACH_LZ(X)
#undef X
    default: throw Error(1, "unsupported pad length");
  }
}
template <typename T>
static void dispatch_yfwd(blr_ctx* c, PadEngine* e, const YFwdArgs<T>& a) {
  switch (e->g.P[1]) {
#define X(LL, A, B) case LL: launch_yfwd<T, WShape<A, B>>(c, e, a); break;
    BLR_FOR_EACH_L(X)
#undef X
    default: throw Error(1, "unsupported pad length");
  }
}
template <typename T>
static void dispatch_xfwd(blr_ctx* c, PadEngine* e, const FwdArgs<T>& a) {
  switch (e->g.P[0]) {
#define X(LL, A, B) case LL: launch_xfwd<T, WShape<A, B>>(c, e, a); break;
    BLR_FOR_EACH_L(X)
#undef X
    default: throw Error(1, "unsupported pad length");
  }
}

// fused forward projection (blr_fwd2.cuh): 3-D grids with equal x / y pad lengths.
// Opt-in (BLR_FWD2=1 or blr_set_fused_forward(1)): bit-identical to the
// two-kernel path, but A/B on the B200 (r02, 128^3 / K=32) it ties it for
// one-job outputs (state GN HVP 5.59 vs 5.43 ms) and loses for the flux
// divergence (2 jobs, 93 KB smem -> 2 CTAs/SM: deformation 11.4 vs 9.76 ms);
// ncu: exposed bulk-load and cluster-barrier waits (no double buffering).
static std::atomic<int> g_fwd2_disabled{-1};  // -1: not yet read from BLR_FWD2
void set_fused_forward(int on) { g_fwd2_disabled.store(on ? 0 : 1); }
template <typename T>
static bool dispatch_fwd2(blr_ctx* c, PadEngine* e, const Fwd2Args<T>& a, int no, int njmax, bool run) {
  int dis = g_fwd2_disabled.load();
  if (dis < 0) {
    const char* env = getenv("BLR_FWD2");
    int expect = -1;
    g_fwd2_disabled.compare_exchange_strong(expect, (env && env[0] == '1') ? 0 : 1);
    dis = g_fwd2_disabled.load();
  }
  const PadGeom& g = e->g;
  if (dis || g.P[0] != g.P[1] || g.P[0] < 2) return false;
  switch (g.P[0]) {
#define X(LL, A, B)                                                  \
  case LL:                                                           \
    if (!fwd2_fits<T, WShape<A, B>>(g)) return false;                \
    if (run) launch_fwd2<T, WShape<A, B>>(c, e, a, no, njmax);       \
    return true;
    BLR_FOR_EACH_LZ(X)
#undef X
    default: return false;
  }
}

// --- realization of band fields on the pad grid (x pass + y pass) ----------------
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

// S[f] = Y(X(field f)) for every spec; derivative multipliers: x before the
// x pass, y / z before the y pass.
template <typename T>
static void inv2d(blr_ctx* c, PadEngine* e, const std::vector<InvSpec<T>>& f, Cx<T>* S) {
  const PadGeom& g = e->g;
  std::vector<std::pair<const Cx<T>*, int>> xf;
  std::vector<std::array<int, 3>> yx(f.size());
  for (size_t i = 0; i < f.size(); ++i)
    for (int t = 0; t < f[i].nterms; ++t) {
      std::pair<const Cx<T>*, int> key(f[i].src[t], f[i].axis[t] == 0 ? 1 : 0);
      int idx = -1;
      for (size_t q = 0; q < xf.size(); ++q)
        if (xf[q] == key) { idx = (int)q; break; }
      if (idx < 0) { idx = (int)xf.size(); xf.push_back(key); }
      yx[i][t] = idx;
    }
  if ((int)xf.size() > kMaxX) throw Error(1, "too many x-pass fields");
  Cx<T>* I = (Cx<T>*)e_scratch(c, e, 0, xf.size() * g.n1 * sizeof(Cx<T>));
  {
    XPassArgs<T> a;
    std::memset(&a, 0, sizeof(a));
    a.nx = (int)xf.size();
    for (int i = 0; i < a.nx; ++i) { a.src[i] = xf[i].first; a.mulx[i] = xf[i].second; }
    a.out = I;
    ProfScope ps(c, "pad_xpass", (double)a.nx * (g.nh + g.n1) * sizeof(Cx<T>));
    dispatch_xinv<T>(c, e, a);
  }
  for (size_t off = 0; off < f.size(); off += kMaxY) {
    YPassArgs<T> a;
    std::memset(&a, 0, sizeof(a));
    a.ny = (int)std::min<size_t>(kMaxY, f.size() - off);
    int nterm = 0;
    for (int i = 0; i < a.ny; ++i) {
      const InvSpec<T>& s = f[off + i];
      a.nterms[i] = s.nterms;
      for (int t = 0; t < 3; ++t) {
        a.xf[i][t] = t < s.nterms ? yx[off + i][t] : 0;
        a.axis[i][t] = (t < s.nterms && (s.axis[t] == 1 || s.axis[t] == 2)) ? s.axis[t] : -1;
      }
      nterm += s.nterms;
    }
    a.in = I;
    a.out = S + (int64_t)off * g.ns;
    ProfScope ps(c, "pad_ypass", ((double)nterm * g.n1 + a.ny * g.ns) * sizeof(Cx<T>));
    dispatch_yinv<T>(c, e, a);
  }
}

// --- z lines -------------------------------------------------------------------------
// ACC-op tables: output index / real-input index / sign per spectral field
template <typename T>
static void acc_tables(int op, LineArgs<T>& a) {
  const int d = a.d, dd = d * d;
  for (int f = 0; f < kMaxLineS; ++f) { a.oi[f] = 0; a.ri[f] = 0; a.sg[f] = 1.0; }
  a.nst = 0;
  if (op == kOpMap || op == kOpMapTC) {
    // staged slots: V_j
    a.nst = d;
    for (int j = 0; j < d; ++j) a.st_idx[j] = (op == kOpMapTC ? dd : 0) + j;
    for (int f = 0; f < dd; ++f) { a.oi[f] = f / d; a.ri[f] = f % d; }
  } else if (op == kOpInvVol) {
    // staged slots: V_0..V_{d-1}, Dv
    a.nst = d + 1;
    for (int j = 0; j <= d; ++j) a.st_idx[j] = j;
    for (int f = 0; f < dd; ++f) { a.oi[f] = f / d; a.ri[f] = f % d; }
    for (int q = 0; q < d; ++q) { a.oi[dd + q] = d; a.ri[dd + q] = q; a.sg[dd + q] = -1.0; }
    a.oi[dd + d] = d; a.ri[dd + d] = d; a.sg[dd + d] = -1.0;
  } else if (op == kOpContract) {
    for (int o = 0; o < 3; ++o)
      for (int j = 0; j < 3; ++j) a.mi[o][j] = (o < d && j < d) ? (a.transpose ? j * d + o : o * d + j) : 0;
  }
}

static const char* const kLineOpName[] = {"pad_zlines_realize", "pad_zlines_map",     "pad_zlines_map_tc",
                                          "pad_zlines_map_tf",  "pad_zlines_inv_vol", "pad_zlines_bwd_vol",
                                          "pad_zlines_outer",   "pad_zlines_outer_pair", "pad_zlines_contract"};

template <typename T, int OP>
static void lines(blr_ctx* c, PadEngine* e, LineArgs<T>& a, double bytes) {
  a.op = OP;
  acc_tables<T>(OP, a);
  ProfScope ps(c, kLineOpName[OP], bytes);
  dispatch_lines<T, OP>(c, e, a);
}

// --- projection back to the band (y pass + x pass + fix-up) ------------------------
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

// kout / RK4 component index = output index
template <typename T>
static void fwd2d(blr_ctx* c, PadEngine* e, const std::vector<FwdSpec<T>>& outs, Cx<T>* kout, const Rk& rk) {
  const PadGeom& g = e->g;
  // forward-y jobs: x-derivative terms stay separate (i k_x after the x pass);
  // the other terms of an output (plain, i k_y, i k_z) fold into one job
  struct Job { int nt; const Cx<T>* s[3]; int ax[3]; };
  std::vector<Job> jobs;
  struct XT { int nt; int f[3]; int ax[3]; };
  std::vector<XT> xt(outs.size());
  for (size_t i = 0; i < outs.size(); ++i) {
    xt[i].nt = 0;
    Job comb{};
    for (int t = 0; t < outs[i].nterms; ++t) {
      if (outs[i].axis[t] == 0) {
        Job jx{};
        jx.nt = 1; jx.s[0] = outs[i].sin[t]; jx.ax[0] = -1;
        jobs.push_back(jx);
        xt[i].f[xt[i].nt] = (int)jobs.size() - 1;
        xt[i].ax[xt[i].nt++] = 0;
      } else {
        comb.s[comb.nt] = outs[i].sin[t];
        comb.ax[comb.nt++] = outs[i].axis[t];
      }
    }
    if (comb.nt) {
      jobs.push_back(comb);
      xt[i].f[xt[i].nt] = (int)jobs.size() - 1;
      xt[i].ax[xt[i].nt++] = -1;
    }
  }
  bool fused = dispatch_fwd2<T>(c, e, Fwd2Args<T>{}, 0, 0, false);
  for (size_t i = 0; i < outs.size() && fused; ++i) fused = xt[i].nt == 1;  // single-job outputs
  if (fused) {
    for (size_t off = 0; off < outs.size(); off += kMaxFwd) {
      Fwd2Args<T> a;
      std::memset(&a, 0, sizeof(a));
      const int no = (int)std::min<size_t>(kMaxFwd, outs.size() - off);
      int njmax = 1, nterm = 0;
      for (int i = 0; i < no; ++i) {
        const FwdSpec<T>& s = outs[off + i];
        const XT& x = xt[off + i];
        a.nj[i] = x.nt;
        njmax = std::max(njmax, x.nt);
        for (int j = 0; j < x.nt; ++j) {
          const Job& jb = jobs[x.f[j]];
          Fwd2Job<T>& J = a.job[i][j];
          J.nt = jb.nt;
          J.xax = x.ax[j];
          for (int t = 0; t < 3; ++t) {
            J.s[t] = t < jb.nt ? jb.s[t] : jb.s[0];
            J.yax[t] = t < jb.nt ? jb.ax[t] : -1;
          }
          nterm += jb.nt;
        }
        a.e.o[i].mode = s.mode;
        a.e.o[i].vt = s.vt;
        a.e.o[i].nterms = x.nt;
      }
      a.e.no = no;
      a.e.scale = (T)(1.0 / (double)g.np);
      const int64_t shift = (int64_t)off * g.nh;
      a.e.kout = kout ? kout + shift : nullptr;
      a.e.rk_s = rk.s;
      a.e.cs = (T)rk.cs;
      a.e.h6 = (T)rk.h6;
      a.e.cur = rk.cur ? (Cx<T>*)rk.cur + shift : nullptr;
      a.e.acc = rk.acc ? (Cx<T>*)rk.acc + shift : nullptr;
      a.e.stage = rk.stage ? (Cx<T>*)rk.stage + shift : nullptr;
      ProfScope ps(c, "pad_fwd2", ((double)nterm * g.ns + no * g.nh * (rk.s ? 4 : 2)) * sizeof(Cx<T>));
      dispatch_fwd2<T>(c, e, a, no, njmax, true);
    }
    return;
  }
  Cx<T>* I = (Cx<T>*)e_scratch(c, e, 1, jobs.size() * g.n1 * sizeof(Cx<T>));
  for (size_t off = 0; off < jobs.size(); off += kMaxYF) {
    YFwdArgs<T> a;
    std::memset(&a, 0, sizeof(a));
    a.nj = (int)std::min<size_t>(kMaxYF, jobs.size() - off);
    int nterm = 0;
    for (int q = 0; q < a.nj; ++q) {
      const Job& jb = jobs[off + q];
      a.nterms[q] = jb.nt;
      for (int t = 0; t < 3; ++t) {
        a.sin[q][t] = t < jb.nt ? jb.s[t] : jb.s[0];
        a.axis[q][t] = t < jb.nt ? jb.ax[t] : -1;
      }
      nterm += jb.nt;
    }
    a.out = I + (int64_t)off * g.n1;
    ProfScope ps(c, "pad_ypass_fwd", ((double)nterm * g.ns + a.nj * g.n1) * sizeof(Cx<T>));
    dispatch_yfwd<T>(c, e, a);
  }
  for (size_t off = 0; off < outs.size(); off += kMaxFwd) {
    FwdArgs<T> a;
    std::memset(&a, 0, sizeof(a));
    a.no = (int)std::min<size_t>(kMaxFwd, outs.size() - off);
    int nterm = 0;
    for (int i = 0; i < a.no; ++i) {
      const FwdSpec<T>& s = outs[off + i];
      const XT& x = xt[off + i];
      for (int t = 0; t < 3; ++t) {
        a.o[i].f[t] = t < x.nt ? x.f[t] : 0;
        a.o[i].axis[t] = t < x.nt ? x.ax[t] : -1;
      }
      a.o[i].nterms = x.nt;
      a.o[i].mode = s.mode;
      a.o[i].vt = s.vt;
      nterm += x.nt;
    }
    a.in = I;
    a.scale = (T)(1.0 / (double)g.np);
    const int64_t shift = (int64_t)off * g.nh;
    a.kout = kout ? kout + shift : nullptr;
    a.rk_s = rk.s;
    a.cs = (T)rk.cs;
    a.h6 = (T)rk.h6;
    a.cur = rk.cur ? (Cx<T>*)rk.cur + shift : nullptr;
    a.acc = rk.acc ? (Cx<T>*)rk.acc + shift : nullptr;
    a.stage = rk.stage ? (Cx<T>*)rk.stage + shift : nullptr;
    {
      ProfScope ps(c, "pad_xpass_fwd", ((double)nterm * g.n1 + a.no * g.nh * (rk.s ? 4 : 2)) * sizeof(Cx<T>));
      dispatch_xfwd<T>(c, e, a);
    }
  }
}

template <typename T>
static void full_to_h(blr_ctx* c, PadEngine* e, const Cx<T>* full, int ncomp, Cx<T>* H) {
  const PadGeom& g = e->g;
  const size_t sm = (size_t)g.Kz1 * g.B[1] * sizeof(Cx<T>);
  if (sm <= 48 * 1024) {
    launch_pdl(k_full_to_h_t<T>, ncomp * g.B[0], 256, sm, c->stream, full, ncomp, g, H);
  } else {
    launch_pdl(k_full_to_h<T>, grid_blocks(g.nh * ncomp, 256), 256, 0, c->stream, full, ncomp, g, H);
  }
  BLR_LAUNCHED();
}

template <typename T>
static void h_to_full(blr_ctx* c, PadEngine* e, const Cx<T>* H, int ncomp, Cx<T>* full) {
  const PadGeom& g = e->g;
  const size_t sm = 2 * (size_t)g.Kz1 * g.B[1] * sizeof(Cx<T>);
  if (sm <= 96 * 1024) {
    ensure_smem(k_h_to_full_t<T>, sm);
    launch_pdl(k_h_to_full_t<T>, ncomp * g.B[0], 256, sm, c->stream, H, ncomp, g, full);
  } else {
    launch_pdl(k_h_to_full<T>, grid_blocks(c->g.nb() * ncomp, 256), 256, 0, c->stream, H, ncomp, g, full);
  }
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
  void* dst;   // full blocks [n_steps+1][ncomp][nb] ([1][ncomp][nb] when final_only)
  bool final_only = false;
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
  const int last = forward ? n : 0;
  auto record = [&](int node) {
    for (const auto& r : rec) {
      if (!r.dst || (r.final_only && node != last)) continue;
      const int64_t slot = r.final_only ? 0 : node;
      h_to_full<T>(c, e, cur + r.comp0 * e->g.nh, r.ncomp, (Cx<T>*)r.dst + slot * r.ncomp * nb);
    }
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
    rk4_v2<T>(c, e, v.n_steps, substeps, true, cur, ncomp, {{du0, d, dphi, (flags & 8) != 0}}, tmp,
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
// D(phi_i) realizations for the contraction: the cache itself (mode 2), filled
// (mode 1) or a temporary (mode 0)
template <typename T>
static T* contract_jacobians(blr_ctx* c, PadEngine* e, const Cx<T>* phi, int n_nodes, T* dphi_cache,
                             int cache_mode, Tmp2& tmp) {
  const Geom& g = c->g;
  const PadGeom& pg = e->g;
  const int d = g.d, dd = d * d;
  const int64_t L = d * g.nb();
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
  return M;
}

// sum_n w_n D(phi_n)^(T) rho_n for nodes [node0, node0 + nn) with the rho
// nodes already realized in S layout (RS [node][d][ns]) -> band H layout Kh
template <typename T>
static void contract_core(blr_ctx* c, PadEngine* e, const Cx<T>* RS, const T* M, int node0, int nn,
                          const double* w, bool transpose, Cx<T>* So, Cx<T>* Kh) {
  const Geom& g = c->g;
  const PadGeom& pg = e->g;
  const int d = g.d, dd = d * d;
  LineArgs<T> la;
  std::memset(&la, 0, sizeof(la));
  la.d = d; la.no = d; la.transpose = transpose ? 1 : 0;
  la.n_nodes = nn;
  la.sin_node_stride = (int64_t)d * pg.ns;
  la.rin_node_stride = (int64_t)dd * pg.np;
  for (int a = 0; a < d; ++a) la.sin[a] = RS + ((int64_t)node0 * d + a) * pg.ns;
  for (int k = 0; k < dd; ++k) la.rin[k] = M + ((int64_t)node0 * dd + k) * pg.np;
  for (int i = 0; i < nn; ++i) la.w[i] = w ? w[i] : 1.0;
  for (int i = 0; i < d; ++i) la.sout[i] = So + i * pg.ns;
  lines<T, kOpContract>(c, e, la,
                        (double)nn * (d * pg.ns * sizeof(Cx<T>) + dd * pg.np * sizeof(T)) +
                            d * pg.ns * sizeof(Cx<T>));
  std::vector<FwdSpec<T>> outs;
  for (int i = 0; i < d; ++i) outs.push_back(fwd1<T>(So + i * pg.ns, kEpiPlain));
  fwd2d<T>(c, e, outs, Kh, Rk());
}

template <typename T>
bool contract_v2(blr_ctx* c, const Cx<T>* phi, const Cx<T>* rho, int n_nodes, const double* weights,
                 bool transpose, T* dphi_cache, int cache_mode, Cx<T>* out) {
  PadEngine* e = engine<T>(c);
  if (!e) return false;
  if (n_nodes > 32) return false;
  const Geom& g = c->g;
  const PadGeom& pg = e->g;
  const int d = g.d;
  const int64_t L = d * g.nb();
  Tmp2 tmp(c);
  const T* M = contract_jacobians<T>(c, e, phi, n_nodes, dphi_cache, cache_mode, tmp);
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
    contract_core<T>(c, e, RS, M, summed ? 0 : run, summed ? n_nodes : 1, summed ? weights : nullptr, transpose,
                     So, Kh);
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

// Backward momentum transport fused with the summed contraction
// sum_n w_n (rho_n + project(D(phi_n)^(T) rho_n)): the sweep's own node-time
// realizations of rho (the first RK4 stage of every step) are written straight
// into the contraction's S-layout node buffer, and sum_n w_n rho_n accumulates
// in H layout, so no rho node record is ever materialized or re-transformed.
template <typename T>
bool momentum_contract_v2(blr_ctx* c, FlowRef v, int substeps, const Cx<T>* rho_end, const Cx<T>* phi,
                          const double* weights, bool transpose, T* dphi_cache, int cache_mode, Cx<T>* out) {
  PadEngine* e = engine<T>(c);
  if (!e) return false;
  const int n = v.n_steps, n_nodes = n + 1;
  if (n_nodes > 32 || !weights) return false;
  const Geom& g = c->g;
  const PadGeom& pg = e->g;
  const int d = g.d, dd = d * d;
  Tmp2 tmp(c);
  const T* M = contract_jacobians<T>(c, e, phi, n_nodes, dphi_cache, cache_mode, tmp);
  VelBank2<T> V(c, e, v, false, tmp);
  Cx<T>* cur = tmp.get<Cx<T>>(d * pg.nh);
  full_to_h<T>(c, e, rho_end, d, cur);
  Cx<T>* RS = tmp.get<Cx<T>>((int64_t)n_nodes * d * pg.ns);
  Cx<T>* S = tmp.get<Cx<T>>(d * pg.ns);
  Cx<T>* So = tmp.get<Cx<T>>(dd * pg.ns);
  Cx<T>* wsum = tmp.get<Cx<T>>(d * pg.nh);  // sum_n w_n rho_n (H layout)
  BLR_CUDA(cudaMemsetAsync(wsum, 0, d * pg.nh * sizeof(Cx<T>), c->stream));
  auto realize = [&](const Cx<T>* s, Cx<T>* dst) {
    std::vector<InvSpec<T>> f;
    for (int a = 0; a < d; ++a) f.push_back(inv1<T>(s + a * pg.nh, -1));
    inv2d<T>(c, e, f, dst);
  };
  const int per_node = 4 * substeps;
  rk4_v2<T>(c, e, n, substeps, false, cur, d, {}, tmp, [&](int si, double t, const Cx<T>* s, const Rk& rk) {
    const auto& vt = V.at(t);
    Cx<T>* Sd = S;
    if (si % per_node == 0) {  // first stage of a step: the state is rho at node n - step
      const int node = n - si / per_node;
      Sd = RS + (int64_t)node * d * pg.ns;
      band_axpby<T>(c, weights[node], s, 1.0, wsum, d * pg.nh);
    }
    realize(s, Sd);
    LineArgs<T> la;
    std::memset(&la, 0, sizeof(la));
    la.d = d; la.ns = d; la.nr = d; la.no = dd;
    for (int i = 0; i < d; ++i) la.sin[i] = Sd + i * pg.ns;
    for (int j = 0; j < d; ++j) la.rin[j] = vt.real + j * pg.np;
    for (int i = 0; i < dd; ++i) la.sout[i] = So + i * pg.ns;
    lines<T, kOpOuter>(c, e, la, sbytes(pg, d, d, dd, 0, sizeof(T)));
    std::vector<FwdSpec<T>> outs;
    push_flux<T>(g, pg, So, outs);
    fwd2d<T>(c, e, outs, nullptr, rk);
  });
  // node 0 (t = 0) is reached only as the sweep's final state
  realize(cur, RS);
  band_axpby<T>(c, weights[0], cur, 1.0, wsum, d * pg.nh);
  Cx<T>* Kh = tmp.get<Cx<T>>(d * pg.nh);
  contract_core<T>(c, e, RS, M, 0, n_nodes, weights, transpose, So, Kh);
  band_axpby<T>(c, 1.0, wsum, 1.0, Kh, d * pg.nh);
  h_to_full<T>(c, e, Kh, d, out);
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
                               Cx<T>*);                                                               \
  template bool momentum_contract_v2<T>(blr_ctx*, FlowRef, int, const Cx<T>*, const Cx<T>*,              \
                                        const double*, bool, T*, int, Cx<T>*);
BLR_PINST(double)
BLR_PINST(float)

}  // namespace blr
