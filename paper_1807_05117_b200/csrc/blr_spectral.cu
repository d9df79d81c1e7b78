// blr_spectral.cu — band-limited spectral algebra on sm_100a.
//
// include  (spectral.py:89-119): band block -> Hermitian half spectrum of the
//          target grid (one fused scatter pass that also writes the zeros and
//          applies i*2*pi*k derivative multipliers) -> cuFFT C2R.
// project  (spectral.py:122-135): cuFFT R2C -> one gather pass that scales by
//          1/prod(G), applies the collision weights and symmetrizes.
// Band-pointwise operators (Helmholtz, Leray, divergence) and the
// deterministic two-pass reductions used by the solver also live here.
#include <cstdint>
#include "blr_internal.cuh"

#include <cmath>
#include <cstring>
#include <cstdio>
#include <mutex>

namespace blr {

// ---------------------------------------------------------------------------
// errors / launch counting
// ---------------------------------------------------------------------------
static std::atomic<int64_t> g_launches{0};
void count_launch(int n) { g_launches += n; }
int64_t launch_count() { return g_launches.load(); }

// ---------------------------------------------------------------------------
// profiler
// ---------------------------------------------------------------------------
namespace {
struct ProfRec {
  std::string name;
  double bytes;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_event_pool;

cudaEvent_t take_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

bool profiling() { return g_prof_on; }
void profile_enable(bool on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_on = on;
}

ProfScope::ProfScope(blr_ctx* c, const char* name, double bytes, cudaStream_t s) {
  if (!g_prof_on) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  ProfRec r{name, bytes, take_event(), take_event()};
  stream = s ? s : c->stream;
  cudaEventRecord(r.a, stream);
  slot = (int)g_prof.size();
  g_prof.push_back(r);
}

ProfScope::~ProfScope() {
  if (slot < 0) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  cudaEventRecord(g_prof[slot].b, stream);
}

std::string profile_report() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  struct Agg { int64_t n = 0; double ms = 0, bytes = 0; };
  std::map<std::string, Agg> agg;
  for (auto& r : g_prof) {
    cudaEventSynchronize(r.b);
    float ms = 0;
    cudaEventElapsedTime(&ms, r.a, r.b);
    auto& a = agg[r.name];
    a.n += 1;
    a.ms += ms;
    a.bytes += r.bytes;
    g_event_pool.push_back(r.a);
    g_event_pool.push_back(r.b);
  }
  g_prof.clear();
  std::string out = "{";
  bool first = true;
  for (auto& kv : agg) {
    char buf[256];
    snprintf(buf, sizeof(buf), "%s\"%s\": [%lld, %.6f, %.1f]", first ? "" : ", ", kv.first.c_str(),
             (long long)kv.second.n, kv.second.ms, kv.second.bytes);
    out += buf;
    first = false;
  }
  return out + "}";
}

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(2, std::string(what) + ": " + cudaGetErrorString(e));
}
void check_fft(cufftResult r, const char* what) {
  if (r != CUFFT_SUCCESS) throw Error(3, std::string(what) + ": cufft error " + std::to_string((int)r));
}

void* scratch(blr_ctx* c, void*& buf, size_t& cap, size_t need) {
  if (need <= cap) return buf;
  if (buf) {
    BLR_CUDA(cudaStreamSynchronize(c->stream));
    BLR_CUDA(cudaFree(buf));
    buf = nullptr;
    cap = 0;
  }
  BLR_CUDA(cudaMalloc(&buf, need));
  cap = need;
  return buf;
}

// ---------------------------------------------------------------------------
// cuFFT plans: rank = d over the trailing axes, batched, shared work area
// ---------------------------------------------------------------------------
cufftHandle get_plan(blr_ctx* c, bool pad, int batch, bool forward) {
  int64_t key = ((int64_t)batch << 2) | ((pad ? 1 : 0) << 1) | (forward ? 1 : 0);
  auto it = c->plans.find(key);
  if (it != c->plans.end()) return it->second;
  const Geom& g = c->g;
  GridDesc gd = g.grid(pad);
  int n[3];
  for (int i = 0; i < g.d; ++i) n[i] = gd.G[3 - g.d + i];
  cufftHandle h;
  BLR_FFT(cufftCreate(&h));
  BLR_FFT(cufftSetAutoAllocation(h, 0));
  cufftType type;
  if (c->dtype == 0) type = forward ? CUFFT_D2Z : CUFFT_Z2D;
  else type = forward ? CUFFT_R2C : CUFFT_C2R;
  size_t ws = 0;
  int idist = forward ? (int)gd.real_size() : (int)gd.half_size();
  int odist = forward ? (int)gd.half_size() : (int)gd.real_size();
  BLR_FFT(cufftMakePlanMany(h, g.d, n, nullptr, 1, idist, nullptr, 1, odist, type, batch, &ws));
  if (ws > c->fft_work_size) {
    if (c->fft_work) {
      BLR_CUDA(cudaStreamSynchronize(c->stream));
      BLR_CUDA(cudaFree(c->fft_work));
    }
    BLR_CUDA(cudaMalloc(&c->fft_work, ws));
    c->fft_work_size = ws;
    for (auto& kv : c->plans) BLR_FFT(cufftSetWorkArea(kv.second, c->fft_work));
  }
  BLR_FFT(cufftSetWorkArea(h, c->fft_work));
  c->plans[key] = h;
  return h;
}

// cuFFT wants 16-byte aligned real arrays; odd pad sizes put slices of the
// D(u) / D(phi) caches (and their batch strides) at 8-byte offsets.
template <typename T>
static bool fft_real_aligned(const T* p, int batch, int64_t rs) {
  return (reinterpret_cast<uintptr_t>(p) % 16) == 0 && (batch == 1 || (rs * sizeof(T)) % 16 == 0);
}

template <typename T>
void exec_c2r(blr_ctx* c, bool pad, int batch, Cx<T>* in, T* out) {
  const int64_t rs = c->g.grid(pad).real_size();
  if (!fft_real_aligned(out, batch, rs)) {  // through an aligned temporary, one field at a time
    T* tmp = nullptr;
    BLR_CUDA(cudaMallocAsync((void**)&tmp, (size_t)rs * sizeof(T), c->stream));
    const int64_t hs = c->g.grid(pad).half_size();
    for (int b = 0; b < batch; ++b) {
      exec_c2r<T>(c, pad, 1, in + b * hs, tmp);
      BLR_CUDA(cudaMemcpyAsync(out + b * rs, tmp, rs * sizeof(T), cudaMemcpyDeviceToDevice, c->stream));
    }
    BLR_CUDA(cudaFreeAsync(tmp, c->stream));
    return;
  }
  cufftHandle h = get_plan(c, pad, batch, false);
  BLR_FFT(cufftSetStream(h, c->stream));
  GridDesc gd = c->g.grid(pad);
  ProfScope ps(c, pad ? "cufft_c2r_pad" : "cufft_c2r_full",
               (double)batch * (gd.half_size() * sizeof(Cx<T>) + gd.real_size() * sizeof(T)));
  if constexpr (sizeof(T) == 8)
    BLR_FFT(cufftExecZ2D(h, (cufftDoubleComplex*)in, (cufftDoubleReal*)out));
  else
    BLR_FFT(cufftExecC2R(h, (cufftComplex*)in, (cufftReal*)out));
  count_launch();
}

template <typename T>
void exec_r2c(blr_ctx* c, bool pad, int batch, T* in, Cx<T>* out) {
  const int64_t rs = c->g.grid(pad).real_size();
  if (!fft_real_aligned(in, batch, rs)) {
    T* tmp = nullptr;
    BLR_CUDA(cudaMallocAsync((void**)&tmp, (size_t)rs * sizeof(T), c->stream));
    const int64_t hs = c->g.grid(pad).half_size();
    for (int b = 0; b < batch; ++b) {
      BLR_CUDA(cudaMemcpyAsync(tmp, in + b * rs, rs * sizeof(T), cudaMemcpyDeviceToDevice, c->stream));
      exec_r2c<T>(c, pad, 1, tmp, out + b * hs);
    }
    BLR_CUDA(cudaFreeAsync(tmp, c->stream));
    return;
  }
  cufftHandle h = get_plan(c, pad, batch, true);
  BLR_FFT(cufftSetStream(h, c->stream));
  GridDesc gd = c->g.grid(pad);
  ProfScope ps(c, pad ? "cufft_r2c_pad" : "cufft_r2c_full",
               (double)batch * (gd.half_size() * sizeof(Cx<T>) + gd.real_size() * sizeof(T)));
  if constexpr (sizeof(T) == 8)
    BLR_FFT(cufftExecD2Z(h, (cufftDoubleReal*)in, (cufftDoubleComplex*)out));
  else
    BLR_FFT(cufftExecR2C(h, (cufftReal*)in, (cufftComplex*)out));
  count_launch();
}

// ---------------------------------------------------------------------------
// scatter: band blocks -> half spectrum (zeros included), derivative fused
// ---------------------------------------------------------------------------
// Sources mapping to bin b on one axis (1 or 2 block indices, ascending).
__device__ inline int bin_sources(int b, int G, int K, int B, int& s0, int& s1) {
  const bool lo = b <= K, hi = b >= G - K;  // frequency b - G in [-K, -1] for hi
  s0 = lo ? b : b - G + B;
  s1 = b - G + B;
  return (lo ? 1 : 0) + (hi ? 1 : 0);
}

template <typename T>
__global__ void __launch_bounds__(256) k_scatter(ScatterArgs<T> a, GridDesc gd, Cx<T>* H) {
  using C = Cx<T>;
  const int64_t hs = gd.half_size();
  const int64_t total = hs * a.nf;
  const bool small = total <= 0x7fffffff;  // 32-bit index decode (64-bit division is ~5x dearer)
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int fi, b0, b1, b2;
    if (small) {
      const int id = (int)idx, h32 = (int)hs;
      fi = id / h32;
      int r = id - fi * h32;
      b2 = r % gd.Gh;
      r /= gd.Gh;
      b1 = r % gd.G[1];
      b0 = r / gd.G[1];
    } else {
      fi = (int)(idx / hs);
      int64_t r = idx - fi * hs;
      b2 = (int)(r % gd.Gh);
      r /= gd.Gh;
      b1 = (int)(r % gd.G[1]);
      b0 = (int)(r / gd.G[1]);
    }
    int s0[2], s1[2], s2[2];
    int n0 = bin_sources(b0, gd.G[0], gd.K[0], gd.B[0], s0[0], s0[1]);
    int n1 = bin_sources(b1, gd.G[1], gd.K[1], gd.B[1], s1[0], s1[1]);
    int n2 = bin_sources(b2, gd.G[2], gd.K[2], gd.B[2], s2[0], s2[1]);
    C acc;
    acc.x = 0;
    acc.y = 0;
    const ScatterField<T>& F = a.f[fi];
    // fixed-trip loops (<= 2 sources per axis) and scalar frequencies: no
    // dynamically indexed local arrays
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (p >= n0 || q >= n1 || s >= n2) continue;
          int i0 = p ? s0[1] : s0[0], i1 = q ? s1[1] : s1[0], i2 = s ? s2[1] : s2[0];
          int64_t off = ((int64_t)i0 * gd.B[1] + i1) * gd.B[2] + i2;
          const int fr0 = freq_of(i0, gd.K[0], gd.B[0]), fr1 = freq_of(i1, gd.K[1], gd.B[1]),
                    fr2 = freq_of(i2, gd.K[2], gd.B[2]);
          C val;
          val.x = 0;
          val.y = 0;
          for (int t = 0; t < F.nterms; ++t) {
            C z = F.src[t][off];
            const int ax = F.axis[t];
            if (ax >= 0) {
              T k = (T)(kTwoPi * (double)(ax == 0 ? fr0 : (ax == 1 ? fr1 : fr2)));
              T re = -(k * z.y), im = k * z.x;  // (i k) * z
              z.x = re;
              z.y = im;
            }
            if (F.coef[t] != (T)1) {
              z.x *= F.coef[t];
              z.y *= F.coef[t];
            }
            val.x += z.x;
            val.y += z.y;
          }
          acc.x += val.x;
          acc.y += val.y;
        }
    H[idx] = acc;
  }
}

// ---------------------------------------------------------------------------
// gather: half spectrum -> symmetrized band blocks (scale 1/prod(G), weights)
// ---------------------------------------------------------------------------
__device__ inline int bin_count(int b, int G, int K) { return (b <= K ? 1 : 0) + (b >= G - K ? 1 : 0); }

template <typename T>
__device__ inline Cx<T> half_value(const Cx<T>* H, const GridDesc& gd, int f0, int f1, int f2) {
  int b2 = pmod(f2, gd.G[2]);
  if (b2 < gd.Gh) {
    int b0 = pmod(f0, gd.G[0]), b1 = pmod(f1, gd.G[1]);
    return H[((int64_t)b0 * gd.G[1] + b1) * gd.Gh + b2];
  }
  int m0 = pmod(-f0, gd.G[0]), m1 = pmod(-f1, gd.G[1]), m2 = pmod(-f2, gd.G[2]);
  Cx<T> z = H[((int64_t)m0 * gd.G[1] + m1) * gd.Gh + m2];
  z.y = -z.y;
  return z;
}

template <typename T>
__global__ void __launch_bounds__(256) k_gather(const Cx<T>* __restrict__ H, GridDesc gd, int nf,
                                                T scale, Cx<T>* __restrict__ out) {
  using C = Cx<T>;
  const int64_t nb = (int64_t)gd.B[0] * gd.B[1] * gd.B[2];
  const int64_t hs = gd.half_size();
  const int64_t total = nb * nf;
  const bool small = total <= 0x7fffffff;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int fi, i0, i1, i2;
    if (small) {
      const int id = (int)idx, n32 = (int)nb;
      fi = id / n32;
      int r = id - fi * n32;
      i2 = r % gd.B[2];
      r /= gd.B[2];
      i1 = r % gd.B[1];
      i0 = r / gd.B[1];
    } else {
      fi = (int)(idx / nb);
      int64_t r = idx - fi * nb;
      i2 = (int)(r % gd.B[2]);
      r /= gd.B[2];
      i1 = (int)(r % gd.B[1]);
      i0 = (int)(r / gd.B[1]);
    }
    int f0 = freq_of(i0, gd.K[0], gd.B[0]), f1 = freq_of(i1, gd.K[1], gd.B[1]),
        f2 = freq_of(i2, gd.K[2], gd.B[2]);
    const C* Hf = H + fi * hs;
    T w = scale;
    int c0 = bin_count(pmod(f0, gd.G[0]), gd.G[0], gd.K[0]);
    int c1 = bin_count(pmod(f1, gd.G[1]), gd.G[1], gd.K[1]);
    int c2 = bin_count(pmod(f2, gd.G[2]), gd.G[2], gd.K[2]);
    if (c0 * c1 * c2 != 1) w = w * ((T)1 / (T)(c0 * c1 * c2));
    C p = half_value<T>(Hf, gd, f0, f1, f2);
    C q = half_value<T>(Hf, gd, -f0, -f1, -f2);
    C o;
    o.x = (T)0.5 * (p.x * w + q.x * w);
    o.y = (T)0.5 * (p.y * w - q.y * w);
    out[idx] = o;
  }
}

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
template <typename T>
void realize(blr_ctx* c, bool pad, const std::vector<ScatterField<T>>& fields, T* out) {
  GridDesc gd = c->g.grid(pad);
  const int64_t hs = gd.half_size(), rs = gd.real_size();
  size_t off = 0;
  while (off < fields.size()) {
    int nf = (int)std::min<size_t>(kMaxScatter, fields.size() - off);
    ScatterArgs<T> a;
    a.nf = nf;
    for (int i = 0; i < nf; ++i) a.f[i] = fields[off + i];
    Cx<T>* H = (Cx<T>*)scratch(c, c->half_buf, c->half_bytes, (size_t)nf * hs * sizeof(Cx<T>));
    int nterms = 0;
    for (int i = 0; i < nf; ++i) nterms += a.f[i].nterms;
    const double band_half = (double)gd.B[0] * gd.B[1] * (gd.K[2] + 1);
    {
      ProfScope ps(c, pad ? "scatter_pad" : "scatter_full",
                   ((double)nf * hs + nterms * band_half) * sizeof(Cx<T>));
      k_scatter<T><<<grid_blocks(hs * nf, 256), 256, 0, c->stream>>>(a, gd, H);
      BLR_LAUNCHED();
    }
    exec_c2r<T>(c, pad, nf, H, out + off * rs);
    off += nf;
  }
}

template <typename T>
void project(blr_ctx* c, bool pad, T* in, int nf, Cx<T>* out) {
  GridDesc gd = c->g.grid(pad);
  const int64_t hs = gd.half_size(), rs = gd.real_size();
  const int64_t nb = c->g.nb();
  const T scale = (T)(1.0 / (double)rs);
  int off = 0;
  while (off < nf) {
    int n = std::min(kMaxScatter, nf - off);
    Cx<T>* H = (Cx<T>*)scratch(c, c->half_buf, c->half_bytes, (size_t)n * hs * sizeof(Cx<T>));
    exec_r2c<T>(c, pad, n, in + (int64_t)off * rs, H);
    ProfScope ps(c, pad ? "gather_pad" : "gather_full",
                 (double)n * ((double)gd.B[0] * gd.B[1] * (gd.K[2] + 1) + nb) * sizeof(Cx<T>));
    k_gather<T><<<grid_blocks(nb * n, 256), 256, 0, c->stream>>>(H, gd, n, scale,
                                                                 out + (int64_t)off * nb);
    BLR_LAUNCHED();
    off += n;
  }
}

template <typename T>
ScatterField<T> fld(const Cx<T>* src, int axis) {
  ScatterField<T> f;
  f.nterms = 1;
  f.src[0] = src;
  f.axis[0] = axis;
  f.coef[0] = (T)1;
  for (int t = 1; t < 3; ++t) { f.src[t] = nullptr; f.axis[t] = -1; f.coef[t] = (T)1; }
  return f;
}

template <typename T>
ScatterField<T> fld_div(const Geom& g, const Cx<T>* vec) {
  ScatterField<T> f;
  f.nterms = g.d;
  for (int t = 0; t < 3; ++t) { f.src[t] = nullptr; f.axis[t] = -1; f.coef[t] = (T)1; }
  for (int c = 0; c < g.d; ++c) {
    f.src[c] = vec + c * g.nb();
    f.axis[c] = g.axis_of(c);
  }
  return f;
}

// ---------------------------------------------------------------------------
// band-pointwise kernels
// ---------------------------------------------------------------------------
struct BandDesc {
  int K[3], B[3];
  int64_t nb;
};

inline BandDesc band_desc(const Geom& g) {
  BandDesc b;
  for (int a = 0; a < 3; ++a) { b.K[a] = g.K[a]; b.B[a] = g.B[a]; }
  b.nb = g.nb();
  return b;
}

__device__ inline void band_freqs(const BandDesc& bd, int64_t r, int* f) {
  int i2 = (int)(r % bd.B[2]);
  r /= bd.B[2];
  int i1 = (int)(r % bd.B[1]);
  int i0 = (int)(r / bd.B[1]);
  f[0] = freq_of(i0, bd.K[0], bd.B[0]);
  f[1] = freq_of(i1, bd.K[1], bd.B[1]);
  f[2] = freq_of(i2, bd.K[2], bd.B[2]);
}

// symbol A(k) = 1 + alpha * (t0[i0] + t1[i1] + t2[i2])  (spectral.py:242-257)
__device__ inline double symbol_at(const double* sym, const BandDesc& bd, int64_t r, double alpha) {
  int i2 = (int)(r % bd.B[2]);
  r /= bd.B[2];
  int i1 = (int)(r % bd.B[1]);
  int i0 = (int)(r / bd.B[1]);
  double acc = 0.0;
  acc = acc + sym[i0];
  acc = acc + sym[bd.B[0] + i1];
  acc = acc + sym[bd.B[0] + bd.B[1] + i2];
  return 1.0 + alpha * acc;
}

template <typename T>
__global__ void k_helmholtz(const Cx<T>* in, int nblocks, BandDesc bd, const double* sym,
                            double alpha, int order, int inverse, Cx<T>* out) {
  int64_t total = bd.nb * nblocks;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = idx % bd.nb;
    double A = symbol_at(sym, bd, r, alpha);
    double m;
    if (!inverse) m = (order == 1) ? A : (order == 2 ? A * A : pow(A, (double)order));
    else m = (order == 1) ? 1.0 / A : pow(A, -(double)order);
    Cx<T> z = in[idx];
    z.x = (T)(z.x * m);
    z.y = (T)(z.y * m);
    out[idx] = z;
  }
}

// Leray projection w = v - grad(lap^-1 div v), p(0) = 0 (spectral.py:312-328).
template <typename T>
__global__ void k_leray(const Cx<T>* in, int nvec, int d, BandDesc bd, Cx<T>* out) {
  int64_t total = bd.nb * nvec;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int vi = (int)(idx / bd.nb);
    int64_t r = idx - vi * bd.nb;
    int f[3];
    band_freqs(bd, r, f);
    const Cx<T>* v = in + (int64_t)vi * d * bd.nb;
    T dre = 0, dim = 0, lap = 0;
    for (int c = 0; c < d; ++c) {
      T k = (T)(kTwoPi * (double)f[3 - d + c]);
      Cx<T> z = v[c * bd.nb + r];
      dre += -(k * z.y);
      dim += k * z.x;
      lap = lap - k * k;
    }
    T pre = 0, pim = 0;
    if (lap != (T)0) { pre = dre / lap; pim = dim / lap; }
    Cx<T>* o = out + (int64_t)vi * d * bd.nb;
    for (int c = 0; c < d; ++c) {
      T k = (T)(kTwoPi * (double)f[3 - d + c]);
      Cx<T> z = v[c * bd.nb + r];
      Cx<T> w;
      w.x = z.x - (-(k * pim));
      w.y = z.y - k * pre;
      o[c * bd.nb + r] = w;
    }
  }
}

template <typename T>
__global__ void k_divergence(const Cx<T>* in, int nvec, int d, BandDesc bd, Cx<T>* out) {
  int64_t total = bd.nb * nvec;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int vi = (int)(idx / bd.nb);
    int64_t r = idx - vi * bd.nb;
    int f[3];
    band_freqs(bd, r, f);
    const Cx<T>* v = in + (int64_t)vi * d * bd.nb;
    T re = 0, im = 0;
    for (int c = 0; c < d; ++c) {
      T k = (T)(kTwoPi * (double)f[3 - d + c]);
      Cx<T> z = v[c * bd.nb + r];
      re += -(k * z.y);
      im += k * z.x;
    }
    Cx<T> o;
    o.x = re;
    o.y = im;
    out[idx] = o;
  }
}

template <typename T>
__global__ void k_symmetrize(const Cx<T>* in, int nblocks, BandDesc bd, Cx<T>* out) {
  int64_t total = bd.nb * nblocks;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int bi = (int)(idx / bd.nb);
    int64_t r = idx - bi * bd.nb;
    int f[3];
    band_freqs(bd, r, f);
    int m0 = pmod(-f[0], bd.B[0]), m1 = pmod(-f[1], bd.B[1]), m2 = pmod(-f[2], bd.B[2]);
    Cx<T> a = in[idx];
    Cx<T> b = in[bi * bd.nb + ((int64_t)m0 * bd.B[1] + m1) * bd.B[2] + m2];
    Cx<T> o;
    o.x = (T)0.5 * (a.x + b.x);
    o.y = (T)0.5 * (a.y - b.y);
    out[idx] = o;
  }
}

// flux divergence: out[i] = -(sum_j i k_j F[i][j])  (transport.py:264-274, negated)
template <typename T>
__global__ void k_flux_div(const Cx<T>* F, int nsets, int d, BandDesc bd, Cx<T>* out) {
  int64_t total = bd.nb * d * nsets;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = idx % bd.nb;
    int64_t q = idx / bd.nb;
    int i = (int)(q % d);
    int s = (int)(q / d);
    int f[3];
    band_freqs(bd, r, f);
    const Cx<T>* Fs = F + (int64_t)s * d * d * bd.nb;
    T re = 0, im = 0;
    for (int j = 0; j < d; ++j) {
      T k = (T)(kTwoPi * (double)f[3 - d + j]);
      Cx<T> z = Fs[(int64_t)(i * d + j) * bd.nb + r];
      re += -(k * z.y);
      im += k * z.x;
    }
    Cx<T> o;
    o.x = -re;
    o.y = -im;
    out[idx] = o;
  }
}

template <typename T>
void band_flux_div(blr_ctx* c, const Cx<T>* F, int nsets, Cx<T>* out) {
  BandDesc bd = band_desc(c->g);
  ProfScope ps(c, "band_epilogue", (double)bd.nb * nsets * (c->g.d * c->g.d + c->g.d) * sizeof(Cx<T>));
  k_flux_div<T><<<grid_blocks(bd.nb * c->g.d * nsets, 256), 256, 0, c->stream>>>(F, nsets, c->g.d,
                                                                                 bd, out);
  BLR_LAUNCHED();
}

template <typename T>
void band_helmholtz(blr_ctx* c, const Cx<T>* in, int nblocks, int inverse, Cx<T>* out) {
  BandDesc bd = band_desc(c->g);
  k_helmholtz<T><<<grid_blocks(bd.nb * nblocks, 256), 256, 0, c->stream>>>(
      in, nblocks, bd, c->d_sym, c->g.alpha, c->g.order, inverse, out);
  BLR_LAUNCHED();
}

template <typename T>
void band_leray(blr_ctx* c, const Cx<T>* in, int nvec, Cx<T>* out) {
  BandDesc bd = band_desc(c->g);
  k_leray<T><<<grid_blocks(bd.nb * nvec, 256), 256, 0, c->stream>>>(in, nvec, c->g.d, bd, out);
  BLR_LAUNCHED();
}

template <typename T>
void band_divergence(blr_ctx* c, const Cx<T>* in, int nvec, Cx<T>* out) {
  BandDesc bd = band_desc(c->g);
  k_divergence<T><<<grid_blocks(bd.nb * nvec, 256), 256, 0, c->stream>>>(in, nvec, c->g.d, bd, out);
  BLR_LAUNCHED();
}

template <typename T>
void band_symmetrize(blr_ctx* c, const Cx<T>* in, int nblocks, Cx<T>* out) {
  BandDesc bd = band_desc(c->g);
  k_symmetrize<T><<<grid_blocks(bd.nb * nblocks, 256), 256, 0, c->stream>>>(in, nblocks, bd, out);
  BLR_LAUNCHED();
}

// ---------------------------------------------------------------------------
// complex elementwise kernels (RK4 stages, PCG)
// ---------------------------------------------------------------------------
// out = -(a + b)
template <typename T>
__global__ void k_neg_add(const Cx<T>* a, const Cx<T>* b, Cx<T>* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    Cx<T> x = a[i], y = b[i], o;
    o.x = -(x.x + y.x);
    o.y = -(x.y + y.y);
    out[i] = o;
  }
}

template <typename T>
void band_neg_add(blr_ctx* c, const Cx<T>* a, const Cx<T>* b, Cx<T>* out, int64_t n) {
  ProfScope ps(c, "band_epilogue", 3.0 * n * sizeof(Cx<T>));
  k_neg_add<T><<<grid_blocks(n, 256), 256, 0, c->stream>>>(a, b, out, n);
  BLR_LAUNCHED();
}

// RK4 stage bookkeeping after k_s is known (transport.py:330-340):
//   s == 1: acc = k;            stage = cur + cs * k
//   s == 2,3: acc = acc + 2 k;  stage = cur + cs * k
//   s == 4: acc = acc + k;      cur = cur + (h/6) * acc
template <typename T>
__global__ void k_rk4(int s, const Cx<T>* k, Cx<T>* cur, Cx<T>* acc, Cx<T>* stage, T cs, T h6,
                      int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    Cx<T> kk = k[i], cc = cur[i], a;
    if (s == 1) {
      a = kk;
    } else {
      a = acc[i];
      if (s < 4) {
        a.x = a.x + (T)2 * kk.x;
        a.y = a.y + (T)2 * kk.y;
      } else {
        a.x = a.x + kk.x;
        a.y = a.y + kk.y;
      }
    }
    if (s < 4) {
      acc[i] = a;
      Cx<T> st;
      st.x = cc.x + cs * kk.x;
      st.y = cc.y + cs * kk.y;
      stage[i] = st;
    } else {
      cc.x = cc.x + h6 * a.x;
      cc.y = cc.y + h6 * a.y;
      cur[i] = cc;
    }
  }
}

template <typename T>
void band_rk4(blr_ctx* c, int s, const Cx<T>* k, Cx<T>* cur, Cx<T>* acc, Cx<T>* stage, double cs,
              double h6, int64_t n) {
  ProfScope ps(c, "rk4_update", (double)n * sizeof(Cx<T>) * (s == 1 ? 3 : (s < 4 ? 5 : 4)));
  k_rk4<T><<<grid_blocks(n, 256), 256, 0, c->stream>>>(s, k, cur, acc, stage, (T)cs, (T)h6, n);
  BLR_LAUNCHED();
}

// out = (1-w) a + w b   (TimeFlow.sample, transport.py:77-86)
template <typename T>
__global__ void k_lerp(const Cx<T>* a, const Cx<T>* b, T w0, T w1, Cx<T>* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    Cx<T> x = a[i], y = b[i], o;
    o.x = w0 * x.x + w1 * y.x;
    o.y = w0 * x.y + w1 * y.y;
    out[i] = o;
  }
}

template <typename T>
void band_lerp(blr_ctx* c, const Cx<T>* a, const Cx<T>* b, double w, Cx<T>* out, int64_t n) {
  k_lerp<T><<<grid_blocks(n, 256), 256, 0, c->stream>>>(a, b, (T)(1.0 - w), (T)w, out, n);
  BLR_LAUNCHED();
}

// y = a x + b y
template <typename T>
__global__ void k_axpby(T a, const Cx<T>* x, T b, Cx<T>* y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    Cx<T> u = x[i], v = y[i];
    v.x = a * u.x + b * v.x;
    v.y = a * u.y + b * v.y;
    y[i] = v;
  }
}

template <typename T>
void band_axpby(blr_ctx* c, double a, const Cx<T>* x, double b, Cx<T>* y, int64_t n) {
  k_axpby<T><<<grid_blocks(n, 256), 256, 0, c->stream>>>((T)a, x, (T)b, y, n);
  BLR_LAUNCHED();
}

template <typename T>
__global__ void k_pcg_update(T a, const Cx<T>* p, const Cx<T>* hp, Cx<T>* x, Cx<T>* r, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    Cx<T> pp = p[i], hh = hp[i], xx = x[i], rr = r[i];
    xx.x = xx.x + a * pp.x;
    xx.y = xx.y + a * pp.y;
    rr.x = rr.x - a * hh.x;
    rr.y = rr.y - a * hh.y;
    x[i] = xx;
    r[i] = rr;
  }
}

template <typename T>
void band_pcg_update(blr_ctx* c, double a, const Cx<T>* p, const Cx<T>* hp, Cx<T>* x, Cx<T>* r,
                     int64_t n) {
  k_pcg_update<T><<<grid_blocks(n, 256), 256, 0, c->stream>>>((T)a, p, hp, x, r, n);
  BLR_LAUNCHED();
}

// ---------------------------------------------------------------------------
// deterministic reductions: fixed grid, per-block partials in double, then a
// single-block pass in index order
// ---------------------------------------------------------------------------
constexpr int kRedBlocks = 296;  // 2 x 148 SMs
constexpr int kRedThreads = 256;

__device__ inline double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// NaN-propagating max (np.max semantics: a NaN anywhere makes the result NaN;
// fmax would drop it and let a NaN gradient read as converged).
__device__ inline double nan_max(double a, double b) { return (a > b || a != a) ? a : b; }
__device__ inline double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) v = nan_max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <int OP>  // 0 sum, 1 max
__device__ inline double block_reduce(double v) {
  __shared__ double sh[32];
  v = OP == 0 ? warp_sum(v) : warp_max(v);
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  int nw = blockDim.x >> 5;
  v = threadIdx.x < nw ? sh[threadIdx.x] : (OP == 0 ? 0.0 : 0.0);
  if (w == 0) v = OP == 0 ? warp_sum(v) : warp_max(v);
  __syncthreads();
  return v;
}

// MODE: 0 inner Re(a conj b) complex, 1 max|f|, 2 sum (a-b)^2, 3 nonfinite count,
//       4 weighted node inner (complex)
template <typename T, int MODE>
__global__ void __launch_bounds__(kRedThreads) k_reduce(const void* pa, const void* pb, int64_t n,
                                                        double* partial) {
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (MODE == 0) {
      Cx<T> a = ((const Cx<T>*)pa)[i], b = ((const Cx<T>*)pb)[i];
      acc += (double)a.x * (double)b.x + (double)a.y * (double)b.y;
    } else if (MODE == 1) {
      acc = nan_max(acc, fabs((double)((const T*)pa)[i]));
    } else if (MODE == 2) {
      double x = (double)((const T*)pa)[i];
      if (pb) x -= (double)((const T*)pb)[i];
      acc += x * x;
    } else if (MODE == 3) {
      double x = (double)((const T*)pa)[i];
      acc += isfinite(x) ? 0.0 : 1.0;
    }
  }
  acc = block_reduce<(MODE == 1) ? 1 : 0>(acc);
  if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

template <int OP>
__global__ void k_reduce_final(const double* partial, int n, double* out) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc = OP == 0 ? acc + partial[i] : nan_max(acc, partial[i]);
  acc = block_reduce<OP>(acc);
  if (threadIdx.x == 0) out[0] = acc;
}

static void ensure_red(blr_ctx* c) {
  if (!c->d_red) {
    BLR_CUDA(cudaMalloc(&c->d_red, (kRedBlocks + 8) * sizeof(double)));
    BLR_CUDA(cudaMallocHost(&c->h_red, 8 * sizeof(double)));
  }
}

template <typename T, int MODE>
double reduce_host(blr_ctx* c, const void* a, const void* b, int64_t n) {
  ensure_red(c);
  int blocks = grid_blocks(n, kRedThreads, kRedBlocks);
  k_reduce<T, MODE><<<blocks, kRedThreads, 0, c->stream>>>(a, b, n, c->d_red);
  BLR_LAUNCHED();
  constexpr int OP = (MODE == 1) ? 1 : 0;
  k_reduce_final<OP><<<1, 256, 0, c->stream>>>(c->d_red, blocks, c->d_red + kRedBlocks);
  BLR_LAUNCHED();
  BLR_CUDA(cudaMemcpyAsync(c->h_red, c->d_red + kRedBlocks, sizeof(double), cudaMemcpyDeviceToHost,
                           c->stream));
  BLR_CUDA(cudaStreamSynchronize(c->stream));
  return c->h_red[0];
}

template double reduce_host<double, 0>(blr_ctx*, const void*, const void*, int64_t);
template double reduce_host<double, 1>(blr_ctx*, const void*, const void*, int64_t);
template double reduce_host<double, 2>(blr_ctx*, const void*, const void*, int64_t);
template double reduce_host<double, 3>(blr_ctx*, const void*, const void*, int64_t);
template double reduce_host<float, 0>(blr_ctx*, const void*, const void*, int64_t);
template double reduce_host<float, 1>(blr_ctx*, const void*, const void*, int64_t);
template double reduce_host<float, 2>(blr_ctx*, const void*, const void*, int64_t);
template double reduce_host<float, 3>(blr_ctx*, const void*, const void*, int64_t);

#define BLR_INST(T)                                                                              \
  template void realize<T>(blr_ctx*, bool, const std::vector<ScatterField<T>>&, T*);             \
  template void project<T>(blr_ctx*, bool, T*, int, Cx<T>*);                                     \
  template ScatterField<T> fld<T>(const Cx<T>*, int);                                            \
  template ScatterField<T> fld_div<T>(const Geom&, const Cx<T>*);                                \
  template void band_flux_div<T>(blr_ctx*, const Cx<T>*, int, Cx<T>*);                           \
  template void band_helmholtz<T>(blr_ctx*, const Cx<T>*, int, int, Cx<T>*);                     \
  template void band_leray<T>(blr_ctx*, const Cx<T>*, int, Cx<T>*);                              \
  template void band_divergence<T>(blr_ctx*, const Cx<T>*, int, Cx<T>*);                         \
  template void band_symmetrize<T>(blr_ctx*, const Cx<T>*, int, Cx<T>*);                         \
  template void band_neg_add<T>(blr_ctx*, const Cx<T>*, const Cx<T>*, Cx<T>*, int64_t);          \
  template void band_rk4<T>(blr_ctx*, int, const Cx<T>*, Cx<T>*, Cx<T>*, Cx<T>*, double, double, \
                            int64_t);                                                            \
  template void band_lerp<T>(blr_ctx*, const Cx<T>*, const Cx<T>*, double, Cx<T>*, int64_t);     \
  template void band_axpby<T>(blr_ctx*, double, const Cx<T>*, double, Cx<T>*, int64_t);          \
  template void band_pcg_update<T>(blr_ctx*, double, const Cx<T>*, const Cx<T>*, Cx<T>*,         \
                                   Cx<T>*, int64_t);                                             \
  template void exec_c2r<T>(blr_ctx*, bool, int, Cx<T>*, T*);                                    \
  template void exec_r2c<T>(blr_ctx*, bool, int, T*, Cx<T>*);
BLR_INST(double)
BLR_INST(float)

}  // namespace blr
