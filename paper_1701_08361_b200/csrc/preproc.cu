// The pre stage on the device (preproc.hpp).
#include "preproc.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numbers>
#include <string>

namespace rtnb {

namespace {

constexpr int kKbWidth = 4;  // kb::kWidth (preproc.hpp:23)
constexpr int kPre = 256;    // threads per block of the pre-stage kernels

// ---- host: the reference's kernel, taps, density weights, roll-off (double) ----------

double kb_beta() {  // kb::beta, preproc.cpp:22-26 (oversampling 2)
  const double w = kKbWidth, sigma = 2.0;
  const double t = (w / sigma) * (sigma - 0.5);
  return std::numbers::pi * std::sqrt(t * t - 0.8);
}

double kb_kernel(double u) {  // preproc.cpp:28-35
  const double half = kKbWidth / 2.0;
  if (std::abs(u) > half) return 0.0;
  const double t = 1.0 - (u / half) * (u / half);
  const double b = kb_beta();
  return std::cyl_bessel_i(0.0, b * std::sqrt(std::max(t, 0.0))) / std::cyl_bessel_i(0.0, b);
}

double kb_kernel_ft(double f) {  // preproc.cpp:37-52
  const double b = kb_beta();
  const double z = std::numbers::pi * kKbWidth * f;
  const double s2 = b * b - z * z;
  double v;
  if (s2 > 1e-12) {
    const double s = std::sqrt(s2);
    v = std::sinh(s) / s;
  } else if (s2 < -1e-12) {
    const double s = std::sqrt(-s2);
    v = std::sin(s) / s;
  } else {
    v = 1.0;
  }
  return v / (std::sinh(b) / b);
}

double kb_mass() {  // preproc.cpp:54-57
  const double b = kb_beta();
  return kKbWidth / std::cyl_bessel_i(0.0, b) * (std::sinh(b) / b);
}

double readout_radius(int i, int S) { return (2.0 * i + 1.0 - S) / (2.0 * S); }  // seqsim.cpp:161

double dcf_ramp(double kx, double ky, int K, int S, int G) {  // preproc.cpp:97-100
  const double plateau = 0.5 / G;
  return std::max(std::hypot(kx, ky), plateau) * (std::numbers::pi / K) * (1.0 / S);
}

void check_coord(double kx, double ky) {  // preproc.cpp:80-84
  if (!(kx >= -0.5 && kx < 0.5 && ky >= -0.5 && ky < 0.5)) {
    fail(3, "gridding: sample coordinate outside [-0.5, 0.5)");
  }
}

struct Taps {  // make_taps, preproc.cpp:68-78
  int idx[kKbWidth];
  double wgt[kKbWidth];
};
Taps make_taps(double kg, int G) {
  Taps t;
  const int base = static_cast<int>(std::floor(kg)) - kKbWidth / 2 + 1;
  for (int i = 0; i < kKbWidth; ++i) {
    const int cell = base + i;
    t.idx[i] = ((cell % G) + G) % G;
    t.wgt[i] = kb_kernel(cell - kg);
  }
  return t;
}

// ---- device kernels ------------------------------------------------------------------------

// one thread per (channel, grid cell): the reference's float products in its order
// (grid.at(ix, iy) += (y_s * float(v_s)) * float(wx * wy), preproc.cpp:123-133, 188-192)
__global__ void __launch_bounds__(kPre) k_grid_gather(int J, int G, int n, const int* __restrict__ ptr,
                                                      const int* __restrict__ sidx, const float* __restrict__ w,
                                                      const float* __restrict__ dcf,
                                                      const float2* __restrict__ samples, float2* __restrict__ out) {
  const long long G2 = static_cast<long long>(G) * G, total = J * G2;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(t / G2);
    const int cell = static_cast<int>(t - j * G2);
    const float2* y = samples + static_cast<size_t>(j) * n;
    float ax = 0.f, ay = 0.f;
    const int e1 = ptr[cell + 1];
    for (int e = ptr[cell]; e < e1; ++e) {
      const int s = sidx[e];
      const float2 v = y[s];
      const float d = dcf[s], ww = w[e];
      ax = __fadd_rn(ax, __fmul_rn(__fmul_rn(v.x, d), ww));
      ay = __fadd_rn(ay, __fmul_rn(__fmul_rn(v.y, d), ww));
    }
    out[t] = make_float2(ax, ay);
  }
}

// z *= float(G) / deapodization, then mask_window (preproc.cpp:193-195); with apply_post,
// then the series' normalisation z *= post (prep_series, nlinv.cpp:390-400) in the same
// float multiply the separate scaling pass would do
__global__ void __launch_bounds__(kPre) k_deapod_mask(int J, int G, const float* __restrict__ f,
                                                      float2* __restrict__ z, int apply_post, float post) {
  const int L = G / 2, lo = (G - L) / 2;
  const long long G2 = static_cast<long long>(G) * G, total = J * G2;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int p = static_cast<int>(t % G2);
    const int r = p / G, c = p - (p / G) * G;
    float2 v = make_float2(0.f, 0.f);
    if (r >= lo && r < lo + L && c >= lo && c < lo + L) {
      const float2 x = z[t];
      v = make_float2(__fmul_rn(x.x, f[p]), __fmul_rn(x.y, f[p]));
    }
    if (apply_post) v = make_float2(__fmul_rn(v.x, post), __fmul_rn(v.y, post));
    z[t] = v;
  }
}

// per-sample phase tables: AX[s][u] = exp(2 pi i kx_s (u - c)), AY[s][w] = v_s exp(2 pi i ky_s (w - c))
// (std::polar, preproc.cpp:239-242)
__global__ void __launch_bounds__(kPre) k_psf_tables(int n, int G, const double* __restrict__ kx,
                                                     const double* __restrict__ ky, const double* __restrict__ v,
                                                     double2* __restrict__ AX, double2* __restrict__ AY) {
  const int c = G / 2;
  const long long total = static_cast<long long>(n) * G;
  const double two_pi = 2.0 * 3.141592653589793238462643383279502884;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int s = static_cast<int>(t / G), u = static_cast<int>(t - static_cast<long long>(s) * G);
    double sx, cx, sy, cy;
    sincos(two_pi * kx[s] * (u - c), &sx, &cx);
    sincos(two_pi * ky[s] * (u - c), &sy, &cy);
    AX[t] = make_double2(cx, sx);
    AY[t] = make_double2(v[s] * cy, v[s] * sy);
  }
}

// Q[u][w] = sum_s AX[s][u] AY[s][w], accumulated per element in sample order with
// the reference's unfused complex products (preproc.cpp:243-246). 16 x 16 tiles,
// samples staged through shared memory in chunks of 16.
__global__ void __launch_bounds__(256) k_psf_gemm(int n, int G, const double2* __restrict__ AX,
                                                  const double2* __restrict__ AY, double2* __restrict__ Q) {
  __shared__ double2 sx[16][16];
  __shared__ double2 sy[16][16];
  const int tu = threadIdx.x / 16, tw = threadIdx.x % 16;
  const int u0 = blockIdx.y * 16, w0 = blockIdx.x * 16;
  const int u = u0 + tu, w = w0 + tw;
  double qr = 0.0, qi = 0.0;
  for (int s0 = 0; s0 < n; s0 += 16) {
    {
      const int ss = s0 + tu;  // row of the chunk this thread stages
      sx[tu][tw] = (ss < n && u0 + tw < G) ? AX[static_cast<size_t>(ss) * G + u0 + tw] : make_double2(0.0, 0.0);
      sy[tu][tw] = (ss < n && w < G) ? AY[static_cast<size_t>(ss) * G + w] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    const int m = min(16, n - s0);
    for (int k = 0; k < m; ++k) {
      const double2 a = sx[k][tu], b = sy[k][tw];
      qr = __dadd_rn(qr, __dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)));
      qi = __dadd_rn(qi, __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
    }
    __syncthreads();
  }
  if (u < G && w < G) Q[static_cast<size_t>(u) * G + w] = make_double2(qr, qi);
}

// zero the unpaired Nyquist edge (row 0, column 0; preproc.cpp:254-257), round to float
__global__ void __launch_bounds__(kPre) k_psf_round(int G, const double2* __restrict__ Q, float2* __restrict__ P) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < G * G; p += gridDim.x * blockDim.x) {
    const int u = p / G, w = p - (p / G) * G;
    const double2 q = Q[p];
    P[p] = (u == 0 || w == 0) ? make_float2(0.f, 0.f)
                              : make_float2(static_cast<float>(q.x), static_cast<float>(q.y));
  }
}

__global__ void __launch_bounds__(kPre) k_scale(int n, float s, float2* __restrict__ x) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    const float2 v = x[p];
    x[p] = make_float2(__fmul_rn(v.x, s), __fmul_rn(v.y, s));
  }
}

// out[jv][s] = sum_jp complex<double>(m[jv][jp]) * complex<double>(in[jp][s]), rounded
// to float (apply_compression, preproc.cpp:459-468)
__global__ void __launch_bounds__(kPre) k_compress(int Jv, int Jp, int n, const float2* __restrict__ m,
                                                   const float2* __restrict__ in, float2* __restrict__ out) {
  const long long total = static_cast<long long>(Jv) * n;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int jv = static_cast<int>(t / n), s = static_cast<int>(t - static_cast<long long>(jv) * n);
    double ar = 0.0, ai = 0.0;
    for (int jp = 0; jp < Jp; ++jp) {
      const float2 a = m[static_cast<size_t>(jv) * Jp + jp];
      const float2 b = in[static_cast<size_t>(jp) * n + s];
      ar = __dadd_rn(ar, __dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)));
      ai = __dadd_rn(ai, __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
    }
    out[t] = make_float2(static_cast<float>(ar), static_cast<float>(ai));
  }
}

int grid_for(long long n) {
  long long b = (n + kPre - 1) / kPre;
  return static_cast<int>(std::max(1LL, std::min(b, 148LL * 16)));
}

}  // namespace

uint64_t psf_angle_key(const double* angles, int K, int S, int G) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&h](uint64_t v) {
    for (int b = 0; b < 8; ++b) {
      h ^= (v >> (8 * b)) & 0xFF;
      h *= 1099511628211ull;
    }
  };
  mix(static_cast<uint64_t>(S));
  mix(static_cast<uint64_t>(G));
  for (int k = 0; k < K; ++k) mix(static_cast<uint64_t>(std::llround(angles[k] * 1e9)));
  return h;
}

Preproc::Preproc(const Plan& plan, int device) : plan_(plan), dev_(device) {
  if (plan.G < 2 || plan.G % 2) fail(2, "preproc: grid side must be even");
  check_cuda(cudaSetDevice(dev_), "set device");
  check_cuda(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking), "stream");
  // deapodization(G) (preproc.cpp:102-118) and the float factor G / d of grid_adjoint
  const int G = plan.G, c = G / 2;
  const double mass = kb_mass();
  std::vector<double> axis(static_cast<size_t>(G));
  for (int r = 0; r < G; ++r) axis[static_cast<size_t>(r)] = mass * kb_kernel_ft((r - c) / static_cast<double>(G));
  std::vector<float> f(static_cast<size_t>(G) * G);
  const float scale = static_cast<float>(G);
  for (int r = 0; r < G; ++r) {
    for (int q = 0; q < G; ++q) {
      const float d = static_cast<float>(axis[static_cast<size_t>(r)] * axis[static_cast<size_t>(q)]);
      f[static_cast<size_t>(r) * G + q] = scale / d;
    }
  }
  check_cuda(cudaMalloc(&deapod_, sizeof(float) * f.size()), "deapod");
  check_cuda(cudaMemcpy(deapod_, f.data(), sizeof(float) * f.size(), cudaMemcpyHostToDevice), "deapod upload");
  check_cuda(cudaMalloc(&psf_q_, sizeof(double2) * G * G), "psf q");
}

Preproc::~Preproc() {
  cudaSetDevice(dev_);
  if (s_) cudaStreamSynchronize(s_);
  for (auto& kv : plans_) {
    cudaFree(kv.second.ptr);
    cudaFree(kv.second.sidx);
    cudaFree(kv.second.w);
    cudaFree(kv.second.dcf);
  }
  for (void* p : {static_cast<void*>(deapod_), static_cast<void*>(psf_tab_), static_cast<void*>(psf_q_), scratch_}) {
    if (p) cudaFree(p);
  }
  if (s_) cudaStreamDestroy(s_);
}

float2* Preproc::scratch(size_t bytes) {
  if (bytes > scratch_bytes_) {
    if (scratch_) {
      check_cuda(cudaStreamSynchronize(s_), "sync");
      cudaFree(scratch_);
    }
    check_cuda(cudaMalloc(&scratch_, bytes), "preproc scratch");
    scratch_bytes_ = bytes;
  }
  return static_cast<float2*>(scratch_);
}

const Preproc::GridPlan& Preproc::grid_plan(const double* angles, int K, int S, double delay) {
  const int G = plan_.G, c = G / 2;
  uint64_t key = psf_angle_key(angles, K, S, G);
  {
    uint64_t d;
    std::memcpy(&d, &delay, sizeof(d));
    key ^= d * 0x9e3779b97f4a7c15ull;
  }
  std::lock_guard<std::mutex> lock(mu_);
  auto it = plans_.find(key);
  if (it != plans_.end()) return it->second;
  const int n = K * S;
  const size_t G2 = static_cast<size_t>(G) * G;
  std::vector<float> dcf(static_cast<size_t>(n));
  std::vector<int> cnt(G2 + 1, 0);
  std::vector<Taps> tx(static_cast<size_t>(n)), ty(static_cast<size_t>(n));
  for (int k = 0; k < K; ++k) {
    const double ca = std::cos(angles[k]), sa = std::sin(angles[k]);
    for (int i = 0; i < S; ++i) {
      const int s = k * S + i;
      const double r = readout_radius(i, S) + delay / S;  // frame_coords, preproc.cpp:86-95
      const double kx = r * ca, ky = r * sa;
      check_coord(kx, ky);
      dcf[static_cast<size_t>(s)] = static_cast<float>(dcf_ramp(kx, ky, K, S, G));
      tx[static_cast<size_t>(s)] = make_taps(kx * G + c, G);
      ty[static_cast<size_t>(s)] = make_taps(ky * G + c, G);
      for (int a = 0; a < kKbWidth; ++a) {
        for (int b = 0; b < kKbWidth; ++b) ++cnt[static_cast<size_t>(tx[s].idx[a]) * G + ty[s].idx[b] + 1];
      }
    }
  }
  for (size_t p = 0; p < G2; ++p) cnt[p + 1] += cnt[p];
  std::vector<int> sidx(static_cast<size_t>(cnt[G2])), fill(cnt.begin(), cnt.end() - 1);
  std::vector<float> w(sidx.size());
  for (int s = 0; s < n; ++s) {  // ascending sample order within every cell
    for (int a = 0; a < kKbWidth; ++a) {
      for (int b = 0; b < kKbWidth; ++b) {
        const size_t cell = static_cast<size_t>(tx[s].idx[a]) * G + ty[s].idx[b];
        const int e = fill[cell]++;
        sidx[static_cast<size_t>(e)] = s;
        w[static_cast<size_t>(e)] = static_cast<float>(tx[s].wgt[a] * ty[s].wgt[b]);
      }
    }
  }
  GridPlan gp;
  gp.n = n;
  check_cuda(cudaSetDevice(dev_), "set device");
  check_cuda(cudaMalloc(&gp.ptr, sizeof(int) * cnt.size()), "grid plan");
  check_cuda(cudaMalloc(&gp.sidx, sizeof(int) * std::max<size_t>(sidx.size(), 1)), "grid plan");
  check_cuda(cudaMalloc(&gp.w, sizeof(float) * std::max<size_t>(w.size(), 1)), "grid plan");
  check_cuda(cudaMalloc(&gp.dcf, sizeof(float) * std::max<size_t>(dcf.size(), 1)), "grid plan");
  check_cuda(cudaMemcpy(gp.ptr, cnt.data(), sizeof(int) * cnt.size(), cudaMemcpyHostToDevice), "grid plan");
  check_cuda(cudaMemcpy(gp.sidx, sidx.data(), sizeof(int) * sidx.size(), cudaMemcpyHostToDevice), "grid plan");
  check_cuda(cudaMemcpy(gp.w, w.data(), sizeof(float) * w.size(), cudaMemcpyHostToDevice), "grid plan");
  check_cuda(cudaMemcpy(gp.dcf, dcf.data(), sizeof(float) * dcf.size(), cudaMemcpyHostToDevice), "grid plan");
  return plans_.emplace(key, gp).first->second;
}

void Preproc::grid_adjoint(const float2* samples, int J, const double* angles, int K, int S, double delay,
                           float2* z_out, cudaStream_t s, bool spread_only, const float* post_scale) {
  if (J < 1 || K < 1 || S < 1) fail(2, "grid_adjoint: empty frame");
  const GridPlan& gp = grid_plan(angles, K, S, delay);
  const int G = plan_.G;
  const long long tot = static_cast<long long>(J) * G * G;
  k_grid_gather<<<grid_for(tot), kPre, 0, s>>>(J, G, gp.n, gp.ptr, gp.sidx, gp.w, gp.dcf, samples, z_out);
  check_cuda(cudaGetLastError(), "grid gather");
  if (spread_only) return;
  fft2_device(z_out, G, J, +1, s);  // fft::inverse per channel (preproc.cpp:193)
  k_deapod_mask<<<grid_for(tot), kPre, 0, s>>>(J, G, deapod_, z_out, post_scale ? 1 : 0,
                                                post_scale ? *post_scale : 1.f);
  check_cuda(cudaGetLastError(), "deapodise");
  fft_book(fft_current_ctx(), static_cast<uint64_t>(J));
}

void Preproc::psf_from_coords(const std::vector<double>& kx, const std::vector<double>& ky,
                              const std::vector<double>& v, float2* P_out, cudaStream_t s) {
  const int G = plan_.G;
  const int n = static_cast<int>(kx.size());
  if (n < 1) fail(2, "build_psf: no samples");
  const size_t tab = static_cast<size_t>(n) * G;
  if (tab > psf_tab_n_) {
    if (psf_tab_) {
      check_cuda(cudaDeviceSynchronize(), "sync");
      cudaFree(psf_tab_);
    }
    check_cuda(cudaMalloc(&psf_tab_, sizeof(double2) * 2 * tab), "psf tables");
    psf_tab_n_ = tab;
  }
  double* coords = nullptr;
  check_cuda(cudaMallocAsync(&coords, sizeof(double) * 3 * n, s), "psf coords");
  check_cuda(cudaMemcpyAsync(coords, kx.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s), "coords");
  check_cuda(cudaMemcpyAsync(coords + n, ky.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s), "coords");
  check_cuda(cudaMemcpyAsync(coords + 2 * n, v.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s), "coords");
  double2* AX = psf_tab_;
  double2* AY = psf_tab_ + tab;
  k_psf_tables<<<grid_for(static_cast<long long>(tab)), kPre, 0, s>>>(n, G, coords, coords + n, coords + 2 * n, AX, AY);
  const dim3 grid((G + 15) / 16, (G + 15) / 16);
  k_psf_gemm<<<grid, 256, 0, s>>>(n, G, AX, AY, psf_q_);
  k_psf_round<<<grid_for(static_cast<long long>(G) * G), kPre, 0, s>>>(G, psf_q_, P_out);
  check_cuda(cudaGetLastError(), "psf kernels");
  fft2_device(P_out, G, 1, -1, s);  // fft::forward (preproc.cpp:264)
  k_scale<<<grid_for(static_cast<long long>(G) * G), kPre, 0, s>>>(G * G, static_cast<float>(G), P_out);
  check_cuda(cudaGetLastError(), "psf scale");
  check_cuda(cudaFreeAsync(coords, s), "psf coords free");
  fft_book(fft_current_ctx(), 1);
}

void Preproc::build_psf(const double* angles, int K, int S, float2* P_out, cudaStream_t s) {
  const int G = plan_.G;
  std::vector<double> kx, ky, v;
  kx.reserve(static_cast<size_t>(K) * S);
  ky.reserve(kx.capacity());
  v.reserve(kx.capacity());
  for (int k = 0; k < K; ++k) {  // build_psf(angles, S, plan), preproc.cpp:269-285
    const double ca = std::cos(angles[k]), sa = std::sin(angles[k]);
    for (int i = 0; i < S; ++i) {
      const double r = readout_radius(i, S);
      kx.push_back(r * ca);
      ky.push_back(r * sa);
      v.push_back(dcf_ramp(r * ca, r * sa, K, S, G));
      check_coord(kx.back(), ky.back());
    }
  }
  psf_from_coords(kx, ky, v, P_out, s);
}

void Preproc::build_psf_coords(const double* coords, const double* weights, int n, float2* P_out,
                               cudaStream_t s) {
  std::vector<double> kx(static_cast<size_t>(n)), ky(static_cast<size_t>(n)), v(weights, weights + n);
  for (int i = 0; i < n; ++i) {
    kx[static_cast<size_t>(i)] = coords[2 * i];
    ky[static_cast<size_t>(i)] = coords[2 * i + 1];
    check_coord(kx[static_cast<size_t>(i)], ky[static_cast<size_t>(i)]);
  }
  psf_from_coords(kx, ky, v, P_out, s);
}

void Preproc::apply_compression(const float2* m, int Jv, int Jp, const float2* in, int n, float2* out,
                                cudaStream_t s) {
  if (Jv < 1 || Jp < 1 || Jv > Jp) fail(2, "apply_compression: virtual channel count out of range");
  k_compress<<<grid_for(static_cast<long long>(Jv) * n), kPre, 0, s>>>(Jv, Jp, n, m, in, out);
  check_cuda(cudaGetLastError(), "compress");
}

// ---- host wrappers --------------------------------------------------------------------------

void Preproc::grid_adjoint_host(const float* samples, int J, const double* angles, int K, int S, double delay,
                                float* z_out, bool spread_only) {
  check_cuda(cudaSetDevice(dev_), "set device");
  const size_t ns = static_cast<size_t>(J) * K * S, nz = static_cast<size_t>(J) * plan_.G * plan_.G;
  float2* buf = scratch(sizeof(float2) * (ns + nz));
  check_cuda(cudaMemcpyAsync(buf, samples, sizeof(float2) * ns, cudaMemcpyHostToDevice, s_), "h2d");
  grid_adjoint(buf, J, angles, K, S, delay, buf + ns, s_, spread_only);
  check_cuda(cudaMemcpyAsync(z_out, buf + ns, sizeof(float2) * nz, cudaMemcpyDeviceToHost, s_), "d2h");
  check_cuda(cudaStreamSynchronize(s_), "sync");
}

void Preproc::build_psf_host(const double* angles, int K, int S, float* P_out) {
  check_cuda(cudaSetDevice(dev_), "set device");
  const size_t G2 = static_cast<size_t>(plan_.G) * plan_.G;
  float2* buf = scratch(sizeof(float2) * G2);
  build_psf(angles, K, S, buf, s_);
  check_cuda(cudaMemcpyAsync(P_out, buf, sizeof(float2) * G2, cudaMemcpyDeviceToHost, s_), "d2h");
  check_cuda(cudaStreamSynchronize(s_), "sync");
}

void Preproc::build_psf_coords_host(const double* coords, const double* weights, int n, float* P_out) {
  check_cuda(cudaSetDevice(dev_), "set device");
  const size_t G2 = static_cast<size_t>(plan_.G) * plan_.G;
  float2* buf = scratch(sizeof(float2) * G2);
  build_psf_coords(coords, weights, n, buf, s_);
  check_cuda(cudaMemcpyAsync(P_out, buf, sizeof(float2) * G2, cudaMemcpyDeviceToHost, s_), "d2h");
  check_cuda(cudaStreamSynchronize(s_), "sync");
}

void Preproc::apply_compression_host(const float* m, int Jv, int Jp, const float* in, int n, float* out) {
  check_cuda(cudaSetDevice(dev_), "set device");
  const size_t nm = static_cast<size_t>(Jv) * Jp, ni = static_cast<size_t>(Jp) * n, no = static_cast<size_t>(Jv) * n;
  float2* buf = scratch(sizeof(float2) * (nm + ni + no));
  check_cuda(cudaMemcpyAsync(buf, m, sizeof(float2) * nm, cudaMemcpyHostToDevice, s_), "h2d");
  check_cuda(cudaMemcpyAsync(buf + nm, in, sizeof(float2) * ni, cudaMemcpyHostToDevice, s_), "h2d");
  apply_compression(buf, Jv, Jp, buf + nm, n, buf + nm + ni, s_);
  check_cuda(cudaMemcpyAsync(out, buf + nm + ni, sizeof(float2) * no, cudaMemcpyDeviceToHost, s_), "d2h");
  check_cuda(cudaStreamSynchronize(s_), "sync");
}

}  // namespace rtnb
