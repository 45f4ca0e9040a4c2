// Grid planning over the device transforms and image postprocessing on the device
// (SURVEY.md §8(f) ranks 3-4).
//
// Planner (planner.cpp:69-185): the reference times one FFTW transform per size and
// picks the fastest even G in [2 gamma_min N, 2 gamma_max N] (Table 2).
// Here the table holds the device time of one batched centered 2D transform of the
// sm_100a line engine (CUDA events, minimum over trials), so the planner picks the
// grids this engine is fast at; select_grid / make_plan / the table file format are
// the reference's.
//
// Postprocessing (pipeline.cpp:60-135): magnitude images, phase-difference images
// of frame pairs, and the per-slice temporal median-of-3 filter, as kernels over
// device-resident image series.
#include "post.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <limits>
#include <sstream>

namespace rtnb {

namespace {

int even_ceil(double x) {  // planner.cpp:41-45
  int v = static_cast<int>(std::ceil(x - 1e-9));
  if (v % 2 != 0) ++v;
  return v;
}

int even_floor(double x) {  // planner.cpp:47-51
  int v = static_cast<int>(std::floor(x + 1e-9));
  if (v % 2 != 0) --v;
  return v;
}

__global__ void k_fill_bench(float2* x, long long n) {
  // the reference's deterministic fill (planner.cpp:84-87)
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    x[i] = make_float2((i % 37) * 0.1f, (i % 11) * -0.2f);
  }
}

// |x| (std::abs(std::complex<float>), pipeline.cpp:66-69)
__global__ void k_magnitude(const float2* __restrict__ x, long long n, float* __restrict__ out) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float2 v = x[i];
    // glibc's hypotf: the sum of squares in double, one rounding to float
    out[i] = static_cast<float>(__dsqrt_rn(__dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y))));
  }
}

// arg(even * conj(odd)) in double (pipeline.cpp:82-85)
__global__ void k_phase_diff(const float2* __restrict__ even, const float2* __restrict__ odd, long long n,
                             float* __restrict__ out) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float2 a = even[i], b = odd[i];
    const double re = __dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y));
    const double im = __dsub_rn(__dmul_rn(a.y, b.x), __dmul_rn(a.x, b.y));
    out[i] = static_cast<float>(atan2(im, re));
  }
}

__device__ __forceinline__ float median3(float a, float b, float c) {  // pipeline.cpp:92-94
  return fmaxf(fminf(a, b), fminf(fmaxf(a, b), c));
}

// MedianFilter3 over a whole per-slice sequence (pipeline.cpp:104-137): frame k gets
// median(m[k-1], m[k], m[k+1]) with the missing neighbour of the first / last frame
// replicated from the frame itself (push: median(h0, h0, img); drain: median(h0, h1, h1)),
// a single frame passes through
__global__ void k_median3_seq(const float* __restrict__ m, int frames, long long npix, float* __restrict__ out) {
  const long long n = frames * npix;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(i / npix);
    const long long p = i - k * npix;
    if (frames == 1) {
      out[i] = m[i];
      continue;
    }
    const float cur = m[i];
    const float prev = k > 0 ? m[(k - 1) * npix + p] : cur;
    const float next = k + 1 < frames ? m[(k + 1) * npix + p] : cur;
    out[i] = median3(prev, cur, next);
  }
}

int grid_for(long long n) { return static_cast<int>(std::max(1LL, std::min((n + 255) / 256, 148LL * 16))); }

}  // namespace

FftTable benchmark_fft_device(const std::vector<int>& sizes, int trials, int batch, int device) {
  if (sizes.empty()) fail(2, "benchmark_fft: bad size range");
  for (int n : sizes) {
    if (n < 2) fail(2, "benchmark_fft: bad size range");
  }
  if (trials < 1) fail(2, "benchmark_fft: trials must be >= 1");
  if (batch < 1) fail(2, "benchmark_fft: batch must be >= 1");
  check_cuda(cudaSetDevice(device), "set device");
  FftTable t;
  cudaDeviceProp prop{};
  check_cuda(cudaGetDeviceProperties(&prop, device), "device properties");
  t.machine_key = std::string(prop.name) + "-sm" + std::to_string(prop.multiProcessorCount);
  t.library_key = "rtnlinv_b200-line-fft-sm100a";
  cudaStream_t s;
  check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  cudaEvent_t a, b;
  check_cuda(cudaEventCreate(&a), "event");
  check_cuda(cudaEventCreate(&b), "event");
  const int prev_ctx = fft_current_ctx();
  fft_set_ctx(CTX_BENCH);  // fft::CtxScope(bench), planner.cpp:80
  float2* x = nullptr;
  try {
    for (int n : sizes) {
      const long long cnt = static_cast<long long>(n) * n * batch;
      check_cuda(cudaMalloc(&x, sizeof(float2) * cnt), "bench buffer");
      k_fill_bench<<<grid_for(cnt), 256, 0, s>>>(x, cnt);
      fft2_device(x, n, batch, -1, s);  // warm-up (kernel attributes, tables)
      float best = std::numeric_limits<float>::infinity();
      for (int r = 0; r < trials; ++r) {
        check_cuda(cudaEventRecord(a, s), "event");
        fft2_device(x, n, batch, -1, s);
        check_cuda(cudaEventRecord(b, s), "event");
        check_cuda(cudaEventSynchronize(b), "event sync");
        float ms = 0;
        check_cuda(cudaEventElapsedTime(&ms, a, b), "elapsed");
        best = std::min(best, ms);
      }
      fft_book(CTX_BENCH, static_cast<uint64_t>(trials + 1) * batch);
      t.entries_us[n] = static_cast<double>(best) * 1000.0;
      cudaFree(x);
      x = nullptr;
    }
  } catch (...) {
    if (x) cudaFree(x);
    fft_set_ctx(prev_ctx);
    throw;
  }
  fft_set_ctx(prev_ctx);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaStreamDestroy(s);
  return t;
}

std::pair<int, double> select_grid(int N, const FftTable& table, double gamma_min, double gamma_max) {
  // planner.cpp:112-131
  if (N < 2) fail(2, "select_grid: N too small");
  const int lo = even_ceil(2.0 * gamma_min * N);
  const int hi = even_floor(2.0 * gamma_max * N);
  if (lo > hi) fail(2, "select_grid: empty grid search interval");
  int best_g = -1;
  double best_t = std::numeric_limits<double>::infinity();
  for (int g = lo; g <= hi; g += 2) {
    auto it = table.entries_us.find(g);
    if (it == table.entries_us.end()) fail(2, "select_grid: lookup table does not cover size " + std::to_string(g));
    if (it->second < best_t) {
      best_t = it->second;
      best_g = g;
    }
  }
  return {best_g, best_g / (2.0 * N)};
}

void save_fft_table(const FftTable& table, const std::string& path) {  // planner.cpp:151-163
  std::ofstream out(path, std::ios::trunc);
  if (!out) fail(3, "cannot write lookup table: " + path);
  out << "# machine:\t" << table.machine_key << "\n";
  out << "# library:\t" << table.library_key << "\n";
  for (const auto& [size, us] : table.entries_us) {
    char line[64];
    std::snprintf(line, sizeof(line), "%d\t%.3f\n", size, us);
    out << line;
  }
  if (!out.good()) fail(3, "write failed for lookup table: " + path);
}

FftTable load_fft_table(const std::string& path) {  // planner.cpp:165-183
  std::ifstream in(path);
  if (!in) fail(3, "cannot open lookup table: " + path);
  FftTable table;
  std::string line;
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    if (line[0] == '#') {
      const auto tab = line.find('\t');
      if (tab == std::string::npos) continue;
      const std::string value = line.substr(tab + 1);
      if (line.rfind("# machine:", 0) == 0) table.machine_key = value;
      if (line.rfind("# library:", 0) == 0) table.library_key = value;
      continue;
    }
    std::istringstream ls(line);
    int size = 0;
    double us = 0;
    if (!(ls >> size >> us) || size < 2 || us <= 0) fail(3, "malformed lookup table line: " + line);
    table.entries_us[size] = us;
  }
  return table;
}

void post_magnitude(const float2* x, long long n, float* out, cudaStream_t s) {
  k_magnitude<<<grid_for(n), 256, 0, s>>>(x, n, out);
  check_cuda(cudaGetLastError(), "magnitude");
}

void post_phase_difference(const float2* even, const float2* odd, long long n, float* out, cudaStream_t s) {
  k_phase_diff<<<grid_for(n), 256, 0, s>>>(even, odd, n, out);
  check_cuda(cudaGetLastError(), "phase difference");
}

void post_median3(const float* mags, int frames, long long npix, float* out, cudaStream_t s) {
  if (frames < 1) fail(2, "median filter: no frames");
  k_median3_seq<<<grid_for(frames * npix), 256, 0, s>>>(mags, frames, npix, out);
  check_cuda(cudaGetLastError(), "median3");
}

}  // namespace rtnb
