// Grid planning over the device transforms and device postprocessing (post.cu).
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <string>
#include <utility>
#include <vector>

#include "engine.hpp"

namespace rtnb {

// rtnlinv::FftLookupTable (planner.hpp:12-18)
struct FftTable {
  std::map<int, double> entries_us;
  std::string machine_key;
  std::string library_key;
};

// device time (us) of one centered 2D forward transform of `batch` n x n images per
// size, minimum over `trials` (benchmark_fft, planner.cpp:69-110)
FftTable benchmark_fft_device(const std::vector<int>& sizes, int trials, int batch, int device);
std::pair<int, double> select_grid(int N, const FftTable& table, double gamma_min = 1.4, double gamma_max = 2.0);
void save_fft_table(const FftTable& table, const std::string& path);
FftTable load_fft_table(const std::string& path);

// pipeline.cpp:60-137 on device buffers (n = elements, npix = pixels per frame)
void post_magnitude(const float2* x, long long n, float* out, cudaStream_t s);
void post_phase_difference(const float2* even, const float2* odd, long long n, float* out, cudaStream_t s);
void post_median3(const float* mags, int frames, long long npix, float* out, cudaStream_t s);

}  // namespace rtnb
