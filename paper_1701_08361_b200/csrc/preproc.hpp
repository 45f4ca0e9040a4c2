// The pre stage on the device: adjoint gridding of raw
// radial samples (grid_adjoint, preproc.cpp:167-199), the Toeplitz kernel of a
// trajectory (build_psf / build_psf_coords, preproc.cpp:223-290) and coil
// compression (apply_compression, preproc.cpp:446-471).
//
// Gridding is a deterministic gather: per (angle set, S, delay) the host builds,
// once, the inverse of the sample -> 4x4 Kaiser-Bessel tap map as a cell-major CSR
// list in ascending sample order with the reference's float tap weights. One thread
// per (channel, grid cell) then accumulates exactly the reference's float products
// in the reference's order (spread_sample, preproc.cpp:123-133), so the gridded
// k-space is bit-identical; the centered inverse FFT, the G / deapodisation scale
// and the window mask follow on the device.
//
// The PSF's trajectory response q(d) = sum_s v_s exp(2 pi i k_s . d) is a complex
// FP64 product Q = AX^T AY of the per-sample phase tables (preproc.cpp:233-246),
// accumulated per element in sample order like the reference; then the Nyquist
// edge is zeroed, Q is rounded to float, transformed and scaled by G.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "engine.hpp"

namespace rtnb {

// PsfCache::angle_key (preproc.cpp:301-313): FNV-1a over S, G and the angles in 1e-9 units
uint64_t psf_angle_key(const double* angles, int K, int S, int G);

class Preproc {
 public:
  Preproc(const Plan& plan, int device);
  ~Preproc();
  Preproc(const Preproc&) = delete;
  Preproc& operator=(const Preproc&) = delete;

  const Plan& plan() const { return plan_; }

  // device-side, stream ordered. samples: J x K x S complex64 (KSpaceFrame::samples)
  // post_scale: the series normalisation applied in the deapodisation pass (nullptr: none)
  void grid_adjoint(const float2* samples, int J, const double* angles, int K, int S, double delay,
                    float2* z_out, cudaStream_t s, bool spread_only = false, const float* post_scale = nullptr);
  void build_psf(const double* angles, int K, int S, float2* P_out, cudaStream_t s);
  void build_psf_coords(const double* coords, const double* weights, int n, float2* P_out, cudaStream_t s);
  // out[jv][s] = sum_jp m[jv][jp] in[jp][s], FP64 accumulation (preproc.cpp:459-468)
  void apply_compression(const float2* m, int Jv, int Jp, const float2* in, int n, float2* out, cudaStream_t s);

  // host in / host out wrappers (parity boundary)
  void grid_adjoint_host(const float* samples, int J, const double* angles, int K, int S, double delay,
                         float* z_out, bool spread_only = false);
  void build_psf_host(const double* angles, int K, int S, float* P_out);
  void build_psf_coords_host(const double* coords, const double* weights, int n, float* P_out);
  void apply_compression_host(const float* m, int Jv, int Jp, const float* in, int n, float* out);

 private:
  struct GridPlan {
    int n = 0;
    int* ptr = nullptr;   // G*G + 1
    int* sidx = nullptr;  // entries: sample index, ascending per cell
    float* w = nullptr;   // entries: float(wx * wy)
    float* dcf = nullptr; // n: float(dcf_ramp)
  };
  const GridPlan& grid_plan(const double* angles, int K, int S, double delay);
  void psf_from_coords(const std::vector<double>& kx, const std::vector<double>& ky, const std::vector<double>& v,
                       float2* P_out, cudaStream_t s);
  float2* scratch(size_t bytes);

  Plan plan_;
  int dev_ = 0;
  cudaStream_t s_ = nullptr;       // host-wrapper stream
  float* deapod_ = nullptr;        // G*G: float(G) / float(deapodization) (preproc.cpp:195)
  std::mutex mu_;
  std::map<uint64_t, GridPlan> plans_;
  double2* psf_tab_ = nullptr;     // per-sample phase tables
  size_t psf_tab_n_ = 0;
  double2* psf_q_ = nullptr;       // G*G FP64 trajectory response
  void* scratch_ = nullptr;
  size_t scratch_bytes_ = 0;
};

}  // namespace rtnb
