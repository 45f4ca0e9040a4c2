// Frame-series drivers: reconstruct_series_plain and
// the temporally decomposed reconstruct_series (nlinv.cpp:412-526) over
// device-resident frames.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "engine.hpp"
#include "group.hpp"
#include "preproc.hpp"
#include "sched.hpp"

namespace rtnb {

struct SeriesOptions {
  TemporalSchedule sched{1, 1};
  int T = 1;            // frames in flight: one worker (stream + workspace) each
  int A = 1;            // channel-decomposition width: each worker is a Group of A devices
  bool chain = true;
  bool normalize = true;
  bool plain = false;   // reconstruct_series_plain semantics (strictly sequential)
  int cluster = -1;     // cluster-fused applications: 1 on, 0 off, -1 auto (on when T == 1)
};

// Raw acquisition input of the end-to-end path (KSpaceFrame per frame, seqsim.hpp:52-65):
// samples count x Jp x K x S complex64 (host), angles count x K; with a compression
// matrix (Jv x Jp, Jv = plan.J) the physical channels are compressed on the device
// first (apply_compression), else Jp = plan.J.
struct RawInput {
  const float* samples = nullptr;
  const double* angles = nullptr;
  int K = 0;
  int S = 0;
  int Jp = 0;
  double delay = 0.0;
  const float* cmat = nullptr;
};

struct SeriesFrameOut {
  FrameAudit audit;
  int cg_iters = 0;
  float gpu_ms = 0;     // frame start -> image ready, CUDA events on the worker stream
};

// Owns the device-resident series store: gridded frames z[F][J][G][G], the PSF set
// (a K-spoke, U-turn trajectory has at most U distinct kernels), per-frame final
// estimates and images. Worker 0 is the caller's engine; T-1 more are created on the
// same device on demand.
class Series {
 public:
  // devices: worker t runs on devices[t % devices.size()] (default: the primary's
  // device); with channel decomposition (SeriesOptions::A > 1) worker t is a Group
  // over devices[(t*A + k) % devices.size()], k < A (hybrid T x A split). With several devices the series store stays on the primary's device and
  // frames, PSFs and estimates move peer to peer (NVLink / NVSwitch, UVA copies):
  // temporal decomposition across GPUs inside one process, the reference's
  // thread-per-compute-worker model.
  Series(Engine& primary, int frames, int n_psf, std::vector<int> devices = {});
  ~Series();
  Series(const Series&) = delete;
  Series& operator=(const Series&) = delete;

  int frames() const { return F_; }
  // Multi-slice acquisitions (pipeline.cpp:315-334, 429-434, 503): the store holds Sl
  // interleaved slice chains, store index g = frame * Sl + slice, as the pipeline
  // numbers its deliveries. Each slice is its own chain (ledger, estimates, temporal
  // schedule) with its own normalisation (frame 0 of the slice scaled to norm 100);
  // the T frame workers take store indices round-robin across slices.
  void set_slices(int Sl);
  int slices() const { return Sl_; }
  double slice_scale(int sl) const { return slice_scale_[static_cast<size_t>(sl)]; }
  void upload_frames(int first, int count, const float* z_host);  // synchronous H2D
  void upload_psf(int k, const float* P_host);
  void set_psf_index(const int* idx);
  // prep_series normalisation (nlinv.cpp:390-400): scale every frame so frame 0 has
  // norm 100; returns the scale. Idempotent per upload.
  double normalize();
  double data_scale() const { return scale_; }

  // Reconstruct frames [first, first + count). Frames before `first` count as
  // complete (their estimates from earlier calls are the chain). When z_host is not
  // null the frames are streamed from host memory inside the call (copy stream,
  // overlapped with compute) and normalised on arrival: the end-to-end path.
  // images_host (count*N*N) receives the images; nullable.
  // raw: the frames arrive as raw radial samples instead (z_host must be null); they
  // are compressed, gridded (grid_adjoint) and their PSFs built or taken from the
  // series' PSF cache on the device, all on the copy stream (rtnlinv's pre stage,
  // pipeline.cpp:420-498)
  void run(const SeriesOptions& o, int first, int count, const float* z_host, float* images_host,
           std::vector<SeriesFrameOut>* out, const RawInput* raw = nullptr);
  int psf_cache_size() const { return static_cast<int>(psf_keys_.size()); }
  // the device PSF cache in the reference's sidecar format (PsfCache::save / load)
  bool save_psf_cache(const std::string& path);
  bool load_psf_cache(const std::string& path);
  // postprocessing of the device-resident images [first, first + count) into host floats:
  // mode 0 magnitude, 1 magnitude + temporal median-of-3 (MedianFilter3 over the range),
  // 2 phase difference of consecutive frame pairs (count/2 images); pipeline.cpp:60-137
  void post(int first, int count, int mode, float* out);

  float2* images_dev() { return images_; }
  // device time of the last run(): CUDA events spanning every worker stream, from
  // before the first frame's first copy to after the last frame's image
  float last_span_ms() const { return span_ms_; }
  float2* estimate_dev(int n) { return ests_ + static_cast<size_t>(n) * D_; }

 private:
  FrameWorker& worker(int t);
  // g: store index (frame g / Sl of slice g % Sl)
  void run_frame(int t, int g, const SeriesOptions& o, SeriesFrameOut& out, cudaEvent_t ready);

  Engine& eng0_;
  std::vector<std::unique_ptr<Engine>> extra_;
  std::vector<std::unique_ptr<Group>> groups_;
  int A_ = 1;  // width of the current run's workers
  std::unique_ptr<Preproc> pre_;           // raw-input path (created on first use)
  std::vector<uint64_t> psf_keys_;         // PsfCache: angle key of each built PSF slot
  float2* raw_ = nullptr;                  // raw-sample staging (frames x Jp x K x S)
  size_t raw_cap_ = 0;
  float2* raw_c_ = nullptr;                // compressed staging (one frame) + matrix
  size_t raw_c_cap_ = 0;
  void produce_frames(const SeriesOptions& o, int first, int count, const float* z_host, const RawInput* raw,
                      std::vector<cudaEvent_t>& ready);
  // The raw-input pre stage of the frames a worker on another device reconstructs runs on
  // that device (its own copy stream, Preproc, staging, PSF cache and gridded frames), so
  // the H2D copies and gridding of a multi-GPU series are spread over the GPUs and the
  // worker reads its frame locally. RTN_PRE_LANES=1 also gives same-device workers t >= 1
  // their own lanes (tests exercise the lane path on one GPU).
  struct PreLane {
    int dev = 0;
    cudaStream_t copy = nullptr;
    std::unique_ptr<Preproc> pre;
    float2* raw = nullptr;
    size_t raw_cap = 0;
    float2* raw_c = nullptr;
    size_t raw_c_cap = 0;
    float2* z = nullptr;       // gridded frames of the current call (count slots)
    size_t z_cap = 0;
    float2* psf = nullptr;     // this lane's PSF cache (n_psf slots)
    std::vector<uint64_t> keys;
    double* nsq = nullptr;
    PreLane() = default;
    PreLane(const PreLane&) = delete;
    PreLane& operator=(const PreLane&) = delete;
    ~PreLane();
  };
  PreLane* lane_for(int t);
  std::vector<std::unique_ptr<PreLane>> lanes_;
  bool force_lanes_ = false;
  std::vector<const float2*> zsrc_, psrc_;  // per frame of the current run (nullptr: the store)
  bool raw_run_ = false;  // the current run's frames came through the device pre stage
  std::vector<int> devices_;
  int F_ = 0, n_psf_ = 0, D_ = 0;
  size_t zsz_ = 0, psz_ = 0, isz_ = 0;
  float2* z_ = nullptr;
  float2* psf_ = nullptr;
  float2* ests_ = nullptr;
  float2* unity_ = nullptr;
  float2* images_ = nullptr;
  double* nsq_ = nullptr;
  std::vector<int> psf_idx_;
  double scale_ = 1.0;
  bool normalized_ = false;
  cudaStream_t copy_ = nullptr;
  cudaEvent_t span0_ = nullptr, span1_ = nullptr;
  float span_ms_ = 0.f;
  bool step_sync_ = false;
  bool safe_mode_ = false;                 // no device-side chaining of closing steps
  int Sl_ = 1;                             // interleaved slice chains
  std::vector<double> slice_scale_{1.0};   // prep normalisation per slice
  std::vector<std::unique_ptr<CompletionLedger>> ledgers_;  // per slice, current run
  std::vector<std::unique_ptr<CompletionLedger>> enqs_;     // per slice: final work enqueued
  int run_first_ = 0;
  std::vector<cudaEvent_t> done_;          // per frame of the current run: estimate published
};

}  // namespace rtnb
