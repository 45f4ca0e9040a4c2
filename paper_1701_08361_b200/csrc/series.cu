// Series drivers over device-resident frames (nlinv.cpp:366-526).
#include "series.hpp"

#include <nvtx3/nvToolsExt.h>

#include "post.hpp"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <exception>
#include <mutex>
#include <thread>

namespace rtnb {

namespace {

struct RedoSeries {};

__global__ void k_nrm2_frame(const float2* __restrict__ z, long long n, double* out) {
  // single block, fixed order: deterministic FP64 |z|^2 of one frame
  __shared__ double red[256];
  double acc = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const float2 v = z[i];
    acc += (double)v.x * v.x + (double)v.y * v.y;
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

__global__ void k_scale_frames(float2* __restrict__ z, long long n, float s) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float2 v = z[i];
    z[i] = make_float2(v.x * s, v.y * s);
  }
}

}  // namespace

Series::Series(Engine& primary, int frames, int n_psf, std::vector<int> devices)
    : eng0_(primary), F_(frames), n_psf_(n_psf), devices_(std::move(devices)) {
  if (frames < 1) fail(2, "reconstruct_series: no frames");
  if (devices_.empty()) devices_.push_back(primary.device());
  if (devices_[0] != primary.device()) devices_.insert(devices_.begin(), primary.device());
  // peer access between every pair of distinct devices used by the workers
  for (int a : devices_) {
    for (int b : devices_) {
      if (a == b) continue;
      int ok = 0;
      check_cuda(cudaDeviceCanAccessPeer(&ok, a, b), "peer query");
      if (!ok) fail(2, "reconstruct_series: devices " + std::to_string(a) + " and " + std::to_string(b) +
                           " have no peer access");
      check_cuda(cudaSetDevice(a), "set device");
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) check_cuda(e, "enable peer access");
      cudaGetLastError();
    }
  }
  if (n_psf < 1) fail(2, "reconstruct_series: need at least one PSF");
  const Plan& p = eng0_.plan();
  D_ = eng0_.D();
  zsz_ = static_cast<size_t>(p.J) * p.G * p.G;
  psz_ = static_cast<size_t>(p.G) * p.G;
  isz_ = static_cast<size_t>(p.N) * p.N;
  check_cuda(cudaSetDevice(eng0_.device()), "set device");
  check_cuda(cudaMalloc(&z_, sizeof(float2) * zsz_ * F_), "series frames");
  check_cuda(cudaMalloc(&psf_, sizeof(float2) * psz_ * n_psf_), "series psf");
  check_cuda(cudaMalloc(&ests_, sizeof(float2) * static_cast<size_t>(D_) * F_), "series estimates");
  check_cuda(cudaMalloc(&unity_, sizeof(float2) * D_), "unity");
  check_cuda(cudaMalloc(&images_, sizeof(float2) * isz_ * F_), "series images");
  check_cuda(cudaMalloc(&nsq_, sizeof(double)), "nsq");
  check_cuda(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking), "copy stream");
  check_cuda(cudaEventCreate(&span0_), "event");
  check_cuda(cudaEventCreate(&span1_), "event");
  // initial_estimate: rho = 1 on the window, coils 0 (nlinv.cpp:60-70)
  std::vector<float2> u(static_cast<size_t>(D_), make_float2(0.f, 0.f));
  const int L = p.G / 2, lo = (p.G - L) / 2;
  for (int r = lo; r < lo + L; ++r) {
    for (int c = lo; c < lo + L; ++c) u[static_cast<size_t>(r) * p.G + c] = make_float2(1.f, 0.f);
  }
  check_cuda(cudaMemcpy(unity_, u.data(), sizeof(float2) * D_, cudaMemcpyHostToDevice), "unity upload");
  if (const char* e = std::getenv("RTN_STEP_SYNC")) step_sync_ = e[0] == '1';
  if (const char* e = std::getenv("RTN_PRE_LANES")) force_lanes_ = e[0] == '1';
  psf_idx_.resize(static_cast<size_t>(F_));
  for (int n = 0; n < F_; ++n) psf_idx_[static_cast<size_t>(n)] = n % n_psf_;
}

Series::PreLane::~PreLane() {
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(dev);
  if (copy) cudaStreamSynchronize(copy);
  pre.reset();
  for (void* b : {static_cast<void*>(raw), static_cast<void*>(raw_c), static_cast<void*>(z), static_cast<void*>(psf),
                  static_cast<void*>(nsq)}) {
    if (b) cudaFree(b);
  }
  if (copy) cudaStreamDestroy(copy);
  cudaSetDevice(cur);
}

Series::~Series() {
  lanes_.clear();
  cudaSetDevice(eng0_.device());
  if (copy_) cudaStreamSynchronize(copy_);
  pre_.reset();
  if (raw_) cudaFree(raw_);
  if (raw_c_) cudaFree(raw_c_);
  for (void* b : {static_cast<void*>(z_), static_cast<void*>(psf_), static_cast<void*>(ests_),
                  static_cast<void*>(unity_), static_cast<void*>(images_), static_cast<void*>(nsq_)}) {
    if (b) cudaFree(b);
  }
  if (copy_) cudaStreamDestroy(copy_);
  if (span0_) cudaEventDestroy(span0_);
  if (span1_) cudaEventDestroy(span1_);
}

FrameWorker& Series::worker(int t) {
  if (A_ > 1) {
    while (static_cast<int>(groups_.size()) <= t) {
      const int k = static_cast<int>(groups_.size());
      std::vector<int> devs;
      for (int a = 0; a < A_; ++a) devs.push_back(devices_[static_cast<size_t>(k * A_ + a) % devices_.size()]);
      groups_.push_back(std::make_unique<Group>(eng0_.plan(), devs));
    }
    return *groups_[static_cast<size_t>(t)];
  }
  if (t == 0) return eng0_;
  while (static_cast<int>(extra_.size()) < t) {
    const int k = static_cast<int>(extra_.size()) + 1;
    extra_.push_back(std::make_unique<Engine>(eng0_.plan(), devices_[static_cast<size_t>(k) % devices_.size()]));
  }
  return *extra_[static_cast<size_t>(t - 1)];
}

void Series::upload_frames(int first, int count, const float* z_host) {
  if (first < 0 || count < 0 || first + count > F_) fail(2, "upload_frames: frame range out of bounds");
  check_cuda(cudaSetDevice(eng0_.device()), "set device");
  check_cuda(cudaMemcpy(z_ + zsz_ * first, z_host, sizeof(float2) * zsz_ * count, cudaMemcpyHostToDevice),
             "frame upload");
  if (first == 0) normalized_ = false;
}

void Series::upload_psf(int k, const float* P_host) {
  if (k < 0 || k >= n_psf_) fail(2, "upload_psf: index out of range");
  check_cuda(cudaMemcpy(psf_ + psz_ * k, P_host, sizeof(float2) * psz_, cudaMemcpyHostToDevice), "psf upload");
}

void Series::set_psf_index(const int* idx) {
  for (int n = 0; n < F_; ++n) {
    if (idx[n] < 0 || idx[n] >= n_psf_) fail(2, "set_psf_index: index out of range");
    psf_idx_[static_cast<size_t>(n)] = idx[n];
  }
}

void Series::set_slices(int Sl) {
  if (Sl < 1 || Sl > F_) fail(2, "reconstruct_series: slice count out of range");
  Sl_ = Sl;
  slice_scale_.assign(static_cast<size_t>(Sl), 1.0);
  normalized_ = false;
}

double Series::normalize() {
  if (normalized_) return scale_;
  check_cuda(cudaSetDevice(eng0_.device()), "set device");
  for (int sl = 0; sl < Sl_; ++sl) {
    // frame 0 of the slice sets its scale (pipeline.cpp:429-434; nlinv.cpp:390-400 for Sl = 1)
    k_nrm2_frame<<<1, 256>>>(z_ + zsz_ * sl, static_cast<long long>(zsz_), nsq_);
    double nsq = 0;
    check_cuda(cudaMemcpy(&nsq, nsq_, sizeof(double), cudaMemcpyDeviceToHost), "nsq read");
    double sc = 1.0;
    if (nsq > 0) {
      sc = 100.0 / std::sqrt(nsq);
      for (int g = sl; g < F_; g += Sl_) {
        k_scale_frames<<<148 * 2, 256>>>(z_ + zsz_ * g, static_cast<long long>(zsz_), static_cast<float>(sc));
      }
    }
    slice_scale_[static_cast<size_t>(sl)] = sc;
  }
  check_cuda(cudaDeviceSynchronize(), "normalise");
  scale_ = slice_scale_[0];
  normalized_ = true;
  return scale_;
}

namespace {
// NVTX range for a profiler timeline (SURVEY.md §5 "tracing"); no-op without a tool
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

void Series::run_frame(int t, int g, const SeriesOptions& o, SeriesFrameOut& out, cudaEvent_t ready) {
  // frame n of slice sl; its chain (ledger, estimates, schedule) is the slice's own
  const int n = g / Sl_, sl = g % Sl_;
  CompletionLedger& ledger = *ledgers_[static_cast<size_t>(sl)];
  CompletionLedger& enq = *enqs_[static_cast<size_t>(sl)];
  auto est_of = [&](int frame) { return estimate_dev(frame * Sl_ + sl); };
  const double scale = slice_scale_[static_cast<size_t>(sl)];
  const std::string label = "frame " + std::to_string(n) + " slice " + std::to_string(sl) + " worker " +
                            std::to_string(t);
  NvtxRange range(label.c_str());
  FrameWorker& e = worker(t);
  const Plan& p = e.plan();
  const int M = p.newton_steps;
  cudaStream_t s = e.stream();
  const bool chained = o.chain && n > 0;
  FrameAudit a;
  a.frame = n;
  a.thread = t;
  a.workers = o.A;
  a.reg_src.assign(static_cast<size_t>(M), -1);
  if (!o.plain) {
    // frames in the strict prefix start only after the predecessor finished
    if (chained && n <= o.sched.l) ledger.wait_complete(n - 1);
    a.start_seq = ledger.next_seq();
  }
  if (chained) a.init_src = o.plain ? n - 1 : h_choose(n, 0, M, o.sched, ledger);
  const float2* init = chained ? est_of(a.init_src) : unity_;

  if (ready) check_cuda(cudaStreamWaitEvent(s, ready, 0), "wait frame upload");
  check_cuda(cudaSetDevice(e.device()), "set device");
  // the frame's gridded data and PSF: the store, or the lane that ran its pre stage
  const size_t kr = static_cast<size_t>(g - run_first_);
  const float2* zl = kr < zsrc_.size() ? zsrc_[kr] : nullptr;
  const float2* pl = kr < psrc_.size() ? psrc_[kr] : nullptr;
  // frames the device pre stage gridded are window-masked by construction (mask_window,
  // preproc.cpp:193-195): no outside-window scan
  e.load_frame(zl ? zl : z_ + zsz_ * g, pl ? pl : psf_ + psz_ * psf_idx_[static_cast<size_t>(g)], raw_run_);
  e.load_x(init);
  cudaEvent_t ev0, ev1;
  check_cuda(cudaEventCreate(&ev0), "event");
  check_cuda(cudaEventCreate(&ev1), "event");
  check_cuda(cudaEventRecord(ev0, s), "event");
  // the image lands in the store directly on the store's device, via the worker's
  // own buffer (then one peer copy) elsewhere
  const bool local = e.device() == eng0_.device();
  float2* img = local ? images_ + isz_ * g : e.image_dev();
  const float iscale = static_cast<float>(1.0 / scale);
  const bool undo = o.normalize && scale != 1.0;
  const bool fixed_reg = o.plain || !chained;  // every step regularises towards init
  const bool chain_events = !safe_mode_ && !o.plain && o.T > 1;
  if (fixed_reg) {
    for (int m = 0; m < M; ++m) a.reg_src[static_cast<size_t>(m)] = chained ? a.init_src : -1;
    e.load_reg(init);
    if (!o.plain && M > 0) a.reg_final_seq = ledger.next_seq();
    if (e.budget_mode()) {
      e.frame_all(img, iscale, undo);
    } else {
      e.frame_begin();
      for (int m = 0; m < M; ++m) e.frame_step(m, nullptr);
      e.frame_image(img, iscale, undo);
    }
  } else {
    e.frame_begin();
    for (int m = 0; m < M; ++m) {
      int src;
      if (m == M - 1 && chain_events) {
        // closing step: pinned to n-1 (decomp.cpp:197-201). The host waits only until
        // n-1's final work is enqueued; the stream waits on n-1's completion event, so
        // the serial chain of closing steps runs device-side with no host round trip.
        src = n - 1;
        const int gp = g - Sl_;  // store index of frame n-1 of this slice
        if (gp >= run_first_) enq.wait_complete(n - 1);
        a.reg_final_seq = ledger.next_seq();
        if (gp >= run_first_) {
          check_cuda(cudaStreamWaitEvent(s, done_[static_cast<size_t>(gp - run_first_)], 0), "chain wait");
        }
      } else {
        src = h_choose(n, m, M, o.sched, ledger);
        if (m == M - 1) a.reg_final_seq = ledger.next_seq();
      }
      a.reg_src[static_cast<size_t>(m)] = src;
      e.frame_step(m, est_of(src));
      // Sources are chosen when a step is enqueued; h_choose blocks the host thread
      // only when Eq. 10 requires it (empty window, closing step), while this frame's
      // queued steps keep the device busy. step_sync_ re-creates the reference's
      // "choose when the step starts" timing at the cost of one host round trip per step.
      if (step_sync_ && o.T > 1) e.sync();
      ledger.mark_step(n, m);
    }
    e.frame_image(img, iscale, undo);
  }
  check_cuda(cudaEventRecord(ev1, s), "event");
  FrameStats fs;
  if (chain_events) {
    // publish the estimate and its completion event before this thread blocks, so the
    // next frame's closing step can be queued behind it on the device
    e.store_x(estimate_dev(g));
    check_cuda(cudaEventRecord(done_[static_cast<size_t>(g - run_first_)], s), "done event");
    a.finish_seq = ledger.next_seq();
    enq.mark_complete(n);
    if (!e.frame_verify(&fs)) throw RedoSeries{};  // consumers may hold the speculative estimate
  } else if (!e.frame_verify(&fs)) {
    // a step met an exactly-zero right-hand side: redo with the true budget split,
    // replaying the recorded regularisation sources
    e.load_x(init);
    const std::vector<int> srcs = a.reg_src;
    const float2* u = unity_;
    RegFn rf = [this, srcs, u, sl](int m) -> const float2* {
      const int sidx = srcs[static_cast<size_t>(m)];
      return sidx >= 0 ? estimate_dev(sidx * Sl_ + sl) : u;
    };
    e.frame_run_sync(rf, img, iscale, undo, &fs);
    check_cuda(cudaEventRecord(ev1, s), "event");
  }
  if (!chain_events) e.store_x(estimate_dev(g));
  if (!local) {
    check_cuda(cudaMemcpyAsync(images_ + isz_ * g, img, sizeof(float2) * isz_, cudaMemcpyDefault, s), "image");
  }
  e.sync();
  float ms = 0;
  check_cuda(cudaEventElapsedTime(&ms, ev0, ev1), "elapsed");
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  a.reg_final_src = chained ? a.reg_src[static_cast<size_t>(M - 1)] : -1;
  if (!o.plain && !chain_events) a.finish_seq = ledger.next_seq();
  out.audit = a;
  out.cg_iters = fs.cg_iters;
  out.gpu_ms = ms;
  ledger.mark_complete(n);
}

// PsfCache::save / load (preproc.cpp:346-388): "PSFC" v1, G, count, then per entry the
// angle key and the G x G complex64 kernel; the file is interchangeable with the reference's
bool Series::save_psf_cache(const std::string& path) {
  const uint32_t magic = 0x43465350u, version = 1, G = static_cast<uint32_t>(eng0_.plan().G);
  const uint32_t count = static_cast<uint32_t>(psf_keys_.size());
  std::vector<float2> host(psz_);
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) return false;
  bool ok = std::fwrite(&magic, 4, 1, f) == 1 && std::fwrite(&version, 4, 1, f) == 1 &&
            std::fwrite(&G, 4, 1, f) == 1 && std::fwrite(&count, 4, 1, f) == 1;
  check_cuda(cudaSetDevice(eng0_.device()), "set device");
  for (uint32_t e = 0; ok && e < count; ++e) {
    check_cuda(cudaMemcpy(host.data(), psf_ + psz_ * e, sizeof(float2) * psz_, cudaMemcpyDeviceToHost), "psf d2h");
    ok = std::fwrite(&psf_keys_[e], 8, 1, f) == 1 && std::fwrite(host.data(), sizeof(float2), psz_, f) == psz_;
  }
  return std::fclose(f) == 0 && ok;
}

bool Series::load_psf_cache(const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) return false;
  uint32_t magic = 0, version = 0, G = 0, count = 0;
  bool ok = std::fread(&magic, 4, 1, f) == 1 && std::fread(&version, 4, 1, f) == 1 && std::fread(&G, 4, 1, f) == 1 &&
            std::fread(&count, 4, 1, f) == 1 && magic == 0x43465350u && version == 1 &&
            G == static_cast<uint32_t>(eng0_.plan().G);
  std::vector<std::pair<uint64_t, std::vector<float2>>> entries;
  for (uint32_t e = 0; ok && e < count; ++e) {
    uint64_t key = 0;
    std::vector<float2> P(psz_);
    ok = std::fread(&key, 8, 1, f) == 1 && std::fread(P.data(), sizeof(float2), psz_, f) == psz_;
    if (ok) entries.emplace_back(key, std::move(P));
  }
  std::fclose(f);
  if (!ok) return false;
  check_cuda(cudaSetDevice(eng0_.device()), "set device");
  for (auto& [key, P] : entries) {  // insert or replace, like the reference's map
    int slot = -1;
    for (size_t i = 0; i < psf_keys_.size(); ++i) {
      if (psf_keys_[i] == key) slot = static_cast<int>(i);
    }
    if (slot < 0) {
      if (static_cast<int>(psf_keys_.size()) >= n_psf_) fail(2, "load_psf_cache: more kernels than PSF slots");
      slot = static_cast<int>(psf_keys_.size());
      psf_keys_.push_back(key);
    }
    check_cuda(cudaMemcpy(psf_ + psz_ * slot, P.data(), sizeof(float2) * psz_, cudaMemcpyHostToDevice), "psf h2d");
  }
  return true;
}

void Series::post(int first, int count, int mode, float* out) {
  if (first < 0 || count < 1 || first + count > F_) fail(2, "series post: frame range out of bounds");
  if (mode < 0 || mode > 2) fail(2, "series post: unknown mode");
  check_cuda(cudaSetDevice(eng0_.device()), "set device");
  const long long npix = static_cast<long long>(isz_);
  float* buf = nullptr;
  check_cuda(cudaMalloc(&buf, sizeof(float) * npix * count * 2), "post buffer");
  const float2* img = images_ + isz_ * first;
  long long n_out = npix * count;
  float* res = buf;
  if (mode == 2) {
    const int pairs = count / 2;
    for (int k = 0; k < pairs; ++k) {
      post_phase_difference(img + 2 * k * isz_, img + (2 * k + 1) * isz_, npix, buf + k * npix, copy_);
    }
    n_out = npix * pairs;
  } else {
    post_magnitude(img, npix * count, buf, copy_);
    if (mode == 1) {
      post_median3(buf, count, npix, buf + npix * count, copy_);
      res = buf + npix * count;
    }
  }
  const cudaError_t e = cudaMemcpyAsync(out, res, sizeof(float) * n_out, cudaMemcpyDeviceToHost, copy_);
  const cudaError_t e2 = cudaStreamSynchronize(copy_);
  cudaFree(buf);
  check_cuda(e, "post d2h");
  check_cuda(e2, "post sync");
}

Series::PreLane* Series::lane_for(int t) {
  if (t == 0) return nullptr;  // worker 0 is the store's engine
  const int dev = worker(t).device();
  if (dev == eng0_.device() && !force_lanes_) return nullptr;
  if (lanes_.size() <= static_cast<size_t>(t)) lanes_.resize(static_cast<size_t>(t) + 1);
  auto& l = lanes_[static_cast<size_t>(t)];
  if (!l || l->dev != dev) {
    l = std::make_unique<PreLane>();
    l->dev = dev;
    check_cuda(cudaSetDevice(dev), "set device");
    check_cuda(cudaStreamCreateWithFlags(&l->copy, cudaStreamNonBlocking), "lane stream");
    l->pre = std::make_unique<Preproc>(eng0_.plan(), dev);
    check_cuda(cudaMalloc(&l->psf, sizeof(float2) * psz_ * n_psf_), "lane psf");
    check_cuda(cudaMalloc(&l->nsq, sizeof(double)), "lane nsq");
    check_cuda(cudaSetDevice(eng0_.device()), "set device");
  }
  return l.get();
}

void Series::produce_frames(const SeriesOptions& o, int first, int count, const float* z_host,
                            const RawInput* raw, std::vector<cudaEvent_t>& ready) {
  NvtxRange range(raw ? "pre stage (raw acquisitions)" : "frame upload");
  const Plan& p = eng0_.plan();
  const size_t nsamp = raw ? static_cast<size_t>(raw->K) * raw->S : 0;
  const int T = o.plain ? 1 : std::min(o.T, count);
  const int Jp = raw && raw->cmat ? raw->Jp : p.J;
  // where frame k's pre stage runs: the store's copy stream (worker 0 and same-device
  // workers), or the lane of the worker that reconstructs it (k mod T) on its own device
  struct View {
    int dev;
    cudaStream_t s;
    Preproc* pre;
    float2* raw;       // this frame's raw staging
    float2* raw_c;     // compression: matrix, then per-frame compressed samples
    float2* z;         // gridded frame destination
    float2* psf;       // PSF slots
    std::vector<uint64_t>* keys;
    double* nsq;
    PreLane* lane;
  };
  zsrc_.assign(static_cast<size_t>(count), nullptr);
  psrc_.assign(static_cast<size_t>(count), nullptr);
  std::vector<PreLane*> lane_of(static_cast<size_t>(T), nullptr);
  if (raw) {
    if (!raw->samples || !raw->angles || raw->K < 1 || raw->S < 1) fail(2, "reconstruct_series: empty raw input");
    if (raw->cmat && Jp < p.J) fail(2, "reconstruct_series: fewer physical than virtual channels");
    if (!pre_) pre_ = std::make_unique<Preproc>(p, eng0_.device());
    const size_t need = static_cast<size_t>(count) * Jp * nsamp;
    const size_t needc = raw->cmat ? static_cast<size_t>(p.J) * nsamp * count + static_cast<size_t>(p.J) * Jp : 0;
    auto grow = [](float2*& b, size_t& cap, size_t n, const char* what) {
      if (n <= cap) return;
      if (b) cudaFree(b);
      check_cuda(cudaMalloc(&b, sizeof(float2) * n), what);
      cap = n;
    };
    grow(raw_, raw_cap_, need, "raw staging");
    if (raw->cmat) {
      grow(raw_c_, raw_c_cap_, needc, "compression staging");
      check_cuda(cudaMemcpyAsync(raw_c_, raw->cmat, sizeof(float2) * p.J * Jp, cudaMemcpyHostToDevice, copy_),
                 "compression matrix");
    }
    for (int t = 1; t < T; ++t) {
      PreLane* l = lane_for(t);
      lane_of[static_cast<size_t>(t)] = l;
      if (!l) continue;
      check_cuda(cudaSetDevice(l->dev), "set device");
      const size_t nk = static_cast<size_t>((count + T - 1) / T);  // frames of this worker
      grow(l->raw, l->raw_cap, nk * Jp * nsamp, "lane raw staging");
      grow(l->z, l->z_cap, nk * zsz_, "lane frames");
      check_cuda(cudaStreamWaitEvent(l->copy, span0_, 0), "lane span wait");
      if (raw->cmat) {
        grow(l->raw_c, l->raw_c_cap, static_cast<size_t>(p.J) * nsamp * nk + static_cast<size_t>(p.J) * Jp,
             "lane compression staging");
        check_cuda(cudaMemcpyAsync(l->raw_c, raw->cmat, sizeof(float2) * p.J * Jp, cudaMemcpyHostToDevice, l->copy),
                   "compression matrix");
      }
      check_cuda(cudaSetDevice(eng0_.device()), "set device");
    }
  }
  auto view_of = [&](int k) {
    const int n = first + k;
    PreLane* l = raw ? lane_of[static_cast<size_t>(k % T)] : nullptr;
    if (!l) {
      return View{eng0_.device(), copy_, pre_.get(), raw ? raw_ + static_cast<size_t>(k) * Jp * nsamp : nullptr,
                  raw_c_, z_ + zsz_ * n, psf_, &psf_keys_, nsq_, nullptr};
    }
    const size_t slot = static_cast<size_t>(k / T);
    return View{l->dev, l->copy, l->pre.get(), l->raw + slot * Jp * nsamp, l->raw_c, l->z + zsz_ * slot, l->psf,
                &l->keys, l->nsq, l};
  };
  // frame k of the call: H2D, compression, gridding and its PSF on the view's stream
  auto produce = [&](int k, const View& v, const float* post) {
    if (!raw) {
      check_cuda(cudaMemcpyAsync(v.z, z_host + 2 * zsz_ * k, sizeof(float2) * zsz_, cudaMemcpyHostToDevice, v.s),
                 "frame upload");
      return;
    }
    float2* smp = v.raw;
    check_cuda(cudaMemcpyAsync(smp, raw->samples + 2 * static_cast<size_t>(k) * Jp * nsamp,
                               sizeof(float2) * Jp * nsamp, cudaMemcpyHostToDevice, v.s),
               "raw upload");
    if (raw->cmat) {
      const size_t slot = v.lane ? static_cast<size_t>(k / T) : static_cast<size_t>(k);
      float2* cs = v.raw_c + static_cast<size_t>(p.J) * Jp + slot * p.J * nsamp;
      v.pre->apply_compression(v.raw_c, p.J, Jp, smp, static_cast<int>(nsamp), cs, v.s);
      smp = cs;
    }
    const double* ang = raw->angles + static_cast<size_t>(k) * raw->K;
    v.pre->grid_adjoint(smp, p.J, ang, raw->K, raw->S, raw->delay, v.z, v.s, false, post);
    // PsfCache::get (preproc.cpp:315-332): one PSF per distinct angle set (per lane)
    const uint64_t key = psf_angle_key(ang, raw->K, raw->S, p.G);
    std::vector<uint64_t>& keys = *v.keys;
    int slot = -1;
    for (size_t i = 0; i < keys.size(); ++i) {
      if (keys[i] == key) slot = static_cast<int>(i);
    }
    if (slot < 0) {
      if (static_cast<int>(keys.size()) >= n_psf_) {
        fail(2, "reconstruct_series: more distinct spoke-angle sets than PSF slots");
      }
      slot = static_cast<int>(keys.size());
      v.pre->build_psf(ang, raw->K, raw->S, v.psf + psz_ * slot, v.s);
      keys.push_back(key);
    }
    if (v.lane) {
      zsrc_[static_cast<size_t>(k)] = v.z;
      psrc_[static_cast<size_t>(k)] = v.psf + psz_ * slot;
    } else {
      psf_idx_[static_cast<size_t>(first + k)] = slot;
    }
  };
  ready.resize(static_cast<size_t>(count));
  if (first == 0) normalized_ = false;
  for (int k = 0; k < count; ++k) {
    const int g = first + k, sl = g % Sl_;
    const View v = view_of(k);
    check_cuda(cudaSetDevice(v.dev), "set device");
    // a raw frame after its slice's first: the known normalisation is applied inside the
    // gridding's deapodisation pass (the same float multiply, one pass over z fewer)
    const float known = static_cast<float>(slice_scale_[static_cast<size_t>(sl)]);
    const bool fold = raw && o.normalize && g >= Sl_ && slice_scale_[static_cast<size_t>(sl)] != 1.0;
    produce(k, v, fold ? &known : nullptr);
    if (g < Sl_) {
      // frame 0 of slice sl arrived: it sets the slice's scale (pipeline.cpp:429-434)
      double sc = 1.0;
      if (o.normalize) {
        k_nrm2_frame<<<1, 256, 0, v.s>>>(v.z, static_cast<long long>(zsz_), v.nsq);
        double nsq = 0;
        check_cuda(cudaMemcpyAsync(&nsq, v.nsq, sizeof(double), cudaMemcpyDeviceToHost, v.s), "nsq");
        check_cuda(cudaStreamSynchronize(v.s), "nsq");
        sc = nsq > 0 ? 100.0 / std::sqrt(nsq) : 1.0;
      }
      slice_scale_[static_cast<size_t>(sl)] = sc;
      if (sl == 0) scale_ = sc;
    }
    const double sc = slice_scale_[static_cast<size_t>(sl)];
    if (o.normalize && sc != 1.0 && !fold) {
      k_scale_frames<<<148 * 2, 256, 0, v.s>>>(v.z, static_cast<long long>(zsz_), static_cast<float>(sc));
    }
    check_cuda(cudaEventCreateWithFlags(&ready[static_cast<size_t>(k)], cudaEventDisableTiming), "event");
    check_cuda(cudaEventRecord(ready[static_cast<size_t>(k)], v.s), "event");
  }
  check_cuda(cudaSetDevice(eng0_.device()), "set device");
  normalized_ = true;
}

void Series::run(const SeriesOptions& o, int first, int count, const float* z_host, float* images_host,
                 std::vector<SeriesFrameOut>* out, const RawInput* raw) {
  if (z_host && raw) fail(2, "reconstruct_series: gridded and raw input are exclusive");
  if (first < 0 || count < 1 || first + count > F_) fail(2, "reconstruct_series: frame range out of bounds");
  if (o.T < 1) fail(2, "reconstruct_series: thread count out of range");
  if (o.A < 1 || o.A > kGroupSizeMaxDevice) fail(2, "reconstruct_series: workers per thread out of range");
  const int dev = eng0_.device();
  check_cuda(cudaSetDevice(dev), "set device");
  const Plan& p = eng0_.plan();
  if (o.A > p.J) fail(2, "reconstruct_series: more channel-group members than channels");
  if (o.A != A_) {
    groups_.clear();
    A_ = o.A;
  }
  const int T = o.plain ? 1 : std::min(o.T, count);
  for (int t = 1; t < T; ++t) worker(t);
  // one frame at a time: the latency-optimised cluster path; several in flight: the
  // five-kernel passes, whose smaller blocks interleave across frames
  const bool cl = o.cluster < 0 ? T == 1 : o.cluster != 0;
  if (A_ == 1) {
    eng0_.set_cluster(cl);
    for (auto& ex : extra_) ex->set_cluster(cl);
  } else {
    for (int t = 0; t < T; ++t) worker(t).set_cluster(cl);
  }
  check_cuda(cudaEventRecord(span0_, copy_), "span event");
  for (int t = 0; t < T; ++t) check_cuda(cudaStreamWaitEvent(worker(t).stream(), span0_, 0), "span wait");

  // end-to-end path: frames produced on the copy stream (H2D, or raw samples through
  // the device pre stage), normalised on arrival
  std::vector<cudaEvent_t> ready;
  zsrc_.clear();
  psrc_.clear();
  raw_run_ = raw != nullptr;
  if (z_host || raw) {
    produce_frames(o, first, count, z_host, raw, ready);
  } else if (o.normalize) {
    normalize();
  } else if (first == 0) {
    scale_ = 1.0;
    slice_scale_.assign(static_cast<size_t>(Sl_), 1.0);
  }

  // one chain per slice; store indices before `first` are complete
  const int Fs = (F_ + Sl_ - 1) / Sl_;
  ledgers_.clear();
  enqs_.clear();
  for (int sl = 0; sl < Sl_; ++sl) {
    ledgers_.push_back(std::make_unique<CompletionLedger>(Fs));
    enqs_.push_back(std::make_unique<CompletionLedger>(Fs));
  }
  for (int g = 0; g < first; ++g) {
    ledgers_[static_cast<size_t>(g % Sl_)]->mark_complete(g / Sl_);
    enqs_[static_cast<size_t>(g % Sl_)]->mark_complete(g / Sl_);
  }
  auto poison_all = [&] {
    for (auto& l : ledgers_) l->poison();
    for (auto& l : enqs_) l->poison();
  };
  run_first_ = first;
  done_.assign(static_cast<size_t>(count), nullptr);
  for (int k = 0; k < count; ++k) {
    check_cuda(cudaSetDevice(worker(k % T).device()), "set device");
    check_cuda(cudaEventCreateWithFlags(&done_[static_cast<size_t>(k)], cudaEventDisableTiming), "event");
  }
  check_cuda(cudaSetDevice(dev), "set device");
  out->assign(static_cast<size_t>(count), SeriesFrameOut{});
  std::mutex err_mu;
  std::exception_ptr first_err;
  std::atomic<bool> redo{false};
  auto thread_main = [&](int t) {
    try {
      check_cuda(cudaSetDevice(worker(t).device()), "set device");
      for (int k = t; k < count; k += T) {
        if (ledgers_[static_cast<size_t>((first + k) % Sl_)]->poisoned()) return;
        run_frame(t, first + k, o, (*out)[static_cast<size_t>(k)],
                  ready.empty() ? nullptr : ready[static_cast<size_t>(k)]);
        if (images_host) {
          FrameWorker& e = worker(t);
          check_cuda(cudaMemcpyAsync(images_host + 2 * isz_ * k, images_ + isz_ * (first + k), sizeof(float2) * isz_,
                                     cudaMemcpyDeviceToHost, e.stream()),
                     "image d2h");
          e.sync();
        }
      }
    } catch (const RedoSeries&) {
      redo = true;
      poison_all();
    } catch (...) {
      // once a worker asked for the safe-mode re-run, the other workers' failures are
      // the poisoned ledgers' "series aborted" faults: the re-run supersedes them
      if (!redo.load()) {
        std::lock_guard<std::mutex> g(err_mu);
        if (!first_err) first_err = std::current_exception();
      }
      poison_all();
    }
  };
  if (T == 1) {
    thread_main(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(thread_main, t);
    thread_main(0);
    for (auto& th : pool) th.join();
  }
  for (cudaEvent_t ev : ready) cudaEventDestroy(ev);
  for (int t = 0; t < T; ++t) worker(t).sync();
  for (cudaEvent_t ev : done_) cudaEventDestroy(ev);
  done_.clear();
  if (redo && !first_err) {
    // a speculative budget split was wrong (exactly-zero right-hand side) while later
    // frames already consumed the estimate: re-run the range with per-frame
    // verification before publication
    safe_mode_ = true;
    try {
      run(o, first, count, z_host, images_host, out, raw);
    } catch (...) {
      safe_mode_ = false;
      throw;
    }
    safe_mode_ = false;
    return;
  }
  if (first_err) std::rethrow_exception(first_err);
  // every worker stream has been synchronised by now; close the span on the copy
  // stream after all of them
  for (int t = 0; t < T; ++t) {
    cudaEvent_t e;
    check_cuda(cudaSetDevice(worker(t).device()), "set device");
    check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    check_cuda(cudaEventRecord(e, worker(t).stream()), "event");
    check_cuda(cudaSetDevice(dev), "set device");
    check_cuda(cudaStreamWaitEvent(copy_, e, 0), "event wait");
    cudaEventDestroy(e);
  }
  check_cuda(cudaEventRecord(span1_, copy_), "span event");
  check_cuda(cudaEventSynchronize(span1_), "span sync");
  check_cuda(cudaEventElapsedTime(&span_ms_, span0_, span1_), "span elapsed");
  (void)p;
}

}  // namespace rtnb
