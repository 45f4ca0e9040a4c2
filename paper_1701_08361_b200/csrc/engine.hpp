// Host-side engine: one device context per (GPU, stream) that owns every device
// buffer of a plan and enqueues the fused kernels of kernels_impl.cuh. The C-ABI
// (capi.cpp) and the C++ drop-in over it (compat/rtnlinv_compat.cpp) are thin layers.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "kernels.cuh"

namespace rtnb {

// Mirrors rtnlinv::ReconPlan (planner.hpp:21-35).
struct Plan {
  int N = 0;
  int G = 0;
  int Gc = 0;
  int J = 1;
  int newton_steps = 6;
  float alpha0 = 1.0f;
  float alpha_q = 0.5f;
  float alpha_min = 1e-6f;
  float cg_tol = 1e-3f;
  int cg_max_iter = 200;
  int cg_iter_budget = 0;
  float prev_damping = 1.0f;
  double gamma = 1.5;
};

// Typed failure carrying the reference's exit-code mapping (types.hpp:12-25,
// rtnlinv_main.cpp:381-391): 2 usage, 3 data, 4 solver / decomposition fault.
struct Error : std::runtime_error {
  int code;
  bool decomp;  // a decomposition fault (DecompFault, decomp.hpp:25-66), reported with code 4
  Error(int c, const std::string& m, bool d = false) : std::runtime_error(m), code(c), decomp(d) {}
};
[[noreturn]] void fail(int code, const std::string& msg);
// DecompFault: a worker missed its deadline or the series ledger was poisoned (status 4)
[[noreturn]] void fail_decomp(const std::string& msg);
void check_cuda(cudaError_t e, const char* what);

bool grid_supported(int G);

// Logical transform accounting (fft.hpp:10-38): a 2D transform is booked against
// the calling thread's context, whatever kernels implement it.
enum FftCtx : int { CTX_OTHER = 0, CTX_NORMAL_OP = 1, CTX_SETUP = 2, CTX_BENCH = 3 };
int fft_current_ctx();
void fft_set_ctx(int c);
void fft_book(int ctx, uint64_t n);
uint64_t fft_count(int ctx);
uint64_t fft_count_total();
void fft_reset_counts();

// centered unitary 2D transform of `batch` n x n images resident on the device
void fft2_device(float2* data, int n, int batch, int sign, cudaStream_t s);

struct FrameStats {
  std::vector<int> cg_per_step;
  int cg_iters = 0;
  double seconds = 0;
};

using RegFn = std::function<const float2*(int m)>;  // device pointer of reg(m), or nullptr = keep reg
// host-side RegProvider (nlinv.hpp:102): host pointer to the regularisation target of
// Newton step m (D complex64), or nullptr = keep the previous step's target
using RegHostFn = std::function<const float*(int m)>;

// What a series driver needs from one frame worker: a single-device Engine, or a
// channel-decomposed device Group (group.hpp). Estimates, frames and PSFs are in
// the full layout (rho then chat_0..chat_{J-1}) wherever they come from; a group
// splits them across its members. Every enqueue is ordered on stream().
class FrameWorker {
 public:
  virtual ~FrameWorker() = default;
  virtual const Plan& plan() const = 0;
  virtual int D() const = 0;
  virtual int device() const = 0;
  virtual cudaStream_t stream() const = 0;
  virtual int width() const { return 1; }  // channel-decomposition width A
  virtual bool budget_mode() const = 0;
  // masked: the data is window-masked by construction (the device pre stage), so the
  // outside-window scan is skipped (st->z_out = 0)
  virtual void load_frame(const float2* z, const float2* P, bool masked = false) = 0;
  virtual void load_x(const float2* src) = 0;
  virtual void load_reg(const float2* src) = 0;
  virtual void store_x(float2* dst) = 0;
  virtual float2* image_dev() = 0;
  virtual void frame_begin() = 0;
  virtual void frame_step(int m, const float2* reg_src) = 0;
  virtual void frame_image(float2* img_dst, float image_scale, bool apply_scale) = 0;
  virtual void frame_all(float2* img_dst, float image_scale, bool apply_scale) = 0;
  virtual bool frame_verify(FrameStats* stats) = 0;
  virtual void frame_run_sync(const RegFn& reg, float2* img_dst, float image_scale, bool apply_scale,
                              FrameStats* stats) = 0;
  virtual void sync() = 0;
  // cluster-fused applications for the CR solve (latency mode), where supported
  virtual void set_cluster(bool on) = 0;
};

class Group;
struct ColsWArgs;  // kernels_impl.cuh

class Engine : public FrameWorker {
 public:
  Engine(const Plan& plan, int device = 0);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  const Plan& plan() const override { return plan_; }
  int D() const override { return D_; }  // complex entries of one Estimate: G*G + J*Gc*Gc
  cudaStream_t stream() const override { return s_; }
  int device() const override { return dev_; }

  // ---- inputs (host, complex64 interleaved) ----
  void set_psf(const float* P);    // G*G
  void set_data(const float* z);   // J*G*G
  void set_psf_device(const float2* P);
  void set_data_device(const float2* z);
  const float* winv_host() const { return winv_host_.data(); }
  // caller-supplied W^-1 weights (Gc*Gc real; the `winv` argument of apply_W_inv /
  // make_step_cache / newton_step / reconstruct_frame, nlinv.hpp:41-116)
  void set_weights(const float* w);
  // a linearisation point given as its decoded parts (StepCache::rho masked, G*G, and
  // StepCache::coils, J*G*G; nlinv.hpp:53-60) instead of an estimate to decode
  void set_step_cache(const float* rho, const float* coils);

  // ---- op-level, synchronous, host in / host out (nlinv.hpp:41-98) ----
  void apply_W_inv(const float* chat, float* out);
  void apply_W_invH(const float* u, float* out);
  void toeplitz_apply(float* x);
  void make_step_cache(const float* x, float* rho_out, float* coils_out);  // sets the linearisation point
  void apply_normal(const float* dx, float* out);                          // at that point
  void cg_solve(const float* rhs, float alpha, float tol, int max_iter, float* x_out, int* iters,
                std::vector<double>* residuals);
  void newton_step(float* x, const float* reg, float alpha, float tol, int cap, int* iters,
                   double* residual0);
  // reg == nullptr: every step regularises towards init (nlinv.cpp:425-429)
  void reconstruct_frame(const float* init, const float* reg, float* image, float* est_out,
                         FrameStats* stats);
  // per-step regularisation targets from a RegProvider (step-by-step path; the target of
  // step 0 defaults to init)
  void reconstruct_frame_regs(const float* init, const RegHostFn& reg, float* image, float* est_out,
                              FrameStats* stats);

  // ---- device-resident frame pipeline ----
  // A frame runs on the engine's own buffers: x (estimate; holds init on entry and
  // the final estimate on exit), reg (regularisation target), z / P (frame data).
  // Budget mode (plan.cg_iter_budget > 0) is enqueued speculatively from CUDA
  // graphs captured once per engine: every step runs its budget cap
  // ceil(remaining / steps_left) (nlinv.cpp:301-306), which is exact unless a step
  // meets an exactly-zero right-hand side; frame_verify() detects that and the
  // caller re-runs the frame with frame_run_sync(). Tolerance mode synchronises per
  // CR iteration and never uses graphs.
  using RegFn = rtnb::RegFn;
  void frame_begin() override;
  void frame_step(int m, const float2* reg_src) override;  // enqueue Newton step m
  void frame_image(float2* img_dst, float image_scale, bool apply_scale) override;
  void frame_all(float2* img_dst, float image_scale, bool apply_scale) override;  // budget mode: one graph
  bool frame_verify(FrameStats* stats) override;           // sync + check the speculative split
  void frame_run_sync(const RegFn& reg, float2* img_dst, float image_scale, bool apply_scale,
                      FrameStats* stats) override;
  bool budget_mode() const override { return plan_.cg_iter_budget > 0; }
  void load_frame(const float2* z, const float2* P, bool masked = false) override;
  void load_x(const float2* src) override;
  void load_reg(const float2* src) override;
  void store_x(float2* dst) override;
  float2* image_dev() override { return img_; }
  const std::vector<int>& budget_caps() const { return caps_; }
  void set_use_graphs(bool on) { use_graphs_ = on; }
  // latency mode: every non-setup application as one thread-block cluster per channel
  // (kernels_cluster.cuh) where the geometry supports it; throughput mode (several
  // frames in flight): the five-kernel passes, which share the SMs better
  void set_cluster(bool on) override;
  bool cluster_supported() const { return RC_ != nullptr; }
  bool fused_crA() const;  // budget-mode CR solves use k_crA on the five-kernel path
  int line_batch() const;  // lines per block of the row passes (channel-group size of k_rows2)

  float2* x_dev() { return x_; }
  float2* reg_dev() { return reg_; }
  float2* z_dev() { return z_; }
  float2* psf_dev() { return P_; }
  DevState* state_dev() { return st_; }
  const DevState& state_host() const { return *st_host_; }
  void read_state();
  void sync() override;

  // isolated timing of one kernel class (bench roofline): average ms per launch of
  // `reps` back-to-back launches on the engine stream, CUDA events
  double time_kernel(const char* which, int reps);
  // algorithmic bytes one launch of that kernel moves
  double kernel_bytes(const char* which) const;

 public:
  struct Ops;  // per-grid-size kernel launchers (engine.cu)

 private:
  friend class Group;
  friend class ProcGroup;
  void alloc();
  void ensure_cr_capacity(int max_iter);
  void enq_step_begin(int m);
  // full: every coil entry (make_step_cache); else the window only when the frame's data is
  // window-masked (st->z_out == 0, decided on the device)
  // setup: also the Newton setup's first row pass (e = rho c_j -> V) on the window rows
  void enq_decode(const float2* est, bool full = false, bool setup = false);
  void enq_apply(const float2* dx, float2* out, int cw_mode, float alpha, int dot_slot, int use_halt,
                 const float2* ap_prev = nullptr);
  // the two halves of an application / a Newton-step setup: everything up to the
  // channel-sum partials (front), and the W^-H column pass + rho sum (back). A
  // channel group puts its all-member barrier between them.
  // skip_colA: U already holds dx's W^-1 column pass (k_crA wrote it)
  void enq_apply_front(const float2* dx, int use_halt, bool skip_colA = false);
  void enq_apply_back(const float2* dx, float2* out, int cw_mode, float alpha, int dot_slot, int use_halt,
                      const float2* ap_prev);
  // the cluster-fused application's halves (use_cluster_): clusters, then k_rho_sum
  ColsWArgs cluster_args(const float2* dx, float2* out, int cw_mode, float alpha, int dot_slot,
                         const float2* ap_prev) const;
  void enq_cluster_front(const float2* dx, float2* out, int cw_mode, float alpha, int dot_slot, int use_halt,
                         const float2* ap_prev);
  void enq_rho_sum(const float2* dx, float2* out, int cw_mode, float alpha, int dot_slot, int use_halt,
                   const float2* ap_prev);
  void enq_setup_front(const float2* x);
  void enq_setup_back(const float2* x, const float2* reg, float alpha);
  void enq_setup(const float2* x, const float2* reg, float alpha);
  // group-member kernels (group.cu)
  void join_group(int rank, const GroupView& gv, const GroupScal& gs);
  void enq_grp_fin(int setup, int op_slot, int cr_slot, float tol, int part = 0);
  // kind 0: k_cr_prime, 1: k_cr_pap(it), 2: k_cr_xr(it), with member partials
  void enq_cr_two_pass_grp(int kind, int it, float tol);
  void enq_cr_fused(int it, float tol, const DeferRed& dr = DeferRed{});
  void enq_crA(int it, float tol, const DeferRed& dr);
  int crA_grid() const;
  // a group member's recurrence forming the member-order totals itself (DeferRed::grp)
  DeferRed group_red() const {
    DeferRed d{};
    d.grp = 1;
    d.gs = gs_;
    return d;
  }
  // blocks of this member's back half (k_rho_sum on the cluster path, else k_colsW)
  int back_grid() const;
  void enq_axpy1();
  void enq_state_reset();
  void enq_z_scan(bool masked = false);  // st->z_out for the data now in z_ (stream ordered)
  void enq_coil_ss();
  void enq_image_grp(float2* img, float scale, bool apply_scale);
  void enq_pg_barrier(int* own_flags, const GroupFlags& f);
  void enq_cr(float alpha, float tol, int cap, bool sync_each);
  void enq_newton_step(int m, float2* x, const float2* reg, float alpha, float tol, int cap,
                       bool sync_each);
  void enq_image(const float2* est, float2* img, float scale, bool apply_scale);
  void raise_status(const char* where);
  void book_frame_ffts(const std::vector<int>& iters);

  Plan plan_;
  Dims dims_{};
  int dev_ = 0;
  int D_ = 0;
  cudaStream_t s_ = nullptr;
  const Ops* ops_ = nullptr;
  int vec_grid_ = 0;
  int nbr_ = 0;

  std::vector<float> winv_host_;
  float* winv_ = nullptr;
  float4* twG_ = nullptr;  // packed twiddles (twiddles_for)
  float2* P_ = nullptr;
  float2* z_ = nullptr;
  float2* x_ = nullptr;
  float2* xcg_ = nullptr;
  float2* r_ = nullptr;
  float2* p_ = nullptr;
  float2* ap_ = nullptr;
  float2* ar_ = nullptr;
  float2* est_scratch_[3] = {nullptr, nullptr, nullptr};
  float2* reg_ = nullptr;
  float2* coils_ = nullptr;
  float2* rhom_ = nullptr;
  float2* U_ = nullptr;
  float2* V_ = nullptr;
  float2* Y_ = nullptr;
  double2* RP_ = nullptr;
  float2* gbuf_ = nullptr;
  float2* img_ = nullptr;
  double* partials_ = nullptr;
  CUtensorMap tmP_{};  // TMA descriptor of P_ for k_colsT's P tiles
  // deferred reductions of the budget-mode CR solve (DeferRed): k_colsW's partials (3 per
  // block) and the recurrences' (2 per block, by iteration parity)
  double* dpart_w_ = nullptr;
  double* dpart_c_[2] = {nullptr, nullptr};
  double* defer_w_ = nullptr;  // set while enqueueing: k_colsW writes deferred partials here
  bool defer_red_ = true;      // RTN_DEFER_RED=0: the grid reductions with last-block tails
  DevState* st_ = nullptr;
  DevState* st_host_ = nullptr;  // pinned mirror
  double* cr_buf_ = nullptr;
  int cr_cap_ = 0;
  CrScalars cr_{};
  // group membership (channel decomposition); grp_rank_ < 0: stand-alone
  int grp_rank_ = -1;
  GroupView gv_{};
  GroupScal gs_{};
  double2* RPO_ = nullptr;
  double* SS_ = nullptr;
  // cluster-fused applications (kernels_cluster.cuh): channel terms rc_j and per-CTA dots
  bool use_cluster_ = false;  // current mode (set_cluster); RC_ != nullptr: supported
  float2* RC_ = nullptr;
  double* kpart_ = nullptr;
  int rho_grid_ = 0;
  bool have_cache_ = false;
  std::vector<int> caps_;       // budget-mode per-step caps
  std::vector<float> alphas_;   // per-step alpha schedule
  bool use_graphs_ = true;
  bool fused_cr_ = true;   // RTN_FUSED_CR=0 selects the two-kernel recurrence in graphs too
  bool fused_crA_ = true;  // RTN_CRA=0: k_cr_fused + k_colA instead of k_crA on the pass path
  int win_only_ok_ = 0;    // the applications being enqueued belong to a fused CR solve
  cudaGraphExec_t step_graph_[kMaxSteps] = {};
  cudaGraphExec_t frame_graph_ = nullptr;
  float2* frame_graph_img_ = nullptr;
  float frame_graph_scale_ = 0.f;
  bool frame_graph_apply_ = false;
};

}  // namespace rtnb
