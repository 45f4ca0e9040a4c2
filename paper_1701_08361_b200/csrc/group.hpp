// Channel decomposition across a device group (the reference's
// WorkerGroup + partition_channels + all_reduce_sum, decomp.cpp:10-39, 103-134, used
// by apply_normal / newton_step / reconstruct_frame, nlinv.cpp:152-335).
//
// A Group owns A member Engines, one per device of its list (members may share a
// device: that is how a single GPU exercises the multi-device path). Member d owns
// the contiguous channel block partition_channels(J, A)[d] and replicates rho, the
// PSF and the weights; its Estimate is rho followed by its own chat_j. Every
// operator application runs the member's front half (W^-1 column pass .. k_rows2:
// the member's window channel-sum partials), an all-member barrier, the back half
// (k_colsW: the rho sum over every member's partials read from peer memory, in
// member order, fused with the W^-H column pass and the CR update), a second
// barrier, and k_grp_fin, which forms the group totals of the CR scalars in member
// order. Every member computes bit-identical totals and takes identical decisions;
// there is no host round trip and no separate collective kernel. Barriers are
// device-side epoch flags (k_pg_barrier: release/acquire over NVLink) when every member
// has its own GPU, CUDA events (stream edges) when members share one; either way a
// frame is captured into one multi-device graph in budget mode.
#pragma once

#include <memory>
#include <utility>
#include <vector>

#include "engine.hpp"
#include "sched.hpp"

namespace rtnb {

class Group : public FrameWorker {
 public:
  Group(const Plan& plan, const std::vector<int>& devices, int a_cap = kGroupSizeMaxDevice);
  ~Group() override;
  Group(const Group&) = delete;
  Group& operator=(const Group&) = delete;

  const Plan& plan() const override { return plan_; }
  int D() const override { return D_; }
  int device() const override { return mem_[0]->device(); }
  cudaStream_t stream() const override { return mem_[0]->stream(); }
  int width() const override { return A_; }
  bool budget_mode() const override { return plan_.cg_iter_budget > 0; }
  const std::vector<std::pair<int, int>>& blocks() const { return blocks_; }
  Engine& member(int d) { return *mem_[static_cast<size_t>(d)]; }

  // FrameWorker (full-layout device sources / destinations)
  void load_frame(const float2* z, const float2* P, bool masked = false) override;
  void load_x(const float2* src) override;
  void load_reg(const float2* src) override;
  void store_x(float2* dst) override;
  float2* image_dev() override { return mem_[0]->image_dev(); }
  void frame_begin() override;
  void frame_step(int m, const float2* reg_src) override;
  void frame_image(float2* img_dst, float image_scale, bool apply_scale) override;
  void frame_all(float2* img_dst, float image_scale, bool apply_scale) override;
  bool frame_verify(FrameStats* stats) override;
  void frame_run_sync(const RegFn& reg, float2* img_dst, float image_scale, bool apply_scale,
                      FrameStats* stats) override;
  void sync() override;
  // members run the cluster-fused applications (one cluster per own channel), then
  // k_rho_sum over every member's channel terms after an all-member barrier
  void set_cluster(bool on) override;
  void set_use_graphs(bool on) { use_graphs_ = on; }

  // host in / host out (parity boundary)
  void set_psf(const float* P);
  void set_weights(const float* w);  // every member (nlinv.hpp `winv`)
  void set_data(const float* z);
  void make_step_cache(const float* x);
  void apply_normal(const float* dx, float* out);
  void reconstruct_frame(const float* init, const float* reg, float* image, float* est_out, FrameStats* stats);
  void reconstruct_frame_regs(const float* init, const RegHostFn& reg, float* image, float* est_out,
                              FrameStats* stats);

 private:
  template <class F>
  void each(F&& f);
  void fork();     // members wait for the leader stream
  void join();     // leader stream waits for every member
  void barrier();  // every member waits for every other member
  void enq_newton_step(int m, float tol, int cap, bool sync_each);
  void enq_image(float2* img, float scale, bool apply_scale);
  void read_state();
  void raise_status(const char* where);
  void book_frame_ffts(const std::vector<int>& iters);
  void split_copy(const float2* src, bool reg);

  Plan plan_;
  int A_ = 1;
  int D_ = 0;
  std::vector<std::pair<int, int>> blocks_;
  std::vector<std::unique_ptr<Engine>> mem_;
  std::vector<cudaEvent_t> ev_;      // per member, created on its device
  std::vector<int*> flags_;          // per member: [0] published epoch, [1] local epoch counter
  GroupFlags gf_{};
  bool flag_barrier_ = false;        // device-side epoch barriers (k_pg_barrier) instead of graph edges
  cudaEvent_t ev_fork_ = nullptr;    // on the leader's device
  std::vector<float> alphas_;
  std::vector<int> caps_;
  float2* h_stage_ = nullptr;        // device staging for host in/out (leader device)
  bool use_graphs_ = true;
  cudaGraphExec_t step_graph_[kMaxSteps] = {};
  cudaGraphExec_t frame_graph_ = nullptr;
  float2* frame_graph_img_ = nullptr;
  float frame_graph_scale_ = 0.f;
  bool frame_graph_apply_ = false;
};

// all_reduce_sum (decomp.cpp:26-39) of n_terms device images of n elements: FP64 sums
// in term order, one cast to float; bit-identical to the reference for any partition
void all_reduce_sum_device(const float2* terms, int n_terms, long long n, float2* out, cudaStream_t s);

}  // namespace rtnb
