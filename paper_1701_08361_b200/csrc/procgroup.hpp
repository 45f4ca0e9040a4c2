// Channel decomposition with one process per GPU (torchrun layout).
//
// The same member-order arithmetic as the in-process Group (group.hpp), with each
// process owning exactly one member: member `rank` of A owns the channel block
// partition_channels(J, A)[rank]. The members' cross-channel partials (window channel
// sums, out-of-window setup sums, CR scalar partials, coil magnitude sums), their
// estimate blocks and the group image are exported as CUDA IPC handles; every member
// maps its peers' buffers and k_colsW / k_grp_fin / k_image_grp read them directly
// (NVLink / NVSwitch loads between GPUs; plain loads when peers share a GPU). The
// all-member barriers between the halves of an application are device-side epoch
// flags (k_pg_barrier: release store of the member's epoch, acquire polling of the
// peers'), so a frame stays one CUDA graph per process with no host round trip and
// no collective library on the data path. Handle exchange is the caller's plumbing
// (torch.distributed in the Python binding).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <utility>
#include <vector>

#include "engine.hpp"
#include "sched.hpp"

namespace rtnb {

class ProcGroup : public FrameWorker {
 public:
  static constexpr int kHandles = 8;  // RP, RPO, state, CR scalars, coil sums, flags, x, image

  ProcGroup(const Plan& plan, int device, int rank, int members, int a_cap = kGroupSizeMaxDevice);
  ~ProcGroup() override;
  ProcGroup(const ProcGroup&) = delete;
  ProcGroup& operator=(const ProcGroup&) = delete;

  // this member's IPC handles (kHandles x cudaIpcMemHandle_t)
  void export_handles(cudaIpcMemHandle_t* out) const;
  // every member's handles in rank order (members x kHandles); maps the peers
  void attach(const cudaIpcMemHandle_t* all);
  int rank() const { return rank_; }
  int members() const { return A_; }
  std::pair<int, int> block() const { return blocks_[static_cast<size_t>(rank_)]; }

  const Plan& plan() const override { return plan_; }
  int D() const override { return D_; }
  int device() const override { return eng_->device(); }
  cudaStream_t stream() const override { return eng_->stream(); }
  int width() const override { return A_; }
  bool budget_mode() const override { return plan_.cg_iter_budget > 0; }
  void load_frame(const float2* z, const float2* P, bool masked = false) override;
  void load_x(const float2* src) override;
  void load_reg(const float2* src) override;
  void store_x(float2* dst) override;
  float2* image_dev() override { return img_full_; }
  void frame_begin() override;
  void frame_step(int m, const float2* reg_src) override;
  void frame_image(float2* img_dst, float image_scale, bool apply_scale) override;
  void frame_all(float2* img_dst, float image_scale, bool apply_scale) override;
  bool frame_verify(FrameStats* stats) override;
  void frame_run_sync(const RegFn& reg, float2* img_dst, float image_scale, bool apply_scale,
                      FrameStats* stats) override;
  void sync() override;
  void set_cluster(bool) override {}  // the IPC members run the five passes

  // host in / host out: full-layout buffers on every member (each uses its block)
  void set_psf(const float* P);
  void set_data(const float* z);
  void reconstruct_frame(const float* init, const float* reg, float* image, float* est_out, FrameStats* stats);

 private:
  void barrier();
  void enq_newton_step(int m, float tol, int cap, bool sync_each);
  void enq_image(float2* img, float scale, bool apply_scale);
  void read_state();
  void book_frame_ffts(const std::vector<int>& iters);
  void require_attached() const;

  Plan plan_;
  int rank_ = 0, A_ = 1, D_ = 0;
  std::vector<std::pair<int, int>> blocks_;
  std::unique_ptr<Engine> eng_;
  int* flags_ = nullptr;                      // [0] published epoch, [1] local epoch counter
  float2* img_full_ = nullptr;                 // this member's copy of the group image
  std::vector<void*> opened_;                  // peer mappings to close
  GroupFlags gf_{};
  std::vector<const float2*> peer_x_;          // every member's estimate (rho + its block)
  const float2* img0_ = nullptr;               // member 0's image
  bool attached_ = false;
  std::vector<float> alphas_;
  std::vector<int> caps_;
  float2* h_stage_ = nullptr;
  cudaGraphExec_t step_graph_[kMaxSteps] = {};
  cudaGraphExec_t frame_graph_ = nullptr;
  float frame_graph_scale_ = 0.f;
  bool frame_graph_apply_ = false;
};

}  // namespace rtnb
