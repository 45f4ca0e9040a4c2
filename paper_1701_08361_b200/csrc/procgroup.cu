// Channel decomposition with one process per GPU (procgroup.hpp).
#include "procgroup.hpp"

#include <algorithm>
#include <cstring>
#include <string>

namespace rtnb {

ProcGroup::ProcGroup(const Plan& plan, int device, int rank, int members, int a_cap)
    : plan_(plan), rank_(rank), A_(members) {
  if (A_ < 1 || A_ > kMaxGroup) fail(2, "process group: need 1 to 8 members");
  if (rank_ < 0 || rank_ >= A_) fail(2, "process group: rank out of range");
  if (A_ > plan.J) fail(2, "process group: more members than channels");
  blocks_ = partition_channels(plan.J, A_, a_cap);
  D_ = plan.G * plan.G + plan.J * plan.Gc * plan.Gc;
  Plan lp = plan;
  lp.J = blocks_[static_cast<size_t>(rank_)].second - blocks_[static_cast<size_t>(rank_)].first;
  eng_ = std::make_unique<Engine>(lp, device);
  Engine& e = *eng_;
  check_cuda(cudaSetDevice(device), "set device");
  const size_t G2 = static_cast<size_t>(plan.G) * plan.G;
  check_cuda(cudaMalloc(&e.RPO_, sizeof(double2) * G2), "group rho partials");
  check_cuda(cudaMemset(e.RPO_, 0, sizeof(double2) * G2), "group rho partials");
  check_cuda(cudaMalloc(&e.SS_, sizeof(double) * static_cast<size_t>(plan.N) * plan.N), "group coil sums");
  check_cuda(cudaMalloc(&flags_, sizeof(int) * 2), "group flags");
  check_cuda(cudaMemset(flags_, 0, sizeof(int) * 2), "group flags");
  check_cuda(cudaMalloc(&img_full_, sizeof(float2) * static_cast<size_t>(plan.N) * plan.N), "group image");
  check_cuda(cudaMalloc(&h_stage_, sizeof(float2) * std::max<size_t>(static_cast<size_t>(D_), 1)), "stage");
  alphas_ = e.alphas_;
  caps_ = e.caps_;
  e.set_cluster(false);  // the group path runs the five passes with the member-order sums
}

ProcGroup::~ProcGroup() {
  if (!eng_) return;
  cudaSetDevice(eng_->device());
  cudaStreamSynchronize(eng_->stream());
  for (auto& g : step_graph_) {
    if (g) cudaGraphExecDestroy(g);
  }
  if (frame_graph_) cudaGraphExecDestroy(frame_graph_);
  for (void* p : opened_) cudaIpcCloseMemHandle(p);
  for (void* p : {static_cast<void*>(flags_), static_cast<void*>(img_full_), static_cast<void*>(h_stage_)}) {
    if (p) cudaFree(p);
  }
}

void ProcGroup::export_handles(cudaIpcMemHandle_t* out) const {
  const Engine& e = *eng_;
  const void* bufs[kHandles] = {e.RP_, e.RPO_, e.st_, e.cr_buf_, e.SS_, flags_, e.x_, e.img_};
  check_cuda(cudaSetDevice(e.device()), "set device");
  for (int k = 0; k < kHandles; ++k) {
    check_cuda(cudaIpcGetMemHandle(&out[k], const_cast<void*>(bufs[k])), "ipc export");
  }
}

void ProcGroup::attach(const cudaIpcMemHandle_t* all) {
  if (attached_) fail(2, "process group: already attached");
  Engine& e = *eng_;
  check_cuda(cudaSetDevice(e.device()), "set device");
  GroupView gv{};
  GroupScal gs{};
  gv.A = gs.A = gf_.A = A_;
  peer_x_.assign(static_cast<size_t>(A_), nullptr);
  const int cap = e.cr_cap_;  // same plan on every member: same CR capacity
  for (int m = 0; m < A_; ++m) {
    void* p[kHandles];
    if (m == rank_) {
      const void* loc[kHandles] = {e.RP_, e.RPO_, e.st_, e.cr_buf_, e.SS_, flags_, e.x_, e.img_};
      for (int k = 0; k < kHandles; ++k) p[k] = const_cast<void*>(loc[k]);
    } else {
      for (int k = 0; k < kHandles; ++k) {
        check_cuda(cudaIpcOpenMemHandle(&p[k], all[static_cast<size_t>(m) * kHandles + k],
                                        cudaIpcMemLazyEnablePeerAccess),
                   "ipc open");
        opened_.push_back(p[k]);
      }
    }
    const int Jm = blocks_[static_cast<size_t>(m)].second - blocks_[static_cast<size_t>(m)].first;
    gv.h[m] = (Jm + e.line_batch() - 1) / e.line_batch();
    gv.rp[m] = static_cast<const double2*>(p[0]);
    gv.rpo[m] = static_cast<const double2*>(p[1]);
    gs.st[m] = static_cast<const DevState*>(p[2]);
    gs.pcw[m] = static_cast<const double*>(p[3]) + 5 * cap;
    gs.pcr[m] = static_cast<const double*>(p[3]) + 8 * cap;
    gs.ss[m] = static_cast<const double*>(p[4]);
    gf_.flag[m] = static_cast<const int*>(p[5]);
    peer_x_[static_cast<size_t>(m)] = static_cast<const float2*>(p[6]);
    if (m == 0) img0_ = static_cast<const float2*>(p[7]);
  }
  e.join_group(rank_, gv, gs);
  attached_ = true;
}

void ProcGroup::require_attached() const {
  if (!attached_) fail(2, "process group: attach the peers' handles first");
}

void ProcGroup::barrier() { eng_->enq_pg_barrier(flags_, gf_); }

void ProcGroup::sync() { eng_->sync(); }

void ProcGroup::read_state() { eng_->read_state(); }

// ---- full-layout <-> member-layout copies -----------------------------------------------

void ProcGroup::load_frame(const float2* z, const float2* P, bool masked) {
  Engine& e = *eng_;
  const size_t G2 = static_cast<size_t>(plan_.G) * plan_.G;
  const size_t j0 = static_cast<size_t>(block().first);
  check_cuda(cudaMemcpyAsync(e.z_, z + j0 * G2, sizeof(float2) * G2 * e.plan_.J, cudaMemcpyDefault, e.s_), "z");
  check_cuda(cudaMemcpyAsync(e.P_, P, sizeof(float2) * G2, cudaMemcpyDefault, e.s_), "psf");
  e.enq_z_scan(masked);
}

void ProcGroup::load_x(const float2* src) {
  Engine& e = *eng_;
  const size_t G2 = static_cast<size_t>(plan_.G) * plan_.G, C2 = static_cast<size_t>(plan_.Gc) * plan_.Gc;
  const size_t j0 = static_cast<size_t>(block().first);
  check_cuda(cudaMemcpyAsync(e.x_, src, sizeof(float2) * G2, cudaMemcpyDefault, e.s_), "rho");
  check_cuda(cudaMemcpyAsync(e.x_ + G2, src + G2 + j0 * C2, sizeof(float2) * C2 * e.plan_.J, cudaMemcpyDefault, e.s_),
             "chat");
}

void ProcGroup::load_reg(const float2* src) {
  Engine& e = *eng_;
  const size_t G2 = static_cast<size_t>(plan_.G) * plan_.G, C2 = static_cast<size_t>(plan_.Gc) * plan_.Gc;
  const size_t j0 = static_cast<size_t>(block().first);
  check_cuda(cudaMemcpyAsync(e.reg_, src, sizeof(float2) * G2, cudaMemcpyDefault, e.s_), "rho");
  check_cuda(cudaMemcpyAsync(e.reg_ + G2, src + G2 + j0 * C2, sizeof(float2) * C2 * e.plan_.J, cudaMemcpyDefault,
                             e.s_),
             "chat");
}

// every member's final block, read from the peers (the caller orders this after a
// barrier that follows the peers' last update)
void ProcGroup::store_x(float2* dst) {
  require_attached();
  Engine& e = *eng_;
  const size_t G2 = static_cast<size_t>(plan_.G) * plan_.G, C2 = static_cast<size_t>(plan_.Gc) * plan_.Gc;
  check_cuda(cudaMemcpyAsync(dst, e.x_, sizeof(float2) * G2, cudaMemcpyDefault, e.s_), "rho gather");
  for (int m = 0; m < A_; ++m) {
    const auto b = blocks_[static_cast<size_t>(m)];
    check_cuda(cudaMemcpyAsync(dst + G2 + static_cast<size_t>(b.first) * C2, peer_x_[static_cast<size_t>(m)] + G2,
                               sizeof(float2) * C2 * (b.second - b.first), cudaMemcpyDefault, e.s_),
               "chat gather");
  }
}

// ---- enqueue (the member-order sequence of Group::enq_newton_step) ---------------------

void ProcGroup::enq_newton_step(int m, float tol, int cap, bool sync_each) {
  Engine& e = *eng_;
  const float alpha = alphas_[static_cast<size_t>(m)];
  e.enq_step_begin(m);
  e.enq_setup_front(e.x_);
  barrier();
  e.enq_setup_back(e.x_, e.reg_, alpha);
  barrier();
  e.enq_grp_fin(1, -1, -1, tol);
  bool run_cr = cap >= 1;
  if (run_cr && sync_each) {
    read_state();
    e.raise_status("cg_solve");
    run_cr = !e.st_host_->cr_halt;
  }
  if (run_cr) {
    e.win_only_ok_ = sync_each ? 0 : 1;  // the two-pass kernels read every entry of ar
    for (int it = 0; it < cap; ++it) {
      e.enq_apply_front(e.r_, 1);
      barrier();
      e.enq_apply_back(e.r_, e.ar_, CW_OPALPHA, alpha, it, 1, it > 0 ? e.ap_ : nullptr);
      barrier();
      if (sync_each) {
        // tolerance mode: the exact two-pass recurrence (as the in-process group)
        e.enq_grp_fin(0, it, -1, tol);
        e.enq_cr_two_pass_grp(it == 0 ? 0 : 1, it, tol);
        barrier();
        e.enq_grp_fin(0, -1, it, tol, 1);
        e.enq_cr_two_pass_grp(2, it + 1, tol);
        barrier();
        e.enq_grp_fin(0, -1, it, tol, 2);
        read_state();
        if (e.st_host_->status || e.st_host_->cr_halt) break;
      } else {
        e.enq_cr_fused(it, tol, e.group_red());  // k_grp_fin's sums inside the recurrence
      }
    }
    if (!sync_each) {
      barrier();
      e.enq_grp_fin(0, -1, cap - 1, tol);
    }
    e.win_only_ok_ = 0;
  } else {
    // no CR iteration follows: a lagging member may still be reading this step's setup
    // partials in its k_grp_fin when the next step's setup_front overwrites them
    barrier();
  }
  e.enq_axpy1();
}

void ProcGroup::enq_image(float2* img, float scale, bool apply_scale) {
  Engine& e = *eng_;
  e.enq_decode(e.x_);
  e.enq_coil_ss();
  barrier();
  const size_t nn = static_cast<size_t>(plan_.N) * plan_.N;
  if (rank_ == 0) {
    e.enq_image_grp(e.img_, scale, apply_scale);
    barrier();
    check_cuda(cudaMemcpyAsync(img, e.img_, sizeof(float2) * nn, cudaMemcpyDefault, e.s_), "image");
  } else {
    barrier();  // member 0's image is complete
    check_cuda(cudaMemcpyAsync(img, img0_, sizeof(float2) * nn, cudaMemcpyDefault, e.s_), "image");
  }
}

void ProcGroup::book_frame_ffts(const std::vector<int>& iters) {
  // this member's share of the frame's transforms (its channels)
  uint64_t n = 0;
  for (int c : iters) n += static_cast<uint64_t>(c);
  const uint64_t J = static_cast<uint64_t>(eng_->plan_.J);
  fft_book(CTX_SETUP, 4ull * J * iters.size() + J);
  fft_book(CTX_NORMAL_OP, 4ull * J * n);
}

void ProcGroup::frame_begin() {
  require_attached();
  eng_->enq_state_reset();
}

void ProcGroup::frame_step(int m, const float2* reg_src) {
  require_attached();
  if (reg_src) load_reg(reg_src);
  if (!budget_mode()) {
    enq_newton_step(m, plan_.cg_tol, plan_.cg_max_iter, true);
    return;
  }
  Engine& e = *eng_;
  const int cap = caps_[static_cast<size_t>(m)];
  if (!step_graph_[m]) {
    cudaGraph_t g = nullptr;
    check_cuda(cudaStreamBeginCapture(e.s_, cudaStreamCaptureModeThreadLocal), "capture begin");
    enq_newton_step(m, 0.0f, cap, false);
    check_cuda(cudaStreamEndCapture(e.s_, &g), "capture end");
    check_cuda(cudaGraphInstantiate(&step_graph_[m], g, 0), "graph instantiate");
    cudaGraphDestroy(g);
  }
  check_cuda(cudaGraphLaunch(step_graph_[m], e.s_), "graph launch");
}

void ProcGroup::frame_image(float2* img_dst, float image_scale, bool apply_scale) {
  require_attached();
  Engine& e = *eng_;
  enq_image(img_full_, image_scale, apply_scale);
  if (img_dst && img_dst != img_full_) {
    check_cuda(cudaMemcpyAsync(img_dst, img_full_, sizeof(float2) * plan_.N * plan_.N, cudaMemcpyDefault, e.s_),
               "image");
  }
  check_cuda(cudaMemcpyAsync(e.st_host_, e.st_, sizeof(DevState), cudaMemcpyDeviceToHost, e.s_), "state read");
}

void ProcGroup::frame_all(float2* img_dst, float image_scale, bool apply_scale) {
  require_attached();
  if (!budget_mode()) fail(2, "frame_all: whole-frame graphs need the CG iteration budget mode");
  Engine& e = *eng_;
  if (frame_graph_ && (frame_graph_scale_ != image_scale || frame_graph_apply_ != apply_scale)) {
    cudaGraphExecDestroy(frame_graph_);
    frame_graph_ = nullptr;
  }
  if (!frame_graph_) {
    cudaGraph_t g = nullptr;
    check_cuda(cudaStreamBeginCapture(e.s_, cudaStreamCaptureModeThreadLocal), "capture begin");
    e.enq_state_reset();
    for (int m = 0; m < plan_.newton_steps; ++m) enq_newton_step(m, 0.0f, caps_[static_cast<size_t>(m)], false);
    enq_image(img_full_, image_scale, apply_scale);
    check_cuda(cudaMemcpyAsync(e.st_host_, e.st_, sizeof(DevState), cudaMemcpyDeviceToHost, e.s_), "state read");
    check_cuda(cudaStreamEndCapture(e.s_, &g), "capture end");
    check_cuda(cudaGraphInstantiate(&frame_graph_, g, 0), "graph instantiate");
    cudaGraphDestroy(g);
    frame_graph_scale_ = image_scale;
    frame_graph_apply_ = apply_scale;
  }
  check_cuda(cudaGraphLaunch(frame_graph_, e.s_), "graph launch");
  if (img_dst && img_dst != img_full_) {
    check_cuda(cudaMemcpyAsync(img_dst, img_full_, sizeof(float2) * plan_.N * plan_.N, cudaMemcpyDefault, e.s_),
               "image");
  }
}

bool ProcGroup::frame_verify(FrameStats* stats) {
  Engine& e = *eng_;
  sync();
  e.raise_status("reconstruct_frame");
  const DevState& st = *e.st_host_;
  const int M = plan_.newton_steps;
  std::vector<int> got(static_cast<size_t>(M));
  bool ok = true;
  for (int m = 0; m < M; ++m) {
    got[static_cast<size_t>(m)] = st.steps[m].iters;
    if (budget_mode() && (st.steps[m].iters != caps_[static_cast<size_t>(m)] || st.steps[m].zero_rhs)) ok = false;
  }
  if (ok) {
    book_frame_ffts(got);
    if (stats) {
      stats->cg_per_step = got;
      stats->cg_iters = 0;
      for (int c : got) stats->cg_iters += c;
    }
  }
  return ok;
}

void ProcGroup::frame_run_sync(const RegFn& reg, float2* img_dst, float image_scale, bool apply_scale,
                               FrameStats* stats) {
  require_attached();
  Engine& e = *eng_;
  const int M = plan_.newton_steps;
  frame_begin();
  int remaining = plan_.cg_iter_budget;
  std::vector<int> per;
  for (int m = 0; m < M; ++m) {
    int cap = plan_.cg_max_iter;
    float tol = plan_.cg_tol;
    if (budget_mode()) {
      const int left = M - m;
      cap = (remaining + left - 1) / left;
      tol = 0.0f;
    }
    const float2* src = reg ? reg(m) : nullptr;
    if (src) load_reg(src);
    enq_newton_step(m, tol, cap, true);
    read_state();
    e.raise_status("reconstruct_frame");
    const int it = e.st_host_->steps[m].iters;
    per.push_back(it);
    if (budget_mode()) remaining -= it;
  }
  frame_image(img_dst, image_scale, apply_scale);
  read_state();
  e.raise_status("reconstruct_frame");
  book_frame_ffts(per);
  if (stats) {
    stats->cg_per_step = per;
    stats->cg_iters = 0;
    for (int c : per) stats->cg_iters += c;
  }
}

// ---- host in / host out --------------------------------------------------------------------

void ProcGroup::set_psf(const float* P) {
  Engine& e = *eng_;
  check_cuda(cudaSetDevice(e.device()), "set device");
  check_cuda(cudaMemcpy(e.P_, P, sizeof(float2) * plan_.G * plan_.G, cudaMemcpyHostToDevice), "psf upload");
}

void ProcGroup::set_data(const float* z) {
  Engine& e = *eng_;
  const size_t G2 = static_cast<size_t>(plan_.G) * plan_.G;
  const size_t j0 = static_cast<size_t>(block().first);
  check_cuda(cudaSetDevice(e.device()), "set device");
  check_cuda(cudaMemcpy(e.z_, z + 2 * j0 * G2, sizeof(float2) * G2 * e.plan_.J, cudaMemcpyHostToDevice),
             "data upload");
  e.enq_z_scan();
  e.sync();
}

void ProcGroup::reconstruct_frame(const float* init, const float* reg, float* image, float* est_out,
                                  FrameStats* stats) {
  require_attached();
  Engine& e = *eng_;
  check_cuda(cudaSetDevice(e.device()), "set device");
  auto stage_in = [&](const float* h, bool to_reg) {
    check_cuda(cudaMemcpyAsync(h_stage_, h, sizeof(float2) * D_, cudaMemcpyHostToDevice, e.s_), "h2d");
    if (to_reg) {
      load_reg(h_stage_);
    } else {
      load_x(h_stage_);
    }
  };
  stage_in(init, false);
  stage_in(reg ? reg : init, true);
  bool ok = false;
  if (budget_mode()) {
    frame_all(nullptr, 1.0f, false);
    ok = frame_verify(stats);
  }
  if (!ok) {
    stage_in(init, false);
    frame_run_sync(nullptr, nullptr, 1.0f, false, stats);
  }
  check_cuda(cudaMemcpyAsync(image, img_full_, sizeof(float2) * plan_.N * plan_.N, cudaMemcpyDeviceToHost, e.s_),
             "d2h");
  if (est_out) {
    store_x(h_stage_);
    check_cuda(cudaMemcpyAsync(est_out, h_stage_, sizeof(float2) * D_, cudaMemcpyDeviceToHost, e.s_), "d2h");
  }
  // no member reloads its estimate before every member has read the blocks
  barrier();
  sync();
}

}  // namespace rtnb
