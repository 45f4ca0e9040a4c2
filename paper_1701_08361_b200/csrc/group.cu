// Channel decomposition across a device group (group.hpp).
#include "group.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

namespace rtnb {

namespace {
struct DeviceRestore {
  int dev = 0;
  DeviceRestore() { cudaGetDevice(&dev); }
  ~DeviceRestore() { cudaSetDevice(dev); }
};
}  // namespace

Group::Group(const Plan& plan, const std::vector<int>& devices, int a_cap) : plan_(plan) {
  A_ = static_cast<int>(devices.size());
  if (A_ < 1 || A_ > kMaxGroup) fail(2, "channel group: need 1 to 8 members");
  if (A_ > plan.J) fail(2, "channel group: more members than channels");
  blocks_ = partition_channels(plan.J, A_, a_cap);
  D_ = plan.G * plan.G + plan.J * plan.Gc * plan.Gc;
  DeviceRestore restore;
  // peer access between distinct member devices (NVLink / NVSwitch loads in k_colsW
  // and k_grp_fin, peer copies of estimate blocks)
  for (int a : devices) {
    for (int b : devices) {
      if (a == b) continue;
      int ok = 0;
      check_cuda(cudaDeviceCanAccessPeer(&ok, a, b), "peer query");
      if (!ok) fail(2, "channel group: devices " + std::to_string(a) + " and " + std::to_string(b) +
                           " have no peer access");
      check_cuda(cudaSetDevice(a), "set device");
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) check_cuda(e, "enable peer access");
      cudaGetLastError();
    }
  }
  for (int d = 0; d < A_; ++d) {
    Plan lp = plan;
    lp.J = blocks_[static_cast<size_t>(d)].second - blocks_[static_cast<size_t>(d)].first;
    mem_.push_back(std::make_unique<Engine>(lp, devices[static_cast<size_t>(d)]));
  }
  GroupView gv{};
  GroupScal gs{};
  gv.A = gs.A = A_;
  const size_t G2 = static_cast<size_t>(plan.G) * plan.G;
  for (int d = 0; d < A_; ++d) {
    Engine& e = *mem_[static_cast<size_t>(d)];
    check_cuda(cudaSetDevice(e.dev_), "set device");
    check_cuda(cudaMalloc(&e.RPO_, sizeof(double2) * G2), "group rho partials");
    check_cuda(cudaMemset(e.RPO_, 0, sizeof(double2) * G2), "group rho partials");
    check_cuda(cudaMalloc(&e.SS_, sizeof(double) * static_cast<size_t>(plan.N) * plan.N), "group coil sums");
    gv.h[d] = e.dims_.H;
    gv.rp[d] = e.RP_;
    gv.rpo[d] = e.RPO_;
    gv.rc[d] = e.RC_;
    gv.jb[d] = blocks_[static_cast<size_t>(d)].first;
    gv.jb[d + 1] = blocks_[static_cast<size_t>(d)].second;
    gs.st[d] = e.st_;
    gs.pcw[d] = e.cr_.pcw;
    gs.pcr[d] = e.cr_.pcr;
    gs.ss[d] = e.SS_;
    cudaEvent_t ev;
    check_cuda(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
    ev_.push_back(ev);
    int* fl = nullptr;
    check_cuda(cudaMalloc(&fl, sizeof(int) * 2), "group flags");
    check_cuda(cudaMemset(fl, 0, sizeof(int) * 2), "group flags");
    flags_.push_back(fl);
    gf_.flag[d] = fl;
  }
  gf_.A = A_;
  // all-member barriers: device-side epoch flags (k_pg_barrier, as the one-process-per-GPU
  // group) when every member has its own GPU; CUDA graph edges between the streams when
  // members share a device, where two spinning branches of one graph are not guaranteed
  // to run concurrently. RTN_GROUP_BARRIER=flags|events overrides (the flag barrier's
  // deadline turns a missing member into a DecompFault, never a hang).
  {
    std::vector<int> dv(devices);
    std::sort(dv.begin(), dv.end());
    flag_barrier_ = std::adjacent_find(dv.begin(), dv.end()) == dv.end();
    if (const char* e = std::getenv("RTN_GROUP_BARRIER")) flag_barrier_ = std::strcmp(e, "flags") == 0;
  }
  for (int d = 0; d < A_; ++d) {
    mem_[static_cast<size_t>(d)]->join_group(d, gv, gs);
    mem_[static_cast<size_t>(d)]->set_cluster(false);  // the five passes unless set_cluster(true)
  }
  check_cuda(cudaSetDevice(mem_[0]->dev_), "set device");
  check_cuda(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming), "event");
  check_cuda(cudaMalloc(&h_stage_, sizeof(float2) * std::max<size_t>(static_cast<size_t>(D_), 1)), "stage");
  alphas_ = mem_[0]->alphas_;
  caps_ = mem_[0]->caps_;
}

Group::~Group() {
  sync();
  for (auto& g : step_graph_) {
    if (g) cudaGraphExecDestroy(g);
  }
  if (frame_graph_) cudaGraphExecDestroy(frame_graph_);
  for (size_t d = 0; d < ev_.size(); ++d) {
    cudaSetDevice(mem_[d]->dev_);
    cudaEventDestroy(ev_[d]);
    if (d < flags_.size()) cudaFree(flags_[d]);
  }
  cudaSetDevice(mem_[0]->dev_);
  if (ev_fork_) cudaEventDestroy(ev_fork_);
  if (h_stage_) cudaFree(h_stage_);
}

template <class F>
void Group::each(F&& f) {
  for (int d = 0; d < A_; ++d) {
    Engine& e = *mem_[static_cast<size_t>(d)];
    check_cuda(cudaSetDevice(e.dev_), "set device");
    f(d, e);
  }
  check_cuda(cudaSetDevice(mem_[0]->dev_), "set device");
}

void Group::fork() {
  check_cuda(cudaSetDevice(mem_[0]->dev_), "set device");
  check_cuda(cudaEventRecord(ev_fork_, mem_[0]->s_), "fork record");
  for (int d = 1; d < A_; ++d) {
    check_cuda(cudaSetDevice(mem_[static_cast<size_t>(d)]->dev_), "set device");
    check_cuda(cudaStreamWaitEvent(mem_[static_cast<size_t>(d)]->s_, ev_fork_, 0), "fork wait");
  }
  check_cuda(cudaSetDevice(mem_[0]->dev_), "set device");
}

void Group::join() {
  for (int d = 1; d < A_; ++d) {
    check_cuda(cudaSetDevice(mem_[static_cast<size_t>(d)]->dev_), "set device");
    check_cuda(cudaEventRecord(ev_[static_cast<size_t>(d)], mem_[static_cast<size_t>(d)]->s_), "join record");
  }
  check_cuda(cudaSetDevice(mem_[0]->dev_), "set device");
  for (int d = 1; d < A_; ++d) {
    check_cuda(cudaStreamWaitEvent(mem_[0]->s_, ev_[static_cast<size_t>(d)], 0), "join wait");
  }
}

void Group::barrier() {
  if (A_ == 1) return;
  if (flag_barrier_) {
    // each member bumps and publishes its epoch after its stream's earlier kernels, then
    // polls every member's: no cross-stream dependency, no host involvement
    each([&](int d, Engine& e) { e.enq_pg_barrier(flags_[static_cast<size_t>(d)], gf_); });
    return;
  }
  each([&](int d, Engine& e) { check_cuda(cudaEventRecord(ev_[static_cast<size_t>(d)], e.s_), "barrier record"); });
  each([&](int d, Engine& e) {
    for (int o = 0; o < A_; ++o) {
      if (o != d) check_cuda(cudaStreamWaitEvent(e.s_, ev_[static_cast<size_t>(o)], 0), "barrier wait");
    }
  });
}

void Group::set_cluster(bool on) {
  bool all = true;
  for (auto& m : mem_) all = all && m->cluster_supported();
  on = on && all;
  if (on == mem_[0]->use_cluster_) return;
  sync();
  // captured graphs embed the kernel choice
  for (auto& g : step_graph_) {
    if (g) cudaGraphExecDestroy(g);
    g = nullptr;
  }
  if (frame_graph_) cudaGraphExecDestroy(frame_graph_);
  frame_graph_ = nullptr;
  DeviceRestore restore;
  for (auto& m : mem_) {
    check_cuda(cudaSetDevice(m->dev_), "set device");
    m->set_cluster(on);
  }
}

void Group::sync() {
  DeviceRestore restore;
  for (auto& m : mem_) {
    check_cuda(cudaSetDevice(m->dev_), "set device");
    m->sync();
  }
}

void Group::read_state() {
  sync();
  Engine& e = *mem_[0];
  check_cuda(cudaSetDevice(e.dev_), "set device");
  e.read_state();
}

void Group::raise_status(const char* where) { mem_[0]->raise_status(where); }

// ---- full-layout <-> member-layout copies, all on the leader stream ------------------

void Group::split_copy(const float2* src, bool reg) {
  const size_t G2 = static_cast<size_t>(plan_.G) * plan_.G, C2 = static_cast<size_t>(plan_.Gc) * plan_.Gc;
  cudaStream_t s = mem_[0]->s_;
  check_cuda(cudaSetDevice(mem_[0]->dev_), "set device");
  for (int d = 0; d < A_; ++d) {
    Engine& e = *mem_[static_cast<size_t>(d)];
    float2* dst = reg ? e.reg_ : e.x_;
    const size_t j0 = static_cast<size_t>(blocks_[static_cast<size_t>(d)].first);
    check_cuda(cudaMemcpyAsync(dst, src, sizeof(float2) * G2, cudaMemcpyDefault, s), "rho split");
    check_cuda(cudaMemcpyAsync(dst + G2, src + G2 + j0 * C2, sizeof(float2) * C2 * e.plan_.J, cudaMemcpyDefault, s),
               "chat split");
  }
}

void Group::load_frame(const float2* z, const float2* P, bool masked) {
  const size_t G2 = static_cast<size_t>(plan_.G) * plan_.G;
  cudaStream_t s = mem_[0]->s_;
  check_cuda(cudaSetDevice(mem_[0]->dev_), "set device");
  for (int d = 0; d < A_; ++d) {
    Engine& e = *mem_[static_cast<size_t>(d)];
    const size_t j0 = static_cast<size_t>(blocks_[static_cast<size_t>(d)].first);
    check_cuda(cudaMemcpyAsync(e.z_, z + j0 * G2, sizeof(float2) * G2 * e.plan_.J, cudaMemcpyDefault, s), "z split");
    check_cuda(cudaMemcpyAsync(e.P_, P, sizeof(float2) * G2, cudaMemcpyDefault, s), "psf");
  }
  // each member scans its own block on its stream, ordered after the copies
  fork();
  each([&](int, Engine& e) { e.enq_z_scan(masked); });
  join();
}

void Group::load_x(const float2* src) { split_copy(src, false); }
void Group::load_reg(const float2* src) { split_copy(src, true); }

void Group::store_x(float2* dst) {
  const size_t G2 = static_cast<size_t>(plan_.G) * plan_.G, C2 = static_cast<size_t>(plan_.Gc) * plan_.Gc;
  cudaStream_t s = mem_[0]->s_;
  check_cuda(cudaSetDevice(mem_[0]->dev_), "set device");
  check_cuda(cudaMemcpyAsync(dst, mem_[0]->x_, sizeof(float2) * G2, cudaMemcpyDefault, s), "rho gather");
  for (int d = 0; d < A_; ++d) {
    Engine& e = *mem_[static_cast<size_t>(d)];
    const size_t j0 = static_cast<size_t>(blocks_[static_cast<size_t>(d)].first);
    check_cuda(cudaMemcpyAsync(dst + G2 + j0 * C2, e.x_ + G2, sizeof(float2) * C2 * e.plan_.J, cudaMemcpyDefault, s),
               "chat gather");
  }
}

// ---- enqueue ----------------------------------------------------------------------------

// One Newton step (nlinv.cpp:236-284) with the CR solve (nlinv.cpp:179-234) in the
// fused single-kernel recurrence; barriers separate each application's halves.
void Group::enq_newton_step(int m, float tol, int cap, bool sync_each) {
  const float alpha = alphas_[static_cast<size_t>(m)];
  each([&](int, Engine& e) {
    e.enq_step_begin(m);
    e.enq_setup_front(e.x_);
  });
  barrier();
  each([&](int, Engine& e) { e.enq_setup_back(e.x_, e.reg_, alpha); });
  barrier();
  each([&](int, Engine& e) { e.enq_grp_fin(1, -1, -1, tol); });
  bool run_cr = cap >= 1;
  if (run_cr && sync_each) {
    read_state();
    raise_status("cg_solve");
    run_cr = !mem_[0]->st_host_->cr_halt;
  }
  if (run_cr) {
    // the fused recurrence handles every CR vector, so the window-only skip is exact (the
    // tolerance mode's two-pass kernels read every entry of ar: no skip there)
    each([&](int, Engine& e) { e.win_only_ok_ = sync_each ? 0 : 1; });
    // budget mode: the back halves leave per-block dot partials, which every member's
    // recurrence sums member by member (DeferRed::grp = 2), in place of their grid
    // reductions and k_grp_fin
    DeferRed gdr = mem_[0]->group_red();
    if (!sync_each) {
      gdr.grp = 2;
      for (int d = 0; d < A_; ++d) {
        Engine& m = *mem_[static_cast<size_t>(d)];
        gdr.gw[d] = m.dpart_w_;
        gdr.gnw[d] = m.back_grid();
      }
      each([&](int, Engine& e) { e.defer_w_ = e.dpart_w_; });
    }
    // the enqueue-time modes are restored even if an enqueue throws
    struct Restore {
      std::vector<std::unique_ptr<Engine>>& m;
      ~Restore() {
        for (auto& e : m) {
          e->win_only_ok_ = 0;
          e->defer_w_ = nullptr;
        }
      }
    } restore{mem_};
    const bool cl = mem_[0]->use_cluster_;
    for (int it = 0; it < cap; ++it) {
      if (cl) {
        // one cluster per own channel, then out.rho over every member's channel terms
        each([&](int, Engine& e) { e.enq_cluster_front(e.r_, e.ar_, CW_OPALPHA, alpha, it, 1, it > 0 ? e.ap_ : nullptr); });
        barrier();
        each([&](int, Engine& e) { e.enq_rho_sum(e.r_, e.ar_, CW_OPALPHA, alpha, it, 1, it > 0 ? e.ap_ : nullptr); });
      } else {
        each([&](int, Engine& e) { e.enq_apply_front(e.r_, 1); });
        barrier();
        each([&](int, Engine& e) { e.enq_apply_back(e.r_, e.ar_, CW_OPALPHA, alpha, it, 1, it > 0 ? e.ap_ : nullptr); });
      }
      barrier();
      if (sync_each) {
        // tolerance mode: the reference's two-pass recurrence with the exact |ap|^2 of the
        // rounded update (nlinv.cpp:204-230), member partials summed by k_grp_fin
        each([&](int, Engine& e) {
          e.enq_grp_fin(0, it, -1, tol);                       // <r, Ar>
          e.enq_cr_two_pass_grp(it == 0 ? 0 : 1, it, tol);     // ap = ar, or p, ap update
        });
        barrier();
        each([&](int, Engine& e) {
          e.enq_grp_fin(0, -1, it, tol, 1);                    // |ap|^2
          e.enq_cr_two_pass_grp(2, it + 1, tol);               // x, r update
        });
        barrier();
        each([&](int, Engine& e) { e.enq_grp_fin(0, -1, it, tol, 2); });  // |r|, stop
        read_state();
        if (mem_[0]->st_host_->status || mem_[0]->st_host_->cr_halt) break;
      } else {
        each([&](int, Engine& e) {
          DeferRed dr = gdr;  // k_grp_fin's sums inside the recurrence
          dr.gs = e.gs_;
          e.enq_cr_fused(it, tol, dr);
        });
      }
    }
    if (!sync_each) {
      barrier();
      each([&](int, Engine& e) { e.enq_grp_fin(0, -1, cap - 1, tol); });
    }

  } else {
    // no CR iteration follows: a lagging member may still be reading this step's setup
    // partials in its k_grp_fin when the next step's setup_front overwrites them
    barrier();
  }
  each([&](int, Engine& e) { e.enq_axpy1(); });
}

void Group::enq_image(float2* img, float scale, bool apply_scale) {
  each([&](int, Engine& e) {
    e.enq_decode(e.x_);
    e.enq_coil_ss();
  });
  barrier();
  check_cuda(cudaSetDevice(mem_[0]->dev_), "set device");
  mem_[0]->enq_image_grp(img, scale, apply_scale);
}

void Group::book_frame_ffts(const std::vector<int>& iters) {
  uint64_t n = 0;
  for (int c : iters) n += static_cast<uint64_t>(c);
  fft_book(CTX_SETUP, 4ull * plan_.J * iters.size() + plan_.J);
  fft_book(CTX_NORMAL_OP, 4ull * plan_.J * n);
}

// ---- frame pipeline ------------------------------------------------------------------

void Group::frame_begin() {
  fork();
  each([&](int, Engine& e) { e.enq_state_reset(); });
  join();
}

void Group::frame_step(int m, const float2* reg_src) {
  if (reg_src) load_reg(reg_src);
  if (!budget_mode()) {
    fork();
    enq_newton_step(m, plan_.cg_tol, plan_.cg_max_iter, true);
    join();
    return;
  }
  const int cap = caps_[static_cast<size_t>(m)];
  if (!use_graphs_) {
    fork();
    enq_newton_step(m, 0.0f, cap, false);
    join();
    return;
  }
  cudaStream_t s = mem_[0]->s_;
  if (!step_graph_[m]) {
    cudaGraph_t g = nullptr;
    check_cuda(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "capture begin");
    fork();
    enq_newton_step(m, 0.0f, cap, false);
    join();
    check_cuda(cudaStreamEndCapture(s, &g), "capture end");
    check_cuda(cudaGraphInstantiate(&step_graph_[m], g, 0), "graph instantiate");
    cudaGraphDestroy(g);
  }
  check_cuda(cudaGraphLaunch(step_graph_[m], s), "graph launch");
}

void Group::frame_image(float2* img_dst, float image_scale, bool apply_scale) {
  Engine& e0 = *mem_[0];
  fork();
  enq_image(img_dst ? img_dst : e0.img_, image_scale, apply_scale);
  join();
  check_cuda(cudaMemcpyAsync(e0.st_host_, e0.st_, sizeof(DevState), cudaMemcpyDeviceToHost, e0.s_), "state read");
}

void Group::frame_all(float2* img_dst, float image_scale, bool apply_scale) {
  if (!budget_mode()) fail(2, "frame_all: whole-frame graphs need the CG iteration budget mode");
  Engine& e0 = *mem_[0];
  float2* img = e0.img_;  // fixed graph destination, copied out below
  auto enqueue = [&] {
    fork();
    each([&](int, Engine& e) { e.enq_state_reset(); });
    for (int m = 0; m < plan_.newton_steps; ++m) enq_newton_step(m, 0.0f, caps_[static_cast<size_t>(m)], false);
    enq_image(img, image_scale, apply_scale);
    join();
    check_cuda(cudaMemcpyAsync(e0.st_host_, e0.st_, sizeof(DevState), cudaMemcpyDeviceToHost, e0.s_), "state read");
  };
  auto deliver = [&] {
    if (img_dst && img_dst != e0.img_) {
      check_cuda(cudaMemcpyAsync(img_dst, e0.img_, sizeof(float2) * plan_.N * plan_.N, cudaMemcpyDefault, e0.s_),
                 "image");
    }
  };
  if (!use_graphs_) {
    enqueue();
    deliver();
    return;
  }
  if (frame_graph_ && (frame_graph_img_ != img || frame_graph_scale_ != image_scale ||
                       frame_graph_apply_ != apply_scale)) {
    cudaGraphExecDestroy(frame_graph_);
    frame_graph_ = nullptr;
  }
  if (!frame_graph_) {
    cudaGraph_t g = nullptr;
    check_cuda(cudaStreamBeginCapture(e0.s_, cudaStreamCaptureModeThreadLocal), "capture begin");
    enqueue();
    check_cuda(cudaStreamEndCapture(e0.s_, &g), "capture end");
    check_cuda(cudaGraphInstantiate(&frame_graph_, g, 0), "graph instantiate");
    cudaGraphDestroy(g);
    frame_graph_img_ = img;
    frame_graph_scale_ = image_scale;
    frame_graph_apply_ = apply_scale;
  }
  check_cuda(cudaGraphLaunch(frame_graph_, e0.s_), "graph launch");
  deliver();
}

bool Group::frame_verify(FrameStats* stats) {
  sync();
  raise_status("reconstruct_frame");
  const DevState& st = *mem_[0]->st_host_;
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

void Group::frame_run_sync(const RegFn& reg, float2* img_dst, float image_scale, bool apply_scale,
                           FrameStats* stats) {
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
    fork();
    enq_newton_step(m, tol, cap, true);
    join();
    read_state();
    raise_status("reconstruct_frame");
    const int it = mem_[0]->st_host_->steps[m].iters;
    per.push_back(it);
    if (budget_mode()) remaining -= it;
  }
  frame_image(img_dst, image_scale, apply_scale);
  read_state();
  raise_status("reconstruct_frame");
  book_frame_ffts(per);
  if (stats) {
    stats->cg_per_step = per;
    stats->cg_iters = 0;
    for (int c : per) stats->cg_iters += c;
  }
}

// ---- host in / host out -----------------------------------------------------------------

void Group::set_psf(const float* P) {
  DeviceRestore restore;
  const size_t G2 = static_cast<size_t>(plan_.G) * plan_.G;
  for (auto& m : mem_) {
    check_cuda(cudaSetDevice(m->dev_), "set device");
    check_cuda(cudaMemcpy(m->P_, P, sizeof(float2) * G2, cudaMemcpyHostToDevice), "psf upload");
  }
}

void Group::set_data(const float* z) {
  DeviceRestore restore;
  const size_t G2 = static_cast<size_t>(plan_.G) * plan_.G;
  for (int d = 0; d < A_; ++d) {
    Engine& e = *mem_[static_cast<size_t>(d)];
    const size_t j0 = static_cast<size_t>(blocks_[static_cast<size_t>(d)].first);
    check_cuda(cudaSetDevice(e.dev_), "set device");
    check_cuda(cudaMemcpy(e.z_, z + 2 * j0 * G2, sizeof(float2) * G2 * e.plan_.J, cudaMemcpyHostToDevice),
               "data upload");
    e.enq_z_scan();
    e.sync();
  }
}

void Group::set_weights(const float* w) {
  DeviceRestore restore;
  for (auto& m : mem_) {
    check_cuda(cudaSetDevice(m->dev_), "set device");
    m->set_weights(w);
  }
}

void Group::make_step_cache(const float* x) {
  DeviceRestore restore;
  Engine& e0 = *mem_[0];
  check_cuda(cudaSetDevice(e0.dev_), "set device");
  check_cuda(cudaMemcpyAsync(h_stage_, x, sizeof(float2) * D_, cudaMemcpyHostToDevice, e0.s_), "h2d");
  split_copy(h_stage_, false);
  fork();
  each([&](int, Engine& e) {
    e.enq_state_reset();
    e.enq_decode(e.x_, true);
  });
  join();
  read_state();
  raise_status("make_step_cache");
  fft_book(fft_current_ctx(), static_cast<uint64_t>(plan_.J));
  for (auto& m : mem_) m->have_cache_ = true;
}

void Group::apply_normal(const float* dx, float* out) {
  if (!mem_[0]->have_cache_) fail(2, "apply_normal: no step cache (call make_step_cache first)");
  DeviceRestore restore;
  Engine& e0 = *mem_[0];
  const size_t G2 = static_cast<size_t>(plan_.G) * plan_.G, C2 = static_cast<size_t>(plan_.Gc) * plan_.Gc;
  check_cuda(cudaSetDevice(e0.dev_), "set device");
  check_cuda(cudaMemcpyAsync(h_stage_, dx, sizeof(float2) * D_, cudaMemcpyHostToDevice, e0.s_), "h2d");
  // operand into each member's scratch 0
  for (int d = 0; d < A_; ++d) {
    Engine& e = *mem_[static_cast<size_t>(d)];
    const size_t j0 = static_cast<size_t>(blocks_[static_cast<size_t>(d)].first);
    check_cuda(cudaMemcpyAsync(e.est_scratch_[0], h_stage_, sizeof(float2) * G2, cudaMemcpyDefault, e0.s_), "split");
    check_cuda(cudaMemcpyAsync(e.est_scratch_[0] + G2, h_stage_ + G2 + j0 * C2, sizeof(float2) * C2 * e.plan_.J,
                               cudaMemcpyDefault, e0.s_),
               "split");
  }
  fork();
  each([&](int, Engine& e) {
    e.enq_state_reset();
    e.enq_apply_front(e.est_scratch_[0], 0);
  });
  barrier();
  each([&](int, Engine& e) {
    e.enq_apply_back(e.est_scratch_[0], e.est_scratch_[1], CW_OP, 0.f, -1, 0, nullptr);
  });
  join();
  check_cuda(cudaMemcpyAsync(h_stage_, e0.est_scratch_[1], sizeof(float2) * G2, cudaMemcpyDefault, e0.s_), "gather");
  for (int d = 0; d < A_; ++d) {
    Engine& e = *mem_[static_cast<size_t>(d)];
    const size_t j0 = static_cast<size_t>(blocks_[static_cast<size_t>(d)].first);
    check_cuda(cudaMemcpyAsync(h_stage_ + G2 + j0 * C2, e.est_scratch_[1] + G2, sizeof(float2) * C2 * e.plan_.J,
                               cudaMemcpyDefault, e0.s_),
               "gather");
  }
  fft_book(fft_current_ctx(), 4ull * plan_.J);
  check_cuda(cudaMemcpyAsync(out, h_stage_, sizeof(float2) * D_, cudaMemcpyDeviceToHost, e0.s_), "d2h");
  read_state();
  raise_status("apply_normal");
}

void Group::reconstruct_frame(const float* init, const float* reg, float* image, float* est_out,
                              FrameStats* stats) {
  DeviceRestore restore;
  Engine& e0 = *mem_[0];
  check_cuda(cudaSetDevice(e0.dev_), "set device");
  auto stage_in = [&](const float* h, bool to_reg) {
    check_cuda(cudaMemcpyAsync(h_stage_, h, sizeof(float2) * D_, cudaMemcpyHostToDevice, e0.s_), "h2d");
    split_copy(h_stage_, to_reg);
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
  check_cuda(cudaMemcpyAsync(image, e0.img_, sizeof(float2) * plan_.N * plan_.N, cudaMemcpyDeviceToHost, e0.s_),
             "d2h");
  if (est_out) {
    store_x(h_stage_);
    check_cuda(cudaMemcpyAsync(est_out, h_stage_, sizeof(float2) * D_, cudaMemcpyDeviceToHost, e0.s_), "d2h");
  }
  sync();
  for (auto& m : mem_) m->have_cache_ = true;
}

void Group::reconstruct_frame_regs(const float* init, const RegHostFn& reg, float* image, float* est_out,
                                   FrameStats* stats) {
  DeviceRestore restore;
  Engine& e0 = *mem_[0];
  check_cuda(cudaSetDevice(e0.dev_), "set device");
  auto stage_in = [&](const float* h, bool to_reg) {
    check_cuda(cudaMemcpyAsync(h_stage_, h, sizeof(float2) * D_, cudaMemcpyHostToDevice, e0.s_), "h2d");
    split_copy(h_stage_, to_reg);
  };
  stage_in(init, false);
  stage_in(init, true);
  const RegFn dev = [&](int m) -> const float2* {
    const float* h = reg ? reg(m) : nullptr;
    if (!h) return nullptr;
    check_cuda(cudaSetDevice(e0.dev_), "set device");
    check_cuda(cudaMemcpyAsync(h_stage_, h, sizeof(float2) * D_, cudaMemcpyHostToDevice, e0.s_), "reg h2d");
    check_cuda(cudaStreamSynchronize(e0.s_), "reg h2d");  // the provider may reuse its buffer
    return h_stage_;  // split to the members by load_reg on the same stream
  };
  frame_run_sync(dev, nullptr, 1.0f, false, stats);
  check_cuda(cudaSetDevice(e0.dev_), "set device");
  check_cuda(cudaMemcpyAsync(image, e0.img_, sizeof(float2) * plan_.N * plan_.N, cudaMemcpyDeviceToHost, e0.s_),
             "d2h");
  if (est_out) {
    store_x(h_stage_);
    check_cuda(cudaMemcpyAsync(est_out, h_stage_, sizeof(float2) * D_, cudaMemcpyDeviceToHost, e0.s_), "d2h");
  }
  sync();
  for (auto& m : mem_) m->have_cache_ = true;
}

namespace {
__global__ void k_all_reduce_sum(const float2* __restrict__ terms, int n_terms, long long n, float2* __restrict__ out) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    double sx = 0.0, sy = 0.0;
    for (int t = 0; t < n_terms; ++t) {
      const float2 v = terms[(size_t)t * n + e];
      sx += (double)v.x;
      sy += (double)v.y;
    }
    out[e] = make_float2((float)sx, (float)sy);
  }
}
}  // namespace

void all_reduce_sum_device(const float2* terms, int n_terms, long long n, float2* out, cudaStream_t s) {
  if (n_terms < 1) fail(2, "all_reduce_sum: no terms");
  const long long blocks = std::min<long long>((n + 255) / 256, 148 * 8);
  k_all_reduce_sum<<<static_cast<unsigned>(std::max<long long>(blocks, 1)), 256, 0, s>>>(terms, n_terms, n, out);
  check_cuda(cudaGetLastError(), "all_reduce_sum");
}

}  // namespace rtnb
