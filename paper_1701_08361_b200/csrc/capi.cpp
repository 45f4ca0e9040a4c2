// extern "C" boundary (include/rtnlinv_b200.h) over the engine.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <memory>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rtnlinv_b200.h"
#include "engine.hpp"
#include "group.hpp"
#include "procgroup.hpp"
#include "preproc.hpp"
#include "post.hpp"
#include "rti.hpp"
#include "sched.hpp"
#include "series.hpp"

struct rtn_ctx {
  rtnb::Engine* eng = nullptr;
  rtnb::Group* grp = nullptr;  // channel-decomposed context (rtn_ctx_create_group)
  rtnb::ProcGroup* pg = nullptr;  // one member of a one-process-per-GPU group
  std::unique_ptr<rtnb::Preproc> pre;  // pre stage, created on first use
};

namespace {

thread_local std::string g_err;
thread_local int g_kind = 0;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const rtnb::Error& e) {
    g_err = e.what();
    g_kind = e.decomp ? 6 : e.code;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of memory";
    g_kind = 5;
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    g_kind = 5;
    return 5;
  }
}

rtnb::Plan to_plan(const rtn_plan_t* p) {
  rtnb::Plan q;
  q.N = p->N;
  q.G = p->G;
  q.Gc = p->Gc;
  q.J = p->J;
  q.newton_steps = p->newton_steps;
  q.alpha0 = p->alpha0;
  q.alpha_q = p->alpha_q;
  q.alpha_min = p->alpha_min;
  q.cg_tol = p->cg_tol;
  q.cg_max_iter = p->cg_max_iter;
  q.cg_iter_budget = p->cg_iter_budget;
  q.prev_damping = p->prev_damping;
  q.gamma = p->gamma;
  return q;
}

rtnb::Engine& eng(rtn_ctx* c) {
  if (c && (c->grp || c->pg)) rtnb::fail(2, "this entry point is not available on a channel-group context");
  if (!c || !c->eng) rtnb::fail(2, "null context");
  return *c->eng;
}

}  // namespace

namespace {
template <typename F>
void with_device_buffers(size_t in_bytes, size_t out_bytes, F&& f) {
  void* a = nullptr;
  void* b = nullptr;
  rtnb::check_cuda(cudaMalloc(&a, std::max<size_t>(in_bytes, 1)), "post buffer");
  const cudaError_t e = cudaMalloc(&b, std::max<size_t>(out_bytes, 1));
  if (e != cudaSuccess) {
    cudaFree(a);
    rtnb::check_cuda(e, "post buffer");
  }
  try {
    f(a, b);
  } catch (...) {
    cudaFree(a);
    cudaFree(b);
    throw;
  }
  cudaFree(a);
  cudaFree(b);
}
}  // namespace

extern "C" {

int rtn_abi_version(void) { return 1; }
const char* rtn_last_error(void) { return g_err.c_str(); }
int rtn_last_error_kind(void) { return g_kind; }
int rtn_grid_supported(int G) { return rtnb::grid_supported(G) ? 1 : 0; }

int rtn_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int rtn_ctx_create(const rtn_plan_t* plan, int device, rtn_ctx** out) {
  return guarded([&] {
    if (!plan || !out) rtnb::fail(2, "rtn_ctx_create: null argument");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) rtnb::fail(5, "no CUDA device available");
    auto* c = new rtn_ctx;
    try {
      c->eng = new rtnb::Engine(to_plan(plan), device);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

int rtn_ctx_create_group(const rtn_plan_t* plan, const int* devices, int n_devices, int a_cap, rtn_ctx** out) {
  return guarded([&] {
    if (!plan || !out || !devices) rtnb::fail(2, "rtn_ctx_create_group: null argument");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) rtnb::fail(5, "no CUDA device available");
    for (int k = 0; k < n_devices; ++k) {
      if (devices[k] < 0 || devices[k] >= n) rtnb::fail(2, "rtn_ctx_create_group: device index out of range");
    }
    auto* c = new rtn_ctx;
    try {
      c->grp = new rtnb::Group(to_plan(plan), std::vector<int>(devices, devices + n_devices), a_cap);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

int rtn_ctx_create_proc_member(const rtn_plan_t* plan, int device, int rank, int members, int a_cap,
                               rtn_ctx** out) {
  return guarded([&] {
    if (!plan || !out) rtnb::fail(2, "rtn_ctx_create_proc_member: null argument");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) rtnb::fail(5, "no CUDA device available");
    if (device < 0 || device >= n) rtnb::fail(2, "rtn_ctx_create_proc_member: device index out of range");
    auto* c = new rtn_ctx;
    try {
      c->pg = new rtnb::ProcGroup(to_plan(plan), device, rank, members, a_cap);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

int rtn_ctx_proc_handles(rtn_ctx* ctx, void* out, int* nbytes) {
  return guarded([&] {
    if (!ctx || !ctx->pg || !nbytes) rtnb::fail(2, "rtn_ctx_proc_handles: not a process-group member");
    const int need = static_cast<int>(sizeof(cudaIpcMemHandle_t)) * rtnb::ProcGroup::kHandles;
    if (out) {
      if (*nbytes < need) rtnb::fail(2, "rtn_ctx_proc_handles: buffer too small");
      ctx->pg->export_handles(static_cast<cudaIpcMemHandle_t*>(out));
    }
    *nbytes = need;
  });
}

int rtn_ctx_proc_attach(rtn_ctx* ctx, const void* all, int nbytes) {
  return guarded([&] {
    if (!ctx || !ctx->pg || !all) rtnb::fail(2, "rtn_ctx_proc_attach: not a process-group member");
    const int need = static_cast<int>(sizeof(cudaIpcMemHandle_t)) * rtnb::ProcGroup::kHandles * ctx->pg->members();
    if (nbytes != need) rtnb::fail(2, "rtn_ctx_proc_attach: expected every member's handles in rank order");
    ctx->pg->attach(static_cast<const cudaIpcMemHandle_t*>(all));
  });
}

int rtn_ctx_group_blocks(rtn_ctx* ctx, int* out_pairs) {
  return guarded([&] {
    if (!ctx || !ctx->grp) rtnb::fail(2, "rtn_ctx_group_blocks: not a channel-group context");
    const auto& b = ctx->grp->blocks();
    for (size_t k = 0; k < b.size(); ++k) {
      out_pairs[2 * k] = b[k].first;
      out_pairs[2 * k + 1] = b[k].second;
    }
  });
}

static rtnb::Preproc& pre(rtn_ctx* c) {
  if (!c || (!c->eng && !c->grp && !c->pg)) rtnb::fail(2, "null context");
  if (!c->pre) {
    if (c->grp) {
      c->pre = std::make_unique<rtnb::Preproc>(c->grp->plan(), c->grp->device());
    } else if (c->pg) {
      c->pre = std::make_unique<rtnb::Preproc>(c->pg->plan(), c->pg->device());
    } else {
      c->pre = std::make_unique<rtnb::Preproc>(c->eng->plan(), c->eng->device());
    }
  }
  return *c->pre;
}

int rtn_grid_adjoint(rtn_ctx* ctx, const float* samples, int J, const double* angles, int K, int S, double delay,
                     float* z_out) {
  return guarded([&] {
    if (!samples || !angles || !z_out) rtnb::fail(2, "grid_adjoint: null buffer");
    pre(ctx).grid_adjoint_host(samples, J, angles, K, S, delay, z_out, false);
  });
}
int rtn_grid_spread(rtn_ctx* ctx, const float* samples, int J, const double* angles, int K, int S, double delay,
                    float* grid_out) {
  return guarded([&] {
    if (!samples || !angles || !grid_out) rtnb::fail(2, "grid_spread: null buffer");
    pre(ctx).grid_adjoint_host(samples, J, angles, K, S, delay, grid_out, true);
  });
}
int rtn_build_psf(rtn_ctx* ctx, const double* angles, int K, int S, float* P_out) {
  return guarded([&] {
    if (!angles || !P_out || K < 1 || S < 1) rtnb::fail(2, "build_psf: bad arguments");
    pre(ctx).build_psf_host(angles, K, S, P_out);
  });
}
int rtn_build_psf_coords(rtn_ctx* ctx, const double* coords, const double* weights, int n, float* P_out) {
  return guarded([&] {
    if (!coords || !weights || !P_out || n < 1) rtnb::fail(2, "build_psf_coords: bad arguments");
    pre(ctx).build_psf_coords_host(coords, weights, n, P_out);
  });
}
int rtn_apply_compression(rtn_ctx* ctx, const float* m, int Jv, int Jp, const float* in, int n, float* out) {
  return guarded([&] {
    if (!m || !in || !out || n < 0) rtnb::fail(2, "apply_compression: bad arguments");
    pre(ctx).apply_compression_host(m, Jv, Jp, in, n, out);
  });
}
// ---- planner.hpp:37-64 over the device transforms ------------------------------------------

int rtn_benchmark_fft(const int* sizes, int n, int trials, int batch, int device, double* out_us) {
  return guarded([&] {
    if (!sizes || !out_us || n < 1) rtnb::fail(2, "benchmark_fft: bad size range");
    const rtnb::FftTable t = rtnb::benchmark_fft_device(std::vector<int>(sizes, sizes + n), trials, batch, device);
    for (int i = 0; i < n; ++i) out_us[i] = t.entries_us.at(sizes[i]);
  });
}

static rtnb::FftTable table_of(const int* sizes, const double* us, int n) {
  rtnb::FftTable t;
  for (int i = 0; i < n; ++i) t.entries_us[sizes[i]] = us[i];
  return t;
}

int rtn_select_grid(int N, const int* sizes, const double* us, int n, double gamma_min, double gamma_max, int* G,
                    double* gamma) {
  return guarded([&] {
    if (n < 0 || (n > 0 && (!sizes || !us))) rtnb::fail(2, "select_grid: bad table");
    const auto g = rtnb::select_grid(N, table_of(sizes, us, n), gamma_min, gamma_max);
    *G = g.first;
    *gamma = g.second;
  });
}

int rtn_fft_table_save(const char* path, const int* sizes, const double* us, int n, const char* machine,
                       const char* library) {
  return guarded([&] {
    rtnb::FftTable t = table_of(sizes, us, n);
    t.machine_key = machine ? machine : "";
    t.library_key = library ? library : "";
    rtnb::save_fft_table(t, path);
  });
}

int rtn_fft_table_load(const char* path, int* sizes, double* us, int max_n, int* n, char* machine, char* library,
                       int key_cap) {
  return guarded([&] {
    const rtnb::FftTable t = rtnb::load_fft_table(path);
    int k = 0;
    for (const auto& [s, v] : t.entries_us) {
      if (k < max_n) {
        sizes[k] = s;
        us[k] = v;
      }
      ++k;
    }
    *n = k;
    if (machine && key_cap > 0) std::snprintf(machine, static_cast<size_t>(key_cap), "%s", t.machine_key.c_str());
    if (library && key_cap > 0) std::snprintf(library, static_cast<size_t>(key_cap), "%s", t.library_key.c_str());
  });
}

// ---- pipeline.cpp:60-137 postprocessing on the device -----------------------------------------


int rtn_all_reduce_sum(const float* terms, int n_terms, int G, float* out) {
  return guarded([&] {
    if (!terms || !out || n_terms < 1 || G < 1) rtnb::fail(2, "all_reduce_sum: no terms or bad size");
    const long long n = static_cast<long long>(G) * G;
    with_device_buffers(sizeof(float2) * n * n_terms, sizeof(float2) * n, [&](void* a, void* b) {
      rtnb::check_cuda(cudaMemcpy(a, terms, sizeof(float2) * n * n_terms, cudaMemcpyHostToDevice), "h2d");
      rtnb::all_reduce_sum_device(static_cast<float2*>(a), n_terms, n, static_cast<float2*>(b), nullptr);
      rtnb::check_cuda(cudaMemcpy(out, b, sizeof(float2) * n, cudaMemcpyDeviceToHost), "d2h");
    });
  });
}

int rtn_post_magnitude(const float* images, long long n, float* out) {
  return guarded([&] {
    if (!images || !out || n < 0) rtnb::fail(2, "magnitude_image: bad arguments");
    with_device_buffers(sizeof(float2) * n, sizeof(float) * n, [&](void* a, void* b) {
      rtnb::check_cuda(cudaMemcpy(a, images, sizeof(float2) * n, cudaMemcpyHostToDevice), "h2d");
      rtnb::post_magnitude(static_cast<float2*>(a), n, static_cast<float*>(b), nullptr);
      rtnb::check_cuda(cudaMemcpy(out, b, sizeof(float) * n, cudaMemcpyDeviceToHost), "d2h");
    });
  });
}

int rtn_post_phase_difference(const float* even, const float* odd, long long n, float* out) {
  return guarded([&] {
    if (!even || !odd || !out || n < 0) rtnb::fail(2, "phase_difference_image: bad arguments");
    with_device_buffers(2 * sizeof(float2) * n, sizeof(float) * n, [&](void* a, void* b) {
      float2* e2 = static_cast<float2*>(a);
      rtnb::check_cuda(cudaMemcpy(e2, even, sizeof(float2) * n, cudaMemcpyHostToDevice), "h2d");
      rtnb::check_cuda(cudaMemcpy(e2 + n, odd, sizeof(float2) * n, cudaMemcpyHostToDevice), "h2d");
      rtnb::post_phase_difference(e2, e2 + n, n, static_cast<float*>(b), nullptr);
      rtnb::check_cuda(cudaMemcpy(out, b, sizeof(float) * n, cudaMemcpyDeviceToHost), "d2h");
    });
  });
}

int rtn_post_median3(const float* mags, int frames, long long npix, float* out) {
  return guarded([&] {
    if (!mags || !out || frames < 1 || npix < 0) rtnb::fail(2, "median filter: bad arguments");
    const size_t n = static_cast<size_t>(frames) * static_cast<size_t>(npix);
    with_device_buffers(sizeof(float) * n, sizeof(float) * n, [&](void* a, void* b) {
      rtnb::check_cuda(cudaMemcpy(a, mags, sizeof(float) * n, cudaMemcpyHostToDevice), "h2d");
      rtnb::post_median3(static_cast<float*>(a), frames, npix, static_cast<float*>(b), nullptr);
      rtnb::check_cuda(cudaMemcpy(out, b, sizeof(float) * n, cudaMemcpyDeviceToHost), "d2h");
    });
  });
}

uint64_t rtn_psf_angle_key(const double* angles, int K, int S, int G) {
  return rtnb::psf_angle_key(angles, K, S, G);
}

void rtn_ctx_destroy(rtn_ctx* ctx) {
  if (!ctx) return;
  ctx->pre.reset();
  delete ctx->pg;
  delete ctx->grp;
  delete ctx->eng;
  delete ctx;
}

int rtn_fft2(float* data, int n, int sign) {
  return guarded([&] {
    if (n < 1) rtnb::fail(2, "fft: side must be positive");
    int nd = 0;
    if (cudaGetDeviceCount(&nd) != cudaSuccess || nd == 0) rtnb::fail(5, "no CUDA device available");
    float2* d = nullptr;
    const size_t bytes = sizeof(float2) * static_cast<size_t>(n) * n;
    rtnb::check_cuda(cudaMalloc(&d, bytes), "fft alloc");
    rtnb::check_cuda(cudaMemcpy(d, data, bytes, cudaMemcpyHostToDevice), "fft h2d");
    rtnb::fft2_device(d, n, 1, sign < 0 ? -1 : +1, nullptr);
    rtnb::check_cuda(cudaMemcpy(data, d, bytes, cudaMemcpyDeviceToHost), "fft d2h");
    cudaFree(d);
    rtnb::fft_book(rtnb::fft_current_ctx(), 1);
  });
}

void rtn_fft_set_ctx(int ctx) { rtnb::fft_set_ctx(ctx & 3); }
int rtn_fft_get_ctx(void) { return rtnb::fft_current_ctx(); }
void rtn_fft_counts(uint64_t out[4]) {
  for (int c = 0; c < 4; ++c) out[c] = rtnb::fft_count(c);
}
void rtn_fft_reset_counts(void) { rtnb::fft_reset_counts(); }

int rtn_make_weights_inv(int Gc, int G, float* out) {
  return guarded([&] {
    if (Gc < 1 || G < Gc) rtnb::fail(2, "make_weights_inv: need 1 <= Gc <= G");
    const int c = Gc / 2;
    for (int r = 0; r < Gc; ++r) {
      for (int q = 0; q < Gc; ++q) {
        const double ky = (r - c) / static_cast<double>(G);
        const double kx = (q - c) / static_cast<double>(G);
        const double w = std::pow(1.0 + 880.0 * (kx * kx + ky * ky), 16.0);
        out[2 * (r * Gc + q)] = static_cast<float>(1.0 / w);
        out[2 * (r * Gc + q) + 1] = 0.0f;
      }
    }
  });
}

int rtn_set_psf(rtn_ctx* ctx, const float* P) {
  return guarded([&] {
    if (ctx && ctx->grp) {
      ctx->grp->set_psf(P);
    } else if (ctx && ctx->pg) {
      ctx->pg->set_psf(P);
    } else {
      eng(ctx).set_psf(P);
    }
  });
}
int rtn_set_data(rtn_ctx* ctx, const float* z) {
  return guarded([&] {
    if (ctx && ctx->grp) {
      ctx->grp->set_data(z);
    } else if (ctx && ctx->pg) {
      ctx->pg->set_data(z);
    } else {
      eng(ctx).set_data(z);
    }
  });
}
int rtn_apply_W_inv(rtn_ctx* ctx, const float* chat, float* out) {
  return guarded([&] { eng(ctx).apply_W_inv(chat, out); });
}
int rtn_apply_W_invH(rtn_ctx* ctx, const float* u, float* out) {
  return guarded([&] { eng(ctx).apply_W_invH(u, out); });
}
int rtn_toeplitz_apply(rtn_ctx* ctx, float* x) {
  return guarded([&] { eng(ctx).toeplitz_apply(x); });
}
int rtn_set_weights(rtn_ctx* ctx, const float* winv) {
  return guarded([&] {
    if (!winv) rtnb::fail(2, "set_weights: null weights");
    if (ctx && ctx->grp) {
      ctx->grp->set_weights(winv);
    } else if (ctx && ctx->pg) {
      rtnb::fail(2, "set_weights: not available on a process-group member");
    } else {
      eng(ctx).set_weights(winv);
    }
  });
}
int rtn_set_step_cache(rtn_ctx* ctx, const float* rho, const float* coils) {
  return guarded([&] {
    if (!rho || !coils) rtnb::fail(2, "set_step_cache: null rho or coils");
    eng(ctx).set_step_cache(rho, coils);
  });
}
int rtn_make_step_cache(rtn_ctx* ctx, const float* x, float* rho_out, float* coils_out) {
  return guarded([&] {
    if (ctx && ctx->grp) {
      if (rho_out || coils_out) rtnb::fail(2, "make_step_cache: a channel group keeps its cache distributed");
      ctx->grp->make_step_cache(x);
    } else {
      eng(ctx).make_step_cache(x, rho_out, coils_out);
    }
  });
}
int rtn_apply_normal(rtn_ctx* ctx, const float* dx, float* out) {
  return guarded([&] {
    if (ctx && ctx->grp) {
      ctx->grp->apply_normal(dx, out);
    } else {
      eng(ctx).apply_normal(dx, out);
    }
  });
}
int rtn_cg_solve(rtn_ctx* ctx, const float* rhs, float alpha, float tol, int max_iter, float* x_out,
                 int* iters, double* residuals) {
  return guarded([&] {
    std::vector<double> res;
    eng(ctx).cg_solve(rhs, alpha, tol, max_iter, x_out, iters, &res);
    if (residuals) std::memcpy(residuals, res.data(), sizeof(double) * res.size());
  });
}
int rtn_newton_step(rtn_ctx* ctx, float* x, const float* reg, float alpha, float cg_tol, int cg_max_iter,
                    int* iters, double* residual0) {
  return guarded([&] { eng(ctx).newton_step(x, reg, alpha, cg_tol, cg_max_iter, iters, residual0); });
}
int rtn_reconstruct_frame(rtn_ctx* ctx, const float* init, const float* reg, float* image, float* est_out,
                          int* cg_per_step, double* seconds) {
  return guarded([&] {
    rtnb::FrameStats st;
    if (ctx && ctx->grp) {
      ctx->grp->reconstruct_frame(init, reg, image, est_out, &st);
    } else if (ctx && ctx->pg) {
      ctx->pg->reconstruct_frame(init, reg, image, est_out, &st);
    } else {
      eng(ctx).reconstruct_frame(init, reg, image, est_out, &st);
    }
    if (cg_per_step) {
      for (size_t m = 0; m < st.cg_per_step.size(); ++m) cg_per_step[m] = st.cg_per_step[m];
    }
    if (seconds) *seconds = st.seconds;
  });
}

int rtn_reconstruct_frame_provider(rtn_ctx* ctx, const float* init, rtn_reg_provider reg, void* user,
                                   float* image, float* est_out, int* cg_per_step, double* seconds) {
  return guarded([&] {
    if (!init || !image) rtnb::fail(2, "reconstruct_frame: null init or image");
    rtnb::FrameStats st;
    const rtnb::RegHostFn fn = [&](int m) -> const float* { return reg ? reg(m, user) : nullptr; };
    if (ctx && ctx->grp) {
      ctx->grp->reconstruct_frame_regs(init, fn, image, est_out, &st);
    } else if (ctx && ctx->pg) {
      rtnb::fail(2, "reconstruct_frame: a RegProvider needs a single-device or in-process group context");
    } else {
      eng(ctx).reconstruct_frame_regs(init, fn, image, est_out, &st);
    }
    if (cg_per_step) {
      for (size_t m = 0; m < st.cg_per_step.size(); ++m) cg_per_step[m] = st.cg_per_step[m];
    }
    if (seconds) *seconds = st.seconds;
  });
}

// ---- series -------------------------------------------------------------------------

struct rtn_series {
  rtn_ctx* ctx = nullptr;
  rtnb::Series* s = nullptr;
};

int rtn_series_create(rtn_ctx* ctx, int frames, int n_psf, rtn_series** out) {
  return guarded([&] {
    auto* s = new rtn_series;
    try {
      s->ctx = ctx;
      s->s = new rtnb::Series(eng(ctx), frames, n_psf);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

int rtn_series_create_multi(rtn_ctx* ctx, int frames, int n_psf, const int* devices, int n_devices,
                            rtn_series** out) {
  return guarded([&] {
    if (n_devices < 1 || !devices) rtnb::fail(2, "rtn_series_create_multi: need at least one device");
    int n = 0;
    rtnb::check_cuda(cudaGetDeviceCount(&n), "device count");
    for (int k = 0; k < n_devices; ++k) {
      if (devices[k] < 0 || devices[k] >= n) rtnb::fail(2, "rtn_series_create_multi: device index out of range");
    }
    auto* s = new rtn_series;
    try {
      s->ctx = ctx;
      s->s = new rtnb::Series(eng(ctx), frames, n_psf, std::vector<int>(devices, devices + n_devices));
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

void rtn_series_destroy(rtn_series* s) {
  if (!s) return;
  delete s->s;
  delete s;
}

static rtnb::Series& ser(rtn_series* s) {
  if (!s || !s->s) rtnb::fail(2, "null series");
  return *s->s;
}

int rtn_series_upload_frames(rtn_series* s, int first, int count, const float* z) {
  return guarded([&] { ser(s).upload_frames(first, count, z); });
}
int rtn_series_upload_psf(rtn_series* s, int k, const float* P) {
  return guarded([&] { ser(s).upload_psf(k, P); });
}
int rtn_series_set_psf_index(rtn_series* s, const int* idx) {
  return guarded([&] { ser(s).set_psf_index(idx); });
}
int rtn_series_set_slices(rtn_series* s, int slices) {
  return guarded([&] { ser(s).set_slices(slices); });
}
int rtn_series_slice_scale(rtn_series* s, int slice, double* scale) {
  return guarded([&] {
    if (slice < 0 || slice >= ser(s).slices()) rtnb::fail(2, "series_slice_scale: slice out of range");
    if (scale) *scale = ser(s).slice_scale(slice);
  });
}
int rtn_series_normalize(rtn_series* s, double* scale) {
  return guarded([&] {
    const double v = ser(s).normalize();
    if (scale) *scale = v;
  });
}

static int series_run_impl(rtn_series* s, const rtn_series_opts_t* o, int first, int count, const float* z_host,
                           const rtnb::RawInput* raw, float* images, int* audit, uint64_t* seqs, int* cg_iters,
                           float* gpu_ms) {
  return guarded([&] {
    if (!o) rtnb::fail(2, "reconstruct_series: null options");
    rtnb::SeriesOptions so;
    so.T = o->T;
    so.A = o->A;
    so.sched = rtnb::TemporalSchedule{o->sched_l, o->sched_o};
    so.chain = o->chain != 0;
    so.normalize = o->normalize != 0;
    so.plain = o->plain != 0;
    so.cluster = o->cluster;
    std::vector<rtnb::SeriesFrameOut> out;
    ser(s).run(so, first, count, z_host, images, &out, raw);
    const int M = s->ctx->eng->plan().newton_steps;
    for (int k = 0; k < count; ++k) {
      const rtnb::SeriesFrameOut& f = out[static_cast<size_t>(k)];
      if (audit) {
        int* row = audit + static_cast<size_t>(k) * (5 + M);
        row[0] = f.audit.frame;
        row[1] = f.audit.thread;
        row[2] = f.audit.workers;
        row[3] = f.audit.init_src;
        row[4] = f.audit.reg_final_src;
        for (int m = 0; m < M; ++m) row[5 + m] = f.audit.reg_src[static_cast<size_t>(m)];
      }
      if (seqs) {
        seqs[3 * k] = f.audit.start_seq;
        seqs[3 * k + 1] = f.audit.reg_final_seq;
        seqs[3 * k + 2] = f.audit.finish_seq;
      }
      if (cg_iters) cg_iters[k] = f.cg_iters;
      if (gpu_ms) gpu_ms[k] = f.gpu_ms;
    }
  });
}

int rtn_series_run(rtn_series* s, const rtn_series_opts_t* o, int first, int count, const float* z_host,
                   float* images, int* audit, uint64_t* seqs, int* cg_iters, float* gpu_ms) {
  return series_run_impl(s, o, first, count, z_host, nullptr, images, audit, seqs, cg_iters, gpu_ms);
}

int rtn_series_run_raw(rtn_series* s, const rtn_series_opts_t* o, int first, int count, const float* samples,
                       const double* angles, int K, int S, double delay, const float* cmat, int Jp, float* images,
                       int* audit, uint64_t* seqs, int* cg_iters, float* gpu_ms) {
  rtnb::RawInput raw;
  raw.samples = samples;
  raw.angles = angles;
  raw.K = K;
  raw.S = S;
  raw.Jp = Jp;
  raw.delay = delay;
  raw.cmat = cmat;
  return series_run_impl(s, o, first, count, nullptr, &raw, images, audit, seqs, cg_iters, gpu_ms);
}

int rtn_series_psf_cache_size(rtn_series* s) { return (s && s->s) ? s->s->psf_cache_size() : 0; }

int rtn_series_psf_cache_save(rtn_series* s, const char* path) {
  return guarded([&] {
    if (!path || !ser(s).save_psf_cache(path)) rtnb::fail(3, "psf cache: cannot write " + std::string(path ? path : ""));
  });
}
int rtn_series_psf_cache_load(rtn_series* s, const char* path) {
  return guarded([&] {
    if (!path || !ser(s).load_psf_cache(path)) rtnb::fail(3, "psf cache: cannot read " + std::string(path ? path : ""));
  });
}

int rtn_series_post(rtn_series* s, int first, int count, int mode, float* out) {
  return guarded([&] { ser(s).post(first, count, mode, out); });
}

struct rtn_rti {
  rtnb::RtiSink* w = nullptr;
};

int rtn_rti_open(const char* path, const int* header9, int strict_order, rtn_rti** out) {
  return guarded([&] {
    if (!path || !header9 || !out) rtnb::fail(2, "rti_open: null argument");
    rtnb::RtiHeader h;
    h.version = header9[0];
    h.N = header9[1];
    h.J_physical = header9[2];
    h.K = header9[3];
    h.U = header9[4];
    h.frames = header9[5];
    h.slices = header9[6];
    h.mode = header9[7];
    h.samples = header9[8];
    auto* r = new rtn_rti;
    try {
      r->w = new rtnb::RtiSink(path, h, strict_order != 0);
    } catch (...) {
      delete r;
      throw;
    }
    *out = r;
  });
}

int rtn_rti_write(rtn_rti* w, int frame, int slice, int kind, const float* pixels) {
  return guarded([&] {
    if (!w || !w->w || !pixels) rtnb::fail(2, "rti_write: null argument");
    w->w->write(frame, slice, kind, pixels);
  });
}

int rtn_rti_count(rtn_rti* w) { return (w && w->w) ? w->w->count() : 0; }

int rtn_rti_close(rtn_rti* w) {
  if (!w) return 0;
  const int st = guarded([&] {
    if (w->w) w->w->close();
  });
  delete w->w;
  delete w;
  return st;
}

int rtn_series_write_rti(rtn_series* s, rtn_rti* w, int first, int count, int mode, int slice) {
  return guarded([&] {
    if (!w || !w->w) rtnb::fail(2, "series_write_rti: null sink");
    const rtnb::Plan& p = s->ctx->eng->plan();
    if (w->w->header().N != p.N) rtnb::fail(2, "series_write_rti: image side does not match the sink header");
    const size_t npix = static_cast<size_t>(p.N) * p.N;
    const int n_out = mode == 2 ? count / 2 : count;
    std::vector<float> host(npix * static_cast<size_t>(std::max(n_out, 1)));
    ser(s).post(first, count, mode, host.data());
    for (int k = 0; k < n_out; ++k) {
      // phase-difference images carry the pair index (pipeline.cpp:98-111)
      const int frame = mode == 2 ? first / 2 + k : first + k;
      w->w->write(frame, slice, mode == 2 ? 1 : 0, host.data() + npix * k);
    }
  });
}

int rtn_series_images(rtn_series* s, int first, int count, float* images) {
  return guarded([&] {
    const rtnb::Plan& p = s->ctx->eng->plan();
    const size_t isz = static_cast<size_t>(p.N) * p.N;
    if (first < 0 || first + count > ser(s).frames()) rtnb::fail(2, "series_images: range out of bounds");
    rtnb::check_cuda(cudaMemcpy(images, ser(s).images_dev() + isz * first, sizeof(float2) * isz * count,
                                cudaMemcpyDeviceToHost),
                     "images d2h");
  });
}

float rtn_series_last_span_ms(rtn_series* s) { return (s && s->s) ? s->s->last_span_ms() : 0.f; }

int rtn_series_estimate(rtn_series* s, int n, float* est) {
  return guarded([&] {
    if (n < 0 || n >= ser(s).frames()) rtnb::fail(2, "series_estimate: frame out of range");
    rtnb::check_cuda(cudaMemcpy(est, ser(s).estimate_dev(n), sizeof(float2) * s->ctx->eng->D(),
                                cudaMemcpyDeviceToHost),
                     "estimate d2h");
  });
}

// ---- decomposition / scheduling ------------------------------------------------------

int rtn_partition_channels(int J, int A, int cap, int* out_pairs) {
  return guarded([&] {
    const auto b = rtnb::partition_channels(J, A, cap);
    for (size_t a = 0; a < b.size(); ++a) {
      out_pairs[2 * a] = b[a].first;
      out_pairs[2 * a + 1] = b[a].second;
    }
  });
}

struct rtn_ledger {
  rtnb::CompletionLedger* l = nullptr;
};

int rtn_ledger_create(int frames, rtn_ledger** out) {
  return guarded([&] {
    auto* l = new rtn_ledger;
    l->l = new rtnb::CompletionLedger(frames);
    *out = l;
  });
}
void rtn_ledger_destroy(rtn_ledger* l) {
  if (!l) return;
  delete l->l;
  delete l;
}
int rtn_ledger_mark_step(rtn_ledger* l, int n, int m) {
  return guarded([&] { l->l->mark_step(n, m); });
}
int rtn_ledger_mark_complete(rtn_ledger* l, int n) {
  return guarded([&] { l->l->mark_complete(n); });
}
int rtn_ledger_completed(rtn_ledger* l, int n) { return l->l->completed(n) ? 1 : 0; }
int rtn_ledger_last_step(rtn_ledger* l, int n, int* out) {
  return guarded([&] { *out = l->l->last_step(n); });
}
int rtn_ledger_wait_complete(rtn_ledger* l, int n, int deadline_ms) {
  return guarded([&] { l->l->wait_complete(n, std::chrono::milliseconds(deadline_ms)); });
}
void rtn_ledger_poison(rtn_ledger* l) { l->l->poison(); }
int rtn_ledger_poisoned(rtn_ledger* l) { return l->l->poisoned() ? 1 : 0; }
uint64_t rtn_ledger_next_seq(rtn_ledger* l) { return l->l->next_seq(); }
int rtn_h_choose(int n, int m, int M, int sched_l, int sched_o, rtn_ledger* l, int* out) {
  return guarded([&] { *out = rtnb::h_choose(n, m, M, rtnb::TemporalSchedule{sched_l, sched_o}, *l->l); });
}

// ---- autotune ----------------------------------------------------------------------------

static std::vector<rtnb::TuningRecord> records(const int* rows, const double* ms, int n) {
  std::vector<rtnb::TuningRecord> db;
  for (int i = 0; i < n; ++i) {
    rtnb::TuningRecord r;
    r.key.mode = static_cast<rtnb::ImagingMode>(rows[6 * i]);
    r.key.N = rows[6 * i + 1];
    r.key.bucket = rows[6 * i + 2];
    r.key.J = rows[6 * i + 3];
    r.T = rows[6 * i + 4];
    r.A = rows[6 * i + 5];
    r.runtime_ms = ms[i];
    db.push_back(r);
  }
  return db;
}

static rtnb::ProtocolKey key_of(const int* k) {
  rtnb::ProtocolKey key;
  key.mode = static_cast<rtnb::ImagingMode>(k[0]);
  key.N = k[1];
  key.bucket = k[2];
  key.J = k[3];
  return key;
}

int rtn_legal_configs(int total, int a_cap, int* out_pairs, int max_pairs) {
  int count = 0;
  const int st = guarded([&] {
    const auto v = rtnb::legal_configs(total, a_cap);
    count = static_cast<int>(v.size());
    for (int i = 0; i < count && i < max_pairs; ++i) {
      out_pairs[2 * i] = v[static_cast<size_t>(i)].first;
      out_pairs[2 * i + 1] = v[static_cast<size_t>(i)].second;
    }
  });
  return st == 0 ? count : -st;
}

int rtn_frames_bucket(int frames, int* out) {
  return guarded([&] { *out = rtnb::frames_bucket(frames); });
}

int rtn_select_config(const int* key4, const int* rows6, const double* ms, int n, int* out_ta) {
  return guarded([&] {
    const auto r = rtnb::select_config(key_of(key4), records(rows6, ms, n));
    out_ta[0] = r.first;
    out_ta[1] = r.second;
  });
}

int rtn_learn_step(const int* key4, const int* rows6, const double* ms, int n, int total, int a_cap,
                   int* out_ta) {
  return guarded([&] {
    const auto r = rtnb::learn_step(key_of(key4), records(rows6, ms, n), total, a_cap);
    out_ta[0] = r.first;
    out_ta[1] = r.second;
  });
}

int rtn_tunedb_append(const char* path, const int* row6, double runtime_ms, int64_t timestamp) {
  return guarded([&] {
    rtnb::TuningRecord r = records(row6, &runtime_ms, 1)[0];
    r.timestamp = timestamp;
    rtnb::TuneDb(path).append(r);
  });
}

int rtn_tunedb_load(const char* path, int* rows6, double* ms, int64_t* ts, int max_rows, int* n_rows,
                    int* skipped) {
  return guarded([&] {
    rtnb::TuneDb db(path);
    const auto v = db.load();
    *n_rows = static_cast<int>(v.size());
    if (skipped) *skipped = static_cast<int>(db.skipped_lines());
    for (int i = 0; i < static_cast<int>(v.size()) && i < max_rows; ++i) {
      const auto& r = v[static_cast<size_t>(i)];
      rows6[6 * i] = static_cast<int>(r.key.mode);
      rows6[6 * i + 1] = r.key.N;
      rows6[6 * i + 2] = r.key.bucket;
      rows6[6 * i + 3] = r.key.J;
      rows6[6 * i + 4] = r.T;
      rows6[6 * i + 5] = r.A;
      ms[i] = r.runtime_ms;
      if (ts) ts[i] = r.timestamp;
    }
  });
}

int rtn_time_kernel(rtn_ctx* ctx, const char* which, int reps, double* ms, double* bytes) {
  return guarded([&] {
    *ms = eng(ctx).time_kernel(which, reps);
    if (bytes) *bytes = eng(ctx).kernel_bytes(which);
  });
}

int rtn_cluster_supported(rtn_ctx* ctx, int* supported) {
  return guarded([&] {
    if (!supported) rtnb::fail(2, "cluster_supported: null output");
    *supported = eng(ctx).cluster_supported() ? 1 : 0;
  });
}

int rtn_fused_cra(rtn_ctx* ctx, int* on) {
  return guarded([&] {
    if (!on) rtnb::fail(2, "fused_cra: null output");
    *on = eng(ctx).fused_crA() ? 1 : 0;
  });
}

}  // extern "C"
