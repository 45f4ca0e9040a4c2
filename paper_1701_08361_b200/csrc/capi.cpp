// extern "C" boundary (include/rtnlinv_b200.h) over the engine.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rtnlinv_b200.h"
#include "engine.hpp"

struct rtn_ctx {
  rtnb::Engine* eng = nullptr;
};

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const rtnb::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of memory";
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
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
  if (!c || !c->eng) rtnb::fail(2, "null context");
  return *c->eng;
}

}  // namespace

extern "C" {

int rtn_abi_version(void) { return 1; }
const char* rtn_last_error(void) { return g_err.c_str(); }
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

void rtn_ctx_destroy(rtn_ctx* ctx) {
  if (!ctx) return;
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
  return guarded([&] { eng(ctx).set_psf(P); });
}
int rtn_set_data(rtn_ctx* ctx, const float* z) {
  return guarded([&] { eng(ctx).set_data(z); });
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
int rtn_make_step_cache(rtn_ctx* ctx, const float* x, float* rho_out, float* coils_out) {
  return guarded([&] { eng(ctx).make_step_cache(x, rho_out, coils_out); });
}
int rtn_apply_normal(rtn_ctx* ctx, const float* dx, float* out) {
  return guarded([&] { eng(ctx).apply_normal(dx, out); });
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
    eng(ctx).reconstruct_frame(init, reg, image, est_out, &st);
    if (cg_per_step) {
      for (size_t m = 0; m < st.cg_per_step.size(); ++m) cg_per_step[m] = st.cg_per_step[m];
    }
    if (seconds) *seconds = st.seconds;
  });
}

}  // extern "C"
