// ORACLE TEST INFRASTRUCTURE — not product code. Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load the library built from
// this file (oracle/_ref/librtnlinv_ref.so).
//
// extern "C" wrapper around the UNMODIFIED reference library compiled in place from
// /root/reference/proj/src (see oracle/Makefile). It exposes the reference's own
// functions with flat buffers so the Python tests can (a) generate the synthetic
// phantom inputs the reference's tests use (seqsim.cpp:294-346, preproc.cpp:311-343,
// 414-430), and (b) run the reference hot path on the same inputs as the CUDA path:
//   make_weights_inv  nlinv.cpp:101-117      apply_W_inv/H   nlinv.cpp:119-133
//   toeplitz_apply    preproc.cpp:436-443    make_step_cache nlinv.cpp:135-150
//   apply_normal      nlinv.cpp:152-177      cg_solve        nlinv.cpp:179-234
//   newton_step       nlinv.cpp:236-284      reconstruct_frame nlinv.cpp:286-335
//   reconstruct_series[_plain] nlinv.cpp:412-526, h_choose decomp.cpp:193-209,
//   partition_channels decomp.cpp:10-24, autotune.cpp:15-152, fft.cpp:41-101.
// Layouts: images row-major complex64; an Estimate is flattened rho (G*G) then
// chat[j] (Gc*Gc each), the order of test_nlinv.cpp:70-79 (est_flatten).
// Status codes follow the CLI mapping (rtnlinv_main.cpp:381-391): 0 ok, 2 UsageError,
// 3 DataError, 4 SolverError / DecompFault, 5 other.
#include <array>
#include <chrono>
#include <mutex>
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "rtnlinv/autotune.hpp"
#include "rtnlinv/decomp.hpp"
#include "rtnlinv/fft.hpp"
#include "rtnlinv/ingest.hpp"
#include "rtnlinv/nlinv.hpp"
#include "rtnlinv/pipeline.hpp"
#include "rtnlinv/planner.hpp"
#include "rtnlinv/preproc.hpp"
#include "rtnlinv/seqsim.hpp"

using namespace rtnlinv;

extern "C" {

struct ref_plan_t {
  int N, G, Gc, J, newton_steps;
  float alpha0, alpha_q, alpha_min, cg_tol;
  int cg_max_iter, cg_iter_budget;
  float prev_damping;
  double gamma;
};

struct ref_series_opts_t {
  int T, A, sched_l, sched_o, chain, normalize;
  double delay_samples;
};

}  // extern "C"

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const UsageError& e) {
    g_err = e.what();
    return 2;
  } catch (const DataError& e) {
    g_err = e.what();
    return 3;
  } catch (const SolverError& e) {
    g_err = e.what();
    return 4;
  } catch (const DecompFault& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

ReconPlan to_plan(const ref_plan_t* p) {
  ReconPlan plan;
  plan.N = p->N;
  plan.G = p->G;
  plan.Gc = p->Gc;
  plan.J = p->J;
  plan.newton_steps = p->newton_steps;
  plan.alpha0 = p->alpha0;
  plan.alpha_q = p->alpha_q;
  plan.alpha_min = p->alpha_min;
  plan.cg_tol = p->cg_tol;
  plan.cg_max_iter = p->cg_max_iter;
  plan.cg_iter_budget = p->cg_iter_budget;
  plan.prev_damping = p->prev_damping;
  plan.gamma = p->gamma;
  return plan;
}

void from_plan(const ReconPlan& plan, ref_plan_t* p) {
  p->N = plan.N;
  p->G = plan.G;
  p->Gc = plan.Gc;
  p->J = plan.J;
  p->newton_steps = plan.newton_steps;
  p->alpha0 = plan.alpha0;
  p->alpha_q = plan.alpha_q;
  p->alpha_min = plan.alpha_min;
  p->cg_tol = plan.cg_tol;
  p->cg_max_iter = plan.cg_max_iter;
  p->cg_iter_budget = plan.cg_iter_budget;
  p->prev_damping = plan.prev_damping;
  p->gamma = plan.gamma;
}

CImage load_img(const float* src, int n) {
  CImage img(n);
  std::memcpy(img.v.data(), src, sizeof(cfloat) * img.v.size());
  return img;
}

void store_img(const CImage& img, float* dst) {
  std::memcpy(dst, img.v.data(), sizeof(cfloat) * img.v.size());
}

Estimate load_est(const float* src, const ReconPlan& plan) {
  Estimate e;
  e.rho = load_img(src, plan.G);
  size_t off = static_cast<size_t>(plan.G) * plan.G * 2;
  for (int j = 0; j < plan.J; ++j) {
    e.chat.push_back(load_img(src + off, plan.Gc));
    off += static_cast<size_t>(plan.Gc) * plan.Gc * 2;
  }
  return e;
}

void store_est(const Estimate& e, float* dst) {
  store_img(e.rho, dst);
  size_t off = e.rho.v.size() * 2;
  for (const CImage& c : e.chat) {
    store_img(c, dst + off);
    off += c.v.size() * 2;
  }
}

GriddedData load_z(const float* src, const ReconPlan& plan) {
  GriddedData z;
  z.J = plan.J;
  z.G = plan.G;
  for (int j = 0; j < plan.J; ++j) {
    z.z.push_back(load_img(src + static_cast<size_t>(j) * plan.G * plan.G * 2, plan.G));
  }
  return z;
}

PsfKernel load_psf(const float* src, int G) {
  PsfKernel psf;
  psf.G = G;
  psf.P = load_img(src, G);
  return psf;
}

KSpaceFrame load_frame(const float* samples, const double* angles, int J, int K, int S, int index) {
  KSpaceFrame fr;
  fr.frame_index = index;
  fr.J = J;
  fr.K = K;
  fr.S = S;
  fr.samples.resize(static_cast<size_t>(J) * K * S);
  std::memcpy(fr.samples.data(), samples, sizeof(cfloat) * fr.samples.size());
  fr.spoke_angles.assign(angles, angles + K);
  return fr;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_make_plan(int N, int J, ref_plan_t* out) {
  return guarded([&] { from_plan(make_plan(N, J), out); });
}

// ---- synthetic acquisition (seqsim.cpp) -------------------------------------------

// frames n = 0..F-1 of default_phantom(J, seed) with noise sigma on a K-spoke, U-turn
// radial trajectory with S = 2N samples per spoke (test_nlinv.cpp:100-111).
// samples: F*J*K*S complex64, angles: F*K doubles.
int ref_phantom_series(int J, int F, int K, int U, int N, double noise, uint64_t seed,
                       float* samples, double* angles) {
  return guarded([&] {
    PhantomSpec ph = default_phantom(J, seed);
    ph.noise_sigma = noise;
    TrajectorySpec traj;
    traj.K = K;
    traj.U = U;
    traj.samples_per_spoke = 2 * N;
    const size_t per = static_cast<size_t>(J) * K * 2 * N;
    for (int n = 0; n < F; ++n) {
      const KSpaceFrame fr = simulate_frame(ph, traj, n);
      std::memcpy(samples + static_cast<size_t>(n) * per * 2, fr.samples.data(),
                  sizeof(cfloat) * per);
      std::memcpy(angles + static_cast<size_t>(n) * K, fr.spoke_angles.data(),
                  sizeof(double) * K);
    }
  });
}

int ref_bandlimited_truth_rss(int J, uint64_t seed, int n, int N, float* out) {
  return guarded([&] {
    const PhantomSpec ph = default_phantom(J, seed);
    store_img(bandlimited_truth_rss(ph, n, N), out);
  });
}

int ref_nrmse_scaled(const float* got, const float* want, int N, double interior, double* out) {
  return guarded([&] { *out = nrmse_scaled(load_img(got, N), load_img(want, N), interior); });
}

// ---- pre stage (preproc.cpp) ---------------------------------------------------------

int ref_grid_adjoint(const ref_plan_t* p, const float* samples, const double* angles, int J,
                     int K, int S, float* z_out) {
  return guarded([&] {
    const ReconPlan plan = to_plan(p);
    const GriddedData z = grid_adjoint(load_frame(samples, angles, J, K, S, 0), plan);
    for (int j = 0; j < J; ++j) store_img(z.z[static_cast<size_t>(j)], z_out + static_cast<size_t>(j) * plan.G * plan.G * 2);
  });
}

int ref_build_psf(const ref_plan_t* p, const double* angles, int K, int S, float* P_out) {
  return guarded([&] {
    const ReconPlan plan = to_plan(p);
    std::vector<double> a(angles, angles + K);
    store_img(build_psf(a, S, plan).P, P_out);
  });
}

// the density-compensated Kaiser-Bessel spread of grid_adjoint before its inverse
// FFT (preproc.cpp:180-192, spread_sample preproc.cpp:120-133), per channel
int ref_grid_spread(const ref_plan_t* p, const float* samples, const double* angles, int J, int K, int S,
                    double delay, float* grid_out) {
  return guarded([&] {
    const ReconPlan plan = to_plan(p);
    const KSpaceFrame fr = load_frame(samples, angles, J, K, S, 0);
    const auto coords = frame_coords(fr, delay);
    const int G = plan.G;
    for (int j = 0; j < J; ++j) {
      CImage g(G);
      size_t s = 0;
      for (int k = 0; k < K; ++k) {
        for (int i = 0; i < S; ++i, ++s) {
          const double v = dcf_ramp(coords[s][0], coords[s][1], K, S, G);
          spread_sample(g, coords[s][0], coords[s][1], fr.at(j, k, i) * static_cast<float>(v));
        }
      }
      store_img(g, grid_out + static_cast<size_t>(j) * G * G * 2);
    }
  });
}

int ref_build_psf_coords(const ref_plan_t* p, const double* coords, const double* weights, int n, float* P_out) {
  return guarded([&] {
    const ReconPlan plan = to_plan(p);
    std::vector<std::array<double, 2>> c(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) c[static_cast<size_t>(i)] = {coords[2 * i], coords[2 * i + 1]};
    std::vector<double> w(weights, weights + n);
    store_img(build_psf_coords(c, w, plan).P, P_out);
  });
}

// calibrate_compression (preproc.cpp:390-444) on F frames: the Jv x Jp matrix
int ref_calibrate_compression(const float* samples_in, const double* angles, int F, int Jp, int K, int S, int Jv,
                              float* m_out, double* energy) {
  return guarded([&] {
    std::vector<KSpaceFrame> frames;
    const size_t per_in = static_cast<size_t>(Jp) * K * S * 2;
    for (int n = 0; n < F; ++n) {
      frames.push_back(load_frame(samples_in + n * per_in, angles + static_cast<size_t>(n) * K, Jp, K, S, n));
    }
    const CompressionMatrix cm = calibrate_compression(frames, Jv);
    if (energy) *energy = cm.energy_fraction;
    std::memcpy(m_out, cm.m.data(), sizeof(cfloat) * cm.m.size());
  });
}

// J_phys -> J_virt PCA compression calibrated on `ncal` frames, then applied to all F
// frames (rtnlinv_main.cpp:125-130). samples_in: F*Jp*K*S, samples_out: F*Jv*K*S.
int ref_compress_series(const float* samples_in, const double* angles, int F, int Jp, int K,
                        int S, int Jv, int ncal, float* samples_out, double* energy) {
  return guarded([&] {
    std::vector<KSpaceFrame> frames;
    const size_t per_in = static_cast<size_t>(Jp) * K * S * 2;
    for (int n = 0; n < F; ++n) {
      frames.push_back(load_frame(samples_in + n * per_in, angles + static_cast<size_t>(n) * K, Jp, K, S, n));
    }
    std::vector<KSpaceFrame> cal(frames.begin(), frames.begin() + std::min(ncal, F));
    const CompressionMatrix cm = calibrate_compression(cal, Jv);
    if (energy) *energy = cm.energy_fraction;
    const size_t per_out = static_cast<size_t>(Jv) * K * S;
    for (int n = 0; n < F; ++n) {
      const KSpaceFrame c = apply_compression(frames[static_cast<size_t>(n)], cm);
      std::memcpy(samples_out + static_cast<size_t>(n) * per_out * 2, c.samples.data(),
                  sizeof(cfloat) * per_out);
    }
  });
}

// ---- planner (planner.cpp:112-183) and postprocessing (pipeline.cpp:60-137) -----------------

int ref_select_grid(int N, const int* sizes, const double* us, int n, double gmin, double gmax, int* G,
                    double* gamma) {
  return guarded([&] {
    FftLookupTable t;
    for (int i = 0; i < n; ++i) t.entries_us[sizes[i]] = us[i];
    const auto g = select_grid(N, t, gmin, gmax);
    *G = g.first;
    *gamma = g.second;
  });
}

int ref_table_roundtrip(const char* path, const int* sizes, const double* us, int n, int* sizes_out,
                        double* us_out, int* n_out) {
  return guarded([&] {
    FftLookupTable t;
    t.machine_key = "m";
    t.library_key = "l";
    for (int i = 0; i < n; ++i) t.entries_us[sizes[i]] = us[i];
    save_table(t, path);
    const FftLookupTable r = load_table(path);
    int k = 0;
    for (const auto& [s, v] : r.entries_us) {
      sizes_out[k] = s;
      us_out[k] = v;
      ++k;
    }
    *n_out = k;
  });
}

int ref_magnitude_image(const float* img, int N, float* out) {
  return guarded([&] {
    const ImageOut o = magnitude_image(load_img(img, N), 0, 0);
    std::memcpy(out, o.pixels.data(), sizeof(float) * o.pixels.size());
  });
}

int ref_phase_difference_image(const float* even, const float* odd, int N, float* out) {
  return guarded([&] {
    const ImageOut o = phase_difference_image(load_img(even, N), load_img(odd, N), 0, 0);
    std::memcpy(out, o.pixels.data(), sizeof(float) * o.pixels.size());
  });
}

// MedianFilter3 push/drain over F magnitude frames of one slice, outputs in order
int ref_median_filter(const float* mags, int F, int N, float* out) {
  return guarded([&] {
    MedianFilter3 f;
    std::vector<ImageOut> got;
    for (int n = 0; n < F; ++n) {
      ImageOut im;
      im.frame_index = n;
      im.n = N;
      im.kind = ImageKind::magnitude;
      im.pixels.assign(mags + static_cast<size_t>(n) * N * N, mags + static_cast<size_t>(n + 1) * N * N);
      for (auto& o : f.push(std::move(im))) got.push_back(std::move(o));
    }
    for (auto& o : f.drain()) got.push_back(std::move(o));
    if (static_cast<int>(got.size()) != F) throw UsageError("median filter: frame count changed");
    for (const ImageOut& o : got) {
      std::memcpy(out + static_cast<size_t>(o.frame_index) * N * N, o.pixels.data(), sizeof(float) * N * N);
    }
  });
}

// PsfCache (preproc.cpp:315-388): build the kernels of `nsets` angle sets, save them
int ref_psf_cache_save(const ref_plan_t* p, const double* angles, int nsets, int K, int S, const char* path) {
  return guarded([&] {
    PsfCache c(to_plan(p));
    for (int n = 0; n < nsets; ++n) c.get(std::vector<double>(angles + static_cast<size_t>(n) * K, angles + static_cast<size_t>(n + 1) * K), S);
    if (!c.save(path)) throw DataError("psf cache save failed");
  });
}
// load a sidecar and return the kernel of one angle set (build it if absent: count hits)
int ref_psf_cache_get(const ref_plan_t* p, const char* path, const double* angles, int K, int S, float* P_out,
                      int* hits, int* size) {
  return guarded([&] {
    PsfCache c(to_plan(p));
    if (!c.load(path)) throw DataError("psf cache load failed");
    const auto k = c.get(std::vector<double>(angles, angles + K), S);
    store_img(k->P, P_out);
    *hits = static_cast<int>(c.hits());
    *size = static_cast<int>(c.size());
  });
}

// ---- primitives ---------------------------------------------------------------------

int ref_fft(float* data, int n, int sign) {
  return guarded([&] {
    if (sign < 0) {
      fft::forward(reinterpret_cast<cfloat*>(data), n);
    } else {
      fft::inverse(reinterpret_cast<cfloat*>(data), n);
    }
  });
}

void ref_fft_counts(uint64_t out[4]) {
  for (int c = 0; c < 4; ++c) out[c] = fft::count(static_cast<fft::Ctx>(c));
}
void ref_fft_reset_counts() { fft::reset_counts(); }

int ref_crop_k(const float* x, int n, int Gc, float* out) {
  return guarded([&] { store_img(crop_k(load_img(x, n), Gc), out); });
}
int ref_pad_k(const float* x, int n, int G, float* out) {
  return guarded([&] { store_img(pad_k(load_img(x, n), G), out); });
}

int ref_make_weights_inv(int Gc, int G, float* out) {
  return guarded([&] { store_img(make_weights_inv(Gc, G), out); });
}

int ref_apply_W_inv(const float* chat, const float* winv, int Gc, int G, float* out) {
  return guarded([&] { store_img(apply_W_inv(load_img(chat, Gc), load_img(winv, Gc), G), out); });
}

int ref_apply_W_invH(const float* u, const float* winv, int G, int Gc, float* out) {
  return guarded([&] { store_img(apply_W_invH(load_img(u, G), load_img(winv, Gc), Gc), out); });
}

int ref_toeplitz_apply(float* x, const float* P, int G) {
  return guarded([&] {
    CImage img = load_img(x, G);
    toeplitz_apply(img, load_psf(P, G));
    store_img(img, x);
  });
}

// decoded step cache of x: masked rho (G*G) and coils (J*G*G)
int ref_make_step_cache(const ref_plan_t* p, const float* x, const float* P, float* rho_out,
                        float* coils_out) {
  return guarded([&] {
    const ReconPlan plan = to_plan(p);
    const PsfKernel psf = load_psf(P, plan.G);
    const CImage winv = make_weights_inv(plan.Gc, plan.G);
    const StepCache sc = make_step_cache(load_est(x, plan), plan, psf, winv, nullptr);
    store_img(sc.rho, rho_out);
    for (int j = 0; j < plan.J; ++j) {
      store_img(sc.coils[static_cast<size_t>(j)], coils_out + static_cast<size_t>(j) * plan.G * plan.G * 2);
    }
  });
}

// out = DF^H DF (dx) at the linearisation point x, A lanes of channel decomposition
int ref_apply_normal(const ref_plan_t* p, const float* x, const float* dx, const float* P, int A,
                     float* out) {
  return guarded([&] {
    const ReconPlan plan = to_plan(p);
    const PsfKernel psf = load_psf(P, plan.G);
    const CImage winv = make_weights_inv(plan.Gc, plan.G);
    std::unique_ptr<WorkerGroup> wg;
    if (A > 1) wg = std::make_unique<WorkerGroup>(A);
    const StepCache sc = make_step_cache(load_est(x, plan), plan, psf, winv, wg.get());
    store_est(apply_normal(load_est(dx, plan), sc), out);
  });
}

int ref_cg_solve(const ref_plan_t* p, const float* x, const float* rhs, const float* P,
                 float alpha, float tol, int max_iter, float* out_x, int* out_iters,
                 double* out_residuals) {
  return guarded([&] {
    const ReconPlan plan = to_plan(p);
    const PsfKernel psf = load_psf(P, plan.G);
    const CImage winv = make_weights_inv(plan.Gc, plan.G);
    const StepCache sc = make_step_cache(load_est(x, plan), plan, psf, winv, nullptr);
    const CgResult r = cg_solve(load_est(rhs, plan), sc, alpha, tol, max_iter);
    store_est(r.x, out_x);
    *out_iters = r.iters;
    for (size_t i = 0; i < r.residuals.size(); ++i) out_residuals[i] = r.residuals[i];
  });
}

int ref_newton_step(const ref_plan_t* p, float* x, const float* reg, float alpha, const float* z,
                    const float* P, float cg_tol, int cg_max_iter, int* out_iters,
                    double* out_residual0) {
  return guarded([&] {
    const ReconPlan plan = to_plan(p);
    const PsfKernel psf = load_psf(P, plan.G);
    const CImage winv = make_weights_inv(plan.Gc, plan.G);
    Estimate est = load_est(x, plan);
    const StepStats st = newton_step(est, load_est(reg, plan), alpha, load_z(z, plan), psf, plan,
                                     winv, nullptr, cg_tol, cg_max_iter);
    store_est(est, x);
    *out_iters = st.cg_iters;
    *out_residual0 = st.residual0;
  });
}

// reg == nullptr: regularise every step towards init (the plain chained solve)
int ref_reconstruct_frame(const ref_plan_t* p, const float* z, const float* P, const float* init,
                          const float* reg, int A, float* out_image, float* out_est,
                          int* out_cg_per_step, double* out_seconds) {
  return guarded([&] {
    const ReconPlan plan = to_plan(p);
    const PsfKernel psf = load_psf(P, plan.G);
    const CImage winv = make_weights_inv(plan.Gc, plan.G);
    const Estimate e0 = load_est(init, plan);
    const Estimate r0 = reg ? load_est(reg, plan) : e0;
    std::unique_ptr<WorkerGroup> wg;
    if (A > 1) wg = std::make_unique<WorkerGroup>(A);
    const RegProvider rp = [&r0](int) -> const Estimate& { return r0; };
    const FrameResult fr =
        reconstruct_frame(load_z(z, plan), psf, plan, winv, e0, rp, wg.get());
    store_img(fr.image, out_image);
    if (out_est) store_est(fr.est, out_est);
    if (out_cg_per_step) {
      for (size_t m = 0; m < fr.cg_per_step.size(); ++m) out_cg_per_step[m] = fr.cg_per_step[m];
    }
    if (out_seconds) *out_seconds = fr.seconds;
  });
}

// per-step regularisation targets regs[m] (M*D): replays a scheduled frame whose
// sources were recorded in an audit (SURVEY.md §7 "audit replay")
int ref_reconstruct_frame_regs(const ref_plan_t* p, const float* z, const float* P, const float* init,
                               const float* regs, int A, float* out_image, float* out_est, int* out_cg_per_step) {
  return guarded([&] {
    const ReconPlan plan = to_plan(p);
    const PsfKernel psf = load_psf(P, plan.G);
    const CImage winv = make_weights_inv(plan.Gc, plan.G);
    const size_t D = static_cast<size_t>(plan.G) * plan.G + static_cast<size_t>(plan.J) * plan.Gc * plan.Gc;
    std::vector<Estimate> r;
    for (int m = 0; m < plan.newton_steps; ++m) r.push_back(load_est(regs + 2 * D * m, plan));
    const RegProvider rp = [&r](int m) -> const Estimate& { return r[static_cast<size_t>(m)]; };
    // A WorkerGroup lanes only speed the replay up: the reference is bit-identical across A
    std::unique_ptr<WorkerGroup> wg;
    if (A > 1) wg = std::make_unique<WorkerGroup>(A);
    const FrameResult fr =
        reconstruct_frame(load_z(z, plan), psf, plan, winv, load_est(init, plan), rp, wg.get());
    store_img(fr.image, out_image);
    if (out_est) store_est(fr.est, out_est);
    if (out_cg_per_step) {
      for (size_t m = 0; m < fr.cg_per_step.size(); ++m) out_cg_per_step[m] = fr.cg_per_step[m];
    }
  });
}

int ref_initial_estimate(const ref_plan_t* p, float* out) {
  return guarded([&] { store_est(initial_estimate(to_plan(p)), out); });
}

// Series drivers. samples: F*J*K*S complex64 (raw k-space), angles F*K. plain != 0
// selects reconstruct_series_plain. Outputs: images F*N*N, audit F*(6+M) ints
// {frame, thread, workers, init_src, reg_final_src, reg_src[M]...} + seq F*3
// {start, reg_final, finish}, stats F*{cg_iters} and seconds F.
int ref_reconstruct_series(const ref_plan_t* p, const ref_series_opts_t* o, const float* samples,
                           const double* angles, int F, int K, int S, int plain, float* images,
                           int* audit, uint64_t* seqs, int* cg_iters, double* seconds,
                           double* data_scale) {
  return guarded([&] {
    const ReconPlan plan = to_plan(p);
    std::vector<KSpaceFrame> frames;
    const size_t per = static_cast<size_t>(plan.J) * K * S * 2;
    for (int n = 0; n < F; ++n) {
      frames.push_back(load_frame(samples + n * per, angles + static_cast<size_t>(n) * K, plan.J, K, S, n));
    }
    SeriesOptions opts;
    opts.T = o->T;
    opts.A = o->A;
    opts.sched = TemporalSchedule{o->sched_l, o->sched_o};
    opts.chain = o->chain != 0;
    opts.normalize = o->normalize != 0;
    opts.delay_samples = o->delay_samples;
    const SeriesResult r = plain ? reconstruct_series_plain(frames, plan, opts)
                                 : reconstruct_series(frames, plan, opts);
    const int M = plan.newton_steps;
    for (int n = 0; n < F; ++n) {
      store_img(r.images[static_cast<size_t>(n)], images + static_cast<size_t>(n) * plan.N * plan.N * 2);
      const FrameAudit& a = r.audit[static_cast<size_t>(n)];
      int* row = audit + static_cast<size_t>(n) * (5 + M);
      row[0] = a.frame;
      row[1] = a.thread;
      row[2] = a.workers;
      row[3] = a.init_src;
      row[4] = a.reg_final_src;
      for (int m = 0; m < M; ++m) row[5 + m] = m < static_cast<int>(a.reg_src.size()) ? a.reg_src[static_cast<size_t>(m)] : -1;
      if (seqs) {
        seqs[3 * n + 0] = a.start_seq;
        seqs[3 * n + 1] = a.reg_final_seq;
        seqs[3 * n + 2] = a.finish_seq;
      }
      if (cg_iters) cg_iters[n] = r.stats[static_cast<size_t>(n)].cg_iters;
      if (seconds) seconds[n] = r.stats[static_cast<size_t>(n)].seconds;
    }
    if (data_scale) *data_scale = r.data_scale;
  });
}

// ---- decomposition / scheduling (decomp.cpp) ----------------------------------------

int ref_partition_channels(int J, int A, int* out_pairs) {
  return guarded([&] {
    const auto b = partition_channels(J, A);
    for (size_t a = 0; a < b.size(); ++a) {
      out_pairs[2 * a] = b[a].first;
      out_pairs[2 * a + 1] = b[a].second;
    }
  });
}

// h_choose against a ledger whose completed set is given; frames that are not complete
// get completed by a helper thread after `delay_ms` only if listed in `late` (-1 ends).
int ref_h_choose(int n, int m, int M, int l, int o, const int* completed, int frames,
                 const int* late, int delay_ms, int* out) {
  return guarded([&] {
    CompletionLedger ledger(frames);
    for (int i = 0; i < frames; ++i) {
      if (completed[i]) ledger.mark_complete(i);
    }
    std::thread helper;
    if (late) {
      helper = std::thread([&] {
        std::this_thread::sleep_for(std::chrono::milliseconds(delay_ms));
        for (const int* q = late; *q >= 0; ++q) ledger.mark_complete(*q);
      });
    }
    try {
      *out = h_choose(n, m, M, TemporalSchedule{l, o}, ledger);
    } catch (...) {
      if (helper.joinable()) helper.join();
      throw;
    }
    if (helper.joinable()) helper.join();
  });
}

// ---- autotune (autotune.cpp) ---------------------------------------------------------

int ref_legal_configs(int total, int* out_pairs, int cap) {
  int count = 0;
  const int st = guarded([&] {
    const auto v = legal_configs(total);
    count = static_cast<int>(v.size());
    for (int i = 0; i < count && i < cap; ++i) {
      out_pairs[2 * i] = v[static_cast<size_t>(i)].first;
      out_pairs[2 * i + 1] = v[static_cast<size_t>(i)].second;
    }
  });
  return st == 0 ? count : -st;
}

int ref_frames_bucket(int frames, int* out) {
  return guarded([&] { *out = frames_bucket(frames); });
}

// records: n rows of {mode, N, bucket, J, T, A} ints + runtime_ms doubles
static std::vector<TuningRecord> load_records(const int* rows, const double* ms, int n) {
  std::vector<TuningRecord> db;
  for (int i = 0; i < n; ++i) {
    TuningRecord r;
    r.key = ProtocolKey{static_cast<ImagingMode>(rows[6 * i]), rows[6 * i + 1], rows[6 * i + 2],
                        rows[6 * i + 3]};
    r.T = rows[6 * i + 4];
    r.A = rows[6 * i + 5];
    r.runtime_ms = ms[i];
    db.push_back(r);
  }
  return db;
}

int ref_select_config(const int* key, const int* rows, const double* ms, int n, int* out_ta) {
  return guarded([&] {
    const auto sel = select_config(
        ProtocolKey{static_cast<ImagingMode>(key[0]), key[1], key[2], key[3]}, load_records(rows, ms, n));
    out_ta[0] = sel.first;
    out_ta[1] = sel.second;
  });
}

int ref_learn_step(const int* key, const int* rows, const double* ms, int n, int total,
                   int* out_ta) {
  return guarded([&] {
    const auto sel =
        learn_step(ProtocolKey{static_cast<ImagingMode>(key[0]), key[1], key[2], key[3]},
                   load_records(rows, ms, n), total);
    out_ta[0] = sel.first;
    out_ta[1] = sel.second;
  });
}

}  // extern "C"

extern "C" {

// Timing leg of bench.py's reference arm (BASELINE.md "CPU-baseline plan"): the
// reference's scheduled series driver (reconstruct_series, nlinv.cpp:446-526: T threads
// taking frames round-robin, h_choose / CompletionLedger, A WorkerGroup lanes per
// thread) on frames that were gridded and normalised beforehand, so PSF construction
// and gridding stay outside the timed region as the plan prescribes. The per-thread
// loop below is the reference's own thread_main with prep_series factored out; it calls
// only the reference's public API (reconstruct_frame, h_choose, CompletionLedger,
// WorkerGroup). z: F*J*G*G (normalised), P: U*G*G, psf_idx: F. Outputs: wall seconds of
// the whole run, per-frame wall latency (start -> finish) and per-frame CR iterations.
// Frames [0, first) count as already reconstructed (a continuing series: their
// estimates come from ests_io, F*D complex64); frames [first, F) are timed and their
// estimates written back to ests_io.
int ref_time_series(const ref_plan_t* p, const float* z, const float* P, int U, const int* psf_idx, int F,
                    int first, int T, int A, int sched_l, int sched_o, float* ests_io, double* out_wall,
                    double* out_latency, int* out_cg) {
  return guarded([&] {
    const ReconPlan plan = to_plan(p);
    if (T < 1 || A < 1 || F < 1 || first < 0 || first >= F) throw UsageError("ref_time_series: bad T, A or range");
    const CImage winv = make_weights_inv(plan.Gc, plan.G);
    std::vector<PsfKernel> psfs;
    for (int u = 0; u < U; ++u) psfs.push_back(load_psf(P + 2 * static_cast<size_t>(plan.G) * plan.G * u, plan.G));
    const size_t zsz = 2 * static_cast<size_t>(plan.J) * plan.G * plan.G;
    std::vector<GriddedData> frames;
    for (int n = 0; n < F; ++n) frames.push_back(n >= first ? load_z(z + zsz * n, plan) : GriddedData{});
    const TemporalSchedule sched{sched_l, sched_o};
    const int M = plan.newton_steps;
    const int TT = std::min(T, F - first);
    const size_t D = static_cast<size_t>(plan.G) * plan.G + static_cast<size_t>(plan.J) * plan.Gc * plan.Gc;
    std::vector<Estimate> ests(static_cast<size_t>(F));
    CompletionLedger ledger(F);
    for (int n = 0; n < first; ++n) {
      ests[static_cast<size_t>(n)] = load_est(ests_io + 2 * D * n, plan);
      ledger.mark_complete(n);
    }
    const Estimate unity = initial_estimate(plan);
    std::mutex err_mu;
    std::exception_ptr first_err;
    const auto t0 = std::chrono::steady_clock::now();
    const auto thread_main = [&](int t) {
      try {
        std::unique_ptr<WorkerGroup> wg;
        if (A > 1) wg = std::make_unique<WorkerGroup>(A);
        for (int n = first + t; n < F; n += TT) {
          if (ledger.poisoned()) return;
          const auto ts = std::chrono::steady_clock::now();
          const bool chained = n > 0;
          if (chained && n <= sched.l) ledger.wait_complete(n - 1);
          const int init_src = chained ? h_choose(n, 0, M, sched, ledger) : -1;
          const Estimate init = init_src >= 0 ? ests[static_cast<size_t>(init_src)] : unity;
          const RegProvider reg = [&](int m) -> const Estimate& {
            if (!chained) return unity;
            return ests[static_cast<size_t>(h_choose(n, m, M, sched, ledger))];
          };
          FrameResult fr = reconstruct_frame(frames[static_cast<size_t>(n)], psfs[static_cast<size_t>(psf_idx[n])],
                                             plan, winv, init, reg, wg.get(),
                                             [&](int m) { ledger.mark_step(n, m); });
          ests[static_cast<size_t>(n)] = std::move(fr.est);
          if (out_cg) out_cg[n] = fr.cg_iters;
          if (out_latency) {
            out_latency[n] = std::chrono::duration<double>(std::chrono::steady_clock::now() - ts).count();
          }
          ledger.mark_complete(n);
        }
      } catch (...) {
        {
          std::lock_guard<std::mutex> lock(err_mu);
          if (!first_err) first_err = std::current_exception();
        }
        ledger.poison();
      }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < TT; ++t) pool.emplace_back(thread_main, t);
    thread_main(0);
    for (std::thread& th : pool) th.join();
    if (first_err) std::rethrow_exception(first_err);
    *out_wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (int n = first; n < F; ++n) store_est(ests[static_cast<size_t>(n)], ests_io + 2 * D * n);
  });
}

}  // extern "C"

extern "C" {

// .rti sink (ingest.cpp:240-320): the reference's RtiWriter / RtiReader on flat
// buffers. header9 = {version, N, J_physical, K, U, frames, slices, mode, samples}.
static DatasetHeader rti_header(const int* h) {
  DatasetHeader d;
  d.version = h[0];
  d.N = h[1];
  d.J_physical = h[2];
  d.K = h[3];
  d.U = h[4];
  d.frames = h[5];
  d.slices = h[6];
  d.mode = h[7] == 1 ? ImagingMode::multi_slice : (h[7] == 2 ? ImagingMode::flow : ImagingMode::single_slice);
  d.samples_per_spoke = h[8];
  return d;
}

int ref_rti_write(const char* path, const int* header9, int n, const int* frames, const int* slices,
                  const int* kinds, const float* pixels) {
  return guarded([&] {
    const DatasetHeader h = rti_header(header9);
    RtiWriter w(path, h);
    const size_t npix = static_cast<size_t>(h.N) * h.N;
    for (int i = 0; i < n; ++i) {
      ImageOut img;
      img.frame_index = frames[i];
      img.slice_id = slices[i];
      img.n = h.N;
      img.kind = kinds[i] == 1 ? ImageKind::phase_difference : ImageKind::magnitude;
      img.pixels.assign(pixels + npix * i, pixels + npix * (i + 1));
      w.write_image(img);
    }
    w.close();
  });
}

// header9 out; records {frame, slice, kind} (3 ints each) and pixels (npix each), at
// most max_records; *n_records = the file's record count
int ref_rti_read(const char* path, int* header9, int max_records, int* n_records, int* records, float* pixels) {
  return guarded([&] {
    RtiReader r(path);
    const DatasetHeader& h = r.header();
    const int hv[9] = {h.version, h.N, h.J_physical, h.K, h.U, h.frames, h.slices,
                       h.mode == ImagingMode::multi_slice ? 1 : (h.mode == ImagingMode::flow ? 2 : 0),
                       h.samples_per_spoke};
    std::memcpy(header9, hv, sizeof(hv));
    *n_records = static_cast<int>(r.records().size());
    const size_t npix = static_cast<size_t>(h.N) * h.N;
    for (int i = 0; i < std::min(*n_records, max_records); ++i) {
      const RtiRecord& rec = r.records()[static_cast<size_t>(i)];
      records[3 * i] = rec.frame_index;
      records[3 * i + 1] = rec.slice_id;
      records[3 * i + 2] = rec.kind == ImageKind::phase_difference ? 1 : 0;
      const ImageOut img = r.read_image(static_cast<size_t>(i));
      std::memcpy(pixels + npix * i, img.pixels.data(), sizeof(float) * npix);
    }
  });
}

}  // extern "C"
