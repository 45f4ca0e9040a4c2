/* rtnlinv_b200 — C ABI of the B200-native NLINV hot path.
 *
 * This is the drop-in boundary for the reference's operator / frame API
 * (proj/include/rtnlinv/nlinv.hpp, fft.hpp, decomp.hpp, autotune.hpp). The
 * reference has no FFI of its own (it links statically, CMakeLists.txt:26-41), so
 * each entry point below names the C++ function it replaces; INTEGRATION.md shows
 * the ctypes binding and the C++ shim that re-throws the reference's exception
 * types from these status codes.
 *
 * Conventions
 *  - Plain pointers and sizes only. Images are row-major complex64 (interleaved
 *    float re, im) exactly like rtnlinv::CImage::v (types.hpp:28-39).
 *  - An Estimate (nlinv.hpp:21-24) is flattened as rho (G*G) followed by chat[j]
 *    (Gc*Gc each, j = 0..J-1): D = G*G + J*Gc*Gc complex entries.
 *  - Buffers are host memory owned by the caller; the context owns every device
 *    buffer, its CUDA stream and its kernels. One context per host thread.
 *  - Return value: 0 ok, 2 UsageError, 3 DataError, 4 SolverError / DecompFault,
 *    5 runtime (CUDA) failure — the reference CLI's exit-code mapping
 *    (rtnlinv_main.cpp:381-391, types.hpp:12-25). rtn_last_error() returns the
 *    message of the calling thread's last failure.
 *  - There is no CPU fallback: every compute entry point runs sm_100a kernels and
 *    fails with status 5 when no CUDA device is usable.
 */
#ifndef RTNLINV_B200_H
#define RTNLINV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* rtnlinv::ReconPlan (planner.hpp:21-35), field for field */
typedef struct rtn_plan_t {
  int N;              /* field of view, pixels per side */
  int G;              /* oversampled grid side (even) */
  int Gc;             /* cropped coil k-space side */
  int J;              /* channels */
  int newton_steps;   /* M */
  float alpha0;
  float alpha_q;
  float alpha_min;
  float cg_tol;       /* relative residual stop; 0 disables */
  int cg_max_iter;
  int cg_iter_budget; /* total CR iterations per frame; 0 = off */
  float prev_damping;
  double gamma;
} rtn_plan_t;

typedef struct rtn_ctx rtn_ctx;

int rtn_abi_version(void);
const char* rtn_last_error(void);
/* 1 if the fused line-FFT kernels cover grid side G (rtnlinv::make_plan sizes) */
int rtn_grid_supported(int G);
int rtn_device_count(void);

/* context = device buffers + stream for one plan on one GPU */
int rtn_ctx_create(const rtn_plan_t* plan, int device, rtn_ctx** out);
void rtn_ctx_destroy(rtn_ctx* ctx);

/* --- fft.hpp:10-38 ------------------------------------------------------------ */
/* centered unitary 2D transform in place; sign -1 = fft::forward, +1 = fft::inverse */
int rtn_fft2(float* data, int n, int sign);
/* transform accounting contexts: 0 other, 1 normal_op, 2 setup, 3 bench */
void rtn_fft_set_ctx(int ctx);
int rtn_fft_get_ctx(void);
void rtn_fft_counts(uint64_t out[4]);
void rtn_fft_reset_counts(void);

/* --- nlinv.hpp:41-59, preproc.hpp:110 -------------------------------------------- */
int rtn_make_weights_inv(int Gc, int G, float* out /* Gc*Gc complex64, real part */);
int rtn_set_psf(rtn_ctx* ctx, const float* P /* G*G */);
int rtn_set_data(rtn_ctx* ctx, const float* z /* J*G*G gridded data (GriddedData::z) */);
int rtn_apply_W_inv(rtn_ctx* ctx, const float* chat /* Gc*Gc */, float* out /* G*G */);
int rtn_apply_W_invH(rtn_ctx* ctx, const float* u /* G*G */, float* out /* Gc*Gc */);
int rtn_toeplitz_apply(rtn_ctx* ctx, float* x /* G*G, in place, uses the context PSF */);

/* --- nlinv.hpp:61-98 ----------------------------------------------------------- */
/* make_step_cache: linearise at estimate x; optional outputs masked rho (G*G), coils (J*G*G) */
int rtn_make_step_cache(rtn_ctx* ctx, const float* x, float* rho_out, float* coils_out);
/* apply_normal at the cached linearisation point */
int rtn_apply_normal(rtn_ctx* ctx, const float* dx, float* out);
/* cg_solve (conjugate residual) at the cached point; residuals: max_iter doubles */
int rtn_cg_solve(rtn_ctx* ctx, const float* rhs, float alpha, float tol, int max_iter, float* x_out,
                 int* iters, double* residuals);
/* newton_step on the context's data (rtn_set_data) and PSF; x updated in place */
int rtn_newton_step(rtn_ctx* ctx, float* x, const float* reg, float alpha, float cg_tol,
                    int cg_max_iter, int* iters, double* residual0);

/* --- nlinv.hpp:102-116 ----------------------------------------------------------- */
/* reconstruct_frame with a fixed regularisation target (reg == NULL: init).
 * image: N*N, est_out: D (nullable), cg_per_step: newton_steps ints (nullable). */
int rtn_reconstruct_frame(rtn_ctx* ctx, const float* init, const float* reg, float* image,
                          float* est_out, int* cg_per_step, double* seconds);

#ifdef __cplusplus
}
#endif

#endif /* RTNLINV_B200_H */
