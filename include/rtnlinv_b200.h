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
/* the exception type behind the calling thread's last failure: 2 UsageError, 3 DataError,
 * 4 SolverError, 6 DecompFault (both reported as status 4), 5 runtime (types.hpp:12-25) */
int rtn_last_error_kind(void);
/* 1 if the fused line-FFT kernels cover grid side G (rtnlinv::make_plan sizes) */
int rtn_grid_supported(int G);
int rtn_device_count(void);

/* context = device buffers + stream for one plan on one GPU */
int rtn_ctx_create(const rtn_plan_t* plan, int device, rtn_ctx** out);
void rtn_ctx_destroy(rtn_ctx* ctx);
/* Channel decomposition (decomp.hpp:25-66 WorkerGroup + partition_channels +
 * all_reduce_sum, passed as `WorkerGroup* wg` to apply_normal / cg_solve /
 * newton_step / reconstruct_frame, nlinv.hpp:73-112): one context over n_devices
 * members (entries may repeat a device), member d owning the channel block
 * partition_channels(J, n_devices, a_cap)[d]. The channel sum is read from peer
 * memory inside the last pass kernel and the CR scalars are summed in member
 * order, so results do not depend on timing. Supports rtn_set_psf, rtn_set_data,
 * rtn_make_step_cache (rho_out = coils_out = NULL), rtn_apply_normal and
 * rtn_reconstruct_frame; the other per-context entry points return 2. */
int rtn_ctx_create_group(const rtn_plan_t* plan, const int* devices, int n_devices, int a_cap, rtn_ctx** out);
/* The same decomposition with one process per GPU (torchrun layout): this process
 * owns member `rank` of `members` on `device`. Each member exports its cross-member
 * buffers as CUDA IPC handles (rtn_ctx_proc_handles: call with out = NULL to get the
 * size), the caller exchanges them (e.g. an all-gather over torch.distributed) and
 * hands every member's handles in rank order to rtn_ctx_proc_attach. Barriers are
 * device-side epoch flags, so every member must make the same calls in the same
 * order. Supports rtn_set_psf, rtn_set_data (full J*G*G arrays; each member takes its
 * block) and rtn_reconstruct_frame (full-layout init / reg; every member returns the
 * full image and estimate). */
int rtn_ctx_create_proc_member(const rtn_plan_t* plan, int device, int rank, int members, int a_cap,
                               rtn_ctx** out);
int rtn_ctx_proc_handles(rtn_ctx* ctx, void* out, int* nbytes);
int rtn_ctx_proc_attach(rtn_ctx* ctx, const void* all, int nbytes);
/* the members' channel blocks, 2*n_devices ints {j0, j1} */
int rtn_ctx_group_blocks(rtn_ctx* ctx, int* out_pairs);

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

/* --- preproc.hpp:81-133: the pre stage on the device ----
 * samples: J*K*S complex64 in KSpaceFrame::samples order [j][k][s]; angles: K
 * spoke angles (rad); S samples per spoke; delay in samples (frame_coords).
 * Out-of-range coordinates return 3 (DataError) like check_coord. */
/* grid_adjoint(frame, plan, delay): density-compensated Kaiser-Bessel gather
 * (bit-identical float accumulation to spread_sample), centered inverse FFT,
 * G / deapodization, window mask. z_out: J*G*G. */
int rtn_grid_adjoint(rtn_ctx* ctx, const float* samples, int J, const double* angles, int K, int S, double delay,
                     float* z_out);
/* the gridded k-space of grid_adjoint before its inverse FFT (J*G*G) */
int rtn_grid_spread(rtn_ctx* ctx, const float* samples, int J, const double* angles, int K, int S, double delay,
                    float* grid_out);
/* build_psf(angles, S, plan) and build_psf_coords(coords, weights, plan): P is G*G */
int rtn_build_psf(rtn_ctx* ctx, const double* angles, int K, int S, float* P_out);
int rtn_build_psf_coords(rtn_ctx* ctx, const double* coords /* 2n: kx, ky */, const double* weights, int n,
                         float* P_out);
/* apply_compression: out (Jv*n) = m (Jv*Jp) x in (Jp*n), FP64 accumulation */
int rtn_apply_compression(rtn_ctx* ctx, const float* m, int Jv, int Jp, const float* in, int n, float* out);
/* --- planner.hpp:37-64 over the device transforms ---------------------------------
 * benchmark_fft: device time (us, CUDA events, min over trials) of one centered 2D
 * forward transform of `batch` images per listed size (the sm_100a line engine;
 * sizes it does not cover run the direct DFT and lose the argmin). select_grid /
 * the table file format are the reference's (planner.cpp:112-183). */
int rtn_benchmark_fft(const int* sizes, int n, int trials, int batch, int device, double* out_us);
int rtn_select_grid(int N, const int* sizes, const double* us, int n, double gamma_min, double gamma_max, int* G,
                    double* gamma);
int rtn_fft_table_save(const char* path, const int* sizes, const double* us, int n, const char* machine,
                       const char* library);
int rtn_fft_table_load(const char* path, int* sizes, double* us, int max_n, int* n, char* machine, char* library,
                       int key_cap);

/* --- pipeline.cpp:60-137 postprocessing on the device (host buffers) ---------------- */
/* magnitude_image: n complex64 -> n float */
int rtn_post_magnitude(const float* images, long long n, float* out);
/* phase_difference_image: arg(even * conj(odd)) */
int rtn_post_phase_difference(const float* even, const float* odd, long long n, float* out);
/* MedianFilter3 over one slice's `frames` magnitude images of npix pixels */
int rtn_post_median3(const float* mags, int frames, long long npix, float* out);

/* PsfCache::angle_key (preproc.cpp:301-313) */
uint64_t rtn_psf_angle_key(const double* angles, int K, int S, int G);

/* --- nlinv.hpp:61-98 ----------------------------------------------------------- */
/* the `winv` argument of the W^-1 functions (nlinv.hpp:41-116): Gc*Gc real weights (the
 * context starts with make_weights_inv(Gc, G)); single-device and in-process group contexts */
int rtn_set_weights(rtn_ctx* ctx, const float* winv);
/* a StepCache given by its parts (nlinv.hpp:53-60): masked rho (G*G) and decoded coils
 * (J*G*G), as make_step_cache returns them; apply_normal / cg_solve then linearise there */
int rtn_set_step_cache(rtn_ctx* ctx, const float* rho, const float* coils);
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
/* reconstruct_frame with a RegProvider (nlinv.hpp:102, `const Estimate& reg(int m)`): the
 * provider returns the host address of step m's regularisation target (D complex64),
 * read before the step starts; NULL keeps the previous step's target (step 0: init).
 * Runs step by step. Not available on process-group members (status 2). */
typedef const float* (*rtn_reg_provider)(int m, void* user);
int rtn_reconstruct_frame_provider(rtn_ctx* ctx, const float* init, rtn_reg_provider reg, void* user,
                                   float* image, float* est_out, int* cg_per_step, double* seconds);

/* --- nlinv.hpp:136-169: series drivers over device-resident frames ------------- */
typedef struct rtn_series rtn_series;
/* SeriesOptions (nlinv.hpp:136-145) + TemporalSchedule (decomp.hpp:70-76).
 * T = frames in flight (one CUDA stream + workspace each); plain != 0 selects
 * reconstruct_series_plain. */
typedef struct rtn_series_opts_t {
  int T;
  int A;
  int sched_l;
  int sched_o;
  int chain;
  int normalize;
  int plain;
  int cluster; /* cluster-fused applications (one thread-block cluster per channel):
                  1 on, 0 off, -1 auto = on when T == 1 (latency mode) */
} rtn_series_opts_t;

int rtn_series_create(rtn_ctx* ctx, int frames, int n_psf, rtn_series** out);
/* temporal decomposition across GPUs in one process: frame worker t runs on
 * devices[t % n_devices]; the store stays on the context's device and estimates,
 * frames and images move peer to peer (needs peer access between the devices) */
int rtn_series_create_multi(rtn_ctx* ctx, int frames, int n_psf, const int* devices, int n_devices,
                            rtn_series** out);
void rtn_series_destroy(rtn_series* s);
/* gridded frames z (count*J*G*G, GriddedData::z per frame) into the device store */
int rtn_series_upload_frames(rtn_series* s, int first, int count, const float* z);
int rtn_series_upload_psf(rtn_series* s, int k, const float* P);
int rtn_series_set_psf_index(rtn_series* s, const int* idx /* frames */);
/* multi-slice acquisitions (pipeline.cpp:315-334, 429-434, 503): the store holds
 * `slices` interleaved chains, store index g = frame * slices + slice (the pipeline's
 * delivery order); each slice has its own ledger, estimates, temporal schedule and
 * normalisation (its frame 0 scaled to norm 100). Frame workers take store indices
 * round-robin across the slices. Default 1. */
int rtn_series_set_slices(rtn_series* s, int slices);
int rtn_series_slice_scale(rtn_series* s, int slice, double* scale);
/* prep_series normalisation: frame 0 scaled to norm 100 (nlinv.cpp:390-400); per slice
 * with rtn_series_set_slices; returns slice 0's scale */
int rtn_series_normalize(rtn_series* s, double* data_scale);
/* reconstruct frames [first, first+count). z_host != NULL streams those frames from
 * host memory inside the call (end-to-end path). Outputs (all nullable):
 * images count*N*N, audit count*(5+M) ints {frame, thread, workers, init_src,
 * reg_final_src, reg_src[M]}, seqs count*3 {start, reg_final, finish}, cg_iters
 * count, gpu_ms count (frame start -> image ready). */
int rtn_series_run(rtn_series* s, const rtn_series_opts_t* opts, int first, int count, const float* z_host,
                   float* images, int* audit, uint64_t* seqs, int* cg_iters, float* gpu_ms);
/* the same series run fed with raw acquisitions (KSpaceFrame per frame,
 * seqsim.hpp:52-65): samples count*Jp*K*S complex64, angles count*K. The pre stage
 * runs on the device on the copy stream: optional coil compression (cmat: J*Jp
 * complex64 apply_compression matrix, NULL when Jp == J), grid_adjoint into the
 * series store, PSFs built once per distinct angle set (PsfCache semantics, at
 * most n_psf of them), prep_series normalisation. */
int rtn_series_run_raw(rtn_series* s, const rtn_series_opts_t* opts, int first, int count, const float* samples,
                       const double* angles, int K, int S, double delay, const float* cmat, int Jp, float* images,
                       int* audit, uint64_t* seqs, int* cg_iters, float* gpu_ms);
/* distinct PSFs built by rtn_series_run_raw so far */
int rtn_series_psf_cache_size(rtn_series* s);
/* PsfCache::save / load (preproc.cpp:346-388): the series' device PSF cache as the
 * reference's "PSFC" v1 sidecar file (interchangeable); 3 on I/O or format errors */
int rtn_series_psf_cache_save(rtn_series* s, const char* path);
int rtn_series_psf_cache_load(rtn_series* s, const char* path);
/* postprocessing of the device-resident images [first, first+count) to host floats:
 * mode 0 magnitude (count*N*N), 1 magnitude + temporal median-of-3 (count*N*N),
 * 2 phase difference of frame pairs (count/2 * N*N) */
int rtn_series_post(rtn_series* s, int first, int count, int mode, float* out);
int rtn_series_images(rtn_series* s, int first, int count, float* images);

/* --- ingest.hpp:105-126: the .rti image sink (RtiWriter format) ---------------------
 * header9 = DatasetHeader {version, N, J_physical, K, U, frames, slices, mode, samples},
 * mode 0 single_slice, 1 multi_slice, 2 flow. Images are N*N float32, kind 0 magnitude,
 * 1 phase_difference; with strict_order frame indices must increase per slice. The
 * files (and the "<path>.idx" sidecar) are interchangeable with the reference's. */
typedef struct rtn_rti rtn_rti;
int rtn_rti_open(const char* path, const int* header9, int strict_order, rtn_rti** out);
int rtn_rti_write(rtn_rti* w, int frame, int slice, int kind, const float* pixels);
int rtn_rti_count(rtn_rti* w);
int rtn_rti_close(rtn_rti* w); /* flushes and frees */
/* the device postprocessing of series images [first, first+count) (mode as
 * rtn_series_post) written to the sink as slice `slice`: frame indices first.., or the
 * pair index first/2.. for phase differences (pipeline.cpp:60-137 + the snk stage) */
int rtn_series_write_rti(rtn_series* s, rtn_rti* w, int first, int count, int mode, int slice);
/* device time (ms) of the last rtn_series_run: CUDA events spanning all worker streams */
float rtn_series_last_span_ms(rtn_series* s);
int rtn_series_estimate(rtn_series* s, int n, float* est /* D */);

/* --- decomp.hpp:25-130: decomposition and scheduling (host logic) ----------------- */
/* cap = largest group (4 = reference kGroupSizeMax, 8 = NVSwitch) */
int rtn_partition_channels(int J, int A, int cap, int* out_pairs /* 2*A */);
/* all_reduce_sum (decomp.hpp:25-30): out = sum of n_terms G*G complex64 images in term
 * order in FP64, one cast to float (bit-identical to the reference), on the device */
int rtn_all_reduce_sum(const float* terms /* n_terms*G*G */, int n_terms, int G, float* out /* G*G */);
typedef struct rtn_ledger rtn_ledger;
int rtn_ledger_create(int frames, rtn_ledger** out);
void rtn_ledger_destroy(rtn_ledger* l);
int rtn_ledger_mark_step(rtn_ledger* l, int n, int m);
int rtn_ledger_mark_complete(rtn_ledger* l, int n);
int rtn_ledger_completed(rtn_ledger* l, int n);
int rtn_ledger_last_step(rtn_ledger* l, int n, int* out);
int rtn_ledger_wait_complete(rtn_ledger* l, int n, int deadline_ms);
void rtn_ledger_poison(rtn_ledger* l);
int rtn_ledger_poisoned(rtn_ledger* l);
uint64_t rtn_ledger_next_seq(rtn_ledger* l);
int rtn_h_choose(int n, int m, int M, int sched_l, int sched_o, rtn_ledger* l, int* out);

/* --- autotune.hpp:13-77 ----------------------------------------------------------- */
/* records: n rows of {mode, N, bucket, J, T, A}; a_cap as in rtn_partition_channels;
 * returns the number of configs (negative status on error) */
int rtn_legal_configs(int total_workers, int a_cap, int* out_pairs, int max_pairs);
int rtn_frames_bucket(int frames, int* out);
int rtn_select_config(const int* key4, const int* rows6, const double* runtime_ms, int n, int* out_ta);
int rtn_learn_step(const int* key4, const int* rows6, const double* runtime_ms, int n, int total_workers,
                   int a_cap, int* out_ta);
int rtn_tunedb_append(const char* path, const int* row6, double runtime_ms, int64_t timestamp);
int rtn_tunedb_load(const char* path, int* rows6, double* runtime_ms, int64_t* timestamps, int max_rows,
                    int* n_rows, int* skipped);

/* --- measurement --------------------------------------------------------------------- */
/* average ms per launch of one kernel class ("colsT", "rows1", "rows2", "colA", "colsW",
 * "cr_fused", "crA", "apply") at the cached linearisation point, and its algorithmic
 * bytes; "<name>:cold" times every launch alone after a write larger than L2 */
int rtn_time_kernel(rtn_ctx* ctx, const char* which, int reps, double* ms, double* bytes);
/* 1 when this plan's grid has the cluster-fused application (latency mode; one
 * thread-block cluster per channel), else 0 (the five-kernel passes always run) */
int rtn_cluster_supported(rtn_ctx* ctx, int* supported);
/* 1 when the budget-mode CR solve on the five-kernel path fuses the recurrence with
 * the next application's W^-1 column pass (k_crA), else 0 */
int rtn_fused_cra(rtn_ctx* ctx, int* on);

#ifdef __cplusplus
}
#endif

#endif /* RTNLINV_B200_H */
