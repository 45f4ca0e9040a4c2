// ORACLE TEST INFRASTRUCTURE — not product code.
//
// Minimal stand-in for the FFTW3 (double) surface the reference uses, so the
// reference sources under /root/reference/proj/src compile unmodified in this
// container (FFTW3 is absent here). Only the calls made by
// the reference are provided:
//   fft.cpp:31  fftw_plan_dft_2d(n, n, p, p, sign, FFTW_ESTIMATE | FFTW_UNALIGNED)
//   fft.cpp:59  fftw_execute_dft(plan, in, out)   (in == out, in place)
//   planner.cpp:65  fftw_version
// The transform is FFTW's unnormalised DFT, X[k] = sum_n x[n] exp(sign*2*pi*i*k*n/N)
// per axis, computed in double by oracle/shim/fftw_shim.cpp (mixed-radix
// Cooley-Tukey with exact-table twiddles, direct DFT for prime factors). The
// reference's own KATs (tests/test_fft.cpp: centered-DFT oracle, unitarity,
// adjointness) run against this shim in tests/test_oracle_ref.py.
#pragma once

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct rtn_fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_UNALIGNED (1U << 1)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_destroy_plan(fftw_plan p);
extern const char fftw_version[];

#ifdef __cplusplus
}
#endif
