// Line transforms for the centered 2D FFT on sm_100a.
//
// The reference runs every transform through FFTW in double with two roll passes
// (fft.cpp:41-77). Here a 2D transform is two passes of 1D line transforms; each
// pass is a tile of LPB lines staged in shared memory, and each length-G line is a
// two-step (four-step) Cooley-Tukey transform G = N1 x N2:
//   step 1: N2 threads per line, each an N1-point DFT in registers over the
//           stride-N2 subsequence, then the inter-step twiddle W_G^{n2 k1};
//   step 2: N1 threads per line, each an N2-point DFT in registers over a
//           contiguous (padded) smem block, results in natural order.
// Column lines interleave across the block (coalesced loads of adjacent columns), so
// their step exchange is a block barrier. Row lines own NMAX consecutive thread slots
// in both steps (idle slots when N1 != N2); when NMAX divides 32 a row line lives in
// one warp and its exchange needs only a warp barrier (kernels_impl.cuh: row_line_sync).
// The small DFTs are fully unrolled mixed-radix recursions (radix 2/3/4 closed
// forms, direct sums for other primes) whose twiddles are compile-time constant
// indices into a __constant__ table, so they become constant-bank FMA operands.
//
// Centering (DC at G/2) for even G is folded into sign flips: the centered DFT
// equals (-1)^{G/2} (-1)^p * DFT[(-1)^t x[t]][p]; the (-1)^{G/2} factors of the
// two passes of a 2D transform cancel, so each pass only flips input and output
// signs by parity. The 1/G scale of the unitary 2D transform is applied once, in
// the pass that finishes it.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace rtnb {

// exp(-2 pi i k / N) for N = 1..32, k = 0..N-1, at offset N(N-1)/2, as float4
// {w.x, w.y, -w.y, w.x}: the two packed operands of a twiddle product (cmul_pk).
// Filled from double-precision values by the host (ops.cuh, once per translation unit).
static __constant__ float4 c_small_tw[528];

__host__ __device__ constexpr int small_tw_offset(int n) { return n * (n - 1) / 2; }

__host__ __device__ constexpr bool is_prime_c(int n) {
  if (n < 2) return false;
  for (int d = 2; d * d <= n; ++d)
    if (n % d == 0) return false;
  return true;
}

__host__ __device__ constexpr int split_factor(int n) {
  if (n % 4 == 0 && n > 4) return 4;
  for (int d = 2; d <= n; ++d)
    if (n % d == 0) return d;
  return n;
}

// Packed FP32 (sm_100a FADD2 / FMUL2 / FFMA2): one instruction per complex add and two
// per twiddle product. RTNB_PACKED=0 selects the scalar forms.
#ifndef RTNB_PACKED
#define RTNB_PACKED 1
#endif
__device__ __forceinline__ unsigned long long pk2(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 upk2(unsigned long long v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  return make_float2(lo, hi);
}

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
#if RTNB_PACKED
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
  return upk2(r);
#else
  return make_float2(a.x + b.x, a.y + b.y);
#endif
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
#if RTNB_PACKED
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
  return upk2(r);
#else
  return make_float2(a.x - b.x, a.y - b.y);
#endif
}
// a * w with the twiddle pre-split as t = {w.x, w.y, -w.y, w.x}:
// a.x * (w.x, w.y) + a.y * (-w.y, w.x), a.x and a.y broadcast into both lanes
__device__ __forceinline__ float2 cmul_pk(float2 a, float4 t) {
#if RTNB_PACKED
  unsigned long long m, r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(m) : "l"(pk2(a.x, a.x)), "l"(pk2(t.x, t.y)));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(a.y, a.y)), "l"(pk2(t.z, t.w)), "l"(m));
  return upk2(r);
#else
  return make_float2(a.x * t.x + a.y * t.z, a.x * t.y + a.y * t.w);
#endif
}
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 cneg(float2 a) { return make_float2(-a.x, -a.y); }

// W_N^k for sign S (S = -1 forward: exp(-2 pi i k/N); S = +1 inverse: conjugate)
// (as the packed operand pair of cmul_pk)
template <int N, int S>
__device__ __forceinline__ float4 small_w(int k) {
  const float4 t = c_small_tw[small_tw_offset(N) + (k % N)];
  // conj(w) = {w.x, -w.y, w.y, w.x}
  return S > 0 ? make_float4(t.x, t.z, t.y, t.w) : t;
}

// multiply by -i*S... i.e. by W_4^1 = exp(S * 2 pi i / 4) = S*i
template <int S>
__device__ __forceinline__ float2 mul_w4(float2 a) {
  // S = -1: multiply by -i -> (a.y, -a.x);  S = +1: multiply by i -> (-a.y, a.x)
  return S < 0 ? make_float2(a.y, -a.x) : make_float2(-a.y, a.x);
}

template <int N, int S>
__device__ __forceinline__ void dft(float2 (&x)[N]);

template <int N, int S>
__device__ __forceinline__ void dft_direct(float2 (&x)[N]) {
  float2 y[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    float2 acc = x[0];
#pragma unroll
    for (int t = 1; t < N; ++t) acc = cadd(acc, cmul_pk(x[t], small_w<N, S>((k * t) % N)));
    y[k] = acc;
  }
#pragma unroll
  for (int k = 0; k < N; ++k) x[k] = y[k];
}

template <int N, int S>
__device__ __forceinline__ void dft(float2 (&x)[N]) {
  if constexpr (N == 1) {
    return;
  } else if constexpr (N == 2) {
    const float2 a = x[0], b = x[1];
    x[0] = cadd(a, b);
    x[1] = csub(a, b);
  } else if constexpr (N == 3) {
    // X0 = a+b+c; X1,2 = a - (b+c)/2 -/+ S*i*(sqrt3/2)(b-c)
    const float2 a = x[0], b = x[1], c = x[2];
    const float2 s = cadd(b, c);
    const float2 d = csub(b, c);
    const float h = 0.86602540378443864676f;  // sqrt(3)/2
    const float2 m = make_float2(a.x - 0.5f * s.x, a.y - 0.5f * s.y);
    // S*i*h*d = S*h*(-d.y, d.x)
    const float2 r = make_float2(-S * h * d.y, S * h * d.x);
    x[0] = cadd(a, s);
    x[1] = cadd(m, r);
    x[2] = csub(m, r);
  } else if constexpr (N == 4) {
    const float2 a = x[0], b = x[1], c = x[2], d = x[3];
    const float2 s0 = cadd(a, c), d0 = csub(a, c);
    const float2 s1 = cadd(b, d), d1 = mul_w4<S>(csub(b, d));
    x[0] = cadd(s0, s1);
    x[2] = csub(s0, s1);
    x[1] = cadd(d0, d1);
    x[3] = csub(d0, d1);
  } else if constexpr (is_prime_c(N)) {
    dft_direct<N, S>(x);
  } else {
    // decimation in time, N = P * Q: sub-DFTs of length Q on the P interleaved
    // subsequences, then P-point butterflies with twiddles W_N^{p k}
    constexpr int P = split_factor(N);
    constexpr int Q = N / P;
    float2 sub[P][Q];
#pragma unroll
    for (int p = 0; p < P; ++p) {
#pragma unroll
      for (int q = 0; q < Q; ++q) sub[p][q] = x[p + P * q];
      dft<Q, S>(sub[p]);
    }
#pragma unroll
    for (int k = 0; k < Q; ++k) {
      float2 t[P];
      t[0] = sub[0][k];
#pragma unroll
      for (int p = 1; p < P; ++p) t[p] = cmul_pk(sub[p][k], small_w<N, S>(p * k));
      dft<P, S>(t);
#pragma unroll
      for (int m = 0; m < P; ++m) x[k + Q * m] = t[m];
    }
  }
}

// ---------------------------------------------------------------------------------
// Pruned small DFTs: dft_m<N, S, IN, OUT> computes only the outputs in the bit mask
// OUT from inputs that may be nonzero only in the bit mask IN. The masks are template
// constants, so the recursion drops every zero term and every unneeded butterfly at
// compile time (the window-supported inputs and window-only outputs of the Toeplitz
// and W passes are half of each line; preproc.cpp:438-442). Outputs outside OUT are
// left undefined.
// ---------------------------------------------------------------------------------
__host__ __device__ constexpr uint32_t full_mask(int n) { return n >= 32 ? 0xffffffffu : ((1u << n) - 1u); }

__host__ __device__ constexpr uint32_t range_mask(int lo, int hi) {  // bits [lo, hi)
  uint32_t m = 0;
  for (int i = lo; i < hi; ++i) m |= 1u << i;
  return m;
}

__host__ __device__ constexpr uint32_t dm_sub_in(int N, int P, uint32_t IN, int p) {
  uint32_t m = 0;
  for (int q = 0; q < N / P; ++q)
    if ((IN >> (p + P * q)) & 1u) m |= 1u << q;
  return m;
}
__host__ __device__ constexpr uint32_t dm_sub_out(int N, int P, uint32_t OUT) {
  const int Q = N / P;
  uint32_t m = 0;
  for (int k = 0; k < Q; ++k)
    for (int mm = 0; mm < P; ++mm)
      if ((OUT >> (k + Q * mm)) & 1u) m |= 1u << k;
  return m;
}
__host__ __device__ constexpr uint32_t dm_comb_out(int N, int P, uint32_t OUT, int k) {
  const int Q = N / P;
  uint32_t m = 0;
  for (int mm = 0; mm < P; ++mm)
    if ((OUT >> (k + Q * mm)) & 1u) m |= 1u << mm;
  return m;
}
__host__ __device__ constexpr uint32_t dm_comb_in(int N, int P, uint32_t IN) {
  uint32_t m = 0;
  for (int p = 0; p < P; ++p)
    if (dm_sub_in(N, P, IN, p)) m |= 1u << p;
  return m;
}

template <int I, int E, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < E) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, E>(f);
  }
}

// v * W_N^e (S sign); quarter-turn exponents are sign flips / swaps, no multiply
template <int N, int S, int E>
__device__ __forceinline__ float2 mul_wn(float2 v) {
  constexpr int e = E % N;
  if constexpr (e == 0) {
    return v;
  } else if constexpr ((4 * e) % N == 0) {
    constexpr int qd = (4 * e) / N;  // quarter turns: W^e = (S i)^qd
    if constexpr (qd == 2) {
      return make_float2(-v.x, -v.y);
    } else if constexpr ((qd == 1) == (S > 0)) {
      return make_float2(-v.y, v.x);  // * i
    } else {
      return make_float2(v.y, -v.x);  // * -i
    }
  } else {
    return cmul_pk(v, small_w<N, S>(e));
  }
}

template <int N, int S, uint32_t IN, uint32_t OUT>
__device__ __forceinline__ void dft_m(float2 (&x)[N]) {
  if constexpr (IN == full_mask(N) && OUT == full_mask(N)) {
    dft<N, S>(x);
  } else if constexpr (OUT == 0) {
    return;
  } else if constexpr (IN == 0) {
#pragma unroll
    for (int k = 0; k < N; ++k) x[k] = make_float2(0.f, 0.f);
  } else if constexpr (N <= 4 || is_prime_c(N)) {
    float2 y[N];
    static_for<0, N>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      if constexpr ((OUT >> k) & 1u) {
        float2 acc = make_float2(0.f, 0.f);
        static_for<0, N>([&](auto tc) {
          constexpr int t = decltype(tc)::value;
          if constexpr ((IN >> t) & 1u) acc = cadd(acc, mul_wn<N, S, k * t>(x[t]));
        });
        y[k] = acc;
      }
    });
    static_for<0, N>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      if constexpr ((OUT >> k) & 1u) x[k] = y[k];
    });
  } else {
    constexpr int P = split_factor(N);
    constexpr int Q = N / P;
    constexpr uint32_t SO = dm_sub_out(N, P, OUT);
    constexpr uint32_t CI = dm_comb_in(N, P, IN);
    float2 sub[P][Q];
    static_for<0, P>([&](auto pc) {
      constexpr int p = decltype(pc)::value;
      constexpr uint32_t SI = dm_sub_in(N, P, IN, p);
      if constexpr (SI != 0) {
#pragma unroll
        for (int q = 0; q < Q; ++q) sub[p][q] = x[p + P * q];
        dft_m<Q, S, SI, SO>(sub[p]);
      }
    });
    static_for<0, Q>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      constexpr uint32_t CO = dm_comb_out(N, P, OUT, k);
      if constexpr (CO != 0) {
        float2 t[P];
        static_for<0, P>([&](auto pc) {
          constexpr int p = decltype(pc)::value;
          if constexpr ((CI >> p) & 1u) {
            t[p] = mul_wn<N, S, p * k>(sub[p][k]);
          } else {
            t[p] = make_float2(0.f, 0.f);
          }
        });
        dft_m<P, S, CI, CO>(t);
        static_for<0, P>([&](auto mc) {
          constexpr int m = decltype(mc)::value;
          if constexpr ((CO >> m) & 1u) x[k + Q * m] = t[m];
        });
      }
    });
  }
}

// ---------------------------------------------------------------------------------
// Tile geometry. A block transforms LPB lines of length G = N1*N2 with
// NT = LPB * max(N1, N2) threads and ONE padded shared tile, reused in place:
//   step 1 items (l, n2): the thread loads x[N2*n1 + n2], n1 = 0..N1-1, straight
//     from global memory (fusing the producer's pointwise work), runs an N1-point
//     DFT in registers, applies W_G^{n2 k1} and parks v[k1] at q = N2*k1 + n2;
//   step 2 items (l, k1): after one barrier the thread reads the contiguous block
//     q = N2*k1 + n2, n2 = 0..N2-1, runs an N2-point DFT and holds X[k1 + N1*k2]
//     in registers for the consumer's pointwise work and global stores.
// Element q of line l lives at l*LS + q + q/N2: one pad slot per N2 block keeps the
// step-2 block reads (stride N2+1 across threads) and the natural-order writes
// (stride 1) conflict-free; LS is odd so column tiles spread over banks.
// Item maps: ROWS tiles put the in-line index fastest across threads (a line is
// contiguous in memory), COLS tiles put the line fastest (lines are adjacent
// columns), so every global access of both passes is coalesced.
// ---------------------------------------------------------------------------------
// RS_ (row geometries only): thread slots per row line, a power of two >= NMAX dividing 32,
// so a line whose NMAX does not divide 32 (20, 24, ...) still lives in one warp; 0 = NMAX.
// RG_ (row geometries only): lines of NMAX slots synchronise in groups of RG_ threads
// (lcm(NMAX, 32): whole warps holding whole lines) on named barriers; 0 = none.
template <int N1_, int N2_, int LPB_, int RS_ = 0, int RG_ = 0>
struct LineGeom {
  static constexpr int N1 = N1_;
  static constexpr int N2 = N2_;
  static constexpr int G = N1 * N2;
  static constexpr int LPB = LPB_;
  static constexpr int NMAX = N1 > N2 ? N1 : N2;
  static constexpr int RS = RS_ ? RS_ : NMAX;
  static constexpr int RG = RG_;
  static constexpr int NT = LPB * RS;
  static constexpr int LS0 = G + G / N2;
  static constexpr int LS = (LS0 % 2 == 1) ? LS0 : LS0 + 1;
  static constexpr int SMEM_FLOAT2 = LPB * LS;
  // The field-of-view window [G/4, 3G/4) in the two-step index space: step-1 inputs
  // x[N2 n1 + n2] lie in it for n1 in WIN_N1 when G/4 is a multiple of N2, step-2
  // outputs X[k1 + N1 k2] for k2 in WIN_K2 when G/4 is a multiple of N1 (else: all).
  static constexpr uint32_t ALL_N1 = full_mask(N1);
  static constexpr uint32_t ALL_N2 = full_mask(N2);
  static constexpr uint32_t WIN_N1 = ((G / 4) % N2 == 0) ? range_mask((G / 4) / N2, (3 * G / 4) / N2) : ALL_N1;
  static constexpr uint32_t WIN_K2 = ((G / 4) % N1 == 0) ? range_mask((G / 4) / N1, (3 * G / 4) / N1) : ALL_N2;
  // The coil band [G/2 - Gc/2, G/2 + Gc/2) of the W^-1 / W^-H transforms for Gc = G/4
  // (coil_grid_side, planner.hpp:66): the step-1 inputs a W^-1 line can have, the step-2
  // outputs a W^-H line needs, when the band lies on the DFT grid (else: all)
  static constexpr int OFFC = G / 2 - (G / 4) / 2;
  static constexpr uint32_t GC_N1 =
      (OFFC % N2 == 0 && (G / 4) % N2 == 0) ? range_mask(OFFC / N2, (OFFC + G / 4) / N2) : ALL_N1;
  static constexpr uint32_t GC_K2 =
      (OFFC % N1 == 0 && (G / 4) % N1 == 0) ? range_mask(OFFC / N1, (OFFC + G / 4) / N1) : ALL_N2;
  __device__ __forceinline__ static int a(int l, int q) { return l * LS + q + q / N2; }
};

// item decomposition of threadIdx.x for a step with `n` slots per line
template <class Geo, bool COLS>
// stride > 0 (row lines): line l owns the thread slots [l*stride, (l+1)*stride) whatever the
// step's slot count n, so a line keeps the same threads in both steps
struct Item {
  int l, k;
  bool on;
  __device__ __forceinline__ Item(int tid, int n, int stride = 0) {
    if (COLS) {
      l = tid % Geo::LPB;
      k = tid / Geo::LPB;
      on = tid < Geo::LPB * n;
    } else {
      const int s = stride > 0 ? stride : n;
      l = tid / s;
      k = tid - l * s;
      on = tid < Geo::LPB * s && k < n;
    }
  }
};

// step 1 on registers: v[n1] = x[N2*n1 + n2] -> DFT_N1 -> twiddle W_G^{n2 k1};
// IN: which n1 may be nonzero
template <class Geo, int S, uint32_t IN = Geo::ALL_N1>
// twG: 2G packed twiddles {w.x, w.y, -w.y, w.x} of W_G^e, e < G, for S = -1, then the
// conjugates for S = +1 (twiddles_for, engine.cu)
__device__ __forceinline__ void fft_step1(float2 (&v)[Geo::N1], int n2, const float4* __restrict__ twG) {
  dft_m<Geo::N1, S, IN, Geo::ALL_N1>(v);
  const float4* tw = twG + (S > 0 ? Geo::G : 0);
#pragma unroll
  for (int k1 = 1; k1 < Geo::N1; ++k1) v[k1] = cmul_pk(v[k1], __ldg(tw + n2 * k1));
}

template <class Geo>
__device__ __forceinline__ void park_step1(float2* A, int l, int n2, const float2 (&v)[Geo::N1]) {
#pragma unroll
  for (int k1 = 0; k1 < Geo::N1; ++k1) A[Geo::a(l, Geo::N2 * k1 + n2)] = v[k1];
}

// step 2: u[n2] = parked block of k1 -> DFT_N2 -> u[k2] = X[k1 + N1*k2];
// OUT: which k2 the caller consumes (the others are left undefined)
template <class Geo, int S, uint32_t OUT = Geo::ALL_N2>
__device__ __forceinline__ void fft_step2(const float2* A, int l, int k1, float2 (&u)[Geo::N2]) {
  const float2* src = A + Geo::a(l, Geo::N2 * k1);
#pragma unroll
  for (int n2 = 0; n2 < Geo::N2; ++n2) u[n2] = src[n2];
  dft_m<Geo::N2, S, Geo::ALL_N2, OUT>(u);
}

// A second transform of a step-2 result without reordering: thread k1 holds w[k1 + N1*k2]
// over k2 (natural order). The transform's inner N2-point DFT over k2 runs in its
// registers (IN: which k2 may be nonzero), then the twiddle W_G^{n2 k1} of sign S; the
// result goes back to the thread's own step-2 block, where get_step1 reads it by n2 for
// the outer N1-point DFT, whose output n1 is element N2*n1 + n2 (in place: every thread
// reads and writes only its own block)
template <class Geo, int S, uint32_t IN = Geo::ALL_N2>
__device__ __forceinline__ void inv_inner(float2* A, int l, int k1, float2 (&u)[Geo::N2],
                                          const float4* __restrict__ twG) {
  dft_m<Geo::N2, S, IN, Geo::ALL_N2>(u);
  const float4* tw = twG + (S > 0 ? Geo::G : 0);
  float2* dst = A + Geo::a(l, Geo::N2 * k1);
  dst[0] = u[0];
#pragma unroll
  for (int n2 = 1; n2 < Geo::N2; ++n2) dst[n2] = cmul_pk(u[n2], __ldg(tw + n2 * k1));
}

// natural-order write / step-1-order read, for chaining two transforms in a block
template <class Geo>
__device__ __forceinline__ void put_natural(float2* A, int l, int k1, const float2 (&u)[Geo::N2]) {
#pragma unroll
  for (int k2 = 0; k2 < Geo::N2; ++k2) A[Geo::a(l, k1 + Geo::N1 * k2)] = u[k2];
}
template <class Geo>
__device__ __forceinline__ void get_step1(const float2* A, int l, int n2, float2 (&v)[Geo::N1]) {
#pragma unroll
  for (int n1 = 0; n1 < Geo::N1; ++n1) v[n1] = A[Geo::a(l, Geo::N2 * n1 + n2)];
}

}  // namespace rtnb
