// sm_100a kernels for the NLINV IRGNM hot path.
//
// Every 2D transform of the reference (fft.cpp:41-77, four per channel per normal
// operator application, nlinv.cpp:152-177) is split into row and column passes of
// line transforms (fft_line.cuh) and the passes are fused with the pointwise work
// around them, so one operator application is five kernels:
//
//   colA   W^-1 column pass: chat_j*winv padded into k-space, inverse line FFT,
//          keep the window rows                                  (nlinv.cpp:119-125)
//   rows1  W^-1 row pass -> t_j = c_j drho + rho (W^-1 dchat_j) on the window,
//          then the forward Toeplitz row pass            (nlinv.cpp:160-165, preproc.cpp:436-443)
//   colsT  forward column pass, * P / G, inverse column pass, keep window rows
//          (the whole k-space part of toeplitz_apply, column-local)
//   rows2  inverse Toeplitz row pass -> T_j; rc_j = conj(c_j) T_j, rt_j = conj(rho) T_j;
//          forward W^-H row pass keeping the Gc coil columns  (nlinv.cpp:166-173)
//   colsW  W^-H column pass * winv -> out.chat_j, plus the fixed-order FP64 channel
//          sum out.rho = sum_j rc_j (decomp.cpp:26-39), fused with the CR "+alpha p"
//          (nlinv.cpp:188-192) and the <p, Ap> partial dot product.
//
// Only the window (G/2 x G/2) of image-domain data is ever read or written: the
// reference masks before and after the Toeplitz kernel (preproc.cpp:438, 442), so
// the skipped values are exactly the ones it zeroes. The Newton-step setup
// (nlinv.cpp:243-270) reuses the same kernels in SETUP mode, and the CR vector
// recurrences (nlinv.cpp:197-232) are two fused kernels per iteration with
// device-resident FP64 scalars.
#pragma once

#include <cuda.h>  // CUtensorMap (the k_colsT P tile)
#include <cuda_runtime.h>
#include <math.h>

#include "fft_line.cuh"
#include "kernels.cuh"

namespace rtnb {


namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ float2 flip(float2 v, int t) {
  return (t & 1) ? make_float2(-v.x, -v.y) : v;
}
__device__ __forceinline__ bool in_win(const Dims& d, int r, int c) {
  return r >= d.lo && r < d.lo + d.L && c >= d.lo && c < d.lo + d.L;
}
// the same with the window of a compile-time grid side (Dims: L = G/2, lo = (G - L)/2 = G/4)
template <int G>
__device__ __forceinline__ bool in_win_c(int r, int c) {
  return r >= G / 4 && r < G / 4 + G / 2 && c >= G / 4 && c < G / 4 + G / 2;
}
// exact IEEE float ops (no contraction) where the reference's rounding is mirrored
__device__ __forceinline__ float2 axpy_rn(float2 y, float a, float2 x) {
  return make_float2(__fadd_rn(y.x, __fmul_rn(a, x.x)), __fadd_rn(y.y, __fmul_rn(a, x.y)));
}
__device__ __forceinline__ float2 cmul_rn(float2 a, float2 b) {
  return make_float2(__fsub_rn(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y)),
                     __fadd_rn(__fmul_rn(a.x, b.y), __fmul_rn(a.y, b.x)));
}
__device__ __forceinline__ float2 cjmul_rn(float2 a, float2 b) {  // conj(a) * b
  return make_float2(__fadd_rn(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y)),
                     __fsub_rn(__fmul_rn(a.x, b.y), __fmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double nrm2(float2 v) { return (double)v.x * v.x + (double)v.y * v.y; }

// Programmatic dependent launch: every hot-path kernel is launched with programmatic
// stream serialisation (engine.cu). It first waits for the previous kernel's grid to
// complete and flush (griddepcontrol.wait; a no-op without the attribute), then lets
// the next kernel start launching, so launch latency and block rasterisation of
// kernel k+1 overlap the tail of kernel k inside the CUDA graph.
#ifndef RTNB_PDL_EARLY
#define RTNB_PDL_EARLY 0
#endif
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
#if RTNB_PDL_EARLY
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Grid-wide deterministic sum of K doubles: per-block partials, then the last
// block to arrive reduces them in a fixed order. Returns true in that block,
// with the totals in tot[] (all threads).
template <int K>
__device__ bool grid_reduce(double (&v)[K], double* partials, unsigned int* counter, double (&tot)[K]) {
  static_assert(K <= kMaxReduce, "partials buffer holds kMaxReduce doubles per block");
  __shared__ double red[K][32];
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double s = warp_sum(v[k]);
    if (lane == 0) red[k][warp] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double s = 0;
      for (int w = 0; w < nw; ++w) s += red[k][w];
      partials[blockIdx.x * K + k] = s;
    }
    __threadfence();
    const unsigned int t = atomicAdd(counter, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double s = 0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) s += __ldcg(partials + b * K + k);
    s = warp_sum(s);
    __syncthreads();
    if (lane == 0) red[k][warp] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double t = 0;
    for (int w = 0; w < nw; ++w) t += red[k][w];
    tot[k] = t;
  }
  if (threadIdx.x == 0) *counter = 0;
  __syncthreads();
  return true;
}

// one partial of K doubles per block, in the fixed order of grid_reduce (warp sums, then
// the warps in order), written to out[blockIdx.x * K + k]: the producer half of a
// deferred reduction (DeferRed)
template <int K>
__device__ void block_partial(double (&v)[K], double* out) {
  __shared__ double red[K][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double s = warp_sum(v[k]);
    if (lane == 0) red[k][warp] = s;
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double s = 0;
    for (int w = 0; w < nw; ++w) s += red[threadIdx.x][w];
    out[blockIdx.x * K + threadIdx.x] = s;
  }
}

}  // namespace

// ---------------------------------------------------------------------------------
// Pass kernels. Lines are batched LPB per block (never straddling channels); block
// size Geo::NT. Loads feed the step-1 registers directly, every transform makes one
// padded shared-memory exchange, and pointwise work is applied where the data sits
// in registers (see fft_line.cuh). Threads whose line is past the tile end still
// take part in every barrier.
// ---------------------------------------------------------------------------------

// resident blocks per SM the pass kernels ask the register allocator for
#ifndef RTNB_MINB
#define RTNB_MINB 3
#endif
// resident blocks for a target of M 256-thread blocks per SM, rounded down: 320-thread
// blocks (G = 320) get 2 blocks and 96 registers, spill-free, instead of 3 and 64 with
// spills (C2 +5 %, profiles/r02/ab_bounds_floor.txt); RTNB_BOUNDS_FLOOR=0 rounds up
#ifndef RTNB_BOUNDS_FLOOR
#define RTNB_BOUNDS_FLOOR 1
#endif
#define RTNB_BLOCKS_FOR(M) (RTNB_BOUNDS_FLOOR ? ((M) * 256 / Geo::NT > 0 ? (M) * 256 / Geo::NT : 1) \
                                              : ((M) * 256 + Geo::NT - 1) / Geo::NT)
#define RTNB_PASS_BOUNDS __launch_bounds__(Geo::NT, RTNB_BLOCKS_FOR(RTNB_MINB))
// per-kernel override for the column passes at the coil resolution and k_rows2: 3 (80
// registers at 256 threads) measured +4.5 % at C3 T = 3, +3 % at C2 over 4 (64 registers:
// k_colsW spilled 40 B)
#ifndef RTNB_MINB_LIGHT
#define RTNB_MINB_LIGHT 3
#endif
#define RTNB_PASS_BOUNDS_LIGHT __launch_bounds__(Geo::NT, RTNB_BLOCKS_FOR(RTNB_MINB_LIGHT))
// per-kernel residency targets (256-thread blocks per SM) of the heavy passes
#ifndef RTNB_MINB_ROWS1
#define RTNB_MINB_ROWS1 RTNB_MINB
#endif
#ifndef RTNB_MINB_CRA
#define RTNB_MINB_CRA RTNB_MINB
#endif
#define RTNB_BOUNDS_N(M) __launch_bounds__(Geo::NT, RTNB_BLOCKS_FOR(M))

template <class Geo, bool COLS>
constexpr int kRowStride = (!COLS && (32 % Geo::RS == 0 || Geo::RG)) ? Geo::RS : 0;

#define RTNB_TILE_SETUP(COLS_)                                  \
  extern __shared__ float2 A[];                                 \
  const Item<Geo, COLS_> i1(threadIdx.x, Geo::N2, kRowStride<Geo, COLS_>); \
  const Item<Geo, COLS_> i2(threadIdx.x, Geo::N1, kRowStride<Geo, COLS_>); \
  constexpr int G = Geo::G, N1 = Geo::N1, N2 = Geo::N2;         \
  constexpr int LO = G / 4, LW = G / 2; /* window (Dims lo, L) */ \
  (void)N1;                                                     \
  (void)N2;                                                     \
  (void)LO;                                                     \
  (void)LW

// Barrier between the steps of a row-pass transform. A row line owns the same RS
// consecutive thread slots in both steps (kRowStride; RS = NMAX, or NMAX rounded up to a
// power of two for the 20- and 24-point geometries); when RS divides 32 every line stays
// inside one warp, so the exchange needs only a warp barrier and the warps of a block run
// their lines independently. Column passes spread a line over the block.
template <bool WARP>
__device__ __forceinline__ void step_sync() {
  if constexpr (WARP) {
    __syncwarp();
  } else {
    __syncthreads();
  }
}
template <class Geo>
__device__ __forceinline__ void row_line_sync() {
  if constexpr (32 % Geo::RS == 0) {
    __syncwarp();
  } else if constexpr (Geo::RG > 0) {
    // the lines of this thread's group of RG threads (whole warps, whole lines): named
    // barrier 1 + group index (0 is __syncthreads')
    asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)threadIdx.x / Geo::RG), "r"(Geo::RG) : "memory");
  } else {
    __syncthreads();
  }
}

// W^-1 column pass. Lines: (channel j, coil k-column q). Input chat_j*winv on the
// Gc centered k-rows, output rows [r0, r0+nr) of U_j (G x Gc, row-major).
template <class Geo>
__global__ void RTNB_PASS_BOUNDS_LIGHT k_colA(Dims d, const float* __restrict__ winv,
                                                  const float4* __restrict__ twG,
                                                  const float2* __restrict__ chat, float2* __restrict__ U,
                                                  int r0, int nr, const DevState* st, int use_halt) {
  pdl_enter();
  // the state flags load with the first operands (their L2 round trips overlap); the
  // kernel returns, before writing anything, once they are in
  const int halt = st->status | (use_halt ? st->cr_halt : 0);
  const int zo = nr < 0 ? st->z_out : 0;
  RTNB_TILE_SETUP(true);
  const int tiles = (d.Gc + Geo::LPB - 1) / Geo::LPB;
  const int j = blockIdx.x / tiles;
  const int q0 = (blockIdx.x - j * tiles) * Geo::LPB;
  const int nl = min(Geo::LPB, d.Gc - q0);
  const float2* src = chat + (size_t)j * d.Gc * d.Gc;
  const bool a1 = i1.on && i1.l < nl;
  float2 v[N1];
  if (a1) {
    const int q = q0 + i1.l;
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      const int t = N2 * n1 + i1.k;
      const int i = t - d.off;
      v[n1] = make_float2(0.f, 0.f);
      if (i >= 0 && i < d.Gc) {
        const float w = winv[i * d.Gc + q];
        const float2 c = src[i * d.Gc + q];
        v[n1] = flip(make_float2(c.x * w, c.y * w), t);  // chat * winv.real() (nlinv.cpp:121)
      }
    }
  }
  if (halt) return;
  if (nr < 0) {  // decode: every row when the data has samples outside the window
    r0 = zo ? 0 : LO;
    nr = zo ? G : LW;
  }
  if (a1) {
    if (d.Gc * 4 == G) {  // pruned: only the coil band can be nonzero
      fft_step1<Geo, +1, Geo::GC_N1>(v, i1.k, twG);
    } else {
      fft_step1<Geo, +1>(v, i1.k, twG);
    }
    park_step1<Geo>(A, i1.l, i1.k, v);
  }
  __syncthreads();
  if (i2.on && i2.l < nl) {
    float2 u[N2];
    if (nr == G) {
      fft_step2<Geo, +1>(A, i2.l, i2.k, u);
    } else {
      fft_step2<Geo, +1, Geo::WIN_K2>(A, i2.l, i2.k, u);  // window rows (r0 = lo, nr = L)
    }
    float2* dst = U + (size_t)j * G * d.Gc + q0 + i2.l;
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) {
      const int p = i2.k + N1 * k2;
      if (p >= r0 && p < r0 + nr) dst[(size_t)p * d.Gc] = flip(u[k2], p);
    }
  }
}

// R1_DECODE_WIN: R1_DECODE on the window rows and columns only, unless the frame's data
// has samples outside the window (st->z_out), when it is R1_DECODE
// R1_DECODE_SETUP: R1_DECODE_WIN and, on the window rows, R1_SETUP from the coil rows just
// decoded (the Newton step's decode and its setup's first pass in one launch)
enum Rows1Mode : int { R1_DECODE = 0, R1_OP = 1, R1_SETUP = 2, R1_DECODE_WIN = 3, R1_DECODE_SETUP = 4 };

// Row pass 1.
//  DECODE: rows 0..G-1 of U_j -> inverse row FFT -> coils_j (full G x G, scaled 1/G);
//          channel 0 blocks also write the masked rho (make_step_cache, nlinv.cpp:135-150).
//  OP:     window rows: W^-1 row pass of U_j, t = c_j*drho + rho*a on the window,
//          forward row FFT -> V_j (L x G).
//  SETUP:  window rows: t = rho*c_j (nlinv.cpp:252) -> forward row FFT -> V_j.
template <class Geo, bool DEC = false>
__global__ void RTNB_BOUNDS_N(RTNB_MINB_ROWS1) k_rows1(Dims d, int mode, const float4* __restrict__ twG,
                                                   const float2* __restrict__ U,
                                                   const float2* __restrict__ coils,
                                                   const float2* __restrict__ rhom,
                                                   const float2* __restrict__ drho, float2* __restrict__ V,
                                                   float2* __restrict__ coils_out,
                                                   const float2* __restrict__ rho_src,
                                                   float2* __restrict__ rhom_out, const DevState* st,
                                                   int use_halt) {
  pdl_enter();
  // the state flags load with the first operands (the decode needs them first: its rows
  // depend on st->z_out)
  const int halt = st->status | (use_halt ? st->cr_halt : 0);
  if (DEC && halt) return;
  RTNB_TILE_SETUP(false);
  // DEC: the decode instantiation (R1_DECODE / R1_DECODE_WIN), else R1_OP / R1_SETUP
  bool wdec = false, fset = false;
  if constexpr (DEC) {
    fset = mode == R1_DECODE_SETUP;
    wdec = (mode == R1_DECODE_WIN || fset) && !st->z_out;
    mode = R1_DECODE;
  } else {
    if (mode == R1_DECODE || mode == R1_DECODE_WIN || mode == R1_DECODE_SETUP) return;
  }
  const int nrows = (mode == R1_DECODE) ? G : LW;
  const int row0 = (mode == R1_DECODE) ? 0 : LO;
  const int tiles = (nrows + Geo::LPB - 1) / Geo::LPB;
  const int j = blockIdx.x / tiles;
  const int rl0 = (blockIdx.x - j * tiles) * Geo::LPB;
  const int nl = min(Geo::LPB, nrows - rl0);
  const float2* Uj = U + (size_t)j * G * d.Gc;
  const float2* cj = coils + (size_t)j * G * G;
  if (wdec && (rl0 + nl <= LO || rl0 >= LO + LW)) return;  // a block of rows outside the window
  const int r1 = row0 + rl0 + i1.l, r2 = row0 + rl0 + i2.l;
  const bool a1 = i1.on && i1.l < nl && !(wdec && (r1 < LO || r1 >= LO + LW));
  const bool a2 = i2.on && i2.l < nl && !(wdec && (r2 < LO || r2 >= LO + LW));
  float2 v[N1];
  if (mode != R1_SETUP) {
    if (a1) {
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        const int t = N2 * n1 + i1.k;
        const int qk = t - d.off;
        v[n1] = (qk >= 0 && qk < d.Gc) ? flip(Uj[(size_t)r1 * d.Gc + qk], t) : make_float2(0.f, 0.f);
      }
    }
    if (!DEC && halt) return;
    if (a1) {
      if (d.Gc * 4 == G) {  // pruned: only the coil band can be nonzero
        fft_step1<Geo, +1, Geo::GC_N1>(v, i1.k, twG);
      } else {
        fft_step1<Geo, +1>(v, i1.k, twG);
      }
      park_step1<Geo>(A, i1.l, i1.k, v);
    }
    row_line_sync<Geo>();
    float2 u[N2];
    if (a2) {
      if (DEC && !wdec) {
        fft_step2<Geo, +1>(A, i2.l, i2.k, u);
      } else {
        fft_step2<Geo, +1, Geo::WIN_K2>(A, i2.l, i2.k, u);
      }
      if constexpr (DEC) {
        float2* out = coils_out + (size_t)j * G * G + (size_t)r2 * G;
        const bool wrow = r2 >= LO && r2 < LO + LW;
#pragma unroll
        for (int k2 = 0; k2 < N2; ++k2) {
          const int p = i2.k + N1 * k2;
          float2 w = make_float2(0.f, 0.f);
          if (!(wdec && (p < LO || p >= LO + LW))) {
            const float2 c = cscale(flip(u[k2], p), d.invG);
            out[p] = c;
            const float2 x = rho_src[(size_t)r2 * G + p];
            const bool win = in_win_c<G>(r2, p);
            if (j == 0) rhom_out[(size_t)r2 * G + p] = win ? x : make_float2(0.f, 0.f);
            // the setup's e = rho * c_j on the window (nlinv.cpp:252), as k_rows1 R1_SETUP
            if (fset && win) w = flip(cmul_rn(x, c), p);
          }
          if (fset) u[k2] = wrow ? w : make_float2(0.f, 0.f);
        }
      } else {
#pragma unroll
        for (int k2 = 0; k2 < N2; ++k2) {
          const int p = i2.k + N1 * k2;
          float2 w = make_float2(0.f, 0.f);
          if (p >= LO && p < LO + LW) {
            const size_t e = (size_t)r2 * G + p;
            const float2 aw = cscale(flip(u[k2], p), d.invG);
            // t = c_j * drho + rho * (W^-1 dchat_j)   (nlinv.cpp:163)
            const float2 s1 = cmul_rn(cj[e], drho[e]);
            const float2 s2 = cmul_rn(rhom[e], aw);
            w = flip(make_float2(__fadd_rn(s1.x, s2.x), __fadd_rn(s1.y, s2.y)), p);
          }
          u[k2] = w;
        }
      }
    }
    if constexpr (DEC) {
      if (!fset) return;  // uniform across the block: no barrier follows
      // R1_DECODE_SETUP: the forward Toeplitz row transform of e on the window rows, in
      // the reverse step order (as R1_OP), into V
      const bool w2 = a2 && r2 >= LO && r2 < LO + LW, w1 = a1 && r1 >= LO && r1 < LO + LW;
      if (w2) inv_inner<Geo, -1, Geo::WIN_K2>(A, i2.l, i2.k, u, twG);
      row_line_sync<Geo>();
      if (w1) {
        get_step1<Geo>(A, i1.l, i1.k, v);
        dft_m<N1, -1, Geo::ALL_N1, Geo::ALL_N1>(v);
        float2* Vr = V + (size_t)j * LW * G + (size_t)(r1 - LO) * G;
#pragma unroll
        for (int n1 = 0; n1 < N1; ++n1) {
          const int t = N2 * n1 + i1.k;
          Vr[t] = flip(v[n1], t);
        }
      }
      return;
    }
    // OP: the forward Toeplitz row transform in the reverse step order (inner DFTs over
    // the window k2 on the registers, one exchange, outer DFT over k1)
    if (a2) inv_inner<Geo, -1, Geo::WIN_K2>(A, i2.l, i2.k, u, twG);
    row_line_sync<Geo>();
    if (a1) {
      get_step1<Geo>(A, i1.l, i1.k, v);
      dft_m<N1, -1, Geo::ALL_N1, Geo::ALL_N1>(v);
      float2* Vr = V + (size_t)j * LW * G + (size_t)(rl0 + i1.l) * G;
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        const int t = N2 * n1 + i1.k;
        Vr[t] = flip(v[n1], t);
      }
    }
  } else {
    // SETUP: e = rho * c_j on the window, forward Toeplitz row transform in the usual
    // step order
    if (a1) {
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        const int t = N2 * n1 + i1.k;
        v[n1] = make_float2(0.f, 0.f);
        if (t >= LO && t < LO + LW) {
          const size_t e = (size_t)r1 * G + t;
          v[n1] = flip(cmul_rn(rhom[e], cj[e]), t);  // e = rho * c_j   (nlinv.cpp:252)
        }
      }
    }
    if (halt) return;
    if (a1) {
      fft_step1<Geo, -1, Geo::WIN_N1>(v, i1.k, twG);
      park_step1<Geo>(A, i1.l, i1.k, v);
    }
    row_line_sync<Geo>();
    if (a2) {
      float2 u[N2];
      fft_step2<Geo, -1>(A, i2.l, i2.k, u);
      float2* Vr = V + (size_t)j * LW * G + (size_t)(rl0 + i2.l) * G;
#pragma unroll
      for (int k2 = 0; k2 < N2; ++k2) {
        const int p = i2.k + N1 * k2;
        Vr[p] = flip(u[k2], p);
      }
    }
  }
}

// Bulk asynchronous copies (sm_90+ copy engine: cp.async.bulk with mbarrier completion).
// Used to stage a block's P columns in shared memory at kernel entry, without registers,
// while the forward column transform runs.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// 2D tensor tile (TMA, cp.async.bulk.tensor) into shared memory, completion on an mbarrier
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// RTNB_COLST_TMAP=1: k_colsT stages its LPB P columns (G rows x LPB x 8 bytes) behind the
// FFT tile with TMA (tensor map over P: 8-byte elements, boxes of LPB columns x up to 256
// rows), issued at kernel entry and waited for just before the k-space multiply. Measured
// (profiles/r02/ab_colsT_tma.txt): k_colsT 9.7 -> 10.1 us, C3 T = 3 -2.6 %, C5 -10 % (the
// 32-48 KB tile per block costs co-residency with the other frames' passes); one bulk copy
// per P row instead of the tensor map: 21 us. Off by default; the direct L2 loads win.
#ifndef RTNB_COLST_TMAP
#define RTNB_COLST_TMAP 0
#endif
template <class Geo>
constexpr bool kColsTTmaP = RTNB_COLST_TMAP && Geo::G % Geo::LPB == 0 && (Geo::LPB * 8) % 16 == 0;
template <class Geo>
constexpr int kColsTBoxRows = Geo::G <= 256 ? Geo::G : Geo::G / 2;
template <class Geo>
constexpr size_t colsT_smem_bytes() {
  // the FFT tile, 128 bytes of alignment slack, the P tile, the mbarrier
  return sizeof(float2) * Geo::SMEM_FLOAT2 + (kColsTTmaP<Geo> ? 128 + sizeof(float2) * Geo::G * Geo::LPB + 16 : 0);
}

// Toeplitz column pass: forward column FFT of the window rows of V_j, * P/G, inverse
// column FFT, keep the window rows (in place in V_j). Lines: (j, column q).
template <class Geo>
__global__ void RTNB_PASS_BOUNDS k_colsT(Dims d, const float4* __restrict__ twG,
                                                   const float2* __restrict__ P, float2* __restrict__ V,
                                                   const DevState* st, int use_halt,
                                                   const __grid_constant__ CUtensorMap tmP) {
  pdl_enter();
  const int halt = st->status | (use_halt ? st->cr_halt : 0);  // consumed after the first loads
  RTNB_TILE_SETUP(true);
  constexpr int tiles = (G + Geo::LPB - 1) / Geo::LPB;
  const int j = blockIdx.x / tiles;
  const int q0 = (blockIdx.x - j * tiles) * Geo::LPB;
  const int nl = min(Geo::LPB, G - q0);
  // the block's P columns: G rows of LPB contiguous entries (a 128-byte aligned tile after
  // the FFT tile), loaded by TMA now and waited for just before the k-space multiply
  float2* Ps = A + Geo::SMEM_FLOAT2;
  if constexpr (kColsTTmaP<Geo>) {
    const uint32_t base = smem_u32(Ps);
    Ps += ((base + 127u) & ~127u) - base >> 3;
  }
  uint64_t* pbar = reinterpret_cast<uint64_t*>(Ps + G * Geo::LPB);
  if constexpr (kColsTTmaP<Geo>) {
    if (threadIdx.x == 0 && !halt) {  // (a halted block must not leave copies in flight)
      mbar_init(pbar, 1);
      mbar_expect_tx(pbar, (uint32_t)(sizeof(float2) * G * Geo::LPB));
      constexpr int R = kColsTBoxRows<Geo>;
#pragma unroll
      for (int r0 = 0; r0 < G; r0 += R) tma_load_2d(Ps + r0 * Geo::LPB, &tmP, q0, r0, pbar);
    }
  }
  const bool a1 = i1.on && i1.l < nl, a2 = i2.on && i2.l < nl;
  float2* Vj = V + (size_t)j * LW * G;
  float2 v[N1];
  if (a1) {
    const float2* col = Vj + q0 + i1.l;
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      const int t = N2 * n1 + i1.k;
      v[n1] = (t >= LO && t < LO + LW) ? flip(col[(size_t)(t - LO) * G], t) : make_float2(0.f, 0.f);
    }
  }
  if (halt) return;
  if (a1) {
    fft_step1<Geo, -1, Geo::WIN_N1>(v, i1.k, twG);
    park_step1<Geo>(A, i1.l, i1.k, v);
  }
  __syncthreads();
  float2 u[N2];
  if constexpr (kColsTTmaP<Geo>) mbar_wait(pbar, 0);
  if (a2) {
    fft_step2<Geo, -1>(A, i2.l, i2.k, u);
    // k-space multiply; the forward pass's output flip cancels the inverse pass's
    // input flip
    if constexpr (kColsTTmaP<Geo>) {
      const float2* Pc = Ps + i2.l;
#pragma unroll
      for (int k2 = 0; k2 < N2; ++k2) {
        const int p = i2.k + N1 * k2;
        u[k2] = cscale(cmul(u[k2], Pc[p * Geo::LPB]), d.invG);
      }
    } else {
      const float2* Pc = P + q0 + i2.l;
#pragma unroll
      for (int k2 = 0; k2 < N2; ++k2) {
        const int p = i2.k + N1 * k2;
        u[k2] = cscale(cmul(u[k2], Pc[(size_t)p * G]), d.invG);
      }
    }
    // the inverse transform in the reverse step order: its N2-point DFTs over k2 act on
    // this thread's registers, so no reordering exchange is needed
    inv_inner<Geo, +1>(A, i2.l, i2.k, u, twG);
  }
  __syncthreads();
  if (a1) {
    // outer N1-point DFT over k1 -> x[N2 n1 + n2], window rows only
    get_step1<Geo>(A, i1.l, i1.k, v);
    dft_m<N1, +1, Geo::ALL_N1, Geo::WIN_N1>(v);
    float2* col = Vj + q0 + i1.l;
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      const int t = N2 * n1 + i1.k;
      if (t >= LO && t < LO + LW) col[(size_t)(t - LO) * G] = flip(v[n1], t);
    }
  }
}


struct ColsWArgs {
  int mode;
  float alpha;      // CW_OPALPHA: out += alpha * dx      (nlinv.cpp:190)
  float a_x;        // CW_SETUP: rhs += a_x * x     (float(-alpha), nlinv.cpp:273)
  float a_reg;      // CW_SETUP: rhs += a_reg * reg (float(alpha*damping), nlinv.cpp:274)
  int dot_slot;     // CW_OP*: index into cr.rar for <dx, out> (-1: scal[0])
  const float2* dx;   // OP: the operand (for +alpha dx and the dot)
  const float2* x;    // SETUP: current estimate
  const float2* reg;  // SETUP: regularisation target
  float2* out;        // OP: result vector; SETUP: r
  float2* out2;       // SETUP: p (= r)
  float2* out3;       // SETUP: x_cg (zeroed)
  const float2* ap_prev;  // fused CR: also reduce |out|^2 and Re<ap_prev, out> (nullable)
  double* defer_out;      // fused CR, one device: per-block partials {acc0, aa, pa} for the
                          // next recurrence (DeferRed) instead of the grid reduction
  int win_only_ok;        // fused CR: rho entries outside the window may be skipped when the
                          // step's setup left them exactly zero (see rho_window_only)
};

// Outside the field-of-view window the normal operator's rho output is zero (T is
// masked, preproc.cpp:442), so if the Newton step's rhs.rho is exactly zero there, every
// CR vector (r, p, ap, ar, x_cg) stays exactly zero there for the whole solve
// (nlinv.cpp:188-232 only combines them linearly). The setup records that (the common
// case: window-masked data and estimates); the fused CR kernels then skip those entries.
__device__ __forceinline__ bool rho_window_only(const DevState* st) {
  return st->rho_out_known && !st->rho_out_nz;
}

// combine the normal-operator value n at flat index e with the CR / rhs terms and
// accumulate the reduction the caller needs (Re<dx,out> or |rhs|^2)
__device__ __forceinline__ float2 finish_elem(const ColsWArgs& a, size_t e, float2 n, double& acc, double& aa,
                                             double& pa) {
  if (a.mode == CW_SETUP) {
    float2 v = axpy_rn(n, a.a_x, a.x[e]);
    v = axpy_rn(v, a.a_reg, a.reg[e]);
    a.out[e] = v;
    a.out2[e] = v;
    a.out3[e] = make_float2(0.f, 0.f);
    acc += nrm2(v);
    return v;
  } else {
    float2 v = n;
    const float2 p = a.dx[e];
    if (a.mode == CW_OPALPHA) v = axpy_rn(v, a.alpha, p);
    a.out[e] = v;
    acc += (double)p.x * v.x + (double)p.y * v.y;  // Re <dx, out>
    aa += nrm2(v);
    if (a.ap_prev) {
      const float2 q = a.ap_prev[e];
      pa += (double)q.x * v.x + (double)q.y * v.y;
    }
    return v;
  }
}

// finish_elem's operator branch with its operands dx[e], ap_prev[e] already loaded
// (issued ahead of the value they combine with)
__device__ __forceinline__ float2 finish_op(const ColsWArgs& a, size_t e, float2 n, float2 p, float2 q,
                                           double& acc, double& aa, double& pa) {
  float2 v = n;
  if (a.mode == CW_OPALPHA) v = axpy_rn(v, a.alpha, p);
  a.out[e] = v;
  acc += (double)p.x * v.x + (double)p.y * v.y;
  aa += nrm2(v);
  if (a.ap_prev) pa += (double)q.x * v.x + (double)q.y * v.y;
  return v;
}

// Row pass 2. Block (window row r, channel group h of Geo::LPB channels): inverse
// Toeplitz row pass -> T (window, 1/G); SETUP: e = z - T and the data residual
// (nlinv.cpp:254-256); rc = conj(c_j) T summed over the group's channels in channel
// order in FP64 in shared memory -> RP[h][r] (double2 partial of all_reduce_sum,
// decomp.cpp:26-39; k_colsW adds the groups in order); rt = conj(rho) T -> forward
// W^-H row pass keeping the Gc coil k-columns -> Y_j (L x Gc).
template <class Geo>
__global__ void RTNB_PASS_BOUNDS_LIGHT k_rows2(Dims d, int setup, const float4* __restrict__ twG,
                                                   const float2* __restrict__ V,
                                                   const float2* __restrict__ coils,
                                                   const float2* __restrict__ rhom,
                                                   const float2* __restrict__ z, float2* __restrict__ Y,
                                                   double2* __restrict__ RP, double* partials, DevState* st,
                                                   int use_halt) {
  pdl_enter();
  const int halt = st->status | (use_halt ? st->cr_halt : 0);  // consumed after the first loads
  RTNB_TILE_SETUP(false);
  constexpr int L = G / 2;
  float2* RCs = A + Geo::SMEM_FLOAT2;  // LPB x L channel terms of this row
  const int rl = blockIdx.x % LW;
  const int h = blockIdx.x / LW;
  const int r = LO + rl;
  const int j0 = h * Geo::LPB;
  const int nl = min(Geo::LPB, d.J - j0);
  const bool a1 = i1.on && i1.l < nl, a2 = i2.on && i2.l < nl;
  double resid = 0.0;
  float2 v[N1];
  if (a1) {
    const float2* Vr = V + (size_t)(j0 + i1.l) * LW * G + (size_t)rl * G;
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      const int t = N2 * n1 + i1.k;
      v[n1] = flip(Vr[t], t);
    }
  }
  if (halt) return;
  if (a1) {
    fft_step1<Geo, +1>(v, i1.k, twG);
    park_step1<Geo>(A, i1.l, i1.k, v);
  }
  row_line_sync<Geo>();
  float2 u[N2];
  if (a2) {
    fft_step2<Geo, +1, Geo::WIN_K2>(A, i2.l, i2.k, u);
    const int j = j0 + i2.l;
    const float2* cj = coils + (size_t)j * G * G + (size_t)r * G;
    const float2* zj = z + (size_t)j * G * G + (size_t)r * G;
    const float2* rr = rhom + (size_t)r * G;
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) {
      const int p = i2.k + N1 * k2;
      float2 w = make_float2(0.f, 0.f);
      if (p >= LO && p < LO + LW) {
        float2 T = cscale(flip(u[k2], p), d.invG);
        if (setup) {
          const float2 zz = zj[p];
          T = make_float2(__fsub_rn(zz.x, T.x), __fsub_rn(zz.y, T.y));
          resid += nrm2(T);
        }
        RCs[i2.l * L + (p - LO)] = cjmul_rn(cj[p], T);
        w = flip(cjmul_rn(rr[p], T), p);
      }
      u[k2] = w;
    }
  }
  if constexpr (32 % Geo::NMAX == 0) {
    // the forward W^-H row transform in the reverse step order: inner DFTs over k2 on the
    // registers (only window k2 nonzero), outer DFT over k1 after one exchange
    if (a2) inv_inner<Geo, -1, Geo::WIN_K2>(A, i2.l, i2.k, u, twG);
    row_line_sync<Geo>();
    if (a1) {
      get_step1<Geo>(A, i1.l, i1.k, v);
      if (d.Gc * 4 == G) {  // pruned: only the coil band is kept
        dft_m<N1, -1, Geo::ALL_N1, Geo::GC_N1>(v);
      } else {
        dft_m<N1, -1, Geo::ALL_N1, Geo::ALL_N1>(v);
      }
      float2* Yr = Y + (size_t)(j0 + i1.l) * LW * d.Gc + (size_t)rl * d.Gc;
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        const int p = N2 * n1 + i1.k;
        const int q = p - d.off;
        if (q >= 0 && q < d.Gc) Yr[q] = flip(v[n1], p);
      }
    }
  } else {
    // 20- and 24-point lines: the usual step order spills less
    row_line_sync<Geo>();
    if (a2) put_natural<Geo>(A, i2.l, i2.k, u);
    row_line_sync<Geo>();
    if (a1) {
      get_step1<Geo>(A, i1.l, i1.k, v);
      fft_step1<Geo, -1, Geo::WIN_N1>(v, i1.k, twG);
      park_step1<Geo>(A, i1.l, i1.k, v);
    }
    row_line_sync<Geo>();
    if (a2) {
      if (d.Gc * 4 == G) {  // pruned: only the coil band is kept
        fft_step2<Geo, -1, Geo::GC_K2>(A, i2.l, i2.k, u);
      } else {
        fft_step2<Geo, -1>(A, i2.l, i2.k, u);
      }
      float2* Yr = Y + (size_t)(j0 + i2.l) * LW * d.Gc + (size_t)rl * d.Gc;
#pragma unroll
      for (int k2 = 0; k2 < N2; ++k2) {
        const int p = i2.k + N1 * k2;
        const int q = p - d.off;
        if (q >= 0 && q < d.Gc) Yr[q] = flip(u[k2], p);
      }
    }
  }
  // the group's channel terms, summed in channel order once every line has written them
  // (the block's only barrier between its lines, placed after both transforms)
  __syncthreads();
  if ((int)threadIdx.x < LW) {
    double sx = 0.0, sy = 0.0;
    for (int l = 0; l < nl; ++l) {
      const float2 t = RCs[l * L + threadIdx.x];
      sx += t.x;
      sy += t.y;
    }
    RP[((size_t)h * LW + rl) * LW + threadIdx.x] = make_double2(sx, sy);
  }
  if (setup) {
    double vv[1] = {resid}, tot[1];
    if (grid_reduce<1>(vv, partials, &st->counter, tot) && threadIdx.x == 0) {
      if (d.grp) {
        st->gp[2] = tot[0];  // member partial, summed by k_grp_fin
      } else {
        st->steps[st->cur_step].resid_win = tot[0];
      }
    }
  }
}

// Last pass of an application: W^-H column pass (blocks [0, nbw)) and out.rho
// outside the window (blocks [nbw, grid)); the window part of out.rho came from
// k_rows2, whose reduction partial (st->scal[1]) is folded into the totals here.
template <class Geo>
__global__ void RTNB_PASS_BOUNDS_LIGHT k_colsW(Dims d, ColsWArgs a, const float* __restrict__ winv,
                                                   const float4* __restrict__ twG,
                                                   const float2* __restrict__ Y,
                                                   const double2* __restrict__ RP,
                                                   const float2* __restrict__ coils,
                                                   const float2* __restrict__ z, int nbw,
                                                   double* partials, DevState* st, CrScalars cr,
                                                   int use_halt, GroupView gv) {
  pdl_enter();
  const int halt = st->status | (use_halt ? st->cr_halt : 0);  // consumed after the first loads
  RTNB_TILE_SETUP(true);
  const int D0 = G * G;
  double acc0 = 0.0, acc1 = 0.0, aa = 0.0, pa = 0.0;
  if ((int)blockIdx.x < nbw) {
    const int tiles = (d.Gc + Geo::LPB - 1) / Geo::LPB;
    const int j = blockIdx.x / tiles;
    const int q0 = (blockIdx.x - j * tiles) * Geo::LPB;
    const int nl = min(Geo::LPB, d.Gc - q0);
    const bool a1 = i1.on && i1.l < nl, a2 = i2.on && i2.l < nl;
    // pruned band (Gc = G/4 on the DFT grid): this thread's outputs are the step-2 slots
    // k2 in [GK0, GK0 + GKN); their CR operands are loaded before the transform
    constexpr bool kBand = Geo::GC_K2 != Geo::ALL_N2;
    constexpr int GK0 = (G / 2 - (G / 4) / 2) / N1, GKN = kBand ? (G / 4) / N1 : 1;
    const bool band = kBand && d.Gc * 4 == G && a.mode != CW_SETUP;
    const size_t cbase = (size_t)D0 + (size_t)j * d.Gc * d.Gc;
    float2 pdx[GKN], pap[GKN];
    if (band && a2) {
      const int q = q0 + i2.l;
#pragma unroll
      for (int kk = 0; kk < GKN; ++kk) {
        const size_t e = cbase + (size_t)(i2.k + N1 * (GK0 + kk) - d.off) * d.Gc + q;
        pdx[kk] = a.dx[e];
        pap[kk] = a.ap_prev ? a.ap_prev[e] : make_float2(0.f, 0.f);
      }
    }
    float2 v[N1];
    if (a1) {
      const float2* col = Y + (size_t)j * LW * d.Gc + q0 + i1.l;
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        const int t = N2 * n1 + i1.k;
        v[n1] = (t >= LO && t < LO + LW) ? flip(col[(size_t)(t - LO) * d.Gc], t) : make_float2(0.f, 0.f);
      }
    }
    if (halt) return;
    if (a1) {
      fft_step1<Geo, -1, Geo::WIN_N1>(v, i1.k, twG);
      park_step1<Geo>(A, i1.l, i1.k, v);
    }
    __syncthreads();
    if (a2) {
      float2 u[N2];
      if (d.Gc * 4 == G) {  // pruned: only the coil band is kept
        fft_step2<Geo, -1, Geo::GC_K2>(A, i2.l, i2.k, u);
      } else {
        fft_step2<Geo, -1>(A, i2.l, i2.k, u);
      }
      const int q = q0 + i2.l;
      if (band) {
#pragma unroll
        for (int kk = 0; kk < GKN; ++kk) {
          const int p = i2.k + N1 * (GK0 + kk);
          const int e = (p - d.off) * d.Gc + q;
          const float w = winv[e];
          const float2 f = cscale(flip(u[GK0 + kk], p), d.invG);
          // crop_k(FFT(u)) * winv   (nlinv.cpp:127-133)
          finish_op(a, cbase + e, make_float2(f.x * w, f.y * w), pdx[kk], pap[kk], acc0, aa, pa);
        }
      } else {
#pragma unroll
        for (int k2 = 0; k2 < N2; ++k2) {
          const int p = i2.k + N1 * k2;
          const int i = p - d.off;
          if (i >= 0 && i < d.Gc) {
            const int e = i * d.Gc + q;
            const float w = winv[e];
            const float2 f = cscale(flip(u[k2], p), d.invG);
            // crop_k(FFT(u)) * winv   (nlinv.cpp:127-133)
            finish_elem(a, cbase + e, make_float2(f.x * w, f.y * w), acc0, aa, pa);
          }
        }
      }
    }
  } else {
    if (halt) return;
    // window: the channel-group partials of k_rows2 added in group order. Outside the
    // window T is masked to zero (preproc.cpp:442), so out.rho there is only the SETUP
    // data term sum_j conj(c_j) z_j, in channel order in FP64
    const int H = d.H;
    double dummy0 = 0.0, dummy1 = 0.0, dummy2 = 0.0;
    const bool win_only = a.mode != CW_SETUP && a.win_only_ok && rho_window_only(st);
    const int nv = win_only ? LW * LW : D0;
    int nz = 0;  // SETUP: a nonzero rhs.rho entry outside the window
    for (int v = (blockIdx.x - nbw) * blockDim.x + threadIdx.x; v < nv; v += (gridDim.x - nbw) * blockDim.x) {
      int e, r, c;
      if (win_only) {
        r = LO + v / LW;
        c = LO + v - (v / LW) * LW;
        e = r * G + c;
      } else {
        e = v;
        r = e / G;
        c = e - (e / G) * G;
      }
      double sx = 0.0, sy = 0.0;
      if (d.grp) {
        // channel decomposition: every member's partials, in member order, loaded
        // from the peers' memory (the all_reduce_sum of decomp.cpp:26-39)
        if (in_win_c<G>(r, c)) {
          const size_t w = (size_t)(r - LO) * LW + (c - LO);
          for (int m = 0; m < gv.A; ++m) {
            for (int h = 0; h < gv.h[m]; ++h) {
              const double2 t = __ldcg(gv.rp[m] + (size_t)h * LW * LW + w);
              sx += t.x;
              sy += t.y;
            }
          }
        } else if (a.mode == CW_SETUP) {
          for (int m = 0; m < gv.A; ++m) {
            const double2 t = __ldcg(gv.rpo[m] + e);
            sx += t.x;
            sy += t.y;
          }
        }
        // the rho part of every dot product is replicated: counted on one member
        float2 o;
        if (d.count_rho) {
          o = finish_elem(a, (size_t)e, make_float2((float)sx, (float)sy), acc0, aa, pa);
        } else {
          o = finish_elem(a, (size_t)e, make_float2((float)sx, (float)sy), dummy0, dummy1, dummy2);
        }
        if (a.mode == CW_SETUP && !in_win_c<G>(r, c) && (o.x != 0.f || o.y != 0.f)) nz = 1;
        continue;
      }
      const bool opm = a.mode != CW_SETUP;
      float2 pdx = make_float2(0.f, 0.f), pap = make_float2(0.f, 0.f);
      if (opm) {
        pdx = a.dx[e];
        if (a.ap_prev) pap = a.ap_prev[e];
      }
      if (in_win_c<G>(r, c)) {
        const double2* src = RP + (size_t)(r - LO) * LW + (c - LO);
        for (int h = 0; h < H; ++h) {
          const double2 t = src[(size_t)h * LW * LW];
          sx += t.x;
          sy += t.y;
        }
      } else if (a.mode == CW_SETUP && st->z_out) {
        for (int j = 0; j < d.J; ++j) {
          const float2 zz = z[(size_t)j * D0 + e];
          const float2 v = cjmul_rn(coils[(size_t)j * D0 + e], zz);
          sx += v.x;
          sy += v.y;
          acc1 += nrm2(zz);
        }
      }
      const float2 n = make_float2((float)sx, (float)sy);
      const float2 o = opm ? finish_op(a, (size_t)e, n, pdx, pap, acc0, aa, pa)
                           : finish_elem(a, (size_t)e, n, acc0, aa, pa);
      if (a.mode == CW_SETUP && !in_win_c<G>(r, c) && (o.x != 0.f || o.y != 0.f)) nz = 1;
    }
    if (a.mode == CW_SETUP && __syncthreads_or(nz) && threadIdx.x == 0) atomicOr(&st->rho_out_nz, 1);
  }
  if (a.defer_out) {
    double dv[3] = {acc0, aa, pa};
    block_partial<3>(dv, a.defer_out);
    return;
  }
  double vv[4] = {acc0, acc1, aa, pa}, tot[4];
  if (grid_reduce<4>(vv, partials, &st->counter, tot) && threadIdx.x == 0) {
    const double total = tot[0];
    if (a.mode == CW_SETUP) st->rho_out_known = 1;  // every block's atomicOr precedes its ticket
    if (d.grp) {
      // member partials; k_grp_fin forms the totals once every member has them
      if (a.mode == CW_SETUP) {
        st->gp[0] = total;
      } else if (a.dot_slot >= 0) {
        cr.pcw[3 * a.dot_slot + 0] = total;
        cr.pcw[3 * a.dot_slot + 1] = tot[2];
        cr.pcw[3 * a.dot_slot + 2] = tot[3];
      } else {
        st->scal[0] = total;
      }
    } else if (a.mode == CW_SETUP) {
      StepRec& s = st->steps[st->cur_step];
      s.rhs_nrm2 = total;
      s.resid_out = tot[1];
      const double rn = sqrt(total);
      // cg_solve entry checks (nlinv.cpp:184-186)
      if (!isfinite(rn)) {
        st->status = ST_SOLVER;
        st->cr_halt = 1;
      } else if (rn == 0.0) {
        s.zero_rhs = 1;
        st->cr_halt = 1;
      }
    } else if (a.dot_slot >= 0) {
      cr.rar[a.dot_slot] = total;
      cr.saa[a.dot_slot] = tot[2];
      cr.spa[a.dot_slot] = tot[3];
    } else {
      st->scal[0] = total;
    }
  }
}

// CR step coefficients of iteration `it` of the fused recurrence (k_cr_fused, k_crA):
// b = rar[it]/rar[it-1] (0 for the priming step), the step denominator |ap|^2 from the
// previous exact norm and the application's dots, and a = rar[it]/|ap|^2. Returns false
// (after recording the decision once) when the iteration must not run.
struct CrCoef {
  double b, a;
  bool upd;
};
__device__ __forceinline__ bool cr_coef(DevState* st, const CrScalars& cr, int it, float tol, CrCoef& c) {
  const double rar_new = cr.rar[it];
  double b = 0.0, denom = cr.saa[0];
  if (it > 0) {
    const double rar_old = cr.rar[it - 1];
    b = (rar_old != 0.0) ? rar_new / rar_old : 0.0;
    denom = b * b * cr.ap2[it - 1] + 2.0 * b * cr.spa[it] + cr.saa[it];
  }
  if (!isfinite(denom) || !isfinite(rar_new)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->status = ST_SOLVER;
      st->cr_halt = 1;
    }
    return false;
  }
  if (denom <= 0.0 && tol > 0.0f) {
    if (blockIdx.x == 0 && threadIdx.x == 0) st->cr_halt = 1;
    return false;
  }
  c.b = b;
  c.upd = denom > 0.0;
  c.a = c.upd ? rar_new / denom : 0.0;
  return true;
}

// member-order sum of one scalar partial over a channel group's members
__device__ __forceinline__ double grp_sum(const GroupScal& g, const double* const* base, int idx) {
  double t = 0.0;
  for (int m = 0; m < g.A; ++m) t += __ldcg(base[m] + idx);
  return t;
}

// Entry of a fused recurrence kernel, all threads of the block: the frame / CR state
// checks, the totals of the deferred reductions (DeferRed) -- the previous iteration's
// tail (|ap|^2 for the denominator, |r|, the iteration count and the tolerance stop,
// as cr_fused_tail) and this iteration's dots -- then the step coefficients (cr_coef).
// The block loads and sums the partials, thread 0 decides (block 0 records), the block
// reads the decision from shared memory. Returns false when the iteration must not run.
// kGrp: the channel-group branch is compiled in (k_crA never runs on a group member).
template <bool kGrp = true>
__device__ inline bool cr_begin(DevState* st, const CrScalars& cr, int it, float tol, const DeferRed& dr, CrCoef& c) {
  if (kGrp && dr.grp) {
    // channel group: k_grp_fin's member-order totals and decisions (the previous
    // iteration's tail, this application's dots), then the step coefficients; every block
    // of every member sums the same member partials in the same order
    __shared__ double g_c[2];
    __shared__ int g_ok;
    __shared__ double g_part[32][3];
    __shared__ double g_tot[3];
    if (dr.grp == 2) {
      // every member's per-block dot partials: each member's blocks summed by the whole
      // block (a stride per thread, the warp trees, thread 0 the warps in order), then
      // the members in order
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      for (int m = 0; m < dr.gs.A; ++m) {
        double t[3] = {0.0, 0.0, 0.0};
        for (int b = threadIdx.x; b < dr.gnw[m]; b += blockDim.x) {
#pragma unroll
          for (int k = 0; k < 3; ++k) t[k] += __ldcg(dr.gw[m] + 3 * b + k);
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const double v = warp_sum(t[k]);
          if (lane == 0) g_part[warp][k] = v;
        }
        __syncthreads();
        if (threadIdx.x < 3) {
          double u = 0.0;
          for (int w = 0; w < (int)((blockDim.x + 31) >> 5); ++w) u += g_part[w][threadIdx.x];
          g_tot[threadIdx.x] = m ? g_tot[threadIdx.x] + u : u;
        }
        __syncthreads();
      }
    }
    if (threadIdx.x == 0) {
      int ok = !(st->status || st->cr_halt);
      const bool rec = blockIdx.x == 0;
      double ap2 = 0.0, rar_old = 0.0;
      if (ok && it > 0) {
        rar_old = cr.rar[it - 1];
        ap2 = grp_sum(dr.gs, dr.gs.pcr, 2 * (it - 1));
        const double rn = sqrt(grp_sum(dr.gs, dr.gs.pcr, 2 * (it - 1) + 1));
        if (rec) {
          cr.ap2[it - 1] = ap2;
          cr.rn[it] = rn;
        }
        if (!isfinite(rn)) {
          if (rec) {
            st->status = ST_SOLVER;
            st->cr_halt = 1;
          }
          ok = 0;
        } else {
          StepRec& s = st->steps[st->cur_step];
          if (rec) s.iters = it;
          if (tol > 0.0f && (rn == 0.0 || rn <= (double)tol * sqrt(s.rhs_nrm2))) {
            if (rec) st->cr_halt = 1;
            ok = 0;
          }
        }
      }
      double a = 0.0, b = 0.0;
      if (ok) {
        const double rar = dr.grp == 2 ? g_tot[0] : grp_sum(dr.gs, dr.gs.pcw, 3 * it + 0);
        const double saa = dr.grp == 2 ? g_tot[1] : grp_sum(dr.gs, dr.gs.pcw, 3 * it + 1);
        const double spa = dr.grp == 2 ? g_tot[2] : grp_sum(dr.gs, dr.gs.pcw, 3 * it + 2);
        if (rec) {
          cr.rar[it] = rar;
          cr.saa[it] = saa;
          cr.spa[it] = spa;
        }
        double denom = saa;
        if (it > 0) {
          b = (rar_old != 0.0) ? rar / rar_old : 0.0;
          denom = b * b * ap2 + 2.0 * b * spa + saa;
        }
        if (!isfinite(denom) || !isfinite(rar)) {
          if (rec) {
            st->status = ST_SOLVER;
            st->cr_halt = 1;
          }
          ok = 0;
        } else if (denom <= 0.0 && tol > 0.0f) {
          if (rec) st->cr_halt = 1;
          ok = 0;
        } else {
          ok = denom > 0.0 ? 2 : 1;
          a = denom > 0.0 ? rar / denom : 0.0;
        }
      }
      g_c[0] = b;
      g_c[1] = a;
      g_ok = ok;
    }
    __syncthreads();
    if (!g_ok) return false;
    c.b = g_c[0];
    c.a = g_c[1];
    c.upd = g_ok == 2;
    return true;
  }
  if (!dr.nw && !dr.nc) {
    if (st->status || st->cr_halt) return false;
    return cr_coef(st, cr, it, tol, c);
  }
  __shared__ double s_c[2];
  __shared__ int s_ok;
  __shared__ double s_part[32][5];
  // the state and scalars thread 0 decides with, loaded before the partials
  int status = 0, halt = 0;
  double rar_old = 0.0, rhs2 = 0.0;
  if (threadIdx.x == 0) {
    status = st->status;
    halt = st->cr_halt;
    rar_old = it > 0 ? cr.rar[it - 1] : 0.0;
    rhs2 = tol > 0.0f ? st->steps[st->cur_step].rhs_nrm2 : 0.0;
  }
  {
    // every thread of the block sums a stride of the partials (one round trip), the warps
    // reduce, thread 0 adds the warp totals in warp order: the same totals in every block
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    {
      double t[3] = {0.0, 0.0, 0.0};
      for (int b = threadIdx.x; b < dr.nw; b += blockDim.x) {
#pragma unroll
        for (int k = 0; k < 3; ++k) t[k] += __ldcg(dr.w + 3 * b + k);
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double v = warp_sum(t[k]);
        if (lane == 0) s_part[warp][k] = v;
      }
    }
    {
      double t[2] = {0.0, 0.0};
      for (int b = threadIdx.x; b < dr.nc; b += blockDim.x) {
#pragma unroll
        for (int k = 0; k < 2; ++k) t[k] += __ldcg(dr.c + 2 * b + k);
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const double v = warp_sum(t[k]);
        if (lane == 0) s_part[warp][3 + k] = v;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    double wt[3] = {0.0, 0.0, 0.0}, ct[2] = {0.0, 0.0};
    if (threadIdx.x == 0) {
      const int nwarp = (blockDim.x + 31) >> 5;
      for (int w = 0; w < nwarp; ++w) {
        wt[0] += s_part[w][0];
        wt[1] += s_part[w][1];
        wt[2] += s_part[w][2];
        ct[0] += s_part[w][3];
        ct[1] += s_part[w][4];
      }
    }
    if (threadIdx.x == 0) {
      const bool rec = blockIdx.x == 0;
      int ok = !(status || halt);
      double ap2_prev = 0.0;
      if (ok && dr.nc) {
        // iteration it-1's tail (cr_fused_tail, nlinv.cpp:205-220)
        ap2_prev = ct[0];
        const double rn = sqrt(ct[1]);
        if (rec) {
          cr.ap2[it - 1] = ap2_prev;
          cr.rn[it] = rn;
        }
        if (!isfinite(rn)) {
          if (rec) {
            st->status = ST_SOLVER;
            st->cr_halt = 1;
          }
          ok = 0;
        } else {
          if (rec) st->steps[st->cur_step].iters = it;
          if (tol > 0.0f && (rn == 0.0 || rn <= (double)tol * sqrt(rhs2))) {
            if (rec) st->cr_halt = 1;
            ok = 0;
          }
        }
      } else if (ok && it > 0) {
        ap2_prev = cr.ap2[it - 1];
      }
      double a = 0.0, b = 0.0;
      if (ok) {
        double rar_new, saa, spa;
        if (dr.nw) {
          rar_new = wt[0];
          saa = wt[1];
          spa = wt[2];
          if (rec) {
            cr.rar[it] = rar_new;
            cr.saa[it] = saa;
            cr.spa[it] = spa;
          }
        } else {
          rar_new = cr.rar[it];
          saa = cr.saa[it];
          spa = cr.spa[it];
        }
        // cr_coef with the totals in registers
        double denom = saa;
        if (it > 0) {
          b = (rar_old != 0.0) ? rar_new / rar_old : 0.0;
          denom = b * b * ap2_prev + 2.0 * b * spa + saa;
        }
        if (!isfinite(denom) || !isfinite(rar_new)) {
          if (rec) {
            st->status = ST_SOLVER;
            st->cr_halt = 1;
          }
          ok = 0;
        } else if (denom <= 0.0 && tol > 0.0f) {
          if (rec) st->cr_halt = 1;
          ok = 0;
        } else {
          ok = denom > 0.0 ? 2 : 1;  // 2: the update runs (upd)
          a = denom > 0.0 ? rar_new / denom : 0.0;
        }
      }
      s_c[0] = b;
      s_c[1] = a;
      s_ok = ok;
    }
  }
  __syncthreads();
  if (!s_ok) return false;
  c.b = s_c[0];
  c.a = s_c[1];
  c.upd = s_ok == 2;
  return true;
}

// the single-device epilogue of the fused recurrence (last block): |ap|^2 for the next
// iteration's denominator, |r|, iteration count, tolerance stop (nlinv.cpp:205-220)
__device__ __forceinline__ void cr_fused_tail(DevState* st, const CrScalars& cr, int it, float tol,
                                              double ap2, double r2) {
  cr.ap2[it] = ap2;
  const double rn = sqrt(r2);
  cr.rn[it + 1] = rn;
  StepRec& s = st->steps[st->cur_step];
  if (!isfinite(rn)) {
    st->status = ST_SOLVER;
    st->cr_halt = 1;
    return;
  }
  s.iters = it + 1;
  const double target = (double)tol * sqrt(s.rhs_nrm2);
  if (tol > 0.0f && (rn == 0.0 || rn <= target)) st->cr_halt = 1;
}

// one CR vector entry of the fused recurrence: p = b p + r; ap = b ap + ar;
// x += a p; r -= a ap (nlinv.cpp:205-230, the reference's float roundings). Returns r.
__device__ __forceinline__ float2 cr_update(float2 pv, float2 apv, float2 rv, float2 arv, float2 xv, float bf,
                                            float af, float naf, bool upd, float2& np, float2& nap,
                                            float2& nx) {
  np = make_float2(__fadd_rn(__fmul_rn(pv.x, bf), rv.x), __fadd_rn(__fmul_rn(pv.y, bf), rv.y));
  nap = make_float2(__fadd_rn(__fmul_rn(apv.x, bf), arv.x), __fadd_rn(__fmul_rn(apv.y, bf), arv.y));
  if (!upd) return rv;
  nx = axpy_rn(xv, af, np);
  return axpy_rn(rv, naf, nap);
}

// Fused CR recurrence of iteration `it` (as k_cr_fused) + the W^-1 column pass (k_colA)
// of the next application, whose operand is the updated residual r. Blocks [0, nbc) own
// one (channel j, coil column tile) as k_colA does: each thread updates the CR vectors on
// the coil entries of its column's step-1 subsequence and transforms r_new * winv
// straight from its registers into U. Blocks [nbc, grid) update the rho entries (the
// window only when the step's setup left them zero outside, rho_window_only). The same
// values as k_cr_fused followed by k_colA: one launch, and the r re-read, fewer per
// iteration.
template <class Geo>
__global__ void RTNB_BOUNDS_N(RTNB_MINB_CRA) k_crA(Dims d, float2* __restrict__ x, float2* __restrict__ r,
                                       float2* __restrict__ p, float2* __restrict__ ap,
                                       const float2* __restrict__ ar, const float* __restrict__ winv,
                                       const float4* __restrict__ twG, float2* __restrict__ U, int nbc,
                                       double* partials, DevState* st, CrScalars cr, int it, float tol,
                                       DeferRed dr) {
  pdl_enter();
  extern __shared__ float2 A[];
  constexpr int G = Geo::G, N1 = Geo::N1, N2 = Geo::N2, LO = G / 4, LW = G / 2;
  const int G2 = G * G;
  // coil blocks: the band's CR operands do not depend on the step coefficients, so their
  // loads are issued before the coefficients are formed (overlapping cr_begin's reads of
  // the deferred partials)
  constexpr uint32_t BAND = Geo::GC_N1;
  constexpr bool kBand = BAND != Geo::ALL_N1;
  constexpr int B0 = kBand ? __builtin_ctz(BAND) : 0, BN = kBand ? __builtin_popcount(BAND) : 1;
  const Item<Geo, true> i1(threadIdx.x, N2), i2(threadIdx.x, N1);
  const int tiles = (d.Gc + Geo::LPB - 1) / Geo::LPB;
  const int j = blockIdx.x / tiles;
  const int q0 = (blockIdx.x - j * tiles) * Geo::LPB;
  const int nl = min(Geo::LPB, d.Gc - q0);
  const size_t cbase = (size_t)G2 + (size_t)j * d.Gc * d.Gc;
  const bool colblk = (int)blockIdx.x < nbc;
  const bool act1 = colblk && i1.on && i1.l < nl;
  const bool band = kBand && d.Gc * 4 == G;
  float2 pv[BN], apv[BN], rv[BN], arv[BN], xv[BN];
  if (band && act1) {
    const int q = q0 + i1.l;
#pragma unroll
    for (int b = 0; b < BN; ++b) {
      const size_t e = cbase + (size_t)(N2 * (B0 + b) + i1.k - d.off) * d.Gc + q;
      pv[b] = p[e];
      apv[b] = ap[e];
      rv[b] = r[e];
      arv[b] = ar[e];
      xv[b] = x[e];
    }
  }
  CrCoef c;
  if (!cr_begin<false>(st, cr, it, tol, dr, c)) return;
  const float bf = (float)c.b, af = (float)c.a, naf = (float)(-c.a);
  double acc_ap = 0.0, acc_r = 0.0;
  if (colblk) {
    if (act1) {
      const int q = q0 + i1.l;
      float2 v[N1];
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) v[n1] = make_float2(0.f, 0.f);
      // the CR update of entry (k-row i, column q), step-1 slot n1; returns r_new * winv
      auto entry = [&](int n1, float2 pv, float2 apv, float2 rv, float2 arv, float2 xv) {
        const int t = N2 * n1 + i1.k;
        const int i = t - d.off;
        const size_t e = cbase + (size_t)i * d.Gc + q;
        float2 np, nap, nx;
        const float2 nr = cr_update(pv, apv, rv, arv, xv, bf, af, naf, c.upd, np, nap, nx);
        p[e] = np;
        ap[e] = nap;
        if (c.upd) {
          x[e] = nx;
          r[e] = nr;
        }
        acc_ap += nrm2(nap);
        acc_r += nrm2(nr);
        const float w = winv[i * d.Gc + q];
        v[n1] = flip(make_float2(nr.x * w, nr.y * w), t);  // chat * winv.real() (nlinv.cpp:121)
      };
      if (band) {
        // the coil band's step-1 slots are compile-time, their operands already loaded
#pragma unroll
        for (int b = 0; b < BN; ++b) entry(B0 + b, pv[b], apv[b], rv[b], arv[b], xv[b]);
        fft_step1<Geo, +1, kBand ? BAND : Geo::ALL_N1>(v, i1.k, twG);
      } else {
#pragma unroll
        for (int n1 = 0; n1 < N1; ++n1) {
          const int i = N2 * n1 + i1.k - d.off;
          if (i >= 0 && i < d.Gc) {
            const size_t e = cbase + (size_t)i * d.Gc + q;
            entry(n1, p[e], ap[e], r[e], ar[e], c.upd ? x[e] : make_float2(0.f, 0.f));
          }
        }
        fft_step1<Geo, +1>(v, i1.k, twG);
      }
      park_step1<Geo>(A, i1.l, i1.k, v);
    }
    __syncthreads();
    if (i2.on && i2.l < nl) {
      float2 u[N2];
      fft_step2<Geo, +1, Geo::WIN_K2>(A, i2.l, i2.k, u);  // window rows of U
      float2* dst = U + (size_t)j * G * d.Gc + q0 + i2.l;
#pragma unroll
      for (int k2 = 0; k2 < N2; ++k2) {
        const int pp = i2.k + N1 * k2;
        if (pp >= LO && pp < LO + LW) dst[(size_t)pp * d.Gc] = flip(u[k2], pp);
      }
    }
  } else {
    const bool win_only = rho_window_only(st);
    const int L = LW, lo = LO;
    const int nv = win_only ? L * L : G2;
    constexpr int kU = 4;
    const int nbr = gridDim.x - nbc;
    const int stride = nbr * blockDim.x;
    for (int v0 = (blockIdx.x - nbc) * blockDim.x + threadIdx.x; v0 < nv; v0 += kU * stride) {
      int idx[kU];
      float2 pv[kU], apv[kU], rv[kU], arv[kU], xv[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int v = v0 + u * stride;
        int i = v < nv ? v : -1;
        if (win_only && i >= 0) i = (lo + v / L) * G + lo + (v - (v / L) * L);
        idx[u] = i;
        if (i >= 0) {
          pv[u] = p[i];
          apv[u] = ap[i];
          rv[u] = r[i];
          arv[u] = ar[i];
          if (c.upd) xv[u] = x[i];
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = idx[u];
        if (i < 0) continue;
        float2 np, nap, nx;
        const float2 nr = cr_update(pv[u], apv[u], rv[u], arv[u], xv[u], bf, af, naf, c.upd, np, nap, nx);
        p[i] = np;
        ap[i] = nap;
        if (c.upd) {
          x[i] = nx;
          r[i] = nr;
        }
        acc_ap += nrm2(nap);
        acc_r += nrm2(nr);
      }
    }
  }
  double vv[2] = {acc_ap, acc_r}, tot[2];
  if (dr.out) {
    block_partial<2>(vv, dr.out);  // the tail runs in the next recurrence (cr_begin)
  } else if (grid_reduce<2>(vv, partials, &st->counter, tot) && threadIdx.x == 0) {
    cr_fused_tail(st, cr, it, tol, tot[0], tot[1]);
  }
}

#ifndef RTNB_PASS_ONLY  // non-template kernels: compiled once (engine.cu)
// ---------------------------------------------------------------------------------
// CR recurrences (nlinv.cpp:197-232). D = G*G + J*Gc*Gc complex entries.
// ---------------------------------------------------------------------------------

// first kernel of every Newton step: reset the step record and the CR halt flag
__global__ void k_step_begin(DevState* st, int m) {
  pdl_enter();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    st->cur_step = m;
    st->cr_halt = 0;
    st->rho_out_known = 0;
    st->rho_out_nz = 0;
    StepRec& s = st->steps[m];
    s.iters = 0;
    s.zero_rhs = 0;
    s.resid_win = 0;
    s.resid_out = 0;
    s.rhs_nrm2 = 0;
  }
}

// after the priming application: r_ar = <r, A r> is in rar[0]; ap = ar, ap2[0] = |ap|^2
// Channel groups (grp != 0) run these with member partials: the norms skip the replicated
// rho entries below rho_skip (counted on member 0 only) and go to cr.pcr (the k_cr_fused
// layout: pcr[2k] = |ap|^2 after update k, pcr[2k+1] = |r|^2 after update k) for
// k_grp_fin, which forms the totals in member order and takes the decisions.
__global__ void __launch_bounds__(kThreads) k_cr_prime(int D, float2* __restrict__ ap,
                                                       const float2* __restrict__ ar, double* partials,
                                                       DevState* st, CrScalars cr, int grp, int rho_skip) {
  pdl_enter();
  if (st->status || st->cr_halt) return;
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < D; i += gridDim.x * blockDim.x) {
    const float2 v = ar[i];
    ap[i] = v;
    if (i >= rho_skip) acc += nrm2(v);
  }
  double v[1] = {acc}, tot[1];
  if (grid_reduce<1>(v, partials, &st->counter, tot) && threadIdx.x == 0) {
    if (grp) {
      cr.pcr[0] = tot[0];
    } else {
      cr.ap2[0] = tot[0];
    }
  }
}

// iteration `it`, first half: a = r_ar / |ap|^2; x += a p; r -= a ap; rn[it] = |r|
__global__ void __launch_bounds__(kThreads) k_cr_xr(int D, float2* __restrict__ x, float2* __restrict__ r,
                                                    const float2* __restrict__ p,
                                                    const float2* __restrict__ ap, double* partials,
                                                    DevState* st, CrScalars cr, int it, float tol, int grp,
                                                    int rho_skip) {
  pdl_enter();
  if (st->status || st->cr_halt) return;
  const double denom = cr.ap2[it - 1];
  const double rar = cr.rar[it - 1];
  if (!isfinite(denom) || !isfinite(rar)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->status = ST_SOLVER;  // "cg_solve: iteration diverged"
      st->cr_halt = 1;
    }
    return;
  }
  if (denom <= 0.0 && tol > 0.0f) {  // residual already exactly zero
    if (blockIdx.x == 0 && threadIdx.x == 0) st->cr_halt = 1;
    return;
  }
  const bool upd = denom > 0.0;
  const double a = upd ? rar / denom : 0.0;
  const float af = (float)a, naf = (float)(-a);
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < D; i += gridDim.x * blockDim.x) {
    float2 rv = r[i];
    if (upd) {
      x[i] = axpy_rn(x[i], af, p[i]);
      rv = axpy_rn(rv, naf, ap[i]);
      r[i] = rv;
    }
    if (i >= rho_skip) acc += nrm2(rv);
  }
  double v[1] = {acc}, tot[1];
  if (grid_reduce<1>(v, partials, &st->counter, tot) && threadIdx.x == 0) {
    if (grp) {  // member partial; k_grp_fin (part 2) forms rn[it] and decides
      cr.pcr[2 * (it - 1) + 1] = tot[0];
      return;
    }
    const double rn = sqrt(tot[0]);
    cr.rn[it] = rn;
    StepRec& s = st->steps[st->cur_step];
    if (!isfinite(rn)) {
      st->status = ST_SOLVER;  // "cg_solve: residual is not finite"
      st->cr_halt = 1;
      return;
    }
    s.iters = it;
    const double target = (double)tol * sqrt(s.rhs_nrm2);
    if (tol > 0.0f && (rn == 0.0 || rn <= target)) st->cr_halt = 1;
  }
}

// iteration `it`, second half: b = <r,Ar>_new / <r,Ar>_old; p = b p + r;
// ap = b ap + ar; ap2[it] = |ap|^2
__global__ void __launch_bounds__(kThreads) k_cr_pap(int D, float2* __restrict__ p, float2* __restrict__ ap,
                                                     const float2* __restrict__ r,
                                                     const float2* __restrict__ ar, double* partials,
                                                     DevState* st, CrScalars cr, int it, int grp, int rho_skip) {
  pdl_enter();
  if (st->status || st->cr_halt) return;
  const double rar_new = cr.rar[it], rar_old = cr.rar[it - 1];
  const double b = (rar_old != 0.0) ? rar_new / rar_old : 0.0;
  const float bf = (float)b;
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < D; i += gridDim.x * blockDim.x) {
    const float2 pv = p[i];
    const float2 apv = ap[i];
    // est_scale(p, b); est_axpy(p, 1.0, r)
    const float2 np = make_float2(__fadd_rn(__fmul_rn(pv.x, bf), r[i].x), __fadd_rn(__fmul_rn(pv.y, bf), r[i].y));
    const float2 arv = ar[i];
    const float2 nap = make_float2(__fadd_rn(__fmul_rn(apv.x, bf), arv.x), __fadd_rn(__fmul_rn(apv.y, bf), arv.y));
    p[i] = np;
    ap[i] = nap;
    if (i >= rho_skip) acc += nrm2(nap);
  }
  double v[1] = {acc}, tot[1];
  if (grid_reduce<1>(v, partials, &st->counter, tot) && threadIdx.x == 0) {
    if (grp) {
      cr.pcr[2 * it] = tot[0];
    } else {
      cr.ap2[it] = tot[0];
    }
  }
}

// Fused CR recurrence for the budget-mode frame graphs: iteration `it` second half
// and iteration it+1 first half in one pass (one kernel and one grid reduction fewer
// per iteration than k_cr_pap + k_cr_xr):
//   b = rar[it]/rar[it-1] (b = 0 for it = 0, the priming step);
//   p = b p + r; ap = b ap + ar;                          (nlinv.cpp:225-230)
//   |ap|^2 = b^2 |ap_prev|^2 + 2b Re<ap_prev, ar> + |ar|^2  from the exact norm of the
//     previous ap and the application's dots (exact for it = 0);
//   a = rar[it]/|ap|^2; x += a p; r -= a ap; rn[it+1] = |r|  (nlinv.cpp:205-220)
// The exact |ap|^2 of this pass is reduced for the next iteration. kGrp: the channel-group
// branches are compiled in (a single engine launches k_cr_fused<false>).
template <bool kGrp>
__global__ void __launch_bounds__(kThreads) k_cr_fused(int D, float2* __restrict__ x, float2* __restrict__ r,
                                                       float2* __restrict__ p, float2* __restrict__ ap,
                                                       const float2* __restrict__ ar, double* partials,
                                                       DevState* st, CrScalars cr, int it, float tol,
                                                       int rho_skip, int grp, int G, DeferRed dr) {
  pdl_enter();
  CrCoef c;
  if (!cr_begin<kGrp>(st, cr, it, tol, dr, c)) return;
  const float bf = (float)c.b, af = (float)c.a, naf = (float)(-c.a);
  double acc_ap = 0.0, acc_r = 0.0;
  // rho entries outside the window are exactly zero in every vector: skip them
  const bool win_only = rho_window_only(st);
  const int L = G / 2, lo = (G - L) / 2, G2 = G * G;
  const int nv = win_only ? D - G2 + L * L : D;
  // four entries per thread per round with every load issued up front (memory-level
  // parallelism); per-thread accumulation order is unchanged
  constexpr int kU = 4;
  const int stride = gridDim.x * blockDim.x;
  for (int v0 = blockIdx.x * blockDim.x + threadIdx.x; v0 < nv; v0 += kU * stride) {
    int idx[kU];
    float2 pv[kU], apv[kU], rv[kU], arv[kU], xv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int v = v0 + u * stride;
      int i = v < nv ? v : -1;
      if (win_only && i >= 0) i = v < L * L ? (lo + v / L) * G + lo + (v - (v / L) * L) : G2 + (v - L * L);
      idx[u] = i;
      if (i >= 0) {
        pv[u] = p[i];
        apv[u] = ap[i];
        rv[u] = r[i];
        arv[u] = ar[i];
        if (c.upd) xv[u] = x[i];
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int i = idx[u];
      if (i < 0) continue;
      float2 np, nap, nx;
      const float2 nr = cr_update(pv[u], apv[u], rv[u], arv[u], xv[u], bf, af, naf, c.upd, np, nap, nx);
      p[i] = np;
      ap[i] = nap;
      if (c.upd) {
        x[i] = nx;
        r[i] = nr;
      }
      if (i >= rho_skip) {  // group members other than the first skip the replicated rho
        acc_ap += nrm2(nap);
        acc_r += nrm2(nr);
      }
    }
  }
  double v[2] = {acc_ap, acc_r}, tot[2];
  if (dr.out) {
    block_partial<2>(v, dr.out);  // the tail runs in the next recurrence (cr_begin)
    return;
  }
  if (grid_reduce<2>(v, partials, &st->counter, tot) && threadIdx.x == 0) {
    if (kGrp && grp) {
      cr.pcr[2 * it + 0] = tot[0];
      cr.pcr[2 * it + 1] = tot[1];
      return;
    }
    cr_fused_tail(st, cr, it, tol, tot[0], tot[1]);
  }
}

// ---------------------------------------------------------------------------------
// Channel decomposition (group mode). Members run the pass kernels on their own
// channel block; the cross-member sums happen at two kinds of points:
//   - vectors: k_colsW reads every member's k_rows2 window partials (and, in SETUP,
//     k_rho_out's out-of-window partials) from peer memory;
//   - scalars: every reduction writes the member's partial, and k_grp_fin (one
//     thread) forms the totals in member order after an all-member event barrier,
//     then runs exactly the decisions the single-device kernels take in their last
//     block (nlinv.cpp:184-186, 205-220). Every member computes identical totals, so
//     every member takes identical decisions.
// ---------------------------------------------------------------------------------

// SETUP, outside the window: partial sum over this member's channels of
// conj(c_j) z_j (the T term is masked to zero there, preproc.cpp:442) and |z_j|^2
__global__ void __launch_bounds__(kThreads) k_rho_out(Dims d, const float2* __restrict__ coils,
                                                      const float2* __restrict__ z, double2* __restrict__ RPO,
                                                      double* partials, DevState* st) {
  pdl_enter();
  if (st->status) return;
  const int G = d.G, D0 = G * G;
  const int zo = st->z_out;
  double acc = 0.0;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < D0; e += gridDim.x * blockDim.x) {
    const int r = e / G, c = e - (e / G) * G;
    if (in_win(d, r, c)) continue;
    double sx = 0.0, sy = 0.0;
    for (int j = 0; zo && j < d.J; ++j) {
      const float2 zz = z[(size_t)j * D0 + e];
      const float2 v = cjmul_rn(coils[(size_t)j * D0 + e], zz);
      sx += v.x;
      sy += v.y;
      acc += nrm2(zz);
    }
    RPO[e] = make_double2(sx, sy);
  }
  double vv[1] = {acc}, tot[1];
  if (grid_reduce<1>(vv, partials, &st->counter, tot) && threadIdx.x == 0) st->gp[1] = tot[0];
}


// Group totals and the decisions that depend on them.
//  setup:       |rhs|^2, resid_out, resid_win of the step; cg_solve entry checks
//  cr_slot >= 0: k_cr_fused(cr_slot): ap2[cr_slot], rn[cr_slot+1], iters, tolerance stop
//  op_slot >= 0: colsW of application op_slot: rar, saa, spa
//  part (cr_slot >= 0): 0 both halves (k_cr_fused), 1 only ap2[cr_slot] (after k_cr_pap /
//               k_cr_prime), 2 only the |r| half (after k_cr_xr(cr_slot + 1))
__global__ void k_grp_fin(GroupScal g, DevState* st, CrScalars cr, int setup, int op_slot, int cr_slot,
                          float tol, int part) {
  pdl_enter();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (st->status) return;
  StepRec& s = st->steps[st->cur_step];
  if (setup) {
    double rhs = 0.0, ro = 0.0, rw = 0.0;
    for (int m = 0; m < g.A; ++m) {
      rhs += __ldcg(&g.st[m]->gp[0]);
      ro += __ldcg(&g.st[m]->gp[1]);
      rw += __ldcg(&g.st[m]->gp[2]);
    }
    s.rhs_nrm2 = rhs;
    s.resid_out = ro;
    s.resid_win = rw;
    const double rn = sqrt(rhs);
    if (!isfinite(rn)) {
      st->status = ST_SOLVER;
      st->cr_halt = 1;
    } else if (rn == 0.0) {
      s.zero_rhs = 1;
      st->cr_halt = 1;
    }
    return;
  }
  if (st->cr_halt) return;
  if (cr_slot >= 0 && part != 2) cr.ap2[cr_slot] = grp_sum(g, g.pcr, 2 * cr_slot);
  if (cr_slot >= 0 && part != 1) {
    const double rn = sqrt(grp_sum(g, g.pcr, 2 * cr_slot + 1));
    cr.rn[cr_slot + 1] = rn;
    if (!isfinite(rn)) {
      st->status = ST_SOLVER;
      st->cr_halt = 1;
      return;
    }
    s.iters = cr_slot + 1;
    const double target = (double)tol * sqrt(s.rhs_nrm2);
    if (tol > 0.0f && (rn == 0.0 || rn <= target)) {
      st->cr_halt = 1;
      return;
    }
  }
  if (op_slot >= 0) {
    cr.rar[op_slot] = grp_sum(g, g.pcw, 3 * op_slot + 0);
    cr.saa[op_slot] = grp_sum(g, g.pcw, 3 * op_slot + 1);
    cr.spa[op_slot] = grp_sum(g, g.pcw, 3 * op_slot + 2);
  }
}

// final image, group mode: this member's sum_j |c_j|^2 over the N x N crop
__global__ void __launch_bounds__(kThreads) k_coil_ss(Dims d, const float2* __restrict__ coils,
                                                      double* __restrict__ ss, const DevState* st) {
  pdl_enter();
  if (st->status) return;
  const int G = d.G, N = d.N;
  const int o = G / 2 - N / 2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < N * N; e += gridDim.x * blockDim.x) {
    const size_t g = (size_t)(e / N + o) * G + (e % N + o);
    double acc = 0.0;
    for (int j = 0; j < d.J; ++j) acc += nrm2(coils[(size_t)j * G * G + g]);
    ss[e] = acc;
  }
}

// final image, group mode (first member): rho * sqrt(sum over members of k_coil_ss)
__global__ void __launch_bounds__(kThreads) k_image_grp(Dims d, const float2* __restrict__ rho, GroupScal g,
                                                        float scale, int apply_scale, float2* __restrict__ img,
                                                        const DevState* st) {
  pdl_enter();
  if (st->status) return;
  const int G = d.G, N = d.N;
  const int o = G / 2 - N / 2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < N * N; e += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int m = 0; m < g.A; ++m) acc += __ldcg(g.ss[m] + e);
    const float s = (float)sqrt(acc);
    const float2 rv = rho[(size_t)(e / N + o) * G + (e % N + o)];
    float2 v = make_float2(rv.x * s, rv.y * s);
    if (apply_scale) v = make_float2(v.x * scale, v.y * scale);
    img[e] = v;
  }
}

// Does the frame's gridded data have a nonzero sample outside the field-of-view
// window? grid_adjoint masks it (preproc.cpp:195), so normally not, and then the
// out-of-window part of rhs.rho (sum_j conj(c_j) z_j, zero there) and of the data
// residual need not be read in every Newton-step setup. st->z_out is cleared by the
// caller before the launch.
__global__ void __launch_bounds__(kThreads) k_z_outside(Dims d, const float2* __restrict__ z, DevState* st) {
  pdl_enter();
  const int G = d.G;
  const long long n = (long long)d.J * G * G;
  int any = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(i % ((long long)G * G));
    const int r = e / G, c = e - (e / G) * G;
    if (in_win(d, r, c)) continue;
    const float2 v = z[i];
    any |= (v.x != 0.f || v.y != 0.f);
  }
  if (__syncthreads_or(any) && threadIdx.x == 0) st->z_out = 1;
}

// All-member barrier of a one-process-per-GPU group (procgroup.hpp): bump this
// member's epoch counter, publish it with a system-scope release (after the stream's
// earlier kernels, whose writes the fence makes visible to the peers), then poll every
// member's published epoch with acquire loads until all have reached it. Every member
// runs the same barrier sequence, so the counters advance in lockstep and captured
// graphs replay correctly.
// A member that does not arrive within the deadline (about 10 s of SM clock) turns the
// wait into the reference's DecompFault (WorkerGroup deadline, decomp.hpp:90-93): the
// status goes to ST_DEADLINE, every later kernel of the frame skips, the host raises.
constexpr long long kBarrierDeadlineCycles = 20000000000LL;
constexpr int kBarrierPoison = 0x7fffffff;
__global__ void k_pg_barrier(int* own, GroupFlags f, DevState* st) {
  pdl_enter();
  __shared__ int epoch;
  if (threadIdx.x == 0) {
    const int e = own[1] + 1;
    own[1] = e;
    __threadfence_system();
    if (own[0] != kBarrierPoison) {  // a poisoned member stays poisoned
      asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(own), "r"(e) : "memory");
    }
    epoch = e;
  }
  __syncthreads();
  // a member whose frame already failed only keeps its epoch count in step
  if ((int)threadIdx.x < f.A && !st->status) {
    const int e = epoch;
    const long long t0 = clock64();
    for (;;) {
      int v;
      asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(f.flag[threadIdx.x]) : "memory");
      if (v == kBarrierPoison) {  // a member missed a deadline: the whole group fails
        atomicExch(&st->status, (int)ST_DEADLINE);
        break;
      }
      if (v >= e) break;
      if (clock64() - t0 > kBarrierDeadlineCycles) {
        atomicExch(&st->status, (int)ST_DEADLINE);
        asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(own), "r"(kBarrierPoison) : "memory");
        break;
      }
      __nanosleep(256);
    }
  }
  __syncthreads();
}

// x += 1.0 * x_cg  (newton_step, nlinv.cpp:281)
__global__ void __launch_bounds__(kThreads) k_axpy1(int D, float2* __restrict__ x, const float2* __restrict__ d,
                                                    const DevState* st) {
  pdl_enter();
  if (st->status) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < D; i += gridDim.x * blockDim.x) {
    const float2 a = x[i], b = d[i];
    x[i] = make_float2(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y));
  }
}

// final image: crop_N(rho * sqrt(sum_j |c_j|^2)) with an FP64 coil sum, then the
// series' undo_scale (nlinv.cpp:317-332, 404-408)
__global__ void __launch_bounds__(kThreads) k_image(Dims d, const float2* __restrict__ rho,
                                                    const float2* __restrict__ coils, float scale,
                                                    int apply_scale, float2* __restrict__ img,
                                                    const DevState* st) {
  pdl_enter();
  if (st->status) return;
  const int G = d.G, N = d.N;
  const int o = G / 2 - N / 2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < N * N; e += gridDim.x * blockDim.x) {
    const int r = e / N + o, c = e % N + o;
    const size_t g = (size_t)r * G + c;
    double acc = 0.0;
    for (int j = 0; j < d.J; ++j) acc += nrm2(coils[(size_t)j * G * G + g]);
    const float s = (float)sqrt(acc);
    const float2 rv = rho[g];
    float2 v = make_float2(rv.x * s, rv.y * s);
    if (apply_scale) v = make_float2(v.x * scale, v.y * scale);
    img[e] = v;
  }
}

#endif  // RTNB_PASS_ONLY

// ---------------------------------------------------------------------------------
// Stand-alone centered 2D transforms (fft::forward / fft::inverse, fft.hpp:22-30).
// ---------------------------------------------------------------------------------

// one pass of a batched 2D transform over `batch` images: rows (COLS = false, axis 1)
// or columns (COLS = true, axis 0); scale applied on output
template <class Geo, int S, bool COLS>
__global__ void __launch_bounds__(Geo::NT) k_fft_pass(float2* __restrict__ data, int batch,
                                                      const float4* __restrict__ twG, float scale) {
  RTNB_TILE_SETUP(COLS);
  constexpr int tiles = (G + Geo::LPB - 1) / Geo::LPB;
  const int img = blockIdx.x / tiles;
  if (img >= batch) return;  // uniform per block
  const int l0 = (blockIdx.x - img * tiles) * Geo::LPB;
  const int nl = min(Geo::LPB, G - l0);
  float2* base = data + (size_t)img * G * G;
  // element t of line l: rows -> base[(l0+l)*G + t], columns -> base[t*G + l0+l]
  const size_t ls = COLS ? 1 : (size_t)G, es = COLS ? (size_t)G : 1;
  if (i1.on && i1.l < nl) {
    float2 v[N1];
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      const int t = N2 * n1 + i1.k;
      v[n1] = flip(base[(l0 + i1.l) * ls + t * es], t);
    }
    fft_step1<Geo, S>(v, i1.k, twG);
    park_step1<Geo>(A, i1.l, i1.k, v);
  }
  step_sync<(kRowStride<Geo, COLS> > 0)>();  // row lines: warp-local exchange
  if (i2.on && i2.l < nl) {
    float2 u[N2];
    fft_step2<Geo, S>(A, i2.l, i2.k, u);
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) {
      const int p = i2.k + N1 * k2;
      base[(l0 + i2.l) * ls + p * es] = cscale(flip(u[k2], p), scale);
    }
  }
}

#ifndef RTNB_PASS_ONLY
// Direct centered DFT along one axis for sizes the line engine does not cover
// (odd sides, large prime factors): X[p] = sum_t x[t] W^{(p-c)(t-c)}, one block per
// line, FP64 accumulation. tw: exp(sign 2 pi i e / n), e = 0..n-1.
__global__ void k_dft_direct(const float2* __restrict__ in, float2* __restrict__ out, int n, int batch,
                             int axis, const double2* __restrict__ tw, float scale) {
  extern __shared__ float2 line[];
  const int img = blockIdx.x / n;
  const int li = blockIdx.x - img * n;
  if (img >= batch) return;
  const float2* src = in + (size_t)img * n * n;
  float2* dst = out + (size_t)img * n * n;
  const size_t stride = (axis == 1) ? 1 : (size_t)n;
  const size_t base = (axis == 1) ? (size_t)li * n : (size_t)li;
  for (int t = threadIdx.x; t < n; t += blockDim.x) line[t] = src[base + t * stride];
  __syncthreads();
  const int c = n / 2;
  for (int p = threadIdx.x; p < n; p += blockDim.x) {
    double ax = 0.0, ay = 0.0;
    for (int t = 0; t < n; ++t) {
      long long e = (long long)(p - c) * (t - c) % n;
      if (e < 0) e += n;
      const double2 w = tw[e];
      const float2 v = line[t];
      ax += v.x * w.x - v.y * w.y;
      ay += v.x * w.y + v.y * w.x;
    }
    dst[base + p * stride] = make_float2((float)(ax * scale), (float)(ay * scale));
  }
}

#endif  // RTNB_PASS_ONLY

}  // namespace rtnb
