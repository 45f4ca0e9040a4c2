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

}  // namespace

// ---------------------------------------------------------------------------------
// Pass kernels. Lines are batched LPB per block and never straddle channels.
// ---------------------------------------------------------------------------------

// W^-1 column pass. Lines: (channel j, coil k-column q). Input chat_j*winv on the
// Gc centered k-rows, output rows [r0, r0+nr) of U_j (G x Gc, row-major).
template <class Geo>
__global__ void __launch_bounds__(kThreads) k_colA(Dims d, const float* __restrict__ winv,
                                                   const float2* __restrict__ twG,
                                                   const float2* __restrict__ chat, float2* __restrict__ U,
                                                   int r0, int nr, const DevState* st, int use_halt) {
  if (st->status || (use_halt && st->cr_halt)) return;
  constexpr int G = Geo::G, LPB = Geo::LPB;
  extern __shared__ float2 sm[];
  float2* A = sm;
  float2* B = sm + LPB * Geo::LSA;
  const int tiles = (d.Gc + LPB - 1) / LPB;
  const int j = blockIdx.x / tiles;
  const int q0 = (blockIdx.x - j * tiles) * LPB;
  const int nl = min(LPB, d.Gc - q0);
  const float2* src = chat + (size_t)j * d.Gc * d.Gc;
  for (int idx = threadIdx.x; idx < G * LPB; idx += blockDim.x) {
    const int t = idx / LPB, l = idx - (idx / LPB) * LPB;
    const int i = t - d.off;
    float2 v = make_float2(0.f, 0.f);
    if (l < nl && i >= 0 && i < d.Gc) {
      const int e = i * d.Gc + q0 + l;
      const float w = winv[e];
      const float2 c = src[e];
      v = flip(make_float2(c.x * w, c.y * w), t);
    }
    A[Geo::a_idx(l, t)] = v;
  }
  tile_fft<Geo, +1>(A, B, nl, twG);
  float2* dst = U + (size_t)j * G * d.Gc;
  for (int idx = threadIdx.x; idx < nr * LPB; idx += blockDim.x) {
    const int pr = idx / LPB, l = idx - pr * LPB;
    if (l < nl) {
      const int p = r0 + pr;
      dst[(size_t)p * d.Gc + q0 + l] = flip(B[Geo::b_idx(l, p)], p);
    }
  }
}

enum Rows1Mode : int { R1_DECODE = 0, R1_OP = 1, R1_SETUP = 2 };

// Row pass 1.
//  DECODE: rows 0..G-1 of U_j -> inverse row FFT -> coils_j (full G x G, scaled 1/G);
//          channel 0 blocks also write the masked rho (make_step_cache, nlinv.cpp:135-150).
//  OP:     window rows: W^-1 row pass of U_j, t = c_j*drho + rho*a on the window,
//          forward row FFT -> V_j (L x G).
//  SETUP:  window rows: t = rho*c_j (nlinv.cpp:252) -> forward row FFT -> V_j.
template <class Geo>
__global__ void __launch_bounds__(kThreads) k_rows1(Dims d, int mode, const float2* __restrict__ twG,
                                                    const float2* __restrict__ U,
                                                    const float2* __restrict__ coils,
                                                    const float2* __restrict__ rhom,
                                                    const float2* __restrict__ drho, float2* __restrict__ V,
                                                    float2* __restrict__ coils_out,
                                                    const float2* __restrict__ rho_src,
                                                    float2* __restrict__ rhom_out, const DevState* st,
                                                    int use_halt) {
  if (st->status || (use_halt && st->cr_halt)) return;
  constexpr int G = Geo::G, LPB = Geo::LPB;
  extern __shared__ float2 sm[];
  float2* A = sm;
  float2* B = sm + LPB * Geo::LSA;
  const int nrows = (mode == R1_DECODE) ? G : d.L;
  const int row0 = (mode == R1_DECODE) ? 0 : d.lo;
  const int tiles = (nrows + LPB - 1) / LPB;
  const int j = blockIdx.x / tiles;
  const int rl0 = (blockIdx.x - j * tiles) * LPB;
  const int nl = min(LPB, nrows - rl0);
  const float2* Uj = U + (size_t)j * G * d.Gc;
  const float2* cj = coils + (size_t)j * G * G;

  if (mode != R1_SETUP) {
    // load U rows into the coil k-columns, inverse row FFT
    for (int idx = threadIdx.x; idx < LPB * G; idx += blockDim.x) {
      const int l = idx / G, t = idx - (idx / G) * G;
      const int q = t - d.off;
      float2 v = make_float2(0.f, 0.f);
      if (l < nl && q >= 0 && q < d.Gc) v = flip(Uj[(size_t)(row0 + rl0 + l) * d.Gc + q], t);
      A[Geo::a_idx(l, t)] = v;
    }
    tile_fft<Geo, +1>(A, B, nl, twG);
    if (mode == R1_DECODE) {
      float2* out = coils_out + (size_t)j * G * G;
      for (int idx = threadIdx.x; idx < LPB * G; idx += blockDim.x) {
        const int l = idx / G, p = idx - (idx / G) * G;
        if (l < nl) {
          const int r = rl0 + l;
          out[(size_t)r * G + p] = cscale(flip(B[Geo::b_idx(l, p)], p), d.invG);
          if (j == 0) {
            const float2 x = rho_src[(size_t)r * G + p];
            rhom_out[(size_t)r * G + p] = in_win(d, r, p) ? x : make_float2(0.f, 0.f);
          }
        }
      }
      return;
    }
  }
  // build t on the window and run the forward Toeplitz row pass
  for (int idx = threadIdx.x; idx < LPB * G; idx += blockDim.x) {
    const int l = idx / G, t = idx - (idx / G) * G;
    float2 v = make_float2(0.f, 0.f);
    if (l < nl && t >= d.lo && t < d.lo + d.L) {
      const size_t e = (size_t)(row0 + rl0 + l) * G + t;
      const float2 rm = rhom[e];
      const float2 c = cj[e];
      if (mode == R1_OP) {
        const float2 a = cscale(flip(B[Geo::b_idx(l, t)], t), d.invG);
        // t = c_j * drho + rho * (W^-1 dchat_j)   (nlinv.cpp:163)
        const float2 s1 = cmul_rn(c, drho[e]);
        const float2 s2 = cmul_rn(rm, a);
        v = make_float2(__fadd_rn(s1.x, s2.x), __fadd_rn(s1.y, s2.y));
      } else {
        v = cmul_rn(rm, c);  // e = rho * c_j   (nlinv.cpp:252)
      }
      v = flip(v, t);
    }
    A[Geo::a_idx(l, t)] = v;
  }
  tile_fft<Geo, -1>(A, B, nl, twG);
  float2* Vj = V + (size_t)j * d.L * G;
  for (int idx = threadIdx.x; idx < LPB * G; idx += blockDim.x) {
    const int l = idx / G, p = idx - (idx / G) * G;
    if (l < nl) Vj[(size_t)(rl0 + l) * G + p] = flip(B[Geo::b_idx(l, p)], p);
  }
}

// Toeplitz column pass: forward column FFT of the window rows of V_j, * P/G, inverse
// column FFT, keep the window rows (in place in V_j). Lines: (j, column q).
template <class Geo>
__global__ void __launch_bounds__(kThreads) k_colsT(Dims d, const float2* __restrict__ twG,
                                                    const float2* __restrict__ P, float2* __restrict__ V,
                                                    const DevState* st, int use_halt) {
  if (st->status || (use_halt && st->cr_halt)) return;
  constexpr int G = Geo::G, LPB = Geo::LPB;
  extern __shared__ float2 sm[];
  float2* A = sm;
  float2* B = sm + LPB * Geo::LSA;
  constexpr int tiles = (G + LPB - 1) / LPB;
  const int j = blockIdx.x / tiles;
  const int q0 = (blockIdx.x - j * tiles) * LPB;
  const int nl = min(LPB, G - q0);
  float2* Vj = V + (size_t)j * d.L * G;
  for (int idx = threadIdx.x; idx < G * LPB; idx += blockDim.x) {
    const int t = idx / LPB, l = idx - (idx / LPB) * LPB;
    float2 v = make_float2(0.f, 0.f);
    if (l < nl && t >= d.lo && t < d.lo + d.L) v = flip(Vj[(size_t)(t - d.lo) * G + q0 + l], t);
    A[Geo::a_idx(l, t)] = v;
  }
  tile_fft<Geo, -1>(A, B, nl, twG);
  // k-space multiply; the output sign flip of the forward pass cancels the input
  // flip of the inverse pass
  for (int idx = threadIdx.x; idx < G * LPB; idx += blockDim.x) {
    const int p = idx / LPB, l = idx - (idx / LPB) * LPB;
    float2 v = make_float2(0.f, 0.f);
    if (l < nl) v = cscale(cmul(B[Geo::b_idx(l, p)], P[(size_t)p * G + q0 + l]), d.invG);
    A[Geo::a_idx(l, p)] = v;
  }
  tile_fft<Geo, +1>(A, B, nl, twG);
  for (int idx = threadIdx.x; idx < d.L * LPB; idx += blockDim.x) {
    const int pr = idx / LPB, l = idx - pr * LPB;
    if (l < nl) {
      const int p = d.lo + pr;
      Vj[(size_t)pr * G + q0 + l] = flip(B[Geo::b_idx(l, p)], p);
    }
  }
}

enum Rows2Mode : int { R2_OP = 0, R2_SETUP = 1 };

// Row pass 2: inverse Toeplitz row pass -> T (window, scaled 1/G). SETUP: e = z - T and
// the data-residual partial (nlinv.cpp:254-256). rc = conj(c) T -> RC_j (the channel
// term of out.rho), rt = conj(rho) T -> forward W^-H row pass keeping the Gc
// coil k-columns -> Y_j (L x Gc).
template <class Geo>
__global__ void __launch_bounds__(kThreads) k_rows2(Dims d, int mode, const float2* __restrict__ twG,
                                                    const float2* __restrict__ V,
                                                    const float2* __restrict__ coils,
                                                    const float2* __restrict__ rhom,
                                                    const float2* __restrict__ z, float2* __restrict__ RC,
                                                    float2* __restrict__ Y, double* partials, DevState* st,
                                                    int use_halt) {
  if (st->status || (use_halt && st->cr_halt)) return;
  constexpr int G = Geo::G, LPB = Geo::LPB;
  extern __shared__ float2 sm[];
  float2* A = sm;
  float2* B = sm + LPB * Geo::LSA;
  const int tiles = (d.L + LPB - 1) / LPB;
  const int j = blockIdx.x / tiles;
  const int rl0 = (blockIdx.x - j * tiles) * LPB;
  const int nl = min(LPB, d.L - rl0);
  const float2* Vj = V + (size_t)j * d.L * G;
  const float2* cj = coils + (size_t)j * G * G;
  const float2* zj = z + (size_t)j * G * G;
  float2* RCj = RC + (size_t)j * d.L * d.L;
  for (int idx = threadIdx.x; idx < LPB * G; idx += blockDim.x) {
    const int l = idx / G, t = idx - (idx / G) * G;
    float2 v = make_float2(0.f, 0.f);
    if (l < nl) v = flip(Vj[(size_t)(rl0 + l) * G + t], t);
    A[Geo::a_idx(l, t)] = v;
  }
  tile_fft<Geo, +1>(A, B, nl, twG);
  double resid = 0.0;
  for (int idx = threadIdx.x; idx < LPB * G; idx += blockDim.x) {
    const int l = idx / G, t = idx - (idx / G) * G;
    float2 v = make_float2(0.f, 0.f);
    if (l < nl && t >= d.lo && t < d.lo + d.L) {
      const int r = d.lo + rl0 + l;
      const size_t e = (size_t)r * G + t;
      float2 T = cscale(flip(B[Geo::b_idx(l, t)], t), d.invG);
      if (mode == R2_SETUP) {
        const float2 zz = zj[e];
        T = make_float2(__fsub_rn(zz.x, T.x), __fsub_rn(zz.y, T.y));
        resid += nrm2(T);
      }
      RCj[(size_t)(rl0 + l) * d.L + (t - d.lo)] = cjmul_rn(cj[e], T);
      v = flip(cjmul_rn(rhom[e], T), t);
    }
    A[Geo::a_idx(l, t)] = v;
  }
  tile_fft<Geo, -1>(A, B, nl, twG);
  float2* Yj = Y + (size_t)j * d.L * d.Gc;
  for (int idx = threadIdx.x; idx < LPB * d.Gc; idx += blockDim.x) {
    const int l = idx / d.Gc, q = idx - (idx / d.Gc) * d.Gc;
    if (l < nl) {
      const int p = d.off + q;
      Yj[(size_t)(rl0 + l) * d.Gc + q] = flip(B[Geo::b_idx(l, p)], p);
    }
  }
  if (mode == R2_SETUP) {
    double v[1] = {resid}, tot[1];
    if (grid_reduce<1>(v, partials, &st->counter, tot) && threadIdx.x == 0) {
      st->steps[st->cur_step].resid_win = tot[0];
    }
  }
}

enum ColsWMode : int { CW_OP = 0, CW_OPALPHA = 1, CW_SETUP = 2 };

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
};

// Last pass of an application: W^-H column pass (blocks [0, nbw)) and the channel
// sum of out.rho over the full G x G grid (blocks [nbw, grid)).
template <class Geo>
__global__ void __launch_bounds__(kThreads) k_colsW(Dims d, ColsWArgs a, const float* __restrict__ winv,
                                                    const float2* __restrict__ twG,
                                                    const float2* __restrict__ Y,
                                                    const float2* __restrict__ RC,
                                                    const float2* __restrict__ coils,
                                                    const float2* __restrict__ z, int nbw,
                                                    double* partials, DevState* st, CrScalars cr,
                                                    int use_halt) {
  if (st->status || (use_halt && st->cr_halt)) return;
  constexpr int G = Geo::G, LPB = Geo::LPB;
  extern __shared__ float2 sm[];
  const int D0 = G * G;
  double acc0 = 0.0, acc1 = 0.0;
  // combine the normal-operator value n at flat index e with the CR / rhs terms
  auto finish = [&](size_t e, float2 n) {
    if (a.mode == CW_SETUP) {
      float2 v = axpy_rn(n, a.a_x, a.x[e]);
      v = axpy_rn(v, a.a_reg, a.reg[e]);
      a.out[e] = v;
      a.out2[e] = v;
      a.out3[e] = make_float2(0.f, 0.f);
      acc0 += nrm2(v);
    } else {
      float2 v = n;
      if (a.mode == CW_OPALPHA) v = axpy_rn(v, a.alpha, a.dx[e]);
      a.out[e] = v;
      const float2 p = a.dx[e];
      acc0 += (double)p.x * v.x + (double)p.y * v.y;  // Re <dx, out>
    }
  };
  if ((int)blockIdx.x < nbw) {
    float2* A = sm;
    float2* B = sm + LPB * Geo::LSA;
    const int tiles = (d.Gc + LPB - 1) / LPB;
    const int j = blockIdx.x / tiles;
    const int q0 = (blockIdx.x - j * tiles) * LPB;
    const int nl = min(LPB, d.Gc - q0);
    const float2* Yj = Y + (size_t)j * d.L * d.Gc;
    for (int idx = threadIdx.x; idx < G * LPB; idx += blockDim.x) {
      const int t = idx / LPB, l = idx - (idx / LPB) * LPB;
      float2 v = make_float2(0.f, 0.f);
      if (l < nl && t >= d.lo && t < d.lo + d.L) v = flip(Yj[(size_t)(t - d.lo) * d.Gc + q0 + l], t);
      A[Geo::a_idx(l, t)] = v;
    }
    tile_fft<Geo, -1>(A, B, nl, twG);
    for (int idx = threadIdx.x; idx < d.Gc * LPB; idx += blockDim.x) {
      const int i = idx / LPB, l = idx - (idx / LPB) * LPB;
      if (l < nl) {
        const int p = d.off + i;
        const int e = i * d.Gc + q0 + l;
        const float w = winv[e];
        const float2 f = cscale(flip(B[Geo::b_idx(l, p)], p), d.invG);
        // crop_k(FFT(u)) * winv   (nlinv.cpp:127-133)
        finish((size_t)D0 + (size_t)j * d.Gc * d.Gc + e, make_float2(f.x * w, f.y * w));
      }
    }
  } else {
    // out.rho: window = fixed-order FP64 sum of rc_j over channels (decomp.cpp:26-39);
    // outside the window T is masked to zero, so only the SETUP data term survives
    for (int e = (blockIdx.x - nbw) * blockDim.x + threadIdx.x; e < D0;
         e += (gridDim.x - nbw) * blockDim.x) {
      const int r = e / G, c = e - (e / G) * G;
      double sx = 0.0, sy = 0.0;
      if (in_win(d, r, c)) {
        const size_t w = (size_t)(r - d.lo) * d.L + (c - d.lo);
        for (int j = 0; j < d.J; ++j) {
          const float2 v = RC[(size_t)j * d.L * d.L + w];
          sx += v.x;
          sy += v.y;
        }
      } else if (a.mode == CW_SETUP) {
        for (int j = 0; j < d.J; ++j) {
          const float2 zz = z[(size_t)j * D0 + e];
          const float2 v = cjmul_rn(coils[(size_t)j * D0 + e], zz);
          sx += v.x;
          sy += v.y;
          acc1 += nrm2(zz);
        }
      }
      finish((size_t)e, make_float2((float)sx, (float)sy));
    }
  }
  double v[2] = {acc0, acc1}, tot[2];
  if (grid_reduce<2>(v, partials, &st->counter, tot) && threadIdx.x == 0) {
    if (a.mode == CW_SETUP) {
      StepRec& s = st->steps[st->cur_step];
      s.rhs_nrm2 = tot[0];
      s.resid_out = tot[1];
      const double rn = sqrt(tot[0]);
      // cg_solve entry checks (nlinv.cpp:184-186)
      if (!isfinite(rn)) {
        st->status = ST_SOLVER;
        st->cr_halt = 1;
      } else if (rn == 0.0) {
        s.zero_rhs = 1;
        st->cr_halt = 1;
      }
    } else if (a.dot_slot >= 0) {
      cr.rar[a.dot_slot] = tot[0];
    } else {
      st->scal[0] = tot[0];
    }
  }
}

// ---------------------------------------------------------------------------------
// CR recurrences (nlinv.cpp:197-232). D = G*G + J*Gc*Gc complex entries.
// ---------------------------------------------------------------------------------

// first kernel of every Newton step: reset the step record and the CR halt flag
__global__ void k_step_begin(DevState* st, int m) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    st->cur_step = m;
    st->cr_halt = 0;
    StepRec& s = st->steps[m];
    s.iters = 0;
    s.zero_rhs = 0;
    s.resid_win = 0;
    s.resid_out = 0;
    s.rhs_nrm2 = 0;
  }
}

// after the priming application: r_ar = <r, A r> is in rar[0]; ap = ar, ap2[0] = |ap|^2
__global__ void __launch_bounds__(kThreads) k_cr_prime(int D, float2* __restrict__ ap,
                                                       const float2* __restrict__ ar, double* partials,
                                                       DevState* st, CrScalars cr) {
  if (st->status || st->cr_halt) return;
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < D; i += gridDim.x * blockDim.x) {
    const float2 v = ar[i];
    ap[i] = v;
    acc += nrm2(v);
  }
  double v[1] = {acc}, tot[1];
  if (grid_reduce<1>(v, partials, &st->counter, tot) && threadIdx.x == 0) cr.ap2[0] = tot[0];
}

// iteration `it`, first half: a = r_ar / |ap|^2; x += a p; r -= a ap; rn[it] = |r|
__global__ void __launch_bounds__(kThreads) k_cr_xr(int D, float2* __restrict__ x, float2* __restrict__ r,
                                                    const float2* __restrict__ p,
                                                    const float2* __restrict__ ap, double* partials,
                                                    DevState* st, CrScalars cr, int it, float tol) {
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
    acc += nrm2(rv);
  }
  double v[1] = {acc}, tot[1];
  if (grid_reduce<1>(v, partials, &st->counter, tot) && threadIdx.x == 0) {
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
                                                     DevState* st, CrScalars cr, int it) {
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
    acc += nrm2(nap);
  }
  double v[1] = {acc}, tot[1];
  if (grid_reduce<1>(v, partials, &st->counter, tot) && threadIdx.x == 0) cr.ap2[it] = tot[0];
}

// x += 1.0 * x_cg  (newton_step, nlinv.cpp:281)
__global__ void __launch_bounds__(kThreads) k_axpy1(int D, float2* __restrict__ x, const float2* __restrict__ d,
                                                    const DevState* st) {
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

// ---------------------------------------------------------------------------------
// Stand-alone centered 2D transforms (fft::forward / fft::inverse, fft.hpp:22-30).
// ---------------------------------------------------------------------------------

// one pass of a batched 2D transform over `batch` images: rows (axis 1) or columns
// (axis 0); scale applied on output
template <class Geo, int S>
__global__ void __launch_bounds__(kThreads) k_fft_pass(float2* __restrict__ data, int batch, int axis,
                                                       const float2* __restrict__ twG, float scale) {
  constexpr int G = Geo::G, LPB = Geo::LPB;
  extern __shared__ float2 sm[];
  float2* A = sm;
  float2* B = sm + LPB * Geo::LSA;
  constexpr int tiles = (G + LPB - 1) / LPB;
  const int img = blockIdx.x / tiles;
  if (img >= batch) return;
  const int l0 = (blockIdx.x - img * tiles) * LPB;
  const int nl = min(LPB, G - l0);
  float2* base = data + (size_t)img * G * G;
  if (axis == 1) {
    for (int idx = threadIdx.x; idx < LPB * G; idx += blockDim.x) {
      const int l = idx / G, t = idx - (idx / G) * G;
      A[Geo::a_idx(l, t)] = (l < nl) ? flip(base[(size_t)(l0 + l) * G + t], t) : make_float2(0.f, 0.f);
    }
  } else {
    for (int idx = threadIdx.x; idx < G * LPB; idx += blockDim.x) {
      const int t = idx / LPB, l = idx - (idx / LPB) * LPB;
      A[Geo::a_idx(l, t)] = (l < nl) ? flip(base[(size_t)t * G + l0 + l], t) : make_float2(0.f, 0.f);
    }
  }
  tile_fft<Geo, S>(A, B, nl, twG);
  if (axis == 1) {
    for (int idx = threadIdx.x; idx < LPB * G; idx += blockDim.x) {
      const int l = idx / G, p = idx - (idx / G) * G;
      if (l < nl) base[(size_t)(l0 + l) * G + p] = cscale(flip(B[Geo::b_idx(l, p)], p), scale);
    }
  } else {
    for (int idx = threadIdx.x; idx < G * LPB; idx += blockDim.x) {
      const int p = idx / LPB, l = idx - (idx / LPB) * LPB;
      if (l < nl) base[(size_t)p * G + l0 + l] = cscale(flip(B[Geo::b_idx(l, p)], p), scale);
    }
  }
}

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

}  // namespace rtnb
