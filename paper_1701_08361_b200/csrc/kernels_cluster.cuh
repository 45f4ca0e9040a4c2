// One normal-operator application per channel in ONE thread-block cluster
// (sm_100a clusters + distributed shared memory), for the fused CR solve.
//
// The five line passes of an application (kernels_impl.cuh: colA, rows1, colsT, rows2,
// colsW) depend only on the same channel's previous pass, so a cluster of C CTAs per
// channel runs all of them with the channel's intermediates U, V, T, Y held in the
// cluster's shared memory: each pass writes its output lines straight into the shared
// memory of the CTA that owns them in the next pass (st.shared::cluster), and a
// cluster barrier separates the passes. Global memory sees only the operands (dchat_j,
// the window rows of c_j, rho, drho, P, the weights) and the results (out.chat_j, the
// channel term rc_j of out.rho, per-CTA dot partials).
//
//   pass A  W^-1 columns   CTA owns Gc/C coil columns     -> U rows   (owner: row block)
//   pass B  rows1          CTA owns L/C window rows       -> V cols   (owner: column block)
//   pass C  Toeplitz cols  CTA owns G/C columns           -> T rows   (owner: row block)
//   pass D  rows2          CTA owns L/C window rows       -> rc_j (global), Y cols
//   pass E  W^-H columns   CTA owns Gc/C coil columns     -> out.chat_j + dots
//
// k_rho_sum then forms out.rho = sum_j rc_j in channel order in FP64 (the reference's
// all_reduce_sum, decomp.cpp:26-39), the CR "+alpha p" and the dot products, and
// reduces every partial in a fixed order. Compiled only where G = 16 x 16 (C3/C4) and
// Gc = G/4; other plans keep the five-kernel path.
#pragma once

#include "kernels_impl.cuh"

namespace rtnb {

namespace {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t cluster_map(uint32_t addr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster(uint32_t addr, float2 v) {
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ int cluster_rank() {
  int r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

}  // namespace

template <class Geo, int C>
struct ClusterGeom {
  static constexpr int G = Geo::G, N1 = Geo::N1, N2 = Geo::N2;
  static constexpr int L = G / 2, LO = G / 4, GC = G / 4, OFF = G / 2 - GC / 2;
  static constexpr int RPC = L / C;     // window rows per CTA (passes B, D)
  static constexpr int CPC = G / C;     // columns per CTA (pass C)
  static constexpr int GCPC = GC / C;   // coil columns per CTA (passes A, E)
  static constexpr int VS = CPC + 1;    // V slab row stride (padded)
  static constexpr int UY_FLOAT2 = (RPC * GC > L * GCPC) ? RPC * GC : L * GCPC;
  static constexpr int V_FLOAT2 = L * VS;
  static constexpr int W_FLOAT2 = RPC * G;
  static constexpr size_t SMEM = sizeof(float2) * (Geo::SMEM_FLOAT2 + UY_FLOAT2 + V_FLOAT2 + W_FLOAT2);
  // step-1 input mask of the coil band t in [OFF, OFF + GC), step-2 output mask of the
  // same band (the W^-1 / W^-H pruning)
  static constexpr uint32_t GC_N1 = range_mask(OFF / N2, (OFF + GC) / N2);
  static constexpr uint32_t GC_K2 = range_mask(OFF / N1, (OFF + GC) / N1);
  static_assert(L % C == 0 && G % C == 0 && GC % C == 0, "cluster split");
  static_assert(OFF % N2 == 0 && GC % N2 == 0 && OFF % N1 == 0 && GC % N1 == 0, "coil band on the DFT grid");
  static_assert(RPC <= Geo::LPB && GCPC <= Geo::LPB && CPC % Geo::LPB == 0, "line batches");
  // step-2 slots k2 of the window outputs p = k1 + N1 k2 in [LO, LO + L) and of the coil
  // band [OFF, OFF + GC): the same for every k1 (prefetch indexing)
  static_assert(LO % N1 == 0 && L % N1 == 0, "window on the DFT grid");
  static constexpr int WK0 = LO / N1, WKN = L / N1, GK0 = OFF / N1, GKN = GC / N1;
};

namespace {
// block-wide FP64 sum of one value per thread (all threads return the total)
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < nw; ++w) t += red[w];
  return t;
}
}  // namespace

template <class Geo, int C>
__global__ void __launch_bounds__(Geo::NT, 2)
    k_apply_cluster(Dims d, ColsWArgs a, const float* __restrict__ winv, const float4* __restrict__ twG,
                    const float2* __restrict__ coils, const float2* __restrict__ rhom,
                    const float2* __restrict__ P, float2* __restrict__ RC, double* __restrict__ kpart,
                    const DevState* st, int use_halt) {
  using CG = ClusterGeom<Geo, C>;
  constexpr int G = CG::G, N1 = CG::N1, N2 = CG::N2, L = CG::L, LO = CG::LO, GC = CG::GC, OFF = CG::OFF;
  constexpr int RPC = CG::RPC, CPC = CG::CPC, GCPC = CG::GCPC, VS = CG::VS;
  pdl_enter();
  // uniform over the cluster: every CTA reads the same state written by earlier kernels
  if (st->status || (use_halt && st->cr_halt)) return;
  extern __shared__ float2 A[];
  float2* UY = A + Geo::SMEM_FLOAT2;
  float2* Vs = UY + CG::UY_FLOAT2;
  float2* Ws = Vs + CG::V_FLOAT2;
  const uint32_t uy_s = smem_addr(UY), vs_s = smem_addr(Vs), ws_s = smem_addr(Ws);
  const int rank = cluster_rank();
  const int j = blockIdx.x / C;
  const float2* dx = a.dx;
  const float2* cj = coils + (size_t)j * G * G;
  const Item<Geo, true> c1(threadIdx.x, N2), c2(threadIdx.x, N1);
  // square factorisations (N1 == N2, C3/C4): a row line is the same warp-local thread slots
  // in both steps, so the row passes exchange under warp barriers (measured: C1's 8 x 16
  // is faster with its packed step-2 slots and block barriers)
  constexpr bool kWarpRows = Geo::N1 == Geo::N2 && 32 % Geo::N1 == 0;
  const Item<Geo, false> r1(threadIdx.x, N2), r2(threadIdx.x, N1);
  float2 v[N1];
  float2 u[N2];

  // ---- pass A: W^-1 column pass of this CTA's coil columns -> U rows -------------------
  {
    const float2* src = dx + (size_t)G * G + (size_t)j * GC * GC;
    const bool a1 = c1.on && c1.l < GCPC, a2 = c2.on && c2.l < GCPC;
    if (a1) {
      const int q = rank * GCPC + c1.l;
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        const int t = N2 * n1 + c1.k;
        const int i = t - OFF;
        v[n1] = make_float2(0.f, 0.f);
        if (i >= 0 && i < GC) {
          const float w = winv[i * GC + q];
          const float2 c = src[i * GC + q];
          v[n1] = flip(make_float2(c.x * w, c.y * w), t);  // chat * winv.real() (nlinv.cpp:121)
        }
      }
      fft_step1<Geo, +1, CG::GC_N1>(v, c1.k, twG);
      park_step1<Geo>(A, c1.l, c1.k, v);
    }
    __syncthreads();
    if (a2) {
      fft_step2<Geo, +1, Geo::WIN_K2>(A, c2.l, c2.k, u);
      const int q = rank * GCPC + c2.l;
#pragma unroll
      for (int k2 = 0; k2 < N2; ++k2) {
        const int p = c2.k + N1 * k2;
        if (p >= LO && p < LO + L) {
          const int r = p - LO;
          st_cluster(cluster_map(uy_s + 8u * (uint32_t)((r % RPC) * GC + q), r / RPC), flip(u[k2], p));
        }
      }
    }
  }
  // pass B's pointwise operands (c_j, drho on its window rows) load while the cluster
  // barrier completes
  constexpr int WK0 = CG::WK0, WKN = CG::WKN;
  float2 pf0[WKN], pf1[WKN];
  cluster_arrive();
  if (r2.on && r2.l < RPC) {
    const size_t row = (size_t)(LO + rank * RPC + r2.l) * G;
#pragma unroll
    for (int kk = 0; kk < WKN; ++kk) {
      const size_t e = row + r2.k + N1 * (WK0 + kk);
      pf0[kk] = cj[e];
      pf1[kk] = dx[e];
    }
  }
  cluster_wait();

  // ---- pass B: rows1 on this CTA's window rows -> V columns ------------------------------
  {
    const bool a1 = r1.on && r1.l < RPC, a2 = r2.on && r2.l < RPC;
    const int R1 = LO + rank * RPC + r1.l, R2 = LO + rank * RPC + r2.l;
    if (a1) {
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        const int t = N2 * n1 + r1.k;
        const int qk = t - OFF;
        v[n1] = (qk >= 0 && qk < GC) ? flip(UY[r1.l * GC + qk], t) : make_float2(0.f, 0.f);
      }
      fft_step1<Geo, +1, CG::GC_N1>(v, r1.k, twG);
      park_step1<Geo>(A, r1.l, r1.k, v);
    }
    step_sync<kWarpRows>();
    if (a2) {
      fft_step2<Geo, +1, Geo::WIN_K2>(A, r2.l, r2.k, u);
#pragma unroll
      for (int k2 = 0; k2 < N2; ++k2) {
        const int p = r2.k + N1 * k2;
        float2 w = make_float2(0.f, 0.f);
        if (p >= LO && p < LO + L) {
          const size_t e = (size_t)R2 * G + p;
          const float2 aw = cscale(flip(u[k2], p), d.invG);
          // t = c_j * drho + rho * (W^-1 dchat_j)   (nlinv.cpp:163)
          const float2 s1 = cmul_rn(pf0[k2 - WK0], pf1[k2 - WK0]);
          const float2 s2 = cmul_rn(rhom[e], aw);
          w = flip(make_float2(__fadd_rn(s1.x, s2.x), __fadd_rn(s1.y, s2.y)), p);
        }
        u[k2] = w;
      }
    }
    if constexpr (kWarpRows) {
      // the forward Toeplitz row transform in the reverse step order (as k_rows1)
      if (a2) inv_inner<Geo, -1, Geo::WIN_K2>(A, r2.l, r2.k, u, twG);
      step_sync<kWarpRows>();
      if (a1) {
        get_step1<Geo>(A, r1.l, r1.k, v);
        dft_m<N1, -1, Geo::ALL_N1, Geo::ALL_N1>(v);
        const int r = rank * RPC + r1.l;
#pragma unroll
        for (int n1 = 0; n1 < N1; ++n1) {
          const int p = N2 * n1 + r1.k;
          st_cluster(cluster_map(vs_s + 8u * (uint32_t)(r * VS + p % CPC), p / CPC), flip(v[n1], p));
        }
      }
    } else {
      step_sync<kWarpRows>();
      if (a2) put_natural<Geo>(A, r2.l, r2.k, u);
      step_sync<kWarpRows>();
      if (a1) {
        get_step1<Geo>(A, r1.l, r1.k, v);
        fft_step1<Geo, -1, Geo::WIN_N1>(v, r1.k, twG);
        park_step1<Geo>(A, r1.l, r1.k, v);
      }
      step_sync<kWarpRows>();
      if (a2) {
        fft_step2<Geo, -1>(A, r2.l, r2.k, u);
        const int r = rank * RPC + r2.l;
#pragma unroll
        for (int k2 = 0; k2 < N2; ++k2) {
          const int p = r2.k + N1 * k2;
          st_cluster(cluster_map(vs_s + 8u * (uint32_t)(r * VS + p % CPC), p / CPC), flip(u[k2], p));
        }
      }
    }
    (void)R1;
  }
  cluster_barrier();

  // ---- pass C: Toeplitz column pass on this CTA's columns -> T rows ----------------------
#pragma unroll 1
  for (int b = 0; b < CPC / Geo::LPB; ++b) {
    const int ql1 = b * Geo::LPB + c1.l, ql2 = b * Geo::LPB + c2.l;
    if (c1.on) {
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        const int t = N2 * n1 + c1.k;
        v[n1] = (t >= LO && t < LO + L) ? flip(Vs[(t - LO) * VS + ql1], t) : make_float2(0.f, 0.f);
      }
      fft_step1<Geo, -1, Geo::WIN_N1>(v, c1.k, twG);
      park_step1<Geo>(A, c1.l, c1.k, v);
    }
    __syncthreads();
    if (c2.on) {
      fft_step2<Geo, -1>(A, c2.l, c2.k, u);
      const float2* Pc = P + rank * CPC + ql2;
#pragma unroll
      for (int k2 = 0; k2 < N2; ++k2) {
        const int p = c2.k + N1 * k2;
        u[k2] = cscale(cmul(u[k2], Pc[(size_t)p * G]), d.invG);
      }
      // inverse in the reverse step order (as k_colsT): inner DFTs in registers
      inv_inner<Geo, +1>(A, c2.l, c2.k, u, twG);
    }
    __syncthreads();
    if (c1.on) {
      get_step1<Geo>(A, c1.l, c1.k, v);
      dft_m<N1, +1, Geo::ALL_N1, Geo::WIN_N1>(v);
      const int q = rank * CPC + ql1;
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        const int t = N2 * n1 + c1.k;
        if (t >= LO && t < LO + L) {
          const int r = t - LO;
          st_cluster(cluster_map(ws_s + 8u * (uint32_t)((r % RPC) * G + q), r / RPC), flip(v[n1], t));
        }
      }
    }
    __syncthreads();
  }
  cluster_arrive();
  if (r2.on && r2.l < RPC) {
    const size_t row = (size_t)(LO + rank * RPC + r2.l) * G;
#pragma unroll
    for (int kk = 0; kk < WKN; ++kk) {
      const size_t e = row + r2.k + N1 * (WK0 + kk);
      pf0[kk] = cj[e];
      pf1[kk] = rhom[e];
    }
  }
  cluster_wait();

  // ---- pass D: rows2 on this CTA's window rows -> rc_j (global), Y columns ---------------
  {
    const bool a1 = r1.on && r1.l < RPC, a2 = r2.on && r2.l < RPC;
    const int r = rank * RPC + r2.l;
    if (a1) {
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        const int t = N2 * n1 + r1.k;
        v[n1] = flip(Ws[r1.l * G + t], t);
      }
      fft_step1<Geo, +1>(v, r1.k, twG);
      park_step1<Geo>(A, r1.l, r1.k, v);
    }
    step_sync<kWarpRows>();
    if (a2) {
      fft_step2<Geo, +1, Geo::WIN_K2>(A, r2.l, r2.k, u);
      float2* rc = RC + (size_t)j * L * L + (size_t)r * L;
#pragma unroll
      for (int k2 = 0; k2 < N2; ++k2) {
        const int p = r2.k + N1 * k2;
        float2 w = make_float2(0.f, 0.f);
        if (p >= LO && p < LO + L) {
          const float2 T = cscale(flip(u[k2], p), d.invG);
          rc[p - LO] = cjmul_rn(pf0[k2 - WK0], T);  // rc_j = conj(c_j) T_j   (nlinv.cpp:166)
          w = flip(cjmul_rn(pf1[k2 - WK0], T), p);  // rt_j = conj(rho) T_j   (nlinv.cpp:167)
        }
        u[k2] = w;
      }
    }
    if constexpr (kWarpRows) {
      // the forward W^-H row transform in the reverse step order (as k_rows2)
      if (a2) inv_inner<Geo, -1, Geo::WIN_K2>(A, r2.l, r2.k, u, twG);
      step_sync<kWarpRows>();
      if (a1) {
        get_step1<Geo>(A, r1.l, r1.k, v);
        dft_m<N1, -1, Geo::ALL_N1, CG::GC_N1>(v);
        const int r1w = rank * RPC + r1.l;
#pragma unroll
        for (int n1 = 0; n1 < N1; ++n1) {
          const int p = N2 * n1 + r1.k;
          const int q = p - OFF;
          if (q >= 0 && q < GC) {
            st_cluster(cluster_map(uy_s + 8u * (uint32_t)(r1w * GCPC + q % GCPC), q / GCPC), flip(v[n1], p));
          }
        }
      }
    } else {
      step_sync<kWarpRows>();
      if (a2) put_natural<Geo>(A, r2.l, r2.k, u);
      step_sync<kWarpRows>();
      if (a1) {
        get_step1<Geo>(A, r1.l, r1.k, v);
        fft_step1<Geo, -1, Geo::WIN_N1>(v, r1.k, twG);
        park_step1<Geo>(A, r1.l, r1.k, v);
      }
      step_sync<kWarpRows>();
      if (a2) {
        fft_step2<Geo, -1, CG::GC_K2>(A, r2.l, r2.k, u);
#pragma unroll
        for (int k2 = 0; k2 < N2; ++k2) {
          const int p = r2.k + N1 * k2;
          const int q = p - OFF;
          if (q >= 0 && q < GC) {
            st_cluster(cluster_map(uy_s + 8u * (uint32_t)(r * GCPC + q % GCPC), q / GCPC), flip(u[k2], p));
          }
        }
      }
    }
  }
  // pass E's CR operands and weights (its outputs are the coil band k2 in [GK0, GK0 + GKN)),
  // requested before the barrier so they land during it
  constexpr int GK0 = CG::GK0, GKN = CG::GKN;
  const size_t cbase = (size_t)G * G + (size_t)j * GC * GC;
  float2 edx[GKN], eap[GKN];
  float ew[GKN];
  if (c2.on && c2.l < GCPC) {
    const int q = rank * GCPC + c2.l;
#pragma unroll
    for (int kk = 0; kk < GKN; ++kk) {
      const int e = (c2.k + N1 * kk) * GC + q;  // k-row i = p - OFF of slot k2 = GK0 + kk
      ew[kk] = winv[e];
      edx[kk] = a.dx[cbase + e];
      eap[kk] = a.ap_prev ? a.ap_prev[cbase + e] : make_float2(0.f, 0.f);
    }
  }
  cluster_barrier();

  // ---- pass E: W^-H column pass of this CTA's coil columns -> out.chat_j + dots ----------
  double acc = 0.0, aa = 0.0, pa = 0.0;
  {
    const bool a1 = c1.on && c1.l < GCPC, a2 = c2.on && c2.l < GCPC;
    if (a1) {
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        const int t = N2 * n1 + c1.k;
        v[n1] = (t >= LO && t < LO + L) ? flip(UY[(t - LO) * GCPC + c1.l], t) : make_float2(0.f, 0.f);
      }
      fft_step1<Geo, -1, Geo::WIN_N1>(v, c1.k, twG);
      park_step1<Geo>(A, c1.l, c1.k, v);
    }
    __syncthreads();
    if (a2) {
      fft_step2<Geo, -1, CG::GC_K2>(A, c2.l, c2.k, u);
      const int q = rank * GCPC + c2.l;
#pragma unroll
      for (int kk = 0; kk < GKN; ++kk) {
        const int p = c2.k + N1 * (GK0 + kk);
        const int e = (p - OFF) * GC + q;
        const float2 f = cscale(flip(u[GK0 + kk], p), d.invG);
        // crop_k(FFT(u)) * winv   (nlinv.cpp:127-133)
        finish_op(a, cbase + e, make_float2(f.x * ew[kk], f.y * ew[kk]), edx[kk], eap[kk], acc, aa, pa);
      }
    }
  }
  __shared__ double red[32];
  const double t0 = block_sum(acc, red);
  const double t1 = block_sum(aa, red);
  const double t2 = block_sum(pa, red);
  if (threadIdx.x == 0) {
    kpart[3 * blockIdx.x + 0] = t0;
    kpart[3 * blockIdx.x + 1] = t1;
    kpart[3 * blockIdx.x + 2] = t2;
  }
}

#ifndef RTNB_PASS_ONLY
// out.rho = sum_j rc_j on the window (zero outside, where T is masked) in FP64 in a
// fixed order, the CR "+alpha dx" and the dots of the rho part, plus the coil-part
// partials of k_apply_cluster (block b takes entries b, b + grid, ...); one grid
// reduction publishes rar / saa / spa. A block takes 32 consecutive entries: lane =
// entry (coalesced channel rows), warp w sums channels w, w + 8, ... (independent loads
// in flight), the 8 warp partials are added in warp order in shared memory. Warp 0
// loads the finish operands (dx, ap_prev) before the channel sums land.
constexpr int kRhoTile = 32;
// Channel decomposition (d.grp): every member runs this kernel after an all-member barrier;
// out.rho reads each channel's term from its owner's RC (peer memory) in the single-device
// channel order, the rho part of the dots is counted on one member, the coil part from the
// member's own cluster partials, and the member's dot partials go to cr.pcw for k_grp_fin.
__global__ void __launch_bounds__(kThreads) k_rho_sum(Dims d, ColsWArgs a, const float2* __restrict__ RC,
                                                      const double* __restrict__ kpart, int nk, double* partials,
                                                      DevState* st, CrScalars cr, int use_halt, GroupView gv) {
  pdl_enter();
  if (st->status || (use_halt && st->cr_halt)) return;
  __shared__ double2 part[kThreads / 32][kRhoTile];
  const int G = d.G, L = d.L, D0 = G * G;
  const bool win_only = a.win_only_ok && rho_window_only(st);
  const int nv = win_only ? L * L : D0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kThreads / 32;
  double acc = 0.0, aa = 0.0, pa = 0.0;
  for (int i = blockIdx.x + threadIdx.x * gridDim.x; i < nk; i += blockDim.x * gridDim.x) {
    acc += __ldcg(kpart + 3 * i);
    aa += __ldcg(kpart + 3 * i + 1);
    pa += __ldcg(kpart + 3 * i + 2);
  }
  for (int v0 = blockIdx.x * kRhoTile; v0 < nv; v0 += gridDim.x * kRhoTile) {
    const int v = v0 + lane;
    int e = -1, r = 0, c = 0;
    if (v < nv) {
      if (win_only) {
        r = d.lo + v / L;
        c = d.lo + v - (v / L) * L;
        e = r * G + c;
      } else {
        e = v;
        r = e / G;
        c = e - (e / G) * G;
      }
    }
    float2 pdx = make_float2(0.f, 0.f), pap = make_float2(0.f, 0.f);
    if (warp == 0 && e >= 0) {
      pdx = a.dx[e];
      if (a.ap_prev) pap = a.ap_prev[e];
    }
    double sx = 0.0, sy = 0.0;
    if (e >= 0 && in_win(d, r, c)) {
      const size_t w = (size_t)(r - d.lo) * L + (c - d.lo);
      const float2* src = RC + w;
      const int Jt = d.grp ? gv.jb[gv.A] : d.J;
      constexpr int kB = 4;
      for (int j0 = warp; j0 < Jt; j0 += kB * nw) {
        float2 t[kB];
#pragma unroll
        for (int q = 0; q < kB; ++q) {
          const int jj = j0 + q * nw;
          if (jj >= Jt) {
            t[q] = make_float2(0.f, 0.f);
          } else if (d.grp) {
            int m = 0;
            while (jj >= gv.jb[m + 1]) ++m;
            t[q] = __ldcg(gv.rc[m] + (size_t)(jj - gv.jb[m]) * L * L + w);
          } else {
            t[q] = __ldcg(src + (size_t)jj * L * L);
          }
        }
#pragma unroll
        for (int q = 0; q < kB; ++q) {
          sx += t[q].x;
          sy += t[q].y;
        }
      }
    }
    part[warp][lane] = make_double2(sx, sy);
    __syncthreads();
    if (warp == 0 && e >= 0) {
      double tx = 0.0, ty = 0.0;
      for (int w = 0; w < nw; ++w) {
        tx += part[w][lane].x;
        ty += part[w][lane].y;
      }
      if (d.count_rho) {
        finish_op(a, (size_t)e, make_float2((float)tx, (float)ty), pdx, pap, acc, aa, pa);
      } else {  // the replicated rho part of the dots is counted on member 0 only
        double z0 = 0.0, z1 = 0.0, z2 = 0.0;
        finish_op(a, (size_t)e, make_float2((float)tx, (float)ty), pdx, pap, z0, z1, z2);
      }
    }
    __syncthreads();
  }
  double vv[3] = {acc, aa, pa}, tot[3];
  if (a.defer_out) {  // per-block partials for the recurrence (DeferRed)
    block_partial<3>(vv, a.defer_out);
    return;
  }
  if (grid_reduce<3>(vv, partials, &st->counter, tot) && threadIdx.x == 0) {
    if (d.grp) {  // member partials; k_grp_fin forms the totals in member order
      if (a.dot_slot >= 0) {
        cr.pcw[3 * a.dot_slot + 0] = tot[0];
        cr.pcw[3 * a.dot_slot + 1] = tot[1];
        cr.pcw[3 * a.dot_slot + 2] = tot[2];
      } else {
        st->scal[0] = tot[0];
      }
      return;
    }
    if (a.dot_slot >= 0) {
      cr.rar[a.dot_slot] = tot[0];
      cr.saa[a.dot_slot] = tot[1];
      cr.spa[a.dot_slot] = tot[2];
    } else {
      st->scal[0] = tot[0];
    }
  }
}
#endif  // RTNB_PASS_ONLY

}  // namespace rtnb
