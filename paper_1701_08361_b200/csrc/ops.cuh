// Per-grid-size kernel launchers (Engine::Ops) and the launch helper shared by the
// engine and the instantiation units inst*.cu (the 14 line-FFT geometries are
// compiled in parallel translation units).
#pragma once

#include <cmath>
#include <numeric>
#include <cstdlib>
#include <utility>
#include <vector>

#include "engine.hpp"
#include "kernels_impl.cuh"
#include "kernels_cluster.cuh"

#ifndef RTNB_LPB_WIDE
#define RTNB_LPB_WIDE 16
#endif
#ifndef RTNB_ROW_NAMED
#define RTNB_ROW_NAMED 0
#endif

namespace rtnb {

struct Engine::Ops {
  // the k_colsT P-tile tensor map's box (kColsTTmaP): LPB columns x colsT_box_rows rows
  int colsT_box_rows = 0;
  // LPB / NT: lines and threads per block of the column passes; LPBR: lines per block of
  // the row passes (k_rows1, k_rows2: fewer, wider-strided lines when NMAX does not divide 32)
  int G = 0, N1 = 0, N2 = 0, LPB = 0, NT = 0, LPBR = 0;
  int crA_N1 = 0;  // first-step length of the k_crA instantiation (it may come from another factorisation)
  size_t smem = 0;
  void (*colA)(cudaStream_t, int, Dims, const float*, const float4*, const float2*, float2*, int, int,
               const DevState*, int) = nullptr;
  void (*rows1)(cudaStream_t, int, Dims, int, const float4*, const float2*, const float2*, const float2*,
                const float2*, float2*, float2*, const float2*, float2*, const DevState*, int) = nullptr;
  void (*colsT)(cudaStream_t, int, Dims, const float4*, const float2*, float2*, const DevState*, int,
                const CUtensorMap*) = nullptr;
  void (*rows2)(cudaStream_t, int, Dims, int, const float4*, const float2*, const float2*,
                const float2*, const float2*, float2*, double2*, double*, DevState*, int) = nullptr;
  void (*colsW)(cudaStream_t, int, Dims, ColsWArgs, const float*, const float4*, const float2*,
                const double2*, const float2*, const float2*, int, double*, DevState*, CrScalars, int,
                const GroupView&) = nullptr;
  void (*fft)(cudaStream_t, int, int, float2*, int, int, const float4*, float) = nullptr;
  // CR recurrence + the next application's W^-1 column pass (k_crA)
  void (*crA)(cudaStream_t, int grid, int nbc, Dims, float2*, float2*, float2*, float2*, const float2*,
              const float*, const float4*, float2*, double*, DevState*, CrScalars, int, float,
              const DeferRed&) = nullptr;
  // whole application per channel in one thread-block cluster (kernels_cluster.cuh);
  // nullptr where not instantiated (grid, tail, CTA count per channel)
  void (*apply_cluster)(cudaStream_t, int J, Dims, ColsWArgs, const float*, const float4*, const float2*,
                        const float2*, const float2*, float2*, double*, const DevState*, int) = nullptr;
  int cluster_ctas = 0;
};

namespace {

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("RTN_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// launch with programmatic stream serialisation (see pdl_enter, kernels_impl.cuh)
template <typename... KArgs, typename... Args>
void launch_k(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(static_cast<unsigned>(block));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  check_cuda(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...), "launch");
}

inline void upload_small_twiddles() {
  float4 tw[528];
  for (int n = 1; n <= 32; ++n) {
    for (int k = 0; k < n; ++k) {
      const double a = -2.0 * 3.14159265358979323846 * k / n;
      const float c = static_cast<float>(std::cos(a)), sn = static_cast<float>(std::sin(a));
      tw[small_tw_offset(n) + k] = make_float4(c, sn, -sn, c);
    }
  }
  check_cuda(cudaMemcpyToSymbol(c_small_tw, tw, sizeof(tw)), "upload small twiddles");
}

template <int N1, int N2>
struct Inst {
  // 16 lines per block, 32 when that keeps the block a whole number of warps; the 20- and
  // 24-point geometries take RTNB_LPB_WIDE (column passes of 320 / 384 or 160 / 192 threads)
  static constexpr int kLpb = ((N1 > N2 ? N1 : N2) >= 20) ? RTNB_LPB_WIDE
                              : ((16 * (N1 > N2 ? N1 : N2)) % 32 == 0) ? 16 : 32;
  using Geo = LineGeom<N1, N2, kLpb>;
  static constexpr size_t kSmem = sizeof(float2) * Geo::SMEM_FLOAT2;
  static constexpr int kNT = Geo::NT;
  // row passes: a line owns RS thread slots, NMAX rounded up to a power of two when it
  // does not divide 32 (every line inside one warp: warp barriers between the transform
  // steps), with at most 256 threads per block
  static constexpr int kNMax = N1 > N2 ? N1 : N2;
  static constexpr int kRS = (32 % kNMax == 0) ? kNMax : (kNMax <= 8 ? 8 : kNMax <= 16 ? 16 : 32);
  // RTNB_ROW_NAMED=1: the 24-point lines keep NMAX slots and synchronise on named barriers
  // over lcm(NMAX, 32) threads (no idle lanes); measured C5 -16 % against the default RS
  // power-of-two slots (idle lanes, warp barriers): profiles/r02/ab_rows_named.txt
  static constexpr int kRG = (kNMax == 24 && RTNB_ROW_NAMED) ? std::lcm(kNMax, 32) : 0;
  static constexpr bool kNamed = kRG > 0 && (kLpb * kNMax) % kRG == 0 && (kLpb * kNMax) / kRG <= 15;
  static constexpr int kLpbR = (32 % kNMax == 0 || kNamed) ? kLpb : (kLpb < 256 / kRS ? kLpb : 256 / kRS);
  using GeoR = LineGeom<N1, N2, kLpbR, (32 % kNMax == 0 || kNamed) ? 0 : kRS, kNamed ? kRG : 0>;
  static constexpr size_t kSmemR = sizeof(float2) * GeoR::SMEM_FLOAT2;
  static constexpr int kNTR = GeoR::NT;
  // row pass 2: one window row x one group of kLpbR channels (+ the channel terms)
  static constexpr size_t kSmem2 = sizeof(float2) * (GeoR::SMEM_FLOAT2 + kLpbR * (N1 * N2 / 2));

  static void set_attrs() {
    // c_small_tw is a per-translation-unit __constant__ (no relocatable device code):
    // every instantiation unit uploads its own copy on the current device
    upload_small_twiddles();
    const int s = static_cast<int>(kSmem);
    check_cuda(cudaFuncSetAttribute(k_colA<Geo>, cudaFuncAttributeMaxDynamicSharedMemorySize, s), "attr colA");
    check_cuda(cudaFuncSetAttribute(k_rows1<GeoR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSmemR)),
               "attr rows1");
    check_cuda(cudaFuncSetAttribute(k_rows1<GeoR, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSmemR)),
               "attr rows1 decode");
    check_cuda(cudaFuncSetAttribute(k_colsT<Geo>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(colsT_smem_bytes<Geo>())),
               "attr colsT");
    check_cuda(cudaFuncSetAttribute(k_rows2<GeoR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSmem2)),
               "attr rows2");
    check_cuda(cudaFuncSetAttribute(k_colsW<Geo>, cudaFuncAttributeMaxDynamicSharedMemorySize, s), "attr colsW");
    check_cuda(cudaFuncSetAttribute(k_crA<Geo>, cudaFuncAttributeMaxDynamicSharedMemorySize, s), "attr crA");
    check_cuda(cudaFuncSetAttribute(k_fft_pass<Geo, -1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, s), "attr fft");
    check_cuda(cudaFuncSetAttribute(k_fft_pass<Geo, +1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, s), "attr ifft");
    check_cuda(cudaFuncSetAttribute(k_fft_pass<Geo, -1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, s), "attr fft");
    check_cuda(cudaFuncSetAttribute(k_fft_pass<Geo, +1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, s), "attr ifft");
  }

  static Engine::Ops make();
  template <int C>
  static void add_cluster(Engine::Ops& o);
};

}  // namespace

template <int N1, int N2>
Engine::Ops Inst<N1, N2>::make() {
  Engine::Ops o;
  o.G = N1 * N2;
  o.N1 = N1;
  o.N2 = N2;
  o.LPB = Geo::LPB;
  o.LPBR = GeoR::LPB;
  o.crA_N1 = N1;
  o.colsT_box_rows = kColsTTmaP<Geo> ? kColsTBoxRows<Geo> : 0;
  o.smem = kSmem;
  o.NT = kNT;
  o.colA = [](cudaStream_t s, int grid, Dims d, const float* winv, const float4* tw, const float2* chat,
              float2* U, int r0, int nr, const DevState* st, int h) {
    launch_k(k_colA<Geo>, grid, kNT, kSmem, s, d, winv, tw, chat, U, r0, nr, st, h);
  };
  o.rows1 = [](cudaStream_t s, int grid, Dims d, int mode, const float4* tw, const float2* U,
               const float2* coils, const float2* rhom, const float2* drho, float2* V, float2* coils_out,
               const float2* rho_src, float2* rhom_out, const DevState* st, int h) {
    launch_k((mode == R1_DECODE || mode == R1_DECODE_WIN || mode == R1_DECODE_SETUP) ? k_rows1<GeoR, true>
                                                                                    : k_rows1<GeoR, false>,
             grid,
             kNTR, kSmemR, s, d, mode, tw, U, coils, rhom, drho, V, coils_out, rho_src,
             rhom_out, st, h);
  };
  o.colsT = [](cudaStream_t s, int grid, Dims d, const float4* tw, const float2* P, float2* V,
               const DevState* st, int h, const CUtensorMap* tmP) {
    launch_k(k_colsT<Geo>, grid, kNT, colsT_smem_bytes<Geo>(), s, d, tw, P, V, st, h, *tmP);
  };
  o.rows2 = [](cudaStream_t s, int grid, Dims d, int setup, const float4* tw, const float2* V,
               const float2* coils, const float2* rhom, const float2* z, float2* Y, double2* RP,
               double* partials, DevState* st, int h) {
    launch_k(k_rows2<GeoR>, grid, kNTR, kSmem2, s, d, setup, tw, V, coils, rhom, z, Y, RP, partials, st, h);
  };
  o.colsW = [](cudaStream_t s, int grid, Dims d, ColsWArgs a, const float* winv, const float4* tw,
               const float2* Y, const double2* RP, const float2* coils, const float2* z, int nbw,
               double* partials, DevState* st, CrScalars cr, int h, const GroupView& gv) {
    launch_k(k_colsW<Geo>, grid, kNT, kSmem, s, d, a, winv, tw, Y, RP, coils, z, nbw, partials, st, cr, h, gv);
  };
  o.crA = [](cudaStream_t s, int grid, int nbc, Dims d, float2* x, float2* r, float2* p, float2* ap,
             const float2* ar, const float* winv, const float4* tw, float2* U, double* partials, DevState* st,
             CrScalars cr, int it, float tol, const DeferRed& dr) {
    launch_k(k_crA<Geo>, grid, kNT, kSmem, s, d, x, r, p, ap, ar, winv, tw, U, nbc, partials, st, cr, it, tol, dr);
  };
  o.fft = [](cudaStream_t s, int grid, int sign, float2* data, int batch, int axis, const float4* tw,
             float scale) {
    if (sign < 0) {
      if (axis == 0) {
        k_fft_pass<Geo, -1, true><<<grid, kNT, kSmem, s>>>(data, batch, tw, scale);
      } else {
        k_fft_pass<Geo, -1, false><<<grid, kNT, kSmem, s>>>(data, batch, tw, scale);
      }
    } else {
      if (axis == 0) {
        k_fft_pass<Geo, +1, true><<<grid, kNT, kSmem, s>>>(data, batch, tw, scale);
      } else {
        k_fft_pass<Geo, +1, false><<<grid, kNT, kSmem, s>>>(data, batch, tw, scale);
      }
    }
  };
  return o;
}


template <int N1, int N2>
template <int C>
void Inst<N1, N2>::add_cluster(Engine::Ops& o) {
  using CG = ClusterGeom<Geo, C>;
  o.cluster_ctas = C;
  o.apply_cluster = [](cudaStream_t s, int J, Dims d, ColsWArgs a, const float* winv, const float4* tw,
                       const float2* coils, const float2* rhom, const float2* P, float2* RC, double* kpart,
                       const DevState* st, int h) {
    static bool attr = [] {
      check_cuda(cudaFuncSetAttribute(k_apply_cluster<Geo, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(CG::SMEM)),
                 "attr cluster");
      return true;
    }();
    (void)attr;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(J * C));
    cfg.blockDim = dim3(static_cast<unsigned>(Geo::NT));
    cfg.dynamicSmemBytes = CG::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    check_cuda(cudaLaunchKernelEx(&cfg, k_apply_cluster<Geo, C>, d, a, winv, tw, coils, rhom, P, RC, kpart, st, h),
               "launch cluster apply");
  };
}

using OpsAttrList = std::vector<std::pair<int, void (*)()>>;
void add_ops_0(std::vector<Engine::Ops>& ops, OpsAttrList& attrs);
void add_ops_1(std::vector<Engine::Ops>& ops, OpsAttrList& attrs);
void add_ops_2(std::vector<Engine::Ops>& ops, OpsAttrList& attrs);
void add_ops_3(std::vector<Engine::Ops>& ops, OpsAttrList& attrs);

#define RTNB_INST(a, b)                  \
  ops.push_back(Inst<a, b>::make());     \
  attrs.push_back({a * b, &Inst<a, b>::set_attrs});

}  // namespace rtnb
