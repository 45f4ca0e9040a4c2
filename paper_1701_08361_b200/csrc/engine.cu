// Engine: device buffers, size dispatch and kernel sequencing for one plan.
#include "engine.hpp"

#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstddef>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <numbers>
#include <string>

#include "ops.cuh"

namespace rtnb {

// ------------------------------------------------------------------------------
// errors, FFT accounting
// ------------------------------------------------------------------------------

void fail(int code, const std::string& msg) { throw Error(code, msg); }
void fail_decomp(const std::string& msg) { throw Error(4, msg, true); }

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(5, std::string(what) + ": " + cudaGetErrorString(e));
}

namespace {
std::atomic<uint64_t> g_counts[4];
thread_local int t_ctx = CTX_OTHER;
}  // namespace

int fft_current_ctx() { return t_ctx; }
void fft_set_ctx(int c) { t_ctx = c; }
void fft_book(int ctx, uint64_t n) { g_counts[ctx & 3].fetch_add(n, std::memory_order_relaxed); }
uint64_t fft_count(int ctx) { return g_counts[ctx & 3].load(); }
uint64_t fft_count_total() {
  uint64_t t = 0;
  for (auto& c : g_counts) t += c.load();
  return t;
}
void fft_reset_counts() {
  for (auto& c : g_counts) c.store(0);
}

// ------------------------------------------------------------------------------
// small pointwise kernels for the op-level primitives
// ------------------------------------------------------------------------------

namespace {

__global__ void k_pad_weight(const float2* __restrict__ chat, const float* __restrict__ winv, int Gc,
                             int G, float2* __restrict__ out) {
  const int off = G / 2 - Gc / 2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < G * G; e += gridDim.x * blockDim.x) {
    const int r = e / G - off, c = e % G - off;
    float2 v = make_float2(0.f, 0.f);
    if (r >= 0 && r < Gc && c >= 0 && c < Gc) {
      const float w = winv[r * Gc + c];
      const float2 x = chat[r * Gc + c];
      v = make_float2(x.x * w, x.y * w);
    }
    out[e] = v;
  }
}

__global__ void k_crop_weight(const float2* __restrict__ in, const float* __restrict__ winv, int Gc,
                              int G, float2* __restrict__ out) {
  const int off = G / 2 - Gc / 2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < Gc * Gc; e += gridDim.x * blockDim.x) {
    const int r = e / Gc, c = e % Gc;
    const float2 x = in[(size_t)(r + off) * G + c + off];
    const float w = winv[e];
    out[e] = make_float2(x.x * w, x.y * w);
  }
}

__global__ void k_mask(float2* __restrict__ x, int G) {
  const int L = G / 2, lo = (G - L) / 2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < G * G; e += gridDim.x * blockDim.x) {
    const int r = e / G, c = e % G;
    if (!(r >= lo && r < lo + L && c >= lo && c < lo + L)) x[e] = make_float2(0.f, 0.f);
  }
}

__global__ void k_mul(float2* __restrict__ x, const float2* __restrict__ P, int n) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    const float2 a = x[e], b = P[e];
    x[e] = make_float2(__fsub_rn(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y)),
                       __fadd_rn(__fmul_rn(a.x, b.y), __fmul_rn(a.y, b.x)));
  }
}

}  // namespace

// ------------------------------------------------------------------------------
// size dispatch
// ------------------------------------------------------------------------------

namespace {

struct Registry {
  std::mutex mu;
  std::vector<Engine::Ops> ops;
  std::vector<std::pair<int, void (*)()>> attrs;  // per G, run once per device
  std::vector<std::vector<int>> attrs_done;       // [device] -> list of G
  std::vector<std::pair<std::pair<int, int>, float4*>> twG;  // (device, G) -> table
  std::vector<std::pair<std::pair<int, int>, double2*>> twD;  // (device, n*sign) -> direct table
};

// TMA descriptor of a G x G complex64 array (8-byte elements, row pitch 8G) read in boxes
// of lpb columns x rows rows (k_colsT's P tiles). cuTensorMapEncodeTiled comes from the
// driver through the runtime's entry-point query (no link against libcuda).
void encode_psf_map(CUtensorMap* map, const float2* P, int G, int lpb, int rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    check_cuda(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q), "tensor map entry");
    if (!fn || q != cudaDriverEntryPointSuccess) fail(5, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  const cuuint64_t dim[2] = {static_cast<cuuint64_t>(G), static_cast<cuuint64_t>(G)};
  const cuuint64_t stride[1] = {static_cast<cuuint64_t>(G) * sizeof(float2)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(lpb), static_cast<cuuint32_t>(rows)};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<float2*>(P), dim, stride, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(5, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
}

Registry& registry() {
  static Registry* r = [] {
    auto* reg = new Registry;
    add_ops_0(reg->ops, reg->attrs);
    add_ops_1(reg->ops, reg->attrs);
    add_ops_2(reg->ops, reg->attrs);
    add_ops_3(reg->ops, reg->attrs);
    // Per-kernel factorisation preferences (measured, scripts/prof_kernels.py): the last
    // registration of a grid side is its default; a kernel may come from another
    // factorisation with the same lines per block (same k_rows2 channel grouping)
    auto alt_of = [&](int G, int N1, int N2, Engine::Ops*& dflt) -> const Engine::Ops* {
      dflt = nullptr;
      const Engine::Ops* alt = nullptr;
      for (auto& o : reg->ops) {
        if (o.G == G) dflt = &o;
        if (o.G == G && o.N1 == N1 && o.N2 == N2) alt = &o;
      }
      return (dflt && alt != dflt) ? alt : nullptr;
    };
    auto prefer_rows2 = [&](int G, int N1, int N2) {
      Engine::Ops* dflt = nullptr;
      const Engine::Ops* alt = alt_of(G, N1, N2, dflt);
      if (alt && dflt->LPBR == alt->LPBR) dflt->rows2 = alt->rows2;
    };
    // a column pass from another factorisation (same lines per block; U / Y layouts do not
    // depend on the factorisation): the 16 x 24 k_colA holds its 16-point first step in
    // registers where the 24 x 16 one spills
    auto prefer_colA = [&](int G, int N1, int N2) {
      Engine::Ops* dflt = nullptr;
      const Engine::Ops* alt = alt_of(G, N1, N2, dflt);
      if (alt && dflt->LPB == alt->LPB) dflt->colA = alt->colA;
    };
    prefer_rows2(320, 20, 16);
    prefer_colA(384, 16, 24);  // spill-free, neutral at C5 (k_crA from 16 x 24 there: -1.5 %)
    // measured per kernel (RTN_GEO_<G>_<kernel>, profiles/r02/ab_geo_per_kernel.txt):
    // G = 320's k_colsW from 20 x 16 (C2 +6 %), G = 384's k_rows1 from 16 x 24 (C5 +0.9 %)
    {
      Engine::Ops* dflt = nullptr;
      if (const Engine::Ops* alt = alt_of(320, 20, 16, dflt); alt && dflt->LPB == alt->LPB) dflt->colsW = alt->colsW;
      if (const Engine::Ops* alt = alt_of(384, 16, 24, dflt); alt && dflt->LPBR == alt->LPBR) dflt->rows1 = alt->rows1;
    }
    // tuning: RTN_GEO_<G>_<kernel>=N1xN2 takes one pass kernel of the default geometry of G
    // from another factorisation with the same lines per block
    for (auto& o : reg->ops) {
      for (const char* k : {"colA", "rows1", "colsT", "rows2", "colsW", "crA"}) {
        const std::string var = "RTN_GEO_" + std::to_string(o.G) + "_" + k;
        const char* e = std::getenv(var.c_str());
        if (!e) continue;
        int n1 = 0, n2 = 0;
        if (std::sscanf(e, "%dx%d", &n1, &n2) != 2) continue;
        Engine::Ops* dflt = nullptr;
        const Engine::Ops* alt = alt_of(o.G, n1, n2, dflt);
        if (!alt || dflt != &o) continue;
        const std::string kk(k);
        if (kk == "colA" && alt->LPB == o.LPB) o.colA = alt->colA;
        if (kk == "colsT" && alt->LPB == o.LPB) o.colsT = alt->colsT;
        if (kk == "colsW" && alt->LPB == o.LPB) o.colsW = alt->colsW;
        if (kk == "crA" && alt->LPB == o.LPB) {
          o.crA = alt->crA;
          o.crA_N1 = alt->crA_N1;
        }
        if (kk == "rows1" && alt->LPBR == o.LPBR) o.rows1 = alt->rows1;
        if (kk == "rows2" && alt->LPBR == o.LPBR) o.rows2 = alt->rows2;
      }
    }
    return reg;
  }();
  return *r;
}

// per-device one-time setup: small-DFT constant table and kernel attributes for G
const Engine::Ops* ops_for(int G, int dev) {
  Registry& r = registry();
  std::lock_guard<std::mutex> lock(r.mu);
  const Engine::Ops* found = nullptr;
  // RTN_GEO_<G>=N1xN2 picks one of several factorisations of G (tuning)
  int want1 = 0, want2 = 0;
  if (const char* e = std::getenv(("RTN_GEO_" + std::to_string(G)).c_str())) std::sscanf(e, "%dx%d", &want1, &want2);
  for (const auto& o : r.ops) {
    if (o.G == G && (!want1 || (o.N1 == want1 && o.N2 == want2))) found = &o;
  }
  if (!found) return nullptr;
  if (dev < 0 || dev >= 64) fail(2, "device index out of range");
  if (r.attrs_done.size() <= static_cast<size_t>(dev)) r.attrs_done.resize(dev + 1);
  bool done = false;
  for (int g : r.attrs_done[dev]) done = done || g == G;
  if (!done) {
    for (auto& a : r.attrs) {
      if (a.first == G) a.second();
    }
    r.attrs_done[dev].push_back(G);
  }
  return found;
}

// W_G^e, e < G, as packed operand pairs {w.x, w.y, -w.y, w.x} (cmul_pk), for the
// forward sign, then their conjugates {w.x, -w.y, w.y, w.x} for the inverse
float4* twiddles_for(int G, int dev) {
  Registry& r = registry();
  std::lock_guard<std::mutex> lock(r.mu);
  for (auto& e : r.twG) {
    if (e.first == std::make_pair(dev, G)) return e.second;
  }
  std::vector<float4> h(2 * static_cast<size_t>(G));
  for (int e = 0; e < G; ++e) {
    const double a = -2.0 * std::numbers::pi * e / G;
    const float c = static_cast<float>(std::cos(a)), sn = static_cast<float>(std::sin(a));
    h[static_cast<size_t>(e)] = make_float4(c, sn, -sn, c);
    h[static_cast<size_t>(G + e)] = make_float4(c, -sn, sn, c);
  }
  float4* d = nullptr;
  check_cuda(cudaMalloc(&d, sizeof(float4) * h.size()), "twiddle alloc");
  check_cuda(cudaMemcpy(d, h.data(), sizeof(float4) * h.size(), cudaMemcpyHostToDevice), "twiddle upload");
  r.twG.push_back({{dev, G}, d});
  return d;
}

double2* direct_table(int n, int sign, int dev) {
  Registry& r = registry();
  std::lock_guard<std::mutex> lock(r.mu);
  const int key = n * (sign < 0 ? -1 : 1);
  for (auto& e : r.twD) {
    if (e.first == std::make_pair(dev, key)) return e.second;
  }
  std::vector<double2> h(static_cast<size_t>(n));
  for (int e = 0; e < n; ++e) {
    const double a = (sign < 0 ? -2.0 : 2.0) * std::numbers::pi * e / n;
    h[static_cast<size_t>(e)] = make_double2(std::cos(a), std::sin(a));
  }
  double2* d = nullptr;
  check_cuda(cudaMalloc(&d, sizeof(double2) * n), "direct table alloc");
  check_cuda(cudaMemcpy(d, h.data(), sizeof(double2) * n, cudaMemcpyHostToDevice), "direct table upload");
  r.twD.push_back({{dev, key}, d});
  return d;
}

int blocks_for(long long n, int cap) {
  long long b = (n + kThreads - 1) / kThreads;
  if (b < 1) b = 1;
  return static_cast<int>(b > cap ? cap : b);
}

}  // namespace

bool grid_supported(int G) {
  for (const auto& o : registry().ops) {
    if (o.G == G) return true;
  }
  return false;
}

void fft2_device(float2* data, int n, int batch, int sign, cudaStream_t s) {
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "get device");
  const Engine::Ops* ops = (n % 2 == 0) ? ops_for(n, dev) : nullptr;
  if (ops) {
    const float4* tw = twiddles_for(n, dev);
    const int grid = batch * ((n + ops->LPB - 1) / ops->LPB);
    ops->fft(s, grid, sign, data, batch, 1, tw, 1.0f);
    ops->fft(s, grid, sign, data, batch, 0, tw, 1.0f / n);
  } else {
    // direct centered DFT per line (any side, including odd; fft.cpp:37-40 convention)
    const double2* tw = direct_table(n, sign, dev);
    float2* tmp = nullptr;
    check_cuda(cudaMallocAsync(&tmp, sizeof(float2) * n * n * batch, s), "fft tmp");
    k_dft_direct<<<batch * n, 128, sizeof(float2) * n, s>>>(data, tmp, n, batch, 1, tw, 1.0f);
    k_dft_direct<<<batch * n, 128, sizeof(float2) * n, s>>>(tmp, data, n, batch, 0, tw, 1.0f / n);
    check_cuda(cudaFreeAsync(tmp, s), "fft tmp free");
  }
  check_cuda(cudaGetLastError(), "fft launch");
}

// ------------------------------------------------------------------------------
// Engine
// ------------------------------------------------------------------------------

Engine::Engine(const Plan& plan, int device) : plan_(plan), dev_(device) {
  if (plan.G < 2 || plan.G % 2 != 0) fail(2, "plan: grid side G must be even and >= 2");
  if (plan.Gc < 1 || plan.Gc > plan.G) fail(2, "make_weights_inv: need 1 <= Gc <= G");
  if (plan.J < 1) fail(2, "plan: need at least one channel");
  if (plan.N < 1 || plan.N > plan.G) fail(2, "plan: image side N must be in [1, G]");
  if (plan.newton_steps < 0 || plan.newton_steps > kMaxSteps) fail(2, "plan: newton_steps out of range");
  check_cuda(cudaSetDevice(dev_), "set device");
  ops_ = ops_for(plan.G, dev_);
  if (!ops_) fail(2, "grid side " + std::to_string(plan.G) + " is not supported by the sm_100a line FFT");
  dims_.G = plan.G;
  dims_.Gc = plan.Gc;
  dims_.J = plan.J;
  dims_.L = plan.G / 2;
  dims_.lo = (plan.G - dims_.L) / 2;
  dims_.off = plan.G / 2 - plan.Gc / 2;
  dims_.N = plan.N;
  dims_.invG = 1.0f / static_cast<float>(plan.G);
  dims_.H = (plan.J + ops_->LPBR - 1) / ops_->LPBR;
  dims_.grp = 0;
  dims_.count_rho = 1;
  D_ = plan.G * plan.G + plan.J * plan.Gc * plan.Gc;
  check_cuda(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking), "stream");
  if (const char* e = std::getenv("RTN_FUSED_CR")) fused_cr_ = e[0] != '0';
  // k_crA by measurement: +4 % at C3 and C4 (16 x 16); the 24-point step-1 geometries
  // (C5's 24 x 16) hold too many CR operands with their DFT and lose 2 %
  fused_crA_ = ops_->crA_N1 <= 16;
  if (const char* e = std::getenv("RTN_CRA")) fused_crA_ = e[0] != '0';
  alloc();
}

Engine::~Engine() {
  cudaSetDevice(dev_);
  cudaStreamSynchronize(s_);
  for (auto& g : step_graph_) {
    if (g) cudaGraphExecDestroy(g);
  }
  if (frame_graph_) cudaGraphExecDestroy(frame_graph_);
  void* bufs[] = {winv_, P_, z_, x_, xcg_, r_, p_, ap_, ar_, reg_, est_scratch_[0], est_scratch_[1],
                  est_scratch_[2], coils_, rhom_, U_, V_, Y_, RP_, gbuf_, img_, partials_, st_, cr_buf_,
                  RPO_, SS_, RC_, kpart_, dpart_w_};
  for (void* b : bufs) {
    if (b) cudaFree(b);
  }
  if (st_host_) cudaFreeHost(st_host_);
  if (s_) cudaStreamDestroy(s_);
}

void Engine::alloc() {
  const size_t G2 = static_cast<size_t>(plan_.G) * plan_.G;
  const size_t J = static_cast<size_t>(plan_.J);
  const size_t L = static_cast<size_t>(dims_.L);
  auto c2 = [](float2** p, size_t n, const char* w) {
    check_cuda(cudaMalloc(p, sizeof(float2) * std::max<size_t>(n, 1)), w);
    check_cuda(cudaMemset(*p, 0, sizeof(float2) * std::max<size_t>(n, 1)), w);
  };
  // W^-1 weights in double, stored as float (make_weights_inv, nlinv.cpp:101-117)
  winv_host_.assign(static_cast<size_t>(plan_.Gc) * plan_.Gc, 0.f);
  const int c = plan_.Gc / 2;
  for (int r = 0; r < plan_.Gc; ++r) {
    for (int q = 0; q < plan_.Gc; ++q) {
      const double ky = (r - c) / static_cast<double>(plan_.G);
      const double kx = (q - c) / static_cast<double>(plan_.G);
      const double w = std::pow(1.0 + 880.0 * (kx * kx + ky * ky), 16.0);
      winv_host_[static_cast<size_t>(r) * plan_.Gc + q] = static_cast<float>(1.0 / w);
    }
  }
  check_cuda(cudaMalloc(&winv_, sizeof(float) * winv_host_.size()), "winv");
  check_cuda(cudaMemcpy(winv_, winv_host_.data(), sizeof(float) * winv_host_.size(), cudaMemcpyHostToDevice),
             "winv upload");
  twG_ = twiddles_for(plan_.G, dev_);
  c2(&P_, G2, "psf");
  c2(&z_, J * G2, "z");
  for (float2** b : {&x_, &xcg_, &r_, &p_, &ap_, &ar_, &reg_, &est_scratch_[0], &est_scratch_[1], &est_scratch_[2]}) {
    c2(b, static_cast<size_t>(D_), "estimate");
  }
  c2(&coils_, J * G2, "coils");
  c2(&rhom_, G2, "rho");
  c2(&U_, J * plan_.G * plan_.Gc, "U");
  c2(&V_, J * L * plan_.G, "V");
  c2(&Y_, J * L * plan_.Gc, "Y");
  check_cuda(cudaMalloc(&RP_, sizeof(double2) * dims_.H * L * L), "RP");
  c2(&gbuf_, G2, "scratch");
  c2(&img_, static_cast<size_t>(plan_.N) * plan_.N, "image");
  // vector-recurrence grids and the out-of-window rho blocks of k_colsW (few blocks,
  // several elements per thread: the grid reduction's ticket/atomic cost scales with
  // the block count); overridable for tuning
  auto env_int = [](const char* k, int dflt) {
    const char* e = std::getenv(k);
    return e ? std::max(1, std::atoi(e)) : dflt;
  };
  // k_cr_fused handles four entries per thread per round
  vec_grid_ = std::min(std::max(1, (D_ + 4 * kThreads - 1) / (4 * kThreads)), env_int("RTN_VEC_BLOCKS", 2 * 148));
  // the CR applications touch only the window part of rho (L^2 entries): about 512
  // entries per block keeps the grid reduction's ticket short (measured best at C3)
  const int L2w = dims_.L * dims_.L;
  nbr_ = std::min(static_cast<int>((G2 + ops_->NT - 1) / ops_->NT),
                  env_int("RTN_RHO_BLOCKS", std::clamp(L2w / 512, 16, 148)));
  // (8 x 148: the largest k_rho_sum grid RTN_RHO_SUM_BLOCKS may ask for)
  const int max_grid = std::max({vec_grid_, plan_.J * ((plan_.G + ops_->LPB - 1) / ops_->LPB) + nbr_ + 8, 8 * 148});
  // grid_reduce<K> writes K doubles per block; K <= kMaxReduce
  check_cuda(cudaMalloc(&partials_, sizeof(double) * kMaxReduce * max_grid), "partials");
  if (ops_->colsT_box_rows > 0) encode_psf_map(&tmP_, P_, plan_.G, ops_->LPB, ops_->colsT_box_rows);
  check_cuda(cudaMalloc(&dpart_w_, sizeof(double) * 7 * max_grid), "deferred partials");
  dpart_c_[0] = dpart_w_ + 3 * max_grid;
  dpart_c_[1] = dpart_w_ + 5 * max_grid;
  if (const char* e = std::getenv("RTN_DEFER_RED")) defer_red_ = e[0] != '0';
  check_cuda(cudaMalloc(&st_, sizeof(DevState)), "state");
  check_cuda(cudaMemset(st_, 0, sizeof(DevState)), "state");
  check_cuda(cudaMallocHost(&st_host_, sizeof(DevState)), "state mirror");
  std::memset(st_host_, 0, sizeof(DevState));
  ensure_cr_capacity(std::max({plan_.cg_max_iter, plan_.cg_iter_budget, 1}));
  // one thread-block cluster per channel for every non-setup application where the
  // geometry is instantiated (G = 16 x 16, Gc = G/4); RTN_CLUSTER=0 keeps five kernels
  {
    const char* e = std::getenv("RTN_CLUSTER");
    use_cluster_ = ops_->apply_cluster && plan_.Gc * 4 == plan_.G && !(e && e[0] == '0');
  }
  if (use_cluster_) {  // supported: latency mode by default
    c2(&RC_, J * L * L, "cluster channel terms");
    check_cuda(cudaMalloc(&kpart_, sizeof(double) * 3 * plan_.J * ops_->cluster_ctas), "cluster partials");
    // 32 window entries (x J channel terms) per block
    rho_grid_ = std::max(1, std::min(static_cast<int>((L * L + kRhoTile - 1) / kRhoTile), 4 * 148));
    if (const char* e = std::getenv("RTN_RHO_SUM_BLOCKS")) rho_grid_ = std::clamp(std::atoi(e), 1, 8 * 148);
  }
  // alpha schedule and budget split are data independent (nlinv.cpp:295-313)
  float alpha = plan_.alpha0;
  int remaining = plan_.cg_iter_budget;
  for (int m = 0; m < plan_.newton_steps; ++m) {
    alphas_.push_back(alpha);
    if (plan_.cg_iter_budget > 0) {
      const int left = plan_.newton_steps - m;
      const int cap = (remaining + left - 1) / left;
      caps_.push_back(cap);
      remaining -= cap;
    }
    alpha = std::max(alpha * plan_.alpha_q, plan_.alpha_min);
  }
}

void Engine::ensure_cr_capacity(int max_iter) {
  if (max_iter + 2 <= cr_cap_) return;
  if (grp_rank_ >= 0) fail(2, "cg capacity of a channel-group member is fixed when the group is built");
  if (cr_buf_) {
    // the cached step / frame graphs captured the CR scalar pointers by value
    check_cuda(cudaStreamSynchronize(s_), "sync");
    for (auto& g : step_graph_) {
      if (g) cudaGraphExecDestroy(g);
      g = nullptr;
    }
    if (frame_graph_) cudaGraphExecDestroy(frame_graph_);
    frame_graph_ = nullptr;
    cudaFree(cr_buf_);
  }
  cr_cap_ = max_iter + 2;
  check_cuda(cudaMalloc(&cr_buf_, sizeof(double) * 10 * cr_cap_), "cr scalars");
  check_cuda(cudaMemset(cr_buf_, 0, sizeof(double) * 10 * cr_cap_), "cr scalars");
  cr_.rar = cr_buf_;
  cr_.ap2 = cr_buf_ + cr_cap_;
  cr_.rn = cr_buf_ + 2 * cr_cap_;
  cr_.saa = cr_buf_ + 3 * cr_cap_;
  cr_.spa = cr_buf_ + 4 * cr_cap_;
  cr_.pcw = cr_buf_ + 5 * cr_cap_;
  cr_.pcr = cr_buf_ + 8 * cr_cap_;
}

void Engine::sync() { check_cuda(cudaStreamSynchronize(s_), "stream sync"); }

int Engine::line_batch() const { return ops_->LPBR; }

void Engine::set_cluster(bool on) {
  on = on && cluster_supported();
  if (on == use_cluster_) return;
  // captured graphs embed the kernel choice
  sync();
  for (auto& g : step_graph_) {
    if (g) cudaGraphExecDestroy(g);
    g = nullptr;
  }
  if (frame_graph_) cudaGraphExecDestroy(frame_graph_);
  frame_graph_ = nullptr;
  use_cluster_ = on;
}

void Engine::read_state() {
  check_cuda(cudaMemcpyAsync(st_host_, st_, sizeof(DevState), cudaMemcpyDeviceToHost, s_), "state read");
  sync();
}

void Engine::raise_status(const char* where) {
  if (st_host_->status == ST_SOLVER) fail(4, std::string(where) + ": iteration diverged or produced non-finite values");
  if (st_host_->status == ST_DEADLINE) fail_decomp(std::string(where) + ": a group member missed the barrier deadline");
  if (st_host_->status != ST_OK) fail(st_host_->status, std::string(where) + ": device error");
}

void Engine::set_psf(const float* P) {
  check_cuda(cudaMemcpyAsync(P_, P, sizeof(float2) * plan_.G * plan_.G, cudaMemcpyHostToDevice, s_), "psf upload");
  sync();
}
void Engine::set_data(const float* z) {
  check_cuda(cudaMemcpyAsync(z_, z, sizeof(float2) * plan_.J * plan_.G * plan_.G, cudaMemcpyHostToDevice, s_),
             "data upload");
  enq_z_scan();
  sync();
}
void Engine::set_psf_device(const float2* P) {
  check_cuda(cudaMemcpyAsync(P_, P, sizeof(float2) * plan_.G * plan_.G, cudaMemcpyDeviceToDevice, s_), "psf copy");
}
void Engine::set_weights(const float* w) {
  std::memcpy(winv_host_.data(), w, sizeof(float) * winv_host_.size());
  check_cuda(cudaMemcpyAsync(winv_, winv_host_.data(), sizeof(float) * winv_host_.size(), cudaMemcpyHostToDevice, s_),
             "weights upload");
  sync();
}
void Engine::set_step_cache(const float* rho, const float* coils) {
  const size_t G2 = static_cast<size_t>(plan_.G) * plan_.G;
  check_cuda(cudaMemcpyAsync(rhom_, rho, sizeof(float2) * G2, cudaMemcpyHostToDevice, s_), "rho upload");
  check_cuda(cudaMemcpyAsync(coils_, coils, sizeof(float2) * G2 * plan_.J, cudaMemcpyHostToDevice, s_),
             "coils upload");
  sync();
  have_cache_ = true;
}
void Engine::set_data_device(const float2* z) {
  check_cuda(cudaMemcpyAsync(z_, z, sizeof(float2) * plan_.J * plan_.G * plan_.G, cudaMemcpyDeviceToDevice, s_),
             "data copy");
  enq_z_scan();
}

// ---- enqueue helpers ---------------------------------------------------------

void Engine::enq_step_begin(int m) {
  launch_k(k_step_begin, 1, 32, 0, s_, st_, m);
}

void Engine::enq_decode(const float2* est, bool full, bool setup) {
  const int J = plan_.J, G = plan_.G, LPB = ops_->LPB, LPBR = ops_->LPBR;
  const int tGc = (plan_.Gc + LPB - 1) / LPB, tGr = (G + LPBR - 1) / LPBR;
  // nr = -1 / R1_DECODE_WIN: all G rows and columns when st->z_out, else the window only
  // (every in-frame consumer of the coils reads them on the window unless the data has
  // samples outside it: k_colsW's / k_rho_out's setup data term)
  ops_->colA(s_, J * tGc, dims_, winv_, twG_, est + static_cast<size_t>(G) * G, U_, 0, full ? G : -1, st_, 0);
  ops_->rows1(s_, J * tGr, dims_, full ? R1_DECODE : setup ? R1_DECODE_SETUP : R1_DECODE_WIN, twG_, U_, nullptr,
              nullptr, nullptr, V_, coils_, est, rhom_,
              st_, 0);
}

// the cluster-fused application's two halves: one 8-CTA cluster per channel (W^-1 ..
// W^-H, the coil part of out and its dots, the channel terms rc_j), then the channel sum
// of out.rho with the CR "+alpha p" and the dots (a channel group puts its all-member
// barrier between them: k_rho_sum reads every member's rc_j)
ColsWArgs Engine::cluster_args(const float2* dx, float2* out, int cw_mode, float alpha, int dot_slot,
                               const float2* ap_prev) const {
  ColsWArgs a{};
  a.mode = cw_mode;
  a.alpha = alpha;
  a.dot_slot = dot_slot;
  a.dx = dx;
  a.out = out;
  a.ap_prev = ap_prev;
  a.win_only_ok = win_only_ok_;
  a.defer_out = defer_w_;
  return a;
}

void Engine::enq_cluster_front(const float2* dx, float2* out, int cw_mode, float alpha, int dot_slot, int use_halt,
                               const float2* ap_prev) {
  const ColsWArgs a = cluster_args(dx, out, cw_mode, alpha, dot_slot, ap_prev);
  ops_->apply_cluster(s_, plan_.J, dims_, a, winv_, twG_, coils_, rhom_, P_, RC_, kpart_, st_, use_halt);
}

void Engine::enq_rho_sum(const float2* dx, float2* out, int cw_mode, float alpha, int dot_slot, int use_halt,
                         const float2* ap_prev) {
  const ColsWArgs a = cluster_args(dx, out, cw_mode, alpha, dot_slot, ap_prev);
  launch_k(k_rho_sum, rho_grid_, kThreads, 0, s_, dims_, a, static_cast<const float2*>(RC_),
           static_cast<const double*>(kpart_), plan_.J * ops_->cluster_ctas, partials_, st_, cr_, use_halt, gv_);
}

void Engine::enq_apply(const float2* dx, float2* out, int cw_mode, float alpha, int dot_slot, int use_halt,
                       const float2* ap_prev) {
  if (use_cluster_ && cw_mode != CW_SETUP) {
    enq_cluster_front(dx, out, cw_mode, alpha, dot_slot, use_halt, ap_prev);
    enq_rho_sum(dx, out, cw_mode, alpha, dot_slot, use_halt, ap_prev);
    return;
  }
  enq_apply_front(dx, use_halt);
  enq_apply_back(dx, out, cw_mode, alpha, dot_slot, use_halt, ap_prev);
}

namespace {
// RTN_DOUBLE=<pass> (diagnostic): the operator applications launch that pass twice, so the
// frame-time difference is the pass's marginal cost in the running mix (rows1, rows2 and
// colsW are idempotent; colsT applies P twice, which stays finite)
int pass_reps(const char* name) {
  static const char* e = std::getenv("RTN_DOUBLE");
  return (e && std::strcmp(e, name) == 0) ? 2 : 1;
}
// RTN_DOUBLE=nop: one empty kernel more per application (the fixed cost of a launch in the chain)
__global__ void k_nop(const DevState* st) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  (void)st;
}
}  // namespace

void Engine::enq_apply_front(const float2* dx, int use_halt, bool skip_colA) {
  const int J = plan_.J, G = plan_.G, LPB = ops_->LPB;
  const int tGc = (plan_.Gc + LPB - 1) / LPB, tG = (G + LPB - 1) / LPB, tL = (dims_.L + ops_->LPBR - 1) / ops_->LPBR;
  if (!skip_colA) {
    ops_->colA(s_, J * tGc, dims_, winv_, twG_, dx + static_cast<size_t>(G) * G, U_, dims_.lo, dims_.L, st_,
               use_halt);
  }
  if (pass_reps("nop") == 2) launch_k(k_nop, 1, 32, 0, s_, static_cast<const DevState*>(st_));
  for (int k = pass_reps("rows1"); k > 0; --k)
    ops_->rows1(s_, J * tL, dims_, R1_OP, twG_, U_, coils_, rhom_, dx, V_, nullptr, nullptr, nullptr, st_, use_halt);
  for (int k = pass_reps("colsT"); k > 0; --k) ops_->colsT(s_, J * tG, dims_, twG_, P_, V_, st_, use_halt, &tmP_);
  for (int k = pass_reps("rows2"); k > 0; --k)
    ops_->rows2(s_, dims_.L * dims_.H, dims_, 0, twG_, V_, coils_, rhom_, z_, Y_, RP_, partials_, st_, use_halt);
}

void Engine::enq_apply_back(const float2* dx, float2* out, int cw_mode, float alpha, int dot_slot, int use_halt,
                            const float2* ap_prev) {
  const int J = plan_.J, LPB = ops_->LPB;
  const int tGc = (plan_.Gc + LPB - 1) / LPB;
  ColsWArgs a{};
  a.mode = cw_mode;
  a.alpha = alpha;
  a.dot_slot = dot_slot;
  a.dx = dx;
  a.out = out;
  a.ap_prev = ap_prev;
  a.win_only_ok = win_only_ok_;
  a.defer_out = defer_w_;
  const int nbw = J * tGc;
  for (int k = pass_reps("colsW"); k > 0; --k)
    ops_->colsW(s_, nbw + nbr_, dims_, a, winv_, twG_, Y_, RP_, coils_, z_, nbw, partials_, st_, cr_, use_halt, gv_);
}

void Engine::enq_setup(const float2* x, const float2* reg, float alpha) {
  enq_setup_front(x);
  enq_setup_back(x, reg, alpha);
}

void Engine::enq_setup_front(const float2* x) {
  const int J = plan_.J, G = plan_.G, LPB = ops_->LPB;
  const int tG = (G + LPB - 1) / LPB;
  // the step's decode and the setup's first row pass in one launch (R1_DECODE_SETUP)
  enq_decode(x, false, true);
  ops_->colsT(s_, J * tG, dims_, twG_, P_, V_, st_, 0, &tmP_);
  ops_->rows2(s_, dims_.L * dims_.H, dims_, 1, twG_, V_, coils_, rhom_, z_, Y_, RP_, partials_, st_, 0);
  if (dims_.grp) launch_k(k_rho_out, nbr_, kThreads, 0, s_, dims_, coils_, z_, RPO_, partials_, st_);
}

void Engine::enq_setup_back(const float2* x, const float2* reg, float alpha) {
  const int J = plan_.J, LPB = ops_->LPB;
  const int tGc = (plan_.Gc + LPB - 1) / LPB;
  ColsWArgs a{};
  a.mode = CW_SETUP;
  a.a_x = static_cast<float>(-static_cast<double>(alpha));
  a.a_reg = static_cast<float>(static_cast<double>(alpha) * plan_.prev_damping);
  a.dot_slot = -1;
  a.x = x;
  a.reg = reg;
  a.out = r_;
  a.out2 = p_;
  a.out3 = xcg_;
  const int nbw = J * tGc;
  ops_->colsW(s_, nbw + nbr_, dims_, a, winv_, twG_, Y_, RP_, coils_, z_, nbw, partials_, st_, cr_, 0, gv_);
}

void Engine::enq_cr(float alpha, float tol, int cap, bool sync_each) {
  ensure_cr_capacity(cap);
  if (!sync_each && fused_cr_) {
    // budget-mode graphs: one fused recurrence kernel per iteration (k_cr_fused)
    // on the pass path the recurrence also runs the next application's W^-1 column pass
    const bool crA = fused_crA() && !use_cluster_;
    // one device: the application's back half (k_colsW, or k_rho_sum on the cluster path)
    // and every recurrence but the step's last leave their reductions to the next
    // recurrence (DeferRed)
    const bool defer = defer_red_ && !dims_.grp;
    const int nbw = back_grid();
    int prev_grid = 0;  // block count of the previous recurrence with deferred partials
    auto red = [&](int it, bool last) {
      DeferRed dr{};
      if (!defer) return dr;
      dr.w = dpart_w_;
      dr.nw = nbw;
      if (it > 0) {
        dr.c = dpart_c_[(it - 1) & 1];
        dr.nc = prev_grid;
      }
      dr.out = last ? nullptr : dpart_c_[it & 1];
      return dr;
    };
    // the enqueue-time modes are restored even if an enqueue throws (the op-level calls
    // that follow must see plain grid reductions)
    struct Restore {
      Engine& e;
      ~Restore() {
        e.defer_w_ = nullptr;
        e.win_only_ok_ = 0;
      }
    } restore{*this};
    win_only_ok_ = 1;
    defer_w_ = defer ? dpart_w_ : nullptr;
    enq_apply(r_, ar_, CW_OPALPHA, alpha, 0, 1, nullptr);
    for (int it = 0; it < cap; ++it) {
      const bool last = it + 1 == cap;
      if (!crA || last) {
        enq_cr_fused(it, tol, red(it, last));
        prev_grid = vec_grid_;
        if (!last) enq_apply(r_, ar_, CW_OPALPHA, alpha, it + 1, 1, ap_);
      } else {
        enq_crA(it, tol, red(it, false));
        prev_grid = crA_grid();
        enq_apply_front(r_, 1, true);
        enq_apply_back(r_, ar_, CW_OPALPHA, alpha, it + 1, 1, ap_);
      }
    }
    return;
  }
  enq_apply(r_, ar_, CW_OPALPHA, alpha, 0, 1);
  launch_k(k_cr_prime, vec_grid_, kThreads, 0, s_, D_, ap_, ar_, partials_, st_, cr_, 0, 0);
  for (int it = 1; it <= cap; ++it) {
    launch_k(k_cr_xr, vec_grid_, kThreads, 0, s_, D_, xcg_, r_, p_, ap_, partials_, st_, cr_, it, tol, 0, 0);
    if (it == cap) break;
    if (sync_each) {
      read_state();
      if (st_host_->status || st_host_->cr_halt) break;
    }
    enq_apply(r_, ar_, CW_OPALPHA, alpha, it, 1);
    launch_k(k_cr_pap, vec_grid_, kThreads, 0, s_, D_, p_, ap_, r_, ar_, partials_, st_, cr_, it, 0, 0);
  }
}

void Engine::enq_newton_step(int m, float2* x, const float2* reg, float alpha, float tol, int cap,
                             bool sync_each) {
  enq_step_begin(m);
  enq_setup(x, reg, alpha);
  if (cap >= 1) {
    if (sync_each) {
      read_state();
      raise_status("cg_solve");
    }
    if (!sync_each || !st_host_->cr_halt) enq_cr(alpha, tol, cap, sync_each);
  }
  launch_k(k_axpy1, vec_grid_, kThreads, 0, s_, D_, x, xcg_, st_);
}

void Engine::enq_image(const float2* est, float2* img, float scale, bool apply_scale) {
  enq_decode(est);
  launch_k(k_image, blocks_for(static_cast<long long>(plan_.N) * plan_.N, 148 * 4), kThreads, 0, s_, dims_,
           est, coils_, scale, apply_scale ? 1 : 0, img, st_);
}

void Engine::enq_cr_fused(int it, float tol, const DeferRed& dr) {
  const int rho_skip = (dims_.grp && !dims_.count_rho) ? plan_.G * plan_.G : 0;
  if (dims_.grp || dr.grp)
    launch_k(k_cr_fused<true>, vec_grid_, kThreads, 0, s_, D_, xcg_, r_, p_, ap_, static_cast<const float2*>(ar_),
             partials_, st_, cr_, it, tol, rho_skip, dims_.grp, plan_.G, dr);
  else
    launch_k(k_cr_fused<false>, vec_grid_, kThreads, 0, s_, D_, xcg_, r_, p_, ap_, static_cast<const float2*>(ar_),
             partials_, st_, cr_, it, tol, rho_skip, 0, plan_.G, dr);
}

bool Engine::fused_crA() const { return fused_crA_ && fused_cr_ && ops_->crA != nullptr && !dims_.grp; }

int Engine::back_grid() const {
  return use_cluster_ ? rho_grid_ : plan_.J * ((plan_.Gc + ops_->LPB - 1) / ops_->LPB) + nbr_;
}

int Engine::crA_grid() const {
  const int nbc = plan_.J * ((plan_.Gc + ops_->LPB - 1) / ops_->LPB);
  // rho part: the window's L^2 entries at four per thread (all G^2 when it is not window-only)
  const int nbr = std::max(1, std::min(vec_grid_, (dims_.L * dims_.L + 4 * kThreads - 1) / (4 * kThreads)));
  return nbc + nbr;
}

void Engine::enq_crA(int it, float tol, const DeferRed& dr) {
  const int nbc = plan_.J * ((plan_.Gc + ops_->LPB - 1) / ops_->LPB);
  ops_->crA(s_, crA_grid(), nbc, dims_, xcg_, r_, p_, ap_, ar_, winv_, twG_, U_, partials_, st_, cr_, it, tol, dr);
}

void Engine::join_group(int rank, const GroupView& gv, const GroupScal& gs) {
  check_cuda(cudaSetDevice(dev_), "set device");
  grp_rank_ = rank;
  dims_.grp = 1;
  dims_.count_rho = rank == 0 ? 1 : 0;
  gv_ = gv;
  gs_ = gs;
}

void Engine::enq_grp_fin(int setup, int op_slot, int cr_slot, float tol, int part) {
  launch_k(k_grp_fin, 1, 32, 0, s_, gs_, st_, cr_, setup, op_slot, cr_slot, tol, part);
}

// a channel-group member's exact two-pass CR kernels (tolerance mode): member partials of
// |ap|^2 and |r|^2, the replicated rho counted on member 0 (k_grp_fin forms the totals)
void Engine::enq_cr_two_pass_grp(int kind, int it, float tol) {
  const int rho_skip = dims_.count_rho ? 0 : plan_.G * plan_.G;
  if (kind == 0) {
    launch_k(k_cr_prime, vec_grid_, kThreads, 0, s_, D_, ap_, ar_, partials_, st_, cr_, 1, rho_skip);
  } else if (kind == 1) {
    launch_k(k_cr_pap, vec_grid_, kThreads, 0, s_, D_, p_, ap_, r_, ar_, partials_, st_, cr_, it, 1, rho_skip);
  } else {
    launch_k(k_cr_xr, vec_grid_, kThreads, 0, s_, D_, xcg_, r_, p_, ap_, partials_, st_, cr_, it, tol, 1, rho_skip);
  }
}

void Engine::enq_axpy1() { launch_k(k_axpy1, vec_grid_, kThreads, 0, s_, D_, x_, static_cast<const float2*>(xcg_), static_cast<const DevState*>(st_)); }

void Engine::enq_z_scan(bool masked) {
  check_cuda(cudaMemsetAsync(&st_->z_out, 0, sizeof(int), s_), "z scan reset");
  if (masked) return;
  launch_k(k_z_outside, blocks_for(static_cast<long long>(plan_.J) * plan_.G * plan_.G, 148 * 4), kThreads, 0, s_,
           dims_, static_cast<const float2*>(z_), st_);
}

void Engine::enq_pg_barrier(int* own_flags, const GroupFlags& f) {
  launch_k(k_pg_barrier, 1, 32, 0, s_, own_flags, f, st_);
}

void Engine::enq_state_reset() { check_cuda(cudaMemsetAsync(st_, 0, sizeof(int) * 4, s_), "state reset"); }

void Engine::enq_coil_ss() {
  launch_k(k_coil_ss, blocks_for(static_cast<long long>(plan_.N) * plan_.N, 148 * 4), kThreads, 0, s_, dims_,
           static_cast<const float2*>(coils_), SS_, static_cast<const DevState*>(st_));
}

void Engine::enq_image_grp(float2* img, float scale, bool apply_scale) {
  launch_k(k_image_grp, blocks_for(static_cast<long long>(plan_.N) * plan_.N, 148 * 4), kThreads, 0, s_, dims_,
           static_cast<const float2*>(x_), gs_, scale, apply_scale ? 1 : 0, img, static_cast<const DevState*>(st_));
}

// ---- FrameWorker: full-layout device buffers in, stream ordered -----------------

void Engine::load_frame(const float2* z, const float2* P, bool masked) {
  check_cuda(cudaMemcpyAsync(z_, z, sizeof(float2) * plan_.J * plan_.G * plan_.G, cudaMemcpyDefault, s_), "z");
  check_cuda(cudaMemcpyAsync(P_, P, sizeof(float2) * plan_.G * plan_.G, cudaMemcpyDefault, s_), "psf");
  enq_z_scan(masked);
}
void Engine::load_x(const float2* src) {
  check_cuda(cudaMemcpyAsync(x_, src, sizeof(float2) * D_, cudaMemcpyDefault, s_), "x");
}
void Engine::load_reg(const float2* src) {
  check_cuda(cudaMemcpyAsync(reg_, src, sizeof(float2) * D_, cudaMemcpyDefault, s_), "reg");
}
void Engine::store_x(float2* dst) {
  check_cuda(cudaMemcpyAsync(dst, x_, sizeof(float2) * D_, cudaMemcpyDefault, s_), "estimate");
}

// ---- op-level API -------------------------------------------------------------

void Engine::apply_W_inv(const float* chat, float* out) {
  const int G = plan_.G, Gc = plan_.Gc;
  check_cuda(cudaMemcpyAsync(est_scratch_[0], chat, sizeof(float2) * Gc * Gc, cudaMemcpyHostToDevice, s_), "h2d");
  k_pad_weight<<<blocks_for(G * G, 1024), kThreads, 0, s_>>>(est_scratch_[0], winv_, Gc, G, gbuf_);
  fft2_device(gbuf_, G, 1, +1, s_);
  fft_book(fft_current_ctx(), 1);
  check_cuda(cudaMemcpyAsync(out, gbuf_, sizeof(float2) * G * G, cudaMemcpyDeviceToHost, s_), "d2h");
  sync();
}

void Engine::apply_W_invH(const float* u, float* out) {
  const int G = plan_.G, Gc = plan_.Gc;
  check_cuda(cudaMemcpyAsync(gbuf_, u, sizeof(float2) * G * G, cudaMemcpyHostToDevice, s_), "h2d");
  fft2_device(gbuf_, G, 1, -1, s_);
  fft_book(fft_current_ctx(), 1);
  k_crop_weight<<<blocks_for(Gc * Gc, 1024), kThreads, 0, s_>>>(gbuf_, winv_, Gc, G, est_scratch_[0]);
  check_cuda(cudaMemcpyAsync(out, est_scratch_[0], sizeof(float2) * Gc * Gc, cudaMemcpyDeviceToHost, s_), "d2h");
  sync();
}

void Engine::toeplitz_apply(float* x) {
  const int G = plan_.G;
  check_cuda(cudaMemcpyAsync(gbuf_, x, sizeof(float2) * G * G, cudaMemcpyHostToDevice, s_), "h2d");
  k_mask<<<blocks_for(G * G, 1024), kThreads, 0, s_>>>(gbuf_, G);
  fft2_device(gbuf_, G, 1, -1, s_);
  k_mul<<<blocks_for(G * G, 1024), kThreads, 0, s_>>>(gbuf_, P_, G * G);
  fft2_device(gbuf_, G, 1, +1, s_);
  k_mask<<<blocks_for(G * G, 1024), kThreads, 0, s_>>>(gbuf_, G);
  fft_book(fft_current_ctx(), 2);
  check_cuda(cudaMemcpyAsync(x, gbuf_, sizeof(float2) * G * G, cudaMemcpyDeviceToHost, s_), "d2h");
  sync();
}

void Engine::make_step_cache(const float* x, float* rho_out, float* coils_out) {
  check_cuda(cudaMemcpyAsync(est_scratch_[2], x, sizeof(float2) * D_, cudaMemcpyHostToDevice, s_), "h2d");
  check_cuda(cudaMemsetAsync(st_, 0, sizeof(int) * 4, s_), "state reset");
  enq_decode(est_scratch_[2], true);
  fft_book(fft_current_ctx(), static_cast<uint64_t>(plan_.J));
  const size_t G2 = static_cast<size_t>(plan_.G) * plan_.G;
  if (rho_out) check_cuda(cudaMemcpyAsync(rho_out, rhom_, sizeof(float2) * G2, cudaMemcpyDeviceToHost, s_), "d2h");
  if (coils_out) {
    check_cuda(cudaMemcpyAsync(coils_out, coils_, sizeof(float2) * G2 * plan_.J, cudaMemcpyDeviceToHost, s_), "d2h");
  }
  sync();
  have_cache_ = true;
}

void Engine::apply_normal(const float* dx, float* out) {
  if (!have_cache_) fail(2, "apply_normal: no step cache (call make_step_cache first)");
  check_cuda(cudaMemsetAsync(st_, 0, sizeof(int) * 4, s_), "state reset");
  check_cuda(cudaMemcpyAsync(est_scratch_[0], dx, sizeof(float2) * D_, cudaMemcpyHostToDevice, s_), "h2d");
  enq_apply(est_scratch_[0], est_scratch_[1], CW_OP, 0.f, -1, 0);
  fft_book(fft_current_ctx(), 4ull * plan_.J);
  check_cuda(cudaMemcpyAsync(out, est_scratch_[1], sizeof(float2) * D_, cudaMemcpyDeviceToHost, s_), "d2h");
  read_state();
  raise_status("apply_normal");
}

void Engine::cg_solve(const float* rhs, float alpha, float tol, int max_iter, float* x_out, int* iters,
                      std::vector<double>* residuals) {
  if (!have_cache_) fail(2, "cg_solve: no step cache (call make_step_cache first)");
  // host-side entry checks mirror nlinv.cpp:182-186 exactly
  double nsq = 0;
  for (int i = 0; i < 2 * D_; ++i) nsq += static_cast<double>(rhs[i]) * rhs[i];
  const double rhs_norm = std::sqrt(nsq);
  if (!std::isfinite(rhs_norm)) fail(4, "cg_solve: right-hand side is not finite");
  *iters = 0;
  if (residuals) residuals->clear();
  if (max_iter < 1 || rhs_norm == 0.0) {
    std::memset(x_out, 0, sizeof(float2) * D_);
    return;
  }
  ensure_cr_capacity(max_iter);
  check_cuda(cudaMemsetAsync(st_, 0, sizeof(int) * 4, s_), "state reset");
  check_cuda(cudaMemcpyAsync(r_, rhs, sizeof(float2) * D_, cudaMemcpyHostToDevice, s_), "h2d");
  check_cuda(cudaMemcpyAsync(p_, r_, sizeof(float2) * D_, cudaMemcpyDeviceToDevice, s_), "d2d");
  check_cuda(cudaMemsetAsync(xcg_, 0, sizeof(float2) * D_, s_), "zero");
  enq_step_begin(0);
  // the step record's rhs norm feeds the tolerance target
  {
    StepRec rec{};
    rec.rhs_nrm2 = nsq;
    check_cuda(cudaMemcpyAsync(reinterpret_cast<char*>(st_) + offsetof(DevState, steps), &rec, sizeof(rec),
                               cudaMemcpyHostToDevice, s_),
               "step record");
    sync();
  }
  const int ctx = fft_current_ctx();
  // the op-level solve keeps the reference's two-pass recurrence exactly
  const bool fused = fused_cr_;
  fused_cr_ = false;
  enq_cr(alpha, tol, max_iter, tol > 0.0f);
  fused_cr_ = fused;
  read_state();
  raise_status("cg_solve");
  const int n = st_host_->steps[0].iters;
  fft_book(ctx, 4ull * plan_.J * static_cast<uint64_t>(n));
  *iters = n;
  if (residuals) {
    std::vector<double> rn(static_cast<size_t>(cr_cap_));
    check_cuda(cudaMemcpy(rn.data(), cr_.rn, sizeof(double) * cr_cap_, cudaMemcpyDeviceToHost), "residuals");
    residuals->assign(rn.begin() + 1, rn.begin() + 1 + n);
  }
  check_cuda(cudaMemcpyAsync(x_out, xcg_, sizeof(float2) * D_, cudaMemcpyDeviceToHost, s_), "d2h");
  sync();
}

void Engine::newton_step(float* x, const float* reg, float alpha, float tol, int cap, int* iters,
                         double* residual0) {
  check_cuda(cudaMemcpyAsync(x_, x, sizeof(float2) * D_, cudaMemcpyHostToDevice, s_), "h2d");
  check_cuda(cudaMemcpyAsync(est_scratch_[1], reg, sizeof(float2) * D_, cudaMemcpyHostToDevice, s_), "h2d");
  check_cuda(cudaMemsetAsync(st_, 0, sizeof(int) * 4, s_), "state reset");
  const int ctx_n = CTX_NORMAL_OP;
  fft_book(CTX_SETUP, 4ull * plan_.J);
  enq_newton_step(0, x_, est_scratch_[1], alpha, tol, cap, true);
  read_state();
  raise_status("newton_step");
  const StepRec& s = st_host_->steps[0];
  *iters = s.iters;
  *residual0 = std::sqrt(s.resid_win + s.resid_out);
  fft_book(ctx_n, 4ull * plan_.J * static_cast<uint64_t>(s.iters));
  check_cuda(cudaMemcpyAsync(x, x_, sizeof(float2) * D_, cudaMemcpyDeviceToHost, s_), "d2h");
  sync();
  have_cache_ = true;
}

// ---- frame pipeline -------------------------------------------------------------

void Engine::book_frame_ffts(const std::vector<int>& iters) {
  // per frame: 4J per step (setup), 4J per CR iteration (normal_op), J final decode
  uint64_t n = 0;
  for (int c : iters) n += static_cast<uint64_t>(c);
  fft_book(CTX_SETUP, 4ull * plan_.J * iters.size() + plan_.J);
  fft_book(CTX_NORMAL_OP, 4ull * plan_.J * n);
}

void Engine::frame_begin() { check_cuda(cudaMemsetAsync(st_, 0, sizeof(int) * 4, s_), "state reset"); }

void Engine::frame_step(int m, const float2* reg_src) {
  if (reg_src && reg_src != reg_) {
    check_cuda(cudaMemcpyAsync(reg_, reg_src, sizeof(float2) * D_, cudaMemcpyDeviceToDevice, s_), "reg copy");
  }
  if (!budget_mode()) {
    // tolerance mode: data-dependent iteration counts, synchronous CR
    enq_newton_step(m, x_, reg_, alphas_[static_cast<size_t>(m)], plan_.cg_tol, plan_.cg_max_iter, true);
    return;
  }
  const int cap = caps_[static_cast<size_t>(m)];
  if (!use_graphs_) {
    enq_newton_step(m, x_, reg_, alphas_[static_cast<size_t>(m)], 0.0f, cap, false);
    return;
  }
  if (!step_graph_[m]) {
    cudaGraph_t g = nullptr;
    check_cuda(cudaStreamBeginCapture(s_, cudaStreamCaptureModeThreadLocal), "capture begin");
    enq_newton_step(m, x_, reg_, alphas_[static_cast<size_t>(m)], 0.0f, cap, false);
    check_cuda(cudaStreamEndCapture(s_, &g), "capture end");
    check_cuda(cudaGraphInstantiate(&step_graph_[m], g, 0), "graph instantiate");
    cudaGraphDestroy(g);
  }
  check_cuda(cudaGraphLaunch(step_graph_[m], s_), "graph launch");
}

void Engine::frame_image(float2* img_dst, float image_scale, bool apply_scale) {
  enq_image(x_, img_dst ? img_dst : img_, image_scale, apply_scale);
  check_cuda(cudaMemcpyAsync(st_host_, st_, sizeof(DevState), cudaMemcpyDeviceToHost, s_), "state read");
}

void Engine::frame_all(float2* img_dst, float image_scale, bool apply_scale) {
  if (!budget_mode()) fail(2, "frame_all: whole-frame graphs need the CG iteration budget mode");
  // the graph always writes the engine's own image buffer (a per-frame destination
  // would force a re-capture per frame); a D2D copy delivers it
  float2* img = img_;
  if (!use_graphs_) {
    frame_begin();
    for (int m = 0; m < plan_.newton_steps; ++m) frame_step(m, nullptr);
    frame_image(img_dst ? img_dst : img_, image_scale, apply_scale);
    return;
  }
  if (frame_graph_ && (frame_graph_img_ != img || frame_graph_scale_ != image_scale ||
                       frame_graph_apply_ != apply_scale)) {
    cudaGraphExecDestroy(frame_graph_);
    frame_graph_ = nullptr;
  }
  if (!frame_graph_) {
    cudaGraph_t g = nullptr;
    check_cuda(cudaStreamBeginCapture(s_, cudaStreamCaptureModeThreadLocal), "capture begin");
    frame_begin();
    for (int m = 0; m < plan_.newton_steps; ++m) {
      enq_newton_step(m, x_, reg_, alphas_[static_cast<size_t>(m)], 0.0f, caps_[static_cast<size_t>(m)], false);
    }
    enq_image(x_, img, image_scale, apply_scale);
    check_cuda(cudaMemcpyAsync(st_host_, st_, sizeof(DevState), cudaMemcpyDeviceToHost, s_), "state read");
    check_cuda(cudaStreamEndCapture(s_, &g), "capture end");
    check_cuda(cudaGraphInstantiate(&frame_graph_, g, 0), "graph instantiate");
    cudaGraphDestroy(g);
    frame_graph_img_ = img;
    frame_graph_scale_ = image_scale;
    frame_graph_apply_ = apply_scale;
  }
  check_cuda(cudaGraphLaunch(frame_graph_, s_), "graph launch");
  if (img_dst && img_dst != img_) {
    check_cuda(cudaMemcpyAsync(img_dst, img_, sizeof(float2) * plan_.N * plan_.N, cudaMemcpyDefault, s_), "image");
  }
}

bool Engine::frame_verify(FrameStats* stats) {
  sync();
  raise_status("reconstruct_frame");
  const int M = plan_.newton_steps;
  std::vector<int> got(static_cast<size_t>(M));
  bool ok = true;
  for (int m = 0; m < M; ++m) {
    got[static_cast<size_t>(m)] = st_host_->steps[m].iters;
    if (budget_mode() && (st_host_->steps[m].iters != caps_[static_cast<size_t>(m)] || st_host_->steps[m].zero_rhs)) {
      ok = false;
    }
  }
  if (ok) {
    book_frame_ffts(got);
    if (stats) {
      stats->cg_per_step = got;
      stats->cg_iters = 0;
      for (int c : got) stats->cg_iters += c;
    }
  }
  return ok;
}

void Engine::frame_run_sync(const RegFn& reg, float2* img_dst, float image_scale, bool apply_scale,
                            FrameStats* stats) {
  const int M = plan_.newton_steps;
  frame_begin();
  int remaining = plan_.cg_iter_budget;
  std::vector<int> per;
  for (int m = 0; m < M; ++m) {
    int cap = plan_.cg_max_iter;
    float tol = plan_.cg_tol;
    if (budget_mode()) {
      const int left = M - m;
      cap = (remaining + left - 1) / left;
      tol = 0.0f;
    }
    const float2* src = reg ? reg(m) : nullptr;
    if (src && src != reg_) {
      check_cuda(cudaMemcpyAsync(reg_, src, sizeof(float2) * D_, cudaMemcpyDeviceToDevice, s_), "reg copy");
    }
    enq_newton_step(m, x_, reg_, alphas_[static_cast<size_t>(m)], tol, cap, true);
    read_state();
    raise_status("reconstruct_frame");
    const int it = st_host_->steps[m].iters;
    per.push_back(it);
    if (budget_mode()) remaining -= it;
  }
  enq_image(x_, img_dst ? img_dst : img_, image_scale, apply_scale);
  read_state();
  raise_status("reconstruct_frame");
  book_frame_ffts(per);
  if (stats) {
    stats->cg_per_step = per;
    stats->cg_iters = 0;
    for (int c : per) stats->cg_iters += c;
  }
}

void Engine::reconstruct_frame(const float* init, const float* reg, float* image, float* est_out,
                               FrameStats* stats) {
  const auto t0 = std::chrono::steady_clock::now();
  check_cuda(cudaMemcpyAsync(x_, init, sizeof(float2) * D_, cudaMemcpyHostToDevice, s_), "h2d");
  check_cuda(cudaMemcpyAsync(reg_, reg ? reg : init, sizeof(float2) * D_, cudaMemcpyHostToDevice, s_), "h2d");
  bool ok = false;
  if (budget_mode()) {
    frame_all(img_, 1.0f, false);
    ok = frame_verify(stats);
  }
  if (!ok) {
    check_cuda(cudaMemcpyAsync(x_, init, sizeof(float2) * D_, cudaMemcpyHostToDevice, s_), "h2d");
    frame_run_sync(nullptr, img_, 1.0f, false, stats);
  }
  check_cuda(cudaMemcpyAsync(image, img_, sizeof(float2) * plan_.N * plan_.N, cudaMemcpyDeviceToHost, s_), "d2h");
  if (est_out) check_cuda(cudaMemcpyAsync(est_out, x_, sizeof(float2) * D_, cudaMemcpyDeviceToHost, s_), "d2h");
  sync();
  have_cache_ = true;
  if (stats) stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void Engine::reconstruct_frame_regs(const float* init, const RegHostFn& reg, float* image, float* est_out,
                                    FrameStats* stats) {
  const auto t0 = std::chrono::steady_clock::now();
  check_cuda(cudaMemcpyAsync(x_, init, sizeof(float2) * D_, cudaMemcpyHostToDevice, s_), "h2d");
  check_cuda(cudaMemcpyAsync(reg_, init, sizeof(float2) * D_, cudaMemcpyHostToDevice, s_), "h2d");
  const RegFn dev = [&](int m) -> const float2* {
    const float* h = reg ? reg(m) : nullptr;
    if (!h) return nullptr;
    check_cuda(cudaMemcpyAsync(reg_, h, sizeof(float2) * D_, cudaMemcpyHostToDevice, s_), "reg h2d");
    sync();  // the provider may reuse its buffer for the next step
    return reg_;
  };
  frame_run_sync(dev, img_, 1.0f, false, stats);
  check_cuda(cudaMemcpyAsync(image, img_, sizeof(float2) * plan_.N * plan_.N, cudaMemcpyDeviceToHost, s_), "d2h");
  if (est_out) check_cuda(cudaMemcpyAsync(est_out, x_, sizeof(float2) * D_, cudaMemcpyDeviceToHost, s_), "d2h");
  sync();
  have_cache_ = true;
  if (stats) stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ---- isolated kernel timing (bench roofline) ------------------------------------------

double Engine::kernel_bytes(const char* which) const {
  // algorithmic bytes: every operand read once, every result written once
  const double c8 = 8.0;
  const double J = plan_.J, G = plan_.G, L = dims_.L, Gc = plan_.Gc;
  const std::string w(which);
  if (w == "colsT") return c8 * (2.0 * J * L * G + G * G);                   // V in + out, P
  if (w == "rows1") return c8 * (J * L * Gc + 2.0 * J * L * L + 2.0 * L * L + J * L * G);  // U, c_j, drho, rho, V
  if (w == "rows2") return c8 * (J * L * G + J * L * L + L * L + J * L * Gc) + 16.0 * dims_.H * L * L;  // V, c_j, rho, Y, RP
  if (w == "colA") return c8 * (J * Gc * Gc + J * L * Gc) + 4.0 * Gc * Gc;
  if (w == "colsW") return c8 * (J * L * Gc + 3.0 * (G * G + J * Gc * Gc)) + 16.0 * dims_.H * L * L + 4.0 * Gc * Gc;
  if (w == "cr_xr" || w == "cr_pap") return c8 * 6.0 * (G * G + J * Gc * Gc);
  if (w == "cr_fused") return c8 * 9.0 * (G * G + J * Gc * Gc);  // x,r,p,ap,ar in; x,r,p,ap out
  // k_crA: the recurrence on the window-only rho and every coil entry, the weights, U's window rows
  if (w == "crA") return c8 * (9.0 * (L * L + J * Gc * Gc) + J * L * Gc) + 4.0 * Gc * Gc;
  if (w == "apply") {
    // one fused normal-operator application (SURVEY.md §8(d) B_op, window pruned)
    return 8.0 * L * L * (J + 3) + 8.0 * G * G + 16.0 * J * Gc * Gc + 4.0 * Gc * Gc;
  }
  return 0.0;
}

double Engine::time_kernel(const char* which, int reps) {
  if (!have_cache_) fail(2, "time_kernel: no step cache");
  // "<kernel>:cold": every launch timed on its own after a write of a buffer larger than
  // L2 (cold-cache operands); otherwise back-to-back launches on L2-resident operands
  std::string w(which);
  const bool cold = w.size() > 5 && w.compare(w.size() - 5, 5, ":cold") == 0;
  if (cold) w.resize(w.size() - 5);
  const int J = plan_.J, G = plan_.G, LPB = ops_->LPB;
  const int tGc = (plan_.Gc + LPB - 1) / LPB, tG = (G + LPB - 1) / LPB, tL = (dims_.L + ops_->LPBR - 1) / ops_->LPBR;
  check_cuda(cudaMemsetAsync(st_, 0, sizeof(int) * 4, s_), "state reset");
  // the recurrences consume deferred partials as in the step (DeferRed): plausible totals
  // (rar = |ar|^2 = |ap|^2 = |r|^2 = 1) so every timed launch runs the full update
  const int nbw = J * tGc + nbr_;
  DeferRed dr{};
  if (defer_red_ && !dims_.grp) {
    std::vector<double> hw(3 * static_cast<size_t>(nbw)), hc(2 * static_cast<size_t>(crA_grid()));
    for (int b = 0; b < nbw; ++b) {
      hw[3 * b] = hw[3 * b + 1] = 1.0 / nbw;
      hw[3 * b + 2] = 0.0;
    }
    for (size_t b = 0; b < hc.size(); ++b) hc[b] = 2.0 / static_cast<double>(hc.size());
    check_cuda(cudaMemcpyAsync(dpart_w_, hw.data(), sizeof(double) * hw.size(), cudaMemcpyHostToDevice, s_), "h2d");
    check_cuda(cudaMemcpyAsync(dpart_c_[0], hc.data(), sizeof(double) * hc.size(), cudaMemcpyHostToDevice, s_), "h2d");
    check_cuda(cudaStreamSynchronize(s_), "sync");
    dr.w = dpart_w_;
    dr.nw = nbw;
    dr.c = dpart_c_[0];
    dr.nc = crA_grid();
  }
  auto launch = [&] {
    if (w == "colsT") {
      ops_->colsT(s_, J * tG, dims_, twG_, P_, V_, st_, 0, &tmP_);
    } else if (w == "rows1") {
      ops_->rows1(s_, J * tL, dims_, R1_OP, twG_, U_, coils_, rhom_, r_, V_, nullptr, nullptr, nullptr, st_, 0);
    } else if (w == "rows2") {
      ops_->rows2(s_, dims_.L * dims_.H, dims_, 0, twG_, V_, coils_, rhom_, z_, Y_, RP_, partials_, st_, 0);
    } else if (w == "colsW") {
      ColsWArgs a{};
      a.mode = CW_OPALPHA;
      a.alpha = 0.5f;
      a.dot_slot = -1;
      a.dx = r_;
      a.out = ar_;
      // as in the CR solve: a scratch output, the partials deferred to the recurrence
      a.defer_out = dr.w ? dpart_w_ : nullptr;
      ops_->colsW(s_, nbw, dims_, a, winv_, twG_, Y_, RP_, coils_, z_, J * tGc, partials_, st_, cr_, 0, gv_);
    } else if (w == "cr_xr") {
      launch_k(k_cr_xr, vec_grid_, kThreads, 0, s_, D_, xcg_, r_, p_, ap_, partials_, st_, cr_, 1, 0.f, 0, 0);
    } else if (w == "cr_fused") {
      // a step's last recurrence: the deferred partials in, its own grid reduction out
      launch_k(k_cr_fused<false>, vec_grid_, kThreads, 0, s_, D_, xcg_, r_, p_, ap_,
               static_cast<const float2*>(ar_), partials_, st_, cr_, 1, 0.f, 0, 0, plan_.G, dr);
    } else if (w == "crA") {
      DeferRed d2 = dr;
      if (d2.w) d2.out = dpart_c_[1];
      ops_->crA(s_, crA_grid(), J * tGc, dims_, xcg_, r_, p_, ap_, ar_, winv_, twG_, U_, partials_, st_, cr_, 1, 0.f,
                d2);
    } else if (w == "cr_pap") {
      launch_k(k_cr_pap, vec_grid_, kThreads, 0, s_, D_, p_, ap_, r_, ar_, partials_, st_, cr_, 1, 0, 0);
    } else if (w == "colA") {
      ops_->colA(s_, J * tGc, dims_, winv_, twG_, r_ + static_cast<size_t>(G) * G, U_, dims_.lo, dims_.L, st_, 0);
    } else if (w == "apply") {
      enq_apply(r_, ar_, CW_OP, 0.f, -1, 0);
    } else {
      fail(2, "time_kernel: unknown kernel " + w);
    }
  };
  if (w.rfind("cr", 0) == 0) {
    // scalars of a stationary iteration (iteration 1: b = rar[1]/rar[0] = 0, step
    // a = rar[1]/|ap|^2 = 0 with |ap|^2 = saa[1] = 1 > 0): every launch runs the full
    // vector pass (loads, update, stores, norms) and the values stay finite however
    // many times it repeats, so no launch exits early on a solver fault
    const double rar[2] = {1.0, 0.0}, one[2] = {1.0, 1.0};
    check_cuda(cudaMemcpyAsync(cr_.rar, rar, sizeof(rar), cudaMemcpyHostToDevice, s_), "scalars");
    for (double* q : {cr_.ap2, cr_.saa, cr_.spa}) {
      check_cuda(cudaMemcpyAsync(q, one, sizeof(one), cudaMemcpyHostToDevice, s_), "scalars");
    }
  }
  // fresh intermediates (U, V, Y, RP, ar) of one application at the linearisation
  // point: the in-place passes (colsT on V) compound over a previous class's repeats
  enq_apply(r_, ar_, CW_OP, 0.f, -1, 0);
  for (int i = 0; i < 3; ++i) launch();
  cudaEvent_t a, b;
  check_cuda(cudaEventCreate(&a), "event");
  check_cuda(cudaEventCreate(&b), "event");
  float ms = 0;
  if (!cold) {
    check_cuda(cudaEventRecord(a, s_), "event");
    for (int i = 0; i < reps; ++i) launch();
    check_cuda(cudaEventRecord(b, s_), "event");
    check_cuda(cudaEventSynchronize(b), "event sync");
    check_cuda(cudaEventElapsedTime(&ms, a, b), "elapsed");
  } else {
    const size_t flush_bytes = size_t(256) << 20;  // 2x the 126 MB L2
    void* flush = nullptr;
    check_cuda(cudaMalloc(&flush, flush_bytes), "l2 flush buffer");
    for (int i = 0; i < reps; ++i) {
      check_cuda(cudaMemsetAsync(flush, i & 0xff, flush_bytes, s_), "l2 flush");
      check_cuda(cudaEventRecord(a, s_), "event");
      launch();
      check_cuda(cudaEventRecord(b, s_), "event");
      check_cuda(cudaEventSynchronize(b), "event sync");
      float one = 0;
      check_cuda(cudaEventElapsedTime(&one, a, b), "elapsed");
      ms += one;
    }
    cudaFree(flush);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  // a launch that returned early on a device fault would time nothing
  read_state();
  if (st_host_->status || st_host_->cr_halt) {
    fail(4, "time_kernel: " + w + " stopped early (device status " + std::to_string(st_host_->status) +
                ", halt " + std::to_string(st_host_->cr_halt) + ")");
  }
  return ms / reps;
}

}  // namespace rtnb
