// ORACLE TEST INFRASTRUCTURE — not product code. See fftw3.h for scope.
//
// Double-precision 2D DFT behind the FFTW plan/execute interface, fast enough that
// the reference's CPU timings are not dominated by the stand-in: per axis a
// Stockham autosort FFT over the factorisation of the length (radix 4, 2, 3, 5 with
// closed-form butterflies; any other prime by a direct DFT), every twiddle read
// from per-stage tables computed once per plan in double. Rows are transformed in
// place; columns are gathered in blocks of 8 into contiguous scratch. Accuracy is
// pinned by the reference's own KATs (tests/test_fft.cpp) run against this shim.
#include "fftw3.h"

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <numbers>
#include <vector>

using cd = std::complex<double>;

extern "C" const char fftw_version[] = "3.3.10-rtnlinv-oracle-shim";

namespace {

struct Stage {
  int p = 0;               // radix
  int ns = 0;              // product of earlier radices
  std::vector<cd> tw;      // ns * (p - 1): exp(sign 2 pi i r k / (ns p)), r = 1..p-1
  std::vector<cd> rootp;   // p: exp(sign 2 pi i t / p) (generic radix)
};

struct Plan1D {
  int n = 0;
  int sign = -1;
  std::vector<Stage> stages;
};

Plan1D make_1d(int n, int sign) {
  Plan1D pl;
  pl.n = n;
  pl.sign = sign;
  std::vector<int> fac;
  int m = n;
  while (m % 4 == 0) {
    fac.push_back(4);
    m /= 4;
  }
  for (int p = 2; p * p <= m; ++p) {
    while (m % p == 0) {
      fac.push_back(p);
      m /= p;
    }
  }
  if (m > 1) fac.push_back(m);
  int ns = 1;
  for (int p : fac) {
    Stage st;
    st.p = p;
    st.ns = ns;
    st.tw.resize(static_cast<size_t>(ns) * (p - 1));
    for (int k = 0; k < ns; ++k) {
      for (int r = 1; r < p; ++r) {
        const double a = sign * 2.0 * std::numbers::pi * r * k / (static_cast<double>(ns) * p);
        st.tw[static_cast<size_t>(k) * (p - 1) + (r - 1)] = cd(std::cos(a), std::sin(a));
      }
    }
    st.rootp.resize(static_cast<size_t>(p));
    for (int t = 0; t < p; ++t) {
      const double a = sign * 2.0 * std::numbers::pi * t / p;
      st.rootp[static_cast<size_t>(t)] = cd(std::cos(a), std::sin(a));
    }
    pl.stages.push_back(std::move(st));
    ns *= p;
  }
  return pl;
}

// one unnormalised 1D transform; x and y are n-element work buffers, the result is
// left in *out (either x or y). Butterflies use explicit double arithmetic (no
// libgcc complex-multiply NaN recovery on the hot path).
void run_1d(const Plan1D& pl, cd* x, cd* y, cd** out) {
  const int n = pl.n;
  double* src = reinterpret_cast<double*>(x);
  double* dst = reinterpret_cast<double*>(y);
  const double s = pl.sign;
  for (const Stage& st : pl.stages) {
    const int p = st.p, ns = st.ns, q = n / p;
    const double* twb = reinterpret_cast<const double*>(st.tw.data());
    if (p == 4) {
      // radix 4: the per-stage branch is hoisted out of the butterfly loops
      for (int b0 = 0; b0 < q; b0 += ns) {
        const double* i0 = src + 2 * b0;
        const double* i1 = i0 + 2 * q;
        const double* i2 = i1 + 2 * q;
        const double* i3 = i2 + 2 * q;
        double* o = dst + 2 * static_cast<size_t>(b0) * 4;
        const double* w = twb;
        for (int k = 0; k < ns; ++k, w += 6) {
          const double a0r = i0[2 * k], a0i = i0[2 * k + 1];
          const double x1r = i1[2 * k], x1i = i1[2 * k + 1];
          const double x2r = i2[2 * k], x2i = i2[2 * k + 1];
          const double x3r = i3[2 * k], x3i = i3[2 * k + 1];
          const double a1r = x1r * w[0] - x1i * w[1], a1i = x1r * w[1] + x1i * w[0];
          const double a2r = x2r * w[2] - x2i * w[3], a2i = x2r * w[3] + x2i * w[2];
          const double a3r = x3r * w[4] - x3i * w[5], a3i = x3r * w[5] + x3i * w[4];
          const double t0r = a0r + a2r, t0i = a0i + a2i, t1r = a0r - a2r, t1i = a0i - a2i;
          const double t2r = a1r + a3r, t2i = a1i + a3i, dr = a1r - a3r, di = a1i - a3i;
          const double t3r = -s * di, t3i = s * dr;
          double* ok = o + 2 * k;
          ok[0] = t0r + t2r;
          ok[1] = t0i + t2i;
          ok[2 * ns] = t1r + t3r;
          ok[2 * ns + 1] = t1i + t3i;
          ok[4 * ns] = t0r - t2r;
          ok[4 * ns + 1] = t0i - t2i;
          ok[6 * ns] = t1r - t3r;
          ok[6 * ns + 1] = t1i - t3i;
        }
      }
      std::swap(src, dst);
      continue;
    }
    for (int b0 = 0; b0 < q; b0 += ns) {
      const int obase = b0 * p;  // (j / ns) * ns * p with j = b0 + k
      for (int k = 0; k < ns; ++k) {
        const int j = b0 + k;
        const double* w = twb + 2 * static_cast<size_t>(k) * (p - 1);
        double* o = dst + 2 * static_cast<size_t>(obase + k);
        if (p == 2) {
          const double* i0 = src + 2 * j;
          const double* i1 = src + 2 * (j + q);
          const double a1r = i1[0] * w[0] - i1[1] * w[1], a1i = i1[0] * w[1] + i1[1] * w[0];
          o[0] = i0[0] + a1r;
          o[1] = i0[1] + a1i;
          o[2 * ns] = i0[0] - a1r;
          o[2 * ns + 1] = i0[1] - a1i;
        } else if (p == 3) {
          const double* i0 = src + 2 * j;
          const double* i1 = src + 2 * (j + q);
          const double* i2 = src + 2 * (j + 2 * q);
          const double a1r = i1[0] * w[0] - i1[1] * w[1], a1i = i1[0] * w[1] + i1[1] * w[0];
          const double a2r = i2[0] * w[2] - i2[1] * w[3], a2i = i2[0] * w[3] + i2[1] * w[2];
          const double tr = a1r + a2r, ti = a1i + a2i;
          const double mr = i0[0] - 0.5 * tr, mi = i0[1] - 0.5 * ti;
          const double h = 0.86602540378443864676 * s;
          const double rr = -h * (a1i - a2i), ri = h * (a1r - a2r);
          o[0] = i0[0] + tr;
          o[1] = i0[1] + ti;
          o[2 * ns] = mr + rr;
          o[2 * ns + 1] = mi + ri;
          o[4 * ns] = mr - rr;
          o[4 * ns + 1] = mi - ri;
        } else {
          double a[2 * 64];
          std::vector<double> big;
          double* av = a;
          if (p > 64) {
            big.resize(2 * static_cast<size_t>(p));
            av = big.data();
          }
          av[0] = src[2 * j];
          av[1] = src[2 * j + 1];
          for (int r = 1; r < p; ++r) {
            const double* ir = src + 2 * (j + r * q);
            av[2 * r] = ir[0] * w[2 * (r - 1)] - ir[1] * w[2 * (r - 1) + 1];
            av[2 * r + 1] = ir[0] * w[2 * (r - 1) + 1] + ir[1] * w[2 * (r - 1)];
          }
          const double* rt = reinterpret_cast<const double*>(st.rootp.data());
          for (int t = 0; t < p; ++t) {
            double accr = av[0], acci = av[1];
            int e = 0;
            for (int r = 1; r < p; ++r) {
              e += t;
              if (e >= p) e -= p;
              accr += av[2 * r] * rt[2 * e] - av[2 * r + 1] * rt[2 * e + 1];
              acci += av[2 * r] * rt[2 * e + 1] + av[2 * r + 1] * rt[2 * e];
            }
            o[2 * t * ns] = accr;
            o[2 * t * ns + 1] = acci;
          }
        }
      }
    }
    std::swap(src, dst);
  }
  *out = reinterpret_cast<cd*>(src);
}

}  // namespace

struct rtn_fftw_plan_s {
  int n0 = 0, n1 = 0;
  Plan1D p0, p1;
};

extern "C" fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex*, fftw_complex*, int sign, unsigned) {
  if (n0 < 1 || n1 < 1) return nullptr;
  auto* p = new rtn_fftw_plan_s;
  p->n0 = n0;
  p->n1 = n1;
  p->p0 = make_1d(n0, sign);
  p->p1 = make_1d(n1, sign);
  return p;
}

extern "C" void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
  const int n0 = p->n0, n1 = p->n1;
  auto* x = reinterpret_cast<cd*>(in);
  auto* y = reinterpret_cast<cd*>(out);
  const int nm = std::max(n0, n1);
  thread_local std::vector<cd> a, b;
  constexpr int kBlk = 8;
  a.resize(static_cast<size_t>(nm) * kBlk);
  b.resize(static_cast<size_t>(nm) * kBlk);
  // rows (axis 1)
  for (int r = 0; r < n0; ++r) {
    std::memcpy(static_cast<void*>(a.data()), x + static_cast<size_t>(r) * n1, sizeof(cd) * n1);
    cd* res = nullptr;
    run_1d(p->p1, a.data(), b.data(), &res);
    std::memcpy(static_cast<void*>(y + static_cast<size_t>(r) * n1), res, sizeof(cd) * n1);
  }
  // columns (axis 0), gathered kBlk at a time
  for (int c0 = 0; c0 < n1; c0 += kBlk) {
    const int nb = std::min(kBlk, n1 - c0);
    for (int r = 0; r < n0; ++r) {
      const cd* row = y + static_cast<size_t>(r) * n1 + c0;
      for (int c = 0; c < nb; ++c) a[static_cast<size_t>(c) * nm + r] = row[c];
    }
    for (int c = 0; c < nb; ++c) {
      cd* res = nullptr;
      run_1d(p->p0, a.data() + static_cast<size_t>(c) * nm, b.data() + static_cast<size_t>(c) * nm, &res);
      if (res != a.data() + static_cast<size_t>(c) * nm) {
        std::memcpy(static_cast<void*>(a.data() + static_cast<size_t>(c) * nm), res, sizeof(cd) * n0);
      }
    }
    for (int r = 0; r < n0; ++r) {
      cd* row = y + static_cast<size_t>(r) * n1 + c0;
      for (int c = 0; c < nb; ++c) row[c] = a[static_cast<size_t>(c) * nm + r];
    }
  }
}

extern "C" void fftw_destroy_plan(fftw_plan p) { delete p; }
