// ORACLE TEST INFRASTRUCTURE — not product code. See fftw3.h for scope.
//
// Double-precision 2D DFT behind the FFTW plan/execute interface. Per axis a
// recursive decimation-in-time Cooley-Tukey over the prime factorisation of
// the length, with every twiddle read from one table exp(sign*2*pi*i*e/N)
// computed once per plan (so no twiddle recurrence error accumulates); prime
// factors use a direct DFT over the same table.
#include "fftw3.h"

#include <cmath>
#include <complex>
#include <cstring>
#include <numbers>
#include <vector>

using cd = std::complex<double>;

extern "C" const char fftw_version[] = "3.3.10-rtnlinv-oracle-shim";

struct rtn_fftw_plan_s {
  int n0 = 0, n1 = 0, sign = -1;
  std::vector<cd> tw0, tw1;         // exp(sign 2 pi i e / n) per axis
  std::vector<int> f0, f1;          // prime factors, ascending
};

namespace {

std::vector<int> factorize(int n) {
  std::vector<int> f;
  for (int p = 2; p * p <= n; ++p) {
    while (n % p == 0) {
      f.push_back(p);
      n /= p;
    }
  }
  if (n > 1) f.push_back(n);
  return f;
}

std::vector<cd> table(int n, int sign) {
  std::vector<cd> t(static_cast<size_t>(n));
  for (int e = 0; e < n; ++e) {
    // reduce to the first octant-free form: angle = 2*pi*e/n exactly once
    const double a = 2.0 * std::numbers::pi * static_cast<double>(e) / n;
    t[static_cast<size_t>(e)] = cd(std::cos(a), sign * std::sin(a));
  }
  return t;
}

// out[k] = sum_j in[j*stride] * w_n^{jk}, n = N / L, w_n^e = tw[(e*L) mod N]
void dft_rec(const cd* in, int stride, cd* out, int n, const int* fac, const std::vector<cd>& tw,
             int L, cd* scratch) {
  const int N = static_cast<int>(tw.size());
  if (n == 1) {
    out[0] = in[0];
    return;
  }
  const int p = fac[0];
  const int m = n / p;
  if (m == 1) {
    // direct DFT of a prime length
    for (int k = 0; k < n; ++k) {
      cd acc(0, 0);
      for (int j = 0; j < n; ++j) {
        const long long e = (static_cast<long long>(j) * k % n) * L % N;
        acc += in[static_cast<size_t>(j) * stride] * tw[static_cast<size_t>(e)];
      }
      out[k] = acc;
    }
    return;
  }
  // p interleaved sub-sequences of length m into out[r*m ...]
  for (int r = 0; r < p; ++r) {
    dft_rec(in + static_cast<size_t>(r) * stride, stride * p, out + static_cast<size_t>(r) * m, m,
            fac + 1, tw, L * p, scratch + n);
  }
  // butterflies: X[k + q m] = sum_r Y_r[k] w_n^{r (k + q m)}
  std::memcpy(static_cast<void*>(scratch), out, sizeof(cd) * static_cast<size_t>(n));
  for (int k = 0; k < m; ++k) {
    for (int q = 0; q < p; ++q) {
      const int kk = k + q * m;
      cd acc(0, 0);
      for (int r = 0; r < p; ++r) {
        const long long e = (static_cast<long long>(r) * kk % n) * L % N;
        acc += scratch[static_cast<size_t>(r) * m + k] * tw[static_cast<size_t>(e)];
      }
      out[kk] = acc;
    }
  }
}

void dft_1d(const cd* in, int stride, cd* out, int n, const std::vector<int>& fac,
            const std::vector<cd>& tw) {
  std::vector<cd> scratch(static_cast<size_t>(4 * n + 8));
  dft_rec(in, stride, out, n, fac.data(), tw, 1, scratch.data());
}

}  // namespace

extern "C" fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex*, fftw_complex*, int sign,
                                      unsigned) {
  if (n0 < 1 || n1 < 1) return nullptr;
  auto* p = new rtn_fftw_plan_s;
  p->n0 = n0;
  p->n1 = n1;
  p->sign = sign;
  p->tw0 = table(n0, sign);
  p->tw1 = table(n1, sign);
  p->f0 = factorize(n0);
  p->f1 = factorize(n1);
  return p;
}

extern "C" void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
  const int n0 = p->n0, n1 = p->n1;
  auto* x = reinterpret_cast<cd*>(in);
  auto* y = reinterpret_cast<cd*>(out);
  std::vector<cd> tmp(static_cast<size_t>(n0) * n1);
  std::vector<cd> line(static_cast<size_t>(std::max(n0, n1)));
  // along axis 1 (contiguous rows)
  for (int r = 0; r < n0; ++r) {
    dft_1d(x + static_cast<size_t>(r) * n1, 1, tmp.data() + static_cast<size_t>(r) * n1, n1, p->f1,
           p->tw1);
  }
  // along axis 0 (columns)
  for (int c = 0; c < n1; ++c) {
    dft_1d(tmp.data() + c, n1, line.data(), n0, p->f0, p->tw0);
    for (int r = 0; r < n0; ++r) y[static_cast<size_t>(r) * n1 + c] = line[static_cast<size_t>(r)];
  }
}

extern "C" void fftw_destroy_plan(fftw_plan p) { delete p; }
