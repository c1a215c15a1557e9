// ORACLE — test infrastructure only (tests/, bench.py cpu_baseline, smoke()).
//
// Restatement of /root/reference/proj/src/fft.cpp without FFTW3 (absent from this
// image; the reference links it unpinned via find_library, CMakeLists.txt:15-19).
// Conventions kept exactly (fft.hpp:10-29, fft.cpp:46-102):
//   forward  = unnormalised sum_j f_j e^{-2 pi i jk/n}
//   inverse  = sum_k F_k e^{+2 pi i jk/n} / n
//   2D       = rows (axis 1) then columns (axis 0)
//   signed_freq(k) = k for k <= (n-1)/2, else k - n; Nyquist bin = n/2 for even n.
// Line transforms: iterative radix-2 for power-of-two n, direct O(n^2) DFT with
// exact (jk mod n) twiddle indexing otherwise.  Twiddle tables are cached per n
// behind a mutex, mirroring the reference's mutex-guarded plan cache (fft.cpp:12-42).

#include <cmath>
#include <complex>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "paratime/fft.hpp"

namespace paratime::detail {

namespace {

using cplx = std::complex<double>;

struct Plan {
  std::size_t n;
  bool pow2;
  std::vector<cplx> w;  // w[k] = exp(-2 pi i k / n), k < n
};

class PlanCache {
 public:
  const Plan& get(std::size_t n) {
    std::lock_guard<std::mutex> lock(mutex_);
    auto it = plans_.find(n);
    if (it != plans_.end()) return *it->second;
    auto p = std::make_unique<Plan>();
    p->n = n;
    p->pow2 = n > 0 && (n & (n - 1)) == 0;
    p->w.resize(n);
    for (std::size_t k = 0; k < n; ++k) {
      const double ang = -2.0 * M_PI * static_cast<double>(k) / static_cast<double>(n);
      p->w[k] = cplx(std::cos(ang), std::sin(ang));
    }
    const Plan& ref = *p;
    plans_.emplace(n, std::move(p));
    return ref;
  }

 private:
  std::mutex mutex_;
  std::map<std::size_t, std::unique_ptr<Plan>> plans_;
};

PlanCache& cache() {
  static PlanCache c;
  return c;
}

void fft_pow2(cplx* a, std::size_t n, const std::vector<cplx>& w, bool inverse) {
  // bit reversal
  for (std::size_t i = 1, j = 0; i < n; ++i) {
    std::size_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(a[i], a[j]);
  }
  for (std::size_t len = 2; len <= n; len <<= 1) {
    const std::size_t half = len / 2, stride = n / len;
    for (std::size_t i = 0; i < n; i += len)
      for (std::size_t k = 0; k < half; ++k) {
        cplx tw = w[k * stride];
        if (inverse) tw = std::conj(tw);
        const cplx t = a[i + k + half] * tw;
        a[i + k + half] = a[i + k] - t;
        a[i + k] = a[i + k] + t;
      }
  }
}

void dft_direct(cplx* a, std::size_t n, const std::vector<cplx>& w, bool inverse) {
  std::vector<cplx> out(n);
  for (std::size_t k = 0; k < n; ++k) {
    cplx acc(0.0, 0.0);
    for (std::size_t j = 0; j < n; ++j) {
      cplx tw = w[(j * k) % n];
      if (inverse) tw = std::conj(tw);
      acc += a[j] * tw;
    }
    out[k] = acc;
  }
  for (std::size_t k = 0; k < n; ++k) a[k] = out[k];
}

}  // namespace

// fft.cpp:46-54
void dft_line(std::complex<double>* data, std::size_t n, bool inverse) {
  const Plan& plan = cache().get(n);
  if (plan.pow2)
    fft_pow2(data, n, plan.w, inverse);
  else
    dft_direct(data, n, plan.w, inverse);
  if (inverse) {
    const double s = 1.0 / static_cast<double>(n);
    for (std::size_t i = 0; i < n; ++i) data[i] *= s;
  }
}

namespace {

// fft.cpp:58-73
void transform_field(std::vector<std::complex<double>>& spec, const Grid& grid, bool inverse) {
  if (grid.dim() == 1) {
    dft_line(spec.data(), grid.points(0), inverse);
    return;
  }
  const std::size_t ny = grid.points(0), nx = grid.points(1);
  for (std::size_t jy = 0; jy < ny; ++jy) dft_line(spec.data() + jy * nx, nx, inverse);
  std::vector<cplx> col(ny);
  for (std::size_t jx = 0; jx < nx; ++jx) {
    for (std::size_t jy = 0; jy < ny; ++jy) col[jy] = spec[jy * nx + jx];
    dft_line(col.data(), ny, inverse);
    for (std::size_t jy = 0; jy < ny; ++jy) spec[jy * nx + jx] = col[jy];
  }
}

}  // namespace

// fft.cpp:77-82
std::vector<std::complex<double>> forward_dft(const std::vector<double>& field, const Grid& grid) {
  std::vector<std::complex<double>> spec(field.begin(), field.end());
  transform_field(spec, grid, false);
  return spec;
}

// fft.cpp:84-90
std::vector<double> inverse_dft_real(std::vector<std::complex<double>> spectrum, const Grid& grid) {
  transform_field(spectrum, grid, true);
  std::vector<double> out(spectrum.size());
  for (std::size_t i = 0; i < out.size(); ++i) out[i] = spectrum[i].real();
  return out;
}

// fft.cpp:92-95
long signed_freq(std::size_t k, std::size_t n) {
  return k <= (n - 1) / 2 ? static_cast<long>(k) : static_cast<long>(k) - static_cast<long>(n);
}

// fft.cpp:97-100
double wavenumber(const Grid& grid, int axis, std::size_t k) {
  const std::size_t n = grid.points(axis);
  return 2.0 * M_PI * static_cast<double>(signed_freq(k, n)) / grid.extent(axis);
}

// fft.cpp:102
bool is_nyquist(std::size_t k, std::size_t n) { return n % 2 == 0 && k == n / 2; }

}  // namespace paratime::detail
