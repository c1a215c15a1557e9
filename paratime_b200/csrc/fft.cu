// Batched complex DFTs along the axes of row-major fields (replaces the reference's
// FFTW wrapper, /root/reference/proj/src/fft.cpp:46-90, with the same conventions):
//   forward = unnormalised sum_j f_j e^{-2 pi i jk/n}; inverse includes 1/n per line;
//   2D = every row (axis 1) first, then every column (axis 0).
// Power-of-two lines use a shared-memory Stockham radix-2 FFT with an exactly tabulated
// twiddle table (host cos/sin of 2 pi k/n); other lengths use a direct O(n^2) DFT with
// (jk mod n) twiddle indexing.  Columns are processed as tiles of adjacent columns so
// global accesses stay coalesced.

#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "ptb_fft.h"

namespace ptb {
namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// One CTA transforms `cols` adjacent lines of length n held as a [n][cols] tile in smem.
// Line l of the tile starts at element (base + l*lstride) with element stride estride.
struct LineJob {
  double2* data;
  int n;            // line length
  long long count;  // number of lines
  // line index -> (outer, inner): offset = outer*outer_stride + inner*inner_stride
  long long inner;  // lines per outer block
  long long outer_stride, inner_stride, elem_stride;
  const double2* tw;  // twiddles w[k] = exp(-2 pi i k/n), k < n
  int inverse;
  int pow2;
};

__device__ __forceinline__ long long line_offset(const LineJob& J, long long l) {
  const long long o = l / J.inner, i = l - o * J.inner;
  return o * J.outer_stride + i * J.inner_stride;
}

// Tile of TC lines, blockDim.x threads.  CONTIG: lines are contiguous in global memory
// (row pass) -> tile stored line-major and threads walk along lines; otherwise (column
// pass) the tile is element-major and threads walk across adjacent lines.  Both keep
// global accesses coalesced and shared-memory accesses conflict-free.
template <int TC, bool CONTIG>
__global__ void k_fft_lines(const LineJob J) {
  extern __shared__ double2 sbuf[];  // [2][n*TC] ping-pong
  const int n = J.n, T = blockDim.x, tid = threadIdx.x;
  const long long l0 = static_cast<long long>(blockIdx.x) * TC;
  double2* A = sbuf;
  double2* B = sbuf + size_t(n) * TC;
  const int es = CONTIG ? 1 : TC, ls = CONTIG ? n : 1;  // smem strides (element, line)
  auto split = [&](int k, int len, int& e, int& c) {   // flat work index -> (element, line)
    if (CONTIG) {
      c = k / len;
      e = k - c * len;
    } else {
      e = k / TC;
      c = k - e * TC;
    }
  };
  for (int k = tid; k < n * TC; k += T) {
    int e, c;
    split(k, n, e, c);
    const long long l = l0 + c;
    A[e * es + c * ls] = l < J.count ? J.data[line_offset(J, l) + e * J.elem_stride] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  if (J.pow2) {
    // Stockham autosort radix-2, sub-transform half-length m = 1, 2, 4, ...
    const int half = n >> 1;
    for (int m = 1; m < n; m <<= 1) {
      for (int k = tid; k < half * TC; k += T) {
        int q, c;
        split(k, half, q, c);
        const int j = q % m, g = q / m;
        double2 w = J.tw[(j * (n / (2 * m))) % n];
        if (J.inverse) w.y = -w.y;
        const double2 a = A[q * es + c * ls];
        const double2 b = cmul(w, A[(q + half) * es + c * ls]);
        B[(2 * g * m + j) * es + c * ls] = make_double2(a.x + b.x, a.y + b.y);
        B[(2 * g * m + j + m) * es + c * ls] = make_double2(a.x - b.x, a.y - b.y);
      }
      __syncthreads();
      double2* t = A;
      A = B;
      B = t;
    }
  } else {
    for (int k = tid; k < n * TC; k += T) {
      int kk, c;
      split(k, n, kk, c);
      double2 acc = make_double2(0.0, 0.0);
      for (int j = 0; j < n; ++j) {
        double2 w = J.tw[(static_cast<long long>(j) * kk) % n];
        if (J.inverse) w.y = -w.y;
        const double2 v = cmul(A[j * es + c * ls], w);
        acc.x += v.x;
        acc.y += v.y;
      }
      B[kk * es + c * ls] = acc;
    }
    __syncthreads();
    double2* t = A;
    A = B;
    B = t;
  }
  const double s = J.inverse ? 1.0 / static_cast<double>(n) : 1.0;
  for (int k = tid; k < n * TC; k += T) {
    int e, c;
    split(k, n, e, c);
    const long long l = l0 + c;
    if (l < J.count) {
      double2 v = A[e * es + c * ls];
      if (J.inverse) {
        v.x *= s;
        v.y *= s;
      }
      J.data[line_offset(J, l) + e * J.elem_stride] = v;
    }
  }
}

struct TwiddleCache {
  std::mutex m;
  std::map<std::pair<int, int>, double2*> tabs;  // (device, n) -> table
  ~TwiddleCache() {}
  const double2* get(int device, int n) {
    std::lock_guard<std::mutex> lock(m);
    auto key = std::make_pair(device, n);
    auto it = tabs.find(key);
    if (it != tabs.end()) return it->second;
    std::vector<double2> w(n);
    for (int k = 0; k < n; ++k) {
      // exact argument: 2 pi k / n
      const long double ang = -2.0L * 3.14159265358979323846264338327950288L * (long double)k / (long double)n;
      w[k] = make_double2(double(std::cos(ang)), double(std::sin(ang)));
    }
    double2* d = nullptr;
    PTB_CUDA_CHECK(cudaMalloc(&d, n * sizeof(double2)));
    PTB_CUDA_CHECK(cudaMemcpy(d, w.data(), n * sizeof(double2), cudaMemcpyHostToDevice));
    tabs.emplace(key, d);
    return d;
  }
};

TwiddleCache& twiddles() {
  static TwiddleCache* c = new TwiddleCache();  // intentionally leaked (process lifetime)
  return *c;
}

void run_lines(ptb_context* ctx, cudaStream_t st, LineJob J) {
  if (J.count == 0) return;
  J.tw = twiddles().get(ctx->device, J.n);
  J.pow2 = (J.n & (J.n - 1)) == 0;
  // lines per CTA: enough to coalesce and fill the CTA, bounded by shared memory
  int tc = 1;
  while (tc < 32 && size_t(J.n) * tc * 2 * 2 * sizeof(double2) <= 96 * 1024 && tc * J.n < 4096) tc *= 2;
  const size_t smem = size_t(J.n) * tc * 2 * sizeof(double2);
  const unsigned blocks = static_cast<unsigned>((J.count + tc - 1) / tc);
  const int threads = 256;
  const bool contig = J.elem_stride == 1;
  switch (tc) {
#define PTB_FFT_CASE(TC)                                                                                   \
  case TC:                                                                                                 \
    if (contig) {                                                                                          \
      PTB_CUDA_CHECK(cudaFuncSetAttribute(k_fft_lines<TC, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                          int(smem)));                                                     \
      k_fft_lines<TC, true><<<blocks, threads, smem, st>>>(J);                                             \
    } else {                                                                                               \
      PTB_CUDA_CHECK(cudaFuncSetAttribute(k_fft_lines<TC, false>,                                          \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));        \
      k_fft_lines<TC, false><<<blocks, threads, smem, st>>>(J);                                            \
    }                                                                                                      \
    break;
    PTB_FFT_CASE(1)
    PTB_FFT_CASE(2)
    PTB_FFT_CASE(4)
    PTB_FFT_CASE(8)
    PTB_FFT_CASE(16)
    PTB_FFT_CASE(32)
#undef PTB_FFT_CASE
    default: fail(PTB_UNSUPPORTED, "fft tile");
  }
  PTB_LAUNCH_CHECK(ctx);
}

}  // namespace

void fft_field(ptb_context* ctx, cudaStream_t st, const ptb_grid& g, size_t batch, double2* data, bool inverse) {
  require(g.n[0] <= 65536 && (g.dim == 1 || g.n[1] <= 65536), "fft: line too long");
  if (g.dim == 1) {
    const int n = int(g.n[0]);
    run_lines(ctx, st, LineJob{data, n, (long long)batch, 1, (long long)n, 0, 1, nullptr, inverse, 0});
    return;
  }
  const int ny = int(g.n[0]), nx = int(g.n[1]);
  // rows: line l = (b*ny + y), contiguous
  run_lines(ctx, st, LineJob{data, nx, (long long)batch * ny, 1, (long long)nx, 0, 1, nullptr, inverse, 0});
  // columns: line l = b*nx + x -> offset b*ny*nx + x, element stride nx
  run_lines(ctx, st,
            LineJob{data, ny, (long long)batch * nx, (long long)nx, (long long)ny * nx, 1, (long long)nx, nullptr,
                    inverse, 0});
}

}  // namespace ptb
