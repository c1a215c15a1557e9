// Internal declarations shared by the paratime_b200 translation units.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <chrono>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

#include "paratime_b200.h"

namespace ptb {

// Exception carrying a ptb_status; converted to a return code at the C ABI.
struct Error : std::runtime_error {
  ptb_status status;
  Error(ptb_status s, const std::string& what) : std::runtime_error(what), status(s) {}
};

extern thread_local std::string g_last_error;

[[noreturn]] inline void fail(ptb_status s, const std::string& what) { throw Error(s, what); }
inline void require(bool ok, const std::string& what) {
  if (!ok) fail(PTB_INVALID_ARGUMENT, what);
}

#define PTB_CUDA_CHECK(expr)                                                           \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess)                                                             \
      ::ptb::fail(PTB_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));      \
  } while (0)

bool sync_check_enabled();  // PTB_SYNC_CHECK=1: synchronise after every launch (debug)

#define PTB_LAUNCH_CHECK(ctx)                                                          \
  do {                                                                                 \
    cudaError_t _e = cudaGetLastError();                                               \
    if (_e == cudaSuccess && ::ptb::sync_check_enabled()) _e = cudaDeviceSynchronize(); \
    if (_e != cudaSuccess)                                                             \
      ::ptb::fail(PTB_CUDA, std::string("kernel launch: ") + cudaGetErrorString(_e) +  \
                                " at " + __FILE__ + ":" + std::to_string(__LINE__));   \
    (ctx)->launches.fetch_add(1, std::memory_order_relaxed);                           \
  } while (0)

// Opt-in host timeline (PTB_PROF=1): mark(label) synchronises the stream and prints the time
// since the previous mark to stderr.  Diagnostics only; off by default (no synchronisation).
struct HostProf {
  bool on = false;
  cudaStream_t st = nullptr;
  std::chrono::steady_clock::time_point t;
  explicit HostProf(cudaStream_t s) : st(s) {
    static const bool env = std::getenv("PTB_PROF") != nullptr;
    on = env;
    if (on) {
      cudaStreamSynchronize(st);
      t = std::chrono::steady_clock::now();
    }
  }
  void mark(const char* label) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[ptb prof] %-28s %9.3f ms\n", label,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// Grow-only device scratch buffer; owns its allocation (move-only, freed on destruction).
struct DeviceBuffer {
  void* ptr = nullptr;
  size_t bytes = 0;
  DeviceBuffer() = default;
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : ptr(o.ptr), bytes(o.bytes) {
    o.ptr = nullptr;
    o.bytes = 0;
  }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      release();
      ptr = o.ptr;
      bytes = o.bytes;
      o.ptr = nullptr;
      o.bytes = 0;
    }
    return *this;
  }
  ~DeviceBuffer() { release(); }
  void* get(size_t need);
  void release();
};

}  // namespace ptb

namespace ptb {
// Programmatic dependent launch (sm_90+): a kernel launched with pdl_attr() may start while its
// predecessor on the stream is still running; it must call pdl_wait() before reading anything the
// predecessor wrote.  pdl_trigger() lets the successor's blocks be scheduled early (they spin in
// pdl_wait until this grid has completed and its writes are visible).  Both are no-ops for
// kernels launched without the attribute.  Used on the latency-bound theta-sweep chain.
__device__ __forceinline__ void pdl_wait() {
#if defined(__CUDA_ARCH__)
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_trigger() {
#if defined(__CUDA_ARCH__)
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#endif
}
bool pdl_enabled();  // PTB_PDL=0 disables the attribute (diagnostics)

// launch `kern` with the programmatic-stream-serialization attribute (the kernel must pdl_wait())
template <typename... Exp, typename... Act>
void launch_pdl(void (*kern)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Act&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Act>(args)...);
  if (e != cudaSuccess) fail(PTB_CUDA, std::string("launch: ") + cudaGetErrorString(e));
}
}  // namespace ptb

struct ptb_context {
  int device = 0;
  cudaStream_t stream = nullptr;      // stream all work is issued on
  cudaStream_t own_stream = nullptr;  // the context's own stream
  int num_sms = 148;
  std::atomic<uint64_t> launches{0};
  std::recursive_mutex mutex;  // serialises host-API calls (reference runs stages concurrently)
  ptb::DeviceBuffer scratch[4];
  ptb::DeviceBuffer flags;
  // host-batch pipeline: three streams/slots so the H2D of chunk i+1, the propagation of chunk i
  // and the D2H of chunk i-1 overlap (separate copy engines for the two directions)
  cudaStream_t aux[3] = {nullptr, nullptr, nullptr};
  // second lane of the wavefront propagator's chunk loop (propagate.cu wave_propagate): alternate
  // chunks run on `stream` and `lane`, so one chunk's last partial round of CTAs overlaps the
  // other's next pass; forked from / joined to `stream` with these events
  cudaStream_t lane = nullptr;
  cudaEvent_t lane_fork = nullptr, lane_join = nullptr;
  ptb::DeviceBuffer slotbuf[3][5];  // per pipeline slot: u, v, su, sv, flags
  // pinned staging for the per-slice flags of the host-batch call: a D2H copy into pageable
  // memory is synchronous and would serialise the pipeline
  int32_t* pinned_flags = nullptr;
  size_t pinned_flags_n = 0;
  ptb::DeviceBuffer gemm_ws;  // split-K partials of ptb::gemm (gemm.cu)
  // parareal driver work buffers kept between runs (driver.cu), so a repeated run neither
  // reallocates nor synchronises on cudaMalloc/cudaFree; freed with the context
  std::shared_ptr<void> driver_cache;
};

namespace ptb {

// Arithmetic parameters of one propagator (host-computed exactly as propagator.cpp).
struct StepParams {
  int dim;              // 1 or 2
  int ny, nx;           // 2D: points(0), points(1); 1D: ny = 1, nx = points(0)
  double ihx2, ihy2;    // 1/(h*h) per axis, propagator.cpp:42-43 (1D: ihx2 = 1/(h0*h0))
  double dt, hd, hdt2;  // dt, 0.5*dt, 0.5*dt*dt (propagator.cpp:64)
  double ry, cc;        // FAST: ry = ihy2/ihx2 (0 in 1D), cc = -2*(1+ry)
};

}  // namespace ptb

struct ptb_propagator {
  ptb_context* ctx = nullptr;
  ptb_grid grid{};
  size_t n = 0;  // points
  size_t steps = 0;
  ptb::StepParams prm{};
  double* c = nullptr;   // speed (N)
  double* c2 = nullptr;  // c*c (N)                — EXACT coefficient
  double* kx = nullptr;  // 0.5*dt*c*c/hx^2 (N)     — FAST coefficient
};

struct ptb_transfer {
  ptb_context* ctx = nullptr;
  ptb_grid coarse{}, fine{};
  int kind = 0;
  size_t ratio[2] = {1, 1};
  // Fourier weights per axis: w[a][rem*nc + j] = weight of coarse node q-j..., see transfer.cu
  double* wx = nullptr;
  double* wy = nullptr;
  // warp-FFT route (2D Fourier, large grids): the x-pass plane (batch x coarse rows x fine cols)
  ptb::DeviceBuffer spec_c;
  ptb::DeviceBuffer nodes_half;  // scratch of interpolate_at_coarse_nodes
  ptb::DeviceBuffer add_work;    // scratch of ptb_interpolate_add_batch (direct routes)
};

namespace ptb {

// Run `fn`, converting exceptions to a status + thread-local message (C ABI boundary).
template <typename Fn>
ptb_status guarded(Fn&& fn) {
  try {
    fn();
    return PTB_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.status;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return PTB_CUDA;
  }
}

// Where a propagation runs: stream + ping-pong scratch (2 x batch*N doubles, or null
// to use the context scratch) + EXACT-mode acceleration scratch for the stream path.
struct LaunchSlot {
  cudaStream_t stream = nullptr;
  double* su = nullptr;
  double* sv = nullptr;
  // optional input state: propagate() then reads (src_u, src_v) and writes (u, v) — the wavefront
  // path's first pass reads the source directly, the other kernel families copy it first
  const double* src_u = nullptr;
  const double* src_v = nullptr;
};

// propagate.cu
// Human-readable launch plan of propagate() (kernels, strip widths, grids).
std::string describe_plan(ptb_propagator* p, size_t steps, size_t batch, int mode);
void propagate(ptb_propagator* p, size_t steps, size_t batch, double* u, double* v, int32_t* flags,
               int mode, const LaunchSlot* slot = nullptr);
void laplacian(ptb_context* ctx, const ptb_grid& g, size_t batch, const double* f, double* out);
void wave_rect_fast(ptb_context* ctx, cudaStream_t st, int S, const StepParams& p, size_t batch, const double* ui,
                    const double* vi, double* uo, double* vo, const double* kx, int32_t* flags, int y0, int rny,
                    int x0, int rnx);
void nonfinite(ptb_context* ctx, size_t n, size_t batch, const double* f, int32_t* flags);

// transfer.cu
void transfer_init(ptb_transfer* t);
void transfer_release(ptb_transfer* t);  // work buffers
void restrict_fields(ptb_transfer* t, size_t batch, const double* fine, double* coarse);
void interpolate_fields(ptb_transfer* t, size_t batch, const double* coarse, double* fine);
// out = base + I(coarse) (base may alias out); scratch: batch fine fields (used off the FFT route)
void interpolate_fields_add(ptb_transfer* t, size_t batch, const double* coarse, const double* base, double* out,
                            double* scratch);
// R(I(coarse)): the interpolant's values at the coarse nodes, bitwise equal to restricting
// the full interpolation (used by the coarse-only sweep)
void interpolate_at_coarse_nodes(ptb_transfer* t, size_t batch, const double* coarse, double* out);

inline size_t grid_size(const ptb_grid& g) { return g.dim == 1 ? g.n[0] : g.n[0] * g.n[1]; }
void validate_grid(const ptb_grid& g);

}  // namespace ptb
