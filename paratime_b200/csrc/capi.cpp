// extern "C" boundary of libparatime_b200 (declared in include/paratime_b200.h).
// Every entry point converts exceptions to a ptb_status plus a thread-local message.

#include <chrono>
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ptb_internal.h"

namespace ptb {

thread_local std::string g_last_error;

bool sync_check_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PTB_SYNC_CHECK");
    return e && *e == '1';
  }();
  return on;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PTB_PDL");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}

void* DeviceBuffer::get(size_t need) {
  if (need == 0) need = 8;
  if (need > bytes) {
    // geometric growth (2x, 2 MiB granules): buffers sized by the corrector rank grow every
    // parareal iteration, and each cudaFree/cudaMalloc pair synchronises the device and costs
    // ~5 ms per 100 MB on a B200 (the Procrustes factors X, Y ping-pong with their spares, so
    // each of the pair must absorb two rank increases per growth)
    size_t want = need;
    if (bytes) want = std::max(need, 2 * bytes);
    want = (want + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
    static const bool prof = std::getenv("PTB_PROF") != nullptr;  // diagnostics: slow (re)allocations
    const auto t0 = std::chrono::steady_clock::now();
    const size_t old = bytes;
    if (ptr) PTB_CUDA_CHECK(cudaFree(ptr));
    ptr = nullptr;
    if (cudaMalloc(&ptr, want) != cudaSuccess) {  // fall back to the exact size under pressure
      (void)cudaGetLastError();
      want = need;
      PTB_CUDA_CHECK(cudaMalloc(&ptr, want));
    }
    bytes = want;
    if (prof) {
      const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      if (ms > 2.0)
        std::fprintf(stderr, "[ptb prof] DeviceBuffer %zu -> %zu MiB: cudaFree + cudaMalloc %.1f ms\n", old >> 20,
                     want >> 20, ms);
    }
  }
  return ptr;
}

void DeviceBuffer::release() {
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  bytes = 0;
}

// Grid constructor checks (grid.cpp:24-33)
void validate_grid(const ptb_grid& g) {
  require(g.dim == 1 || g.dim == 2, "Grid: dimension must be 1 or 2 with matching spacing");
  for (int a = 0; a < g.dim; ++a) {
    require(g.n[a] >= 4, "Grid: need at least 4 points per axis");
    require(g.h[a] > 0.0 && std::isfinite(g.h[a]), "Grid: spacing must be positive");
  }
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace ptb

using namespace ptb;

extern "C" {

const char* ptb_last_error(void) { return g_last_error.c_str(); }
const char* ptb_version(void) { return "paratime_b200 0.1 (sm_100a)"; }

ptb_status ptb_context_create(int device, ptb_context** out) {
  return guarded([&] {
    require(out != nullptr, "context: null output");
    int count = 0;
    PTB_CUDA_CHECK(cudaGetDeviceCount(&count));
    require(device >= 0 && device < count, "context: no such CUDA device");
    DeviceGuard g(device);
    auto* ctx = new ptb_context();
    ctx->device = device;
    cudaDeviceProp prop{};
    PTB_CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
    ctx->num_sms = prop.multiProcessorCount;
    PTB_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
    ctx->stream = ctx->own_stream;
    *out = ctx;
  });
}

ptb_status ptb_context_destroy(ptb_context* ctx) {
  return guarded([&] {
    if (!ctx) return;
    DeviceGuard g(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto& b : ctx->scratch) b.release();
    for (auto& slot : ctx->slotbuf)
      for (auto& b : slot) b.release();
    for (auto& st : ctx->aux)
      if (st) cudaStreamDestroy(st);
    if (ctx->lane) cudaStreamDestroy(ctx->lane);
    if (ctx->lane_fork) cudaEventDestroy(ctx->lane_fork);
    if (ctx->lane_join) cudaEventDestroy(ctx->lane_join);
    ctx->flags.release();
    ctx->driver_cache.reset();  // parareal work buffers
    if (ctx->pinned_flags) cudaFreeHost(ctx->pinned_flags);
    ctx->gemm_ws.release();
    cudaStreamDestroy(ctx->own_stream);
    delete ctx;
  });
}

ptb_status ptb_context_synchronize(ptb_context* ctx) {
  return guarded([&] { PTB_CUDA_CHECK(cudaStreamSynchronize(ctx->stream)); });
}

void* ptb_context_stream(ptb_context* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }
ptb_status ptb_context_set_stream(ptb_context* ctx, void* stream) {
  return guarded([&] {
    require(ctx != nullptr, "context: null");
    ctx->stream = static_cast<cudaStream_t>(stream);
  });
}

ptb_status ptb_context_use_own_stream(ptb_context* ctx) {
  return guarded([&] {
    require(ctx != nullptr, "context: null");
    ctx->stream = ctx->own_stream;
  });
}

int ptb_context_device(ptb_context* ctx) { return ctx ? ctx->device : -1; }
uint64_t ptb_context_launches(ptb_context* ctx) { return ctx ? ctx->launches.load() : 0; }

ptb_status ptb_device_alloc(ptb_context* ctx, size_t bytes, void** out) {
  return guarded([&] {
    DeviceGuard g(ctx->device);
    PTB_CUDA_CHECK(cudaMalloc(out, std::max<size_t>(bytes, 8)));
  });
}

ptb_status ptb_device_free(ptb_context* ctx, void* p) {
  return guarded([&] {
    DeviceGuard g(ctx->device);
    if (p) PTB_CUDA_CHECK(cudaFree(p));
  });
}

ptb_status ptb_memcpy_h2d(ptb_context* ctx, void* dst, const void* src, size_t bytes) {
  return guarded([&] {
    DeviceGuard g(ctx->device);
    PTB_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    PTB_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  });
}

ptb_status ptb_memcpy_d2h(ptb_context* ctx, void* dst, const void* src, size_t bytes) {
  return guarded([&] {
    DeviceGuard g(ctx->device);
    PTB_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    PTB_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  });
}

// PropagatorConfig (propagator.cpp:11-27) + SpeedField (grid.cpp:91-98) checks.
ptb_status ptb_propagator_create(ptb_context* ctx, const ptb_grid* grid, const double* c_host, double dt,
                                 size_t steps, ptb_propagator** out) {
  return guarded([&] {
    require(ctx && grid && c_host && out, "PropagatorConfig: null argument");
    validate_grid(*grid);
    const size_t n = grid_size(*grid);
    for (size_t i = 0; i < n; ++i)
      require(c_host[i] > 0.0 && std::isfinite(c_host[i]),
              "SpeedField: wave speed must be strictly positive and finite");
    require(dt > 0.0 && std::isfinite(dt), "PropagatorConfig: dt must be positive");
    require(steps > 0, "PropagatorConfig: steps_per_coupling must be positive");
    const double cmax = *std::max_element(c_host, c_host + n);
    double hmin = grid->h[0];
    for (int a = 1; a < grid->dim; ++a) hmin = std::min(hmin, grid->h[a]);
    const double cfl = dt * cmax / hmin;
    const double bound = 1.0 / std::sqrt(static_cast<double>(grid->dim));
    if (cfl > bound * (1.0 + 1e-12))
      fail(PTB_INVALID_ARGUMENT, "PropagatorConfig: CFL violated, dt*max(c)/min(h) = " + std::to_string(cfl) +
                                     " > " + std::to_string(bound));
    DeviceGuard g(ctx->device);
    auto* p = new ptb_propagator();
    p->ctx = ctx;
    p->grid = *grid;
    p->n = n;
    p->steps = steps;
    StepParams& s = p->prm;
    s.dim = grid->dim;
    if (grid->dim == 1) {
      s.ny = 1;
      s.nx = int(grid->n[0]);
      s.ihx2 = 1.0 / (grid->h[0] * grid->h[0]);
      s.ihy2 = 0.0;
      s.ry = 0.0;
    } else {
      s.ny = int(grid->n[0]);
      s.nx = int(grid->n[1]);
      s.ihy2 = 1.0 / (grid->h[0] * grid->h[0]);
      s.ihx2 = 1.0 / (grid->h[1] * grid->h[1]);
      s.ry = s.ihy2 / s.ihx2;
    }
    s.cc = -2.0 * (1.0 + s.ry);
    s.dt = dt;
    s.hd = 0.5 * dt;
    s.hdt2 = 0.5 * dt * dt;
    std::vector<double> c2(n), kx(n);
    for (size_t i = 0; i < n; ++i) {
      c2[i] = c_host[i] * c_host[i];
      kx[i] = s.hd * c2[i] * s.ihx2;
    }
    PTB_CUDA_CHECK(cudaMalloc(&p->c, n * sizeof(double)));
    PTB_CUDA_CHECK(cudaMalloc(&p->c2, n * sizeof(double)));
    PTB_CUDA_CHECK(cudaMalloc(&p->kx, n * sizeof(double)));
    PTB_CUDA_CHECK(cudaMemcpy(p->c, c_host, n * sizeof(double), cudaMemcpyHostToDevice));
    PTB_CUDA_CHECK(cudaMemcpy(p->c2, c2.data(), n * sizeof(double), cudaMemcpyHostToDevice));
    PTB_CUDA_CHECK(cudaMemcpy(p->kx, kx.data(), n * sizeof(double), cudaMemcpyHostToDevice));
    *out = p;
  });
}

ptb_status ptb_propagator_destroy(ptb_propagator* p) {
  return guarded([&] {
    if (!p) return;
    DeviceGuard g(p->ctx->device);
    cudaFree(p->c);
    cudaFree(p->c2);
    cudaFree(p->kx);
    delete p;
  });
}

const double* ptb_propagator_speed(ptb_propagator* p) { return p ? p->c : nullptr; }

ptb_status ptb_propagate_steps_batch(ptb_propagator* p, size_t steps, size_t batch, double* u, double* v,
                                     int32_t* flags, int mode) {
  return guarded([&] {
    require(p && (batch == 0 || (u && v)), "propagate: null argument");
    require(mode == PTB_MODE_FAST || mode == PTB_MODE_EXACT, "propagate: unknown mode");
    DeviceGuard g(p->ctx->device);
    std::lock_guard<std::recursive_mutex> lock(p->ctx->mutex);
    propagate(p, steps, batch, u, v, flags, mode);
  });
}

ptb_status ptb_propagate_plan(ptb_propagator* p, size_t steps, size_t batch, int mode, char* buf, size_t len) {
  return guarded([&] {
    require(p && buf && len > 0, "propagate_plan: null argument");
    DeviceGuard g(p->ctx->device);
    std::lock_guard<std::recursive_mutex> lock(p->ctx->mutex);
    const std::string d = describe_plan(p, steps, batch, mode);
    const size_t k = std::min(len - 1, d.size());
    std::memcpy(buf, d.data(), k);
    buf[k] = 0;
  });
}

ptb_status ptb_propagate_batch(ptb_propagator* p, size_t batch, double* u, double* v, int32_t* flags, int mode) {
  if (!p) return PTB_INVALID_ARGUMENT;
  return ptb_propagate_steps_batch(p, p->steps, batch, u, v, flags, mode);
}

// propagate_coupling on host buffers (propagator.cpp:95-105).
ptb_status ptb_propagate_coupling_host(ptb_propagator* p, const double* u_in, const double* v_in, double* u_out,
                                       double* v_out, int mode) {
  return guarded([&] {
    require(p && u_in && v_in && u_out && v_out, "propagate_coupling: null argument");
    ptb_context* ctx = p->ctx;
    DeviceGuard g(ctx->device);
    std::lock_guard<std::recursive_mutex> lock(ctx->mutex);
    const size_t bytes = p->n * sizeof(double);
    // dedicated buffers (scratch[0..1] are used inside propagate)
    static thread_local DeviceBuffer bu, bv, bf;
    double* du = static_cast<double*>(bu.get(bytes));
    double* dv = static_cast<double*>(bv.get(bytes));
    int32_t* df = static_cast<int32_t*>(bf.get(sizeof(int32_t)));
    PTB_CUDA_CHECK(cudaMemcpyAsync(du, u_in, bytes, cudaMemcpyHostToDevice, ctx->stream));
    PTB_CUDA_CHECK(cudaMemcpyAsync(dv, v_in, bytes, cudaMemcpyHostToDevice, ctx->stream));
    PTB_CUDA_CHECK(cudaMemsetAsync(df, 0, sizeof(int32_t), ctx->stream));
    propagate(p, p->steps, 1, du, dv, df, mode);
    int32_t flag = 0;
    PTB_CUDA_CHECK(cudaMemcpyAsync(u_out, du, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    PTB_CUDA_CHECK(cudaMemcpyAsync(v_out, dv, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    PTB_CUDA_CHECK(cudaMemcpyAsync(&flag, df, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    PTB_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    if (flag) fail(PTB_DIVERGED, "propagate_coupling: non-finite state produced");
  });
}

// Batched propagate_coupling on host buffers, chunked over two streams so the PCIe
// copies of one chunk overlap the kernels of the other.
ptb_status ptb_propagate_batch_host(ptb_propagator* p, size_t batch, const double* u_in, const double* v_in,
                                    double* u_out, double* v_out, int32_t* flags_host, int mode) {
  return guarded([&] {
    require(p && (batch == 0 || (u_in && v_in && u_out && v_out)), "propagate_batch_host: null argument");
    if (batch == 0) return;
    ptb_context* ctx = p->ctx;
    DeviceGuard g(ctx->device);
    std::lock_guard<std::recursive_mutex> lock(ctx->mutex);
    const size_t n = p->n, slice_bytes = n * sizeof(double);
    const size_t target = size_t(128) << 20;  // ~128 MiB of u per chunk
    size_t chunk = std::max<size_t>(1, target / slice_bytes);
    if (batch > 1) chunk = std::min(chunk, (batch + 2) / 3);  // at least three chunks to overlap
    for (auto& st : ctx->aux)
      if (!st) PTB_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    if (flags_host && ctx->pinned_flags_n < batch) {
      if (ctx->pinned_flags) cudaFreeHost(ctx->pinned_flags);
      ctx->pinned_flags = nullptr;
      ctx->pinned_flags_n = 0;
      PTB_CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&ctx->pinned_flags), batch * sizeof(int32_t),
                                   cudaHostAllocDefault));
      ctx->pinned_flags_n = batch;
    }
    for (size_t b0 = 0, c = 0; b0 < batch; b0 += chunk, ++c) {
      const size_t nb = std::min(chunk, batch - b0);
      const int k = int(c % 3);
      cudaStream_t st = ctx->aux[k];
      auto& sb = ctx->slotbuf[k];
      double* du = static_cast<double*>(sb[0].get(chunk * slice_bytes));
      double* dv = static_cast<double*>(sb[1].get(chunk * slice_bytes));
      LaunchSlot slot;
      slot.stream = st;
      slot.su = static_cast<double*>(sb[2].get(chunk * slice_bytes));
      slot.sv = static_cast<double*>(sb[3].get(chunk * slice_bytes));
      int32_t* df = static_cast<int32_t*>(sb[4].get(chunk * sizeof(int32_t)));
      PTB_CUDA_CHECK(cudaMemcpyAsync(du, u_in + b0 * n, nb * slice_bytes, cudaMemcpyHostToDevice, st));
      PTB_CUDA_CHECK(cudaMemcpyAsync(dv, v_in + b0 * n, nb * slice_bytes, cudaMemcpyHostToDevice, st));
      PTB_CUDA_CHECK(cudaMemsetAsync(df, 0, nb * sizeof(int32_t), st));
      propagate(p, p->steps, nb, du, dv, df, mode, &slot);
      PTB_CUDA_CHECK(cudaMemcpyAsync(u_out + b0 * n, du, nb * slice_bytes, cudaMemcpyDeviceToHost, st));
      PTB_CUDA_CHECK(cudaMemcpyAsync(v_out + b0 * n, dv, nb * slice_bytes, cudaMemcpyDeviceToHost, st));
      if (flags_host)
        PTB_CUDA_CHECK(
            cudaMemcpyAsync(ctx->pinned_flags + b0, df, nb * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    }
    for (auto& st : ctx->aux) PTB_CUDA_CHECK(cudaStreamSynchronize(st));
    if (flags_host) std::memcpy(flags_host, ctx->pinned_flags, batch * sizeof(int32_t));
  });
}

ptb_status ptb_laplacian_batch(ptb_context* ctx, const ptb_grid* grid, size_t batch, const double* f, double* out) {
  return guarded([&] {
    require(ctx && grid, "laplacian: null argument");
    validate_grid(*grid);
    DeviceGuard g(ctx->device);
    laplacian(ctx, *grid, batch, f, out);
  });
}

// GridTransfer (grid.cpp:100-119)
ptb_status ptb_transfer_create(ptb_context* ctx, const ptb_grid* coarse, const ptb_grid* fine, int kind,
                               ptb_transfer** out) {
  return guarded([&] {
    require(ctx && coarse && fine && out, "GridTransfer: null argument");
    validate_grid(*coarse);
    validate_grid(*fine);
    require(coarse->dim == fine->dim, "GridTransfer: dimension mismatch");
    require(kind == PTB_INTERP_FOURIER || kind == PTB_INTERP_LINEAR, "GridTransfer: unknown kind");
    auto* t = new ptb_transfer();
    t->ctx = ctx;
    t->coarse = *coarse;
    t->fine = *fine;
    t->kind = kind;
    for (int a = 0; a < coarse->dim; ++a) {
      const size_t nc = coarse->n[a], nf = fine->n[a];
      if (nf % nc != 0) {
        delete t;
        fail(PTB_INVALID_ARGUMENT, "GridTransfer: fine points must be an integer multiple of coarse points");
      }
      t->ratio[a] = nf / nc;
      const double ec = double(nc) * coarse->h[a], ef = double(nf) * fine->h[a];
      if (std::abs(ec - ef) > 1e-12 * std::max(ec, ef)) {
        delete t;
        fail(PTB_INVALID_ARGUMENT, "GridTransfer: coarse and fine extents differ; grids are not nested");
      }
    }
    DeviceGuard g(ctx->device);
    transfer_init(t);
    *out = t;
  });
}

ptb_status ptb_transfer_destroy(ptb_transfer* t) {
  return guarded([&] {
    if (!t) return;
    DeviceGuard g(t->ctx->device);
    if (t->wx) cudaFree(t->wx);
    if (t->wy) cudaFree(t->wy);
    transfer_release(t);
    t->nodes_half.release();
    delete t;
  });
}

ptb_status ptb_restrict_batch(ptb_transfer* t, size_t batch, const double* fine, double* coarse) {
  return guarded([&] {
    require(t, "restrict: null transfer");
    DeviceGuard g(t->ctx->device);
    restrict_fields(t, batch, fine, coarse);
  });
}

ptb_status ptb_interpolate_batch(ptb_transfer* t, size_t batch, const double* coarse, double* fine) {
  return guarded([&] {
    require(t, "interpolate: null transfer");
    DeviceGuard g(t->ctx->device);
    std::lock_guard<std::recursive_mutex> lock(t->ctx->mutex);
    interpolate_fields(t, batch, coarse, fine);
  });
}

ptb_status ptb_interpolate_add_batch(ptb_transfer* t, size_t batch, const double* coarse, const double* base,
                                     double* out) {
  return guarded([&] {
    require(t && (batch == 0 || (coarse && base && out)), "interpolate_add: null argument");
    DeviceGuard g(t->ctx->device);
    std::lock_guard<std::recursive_mutex> lock(t->ctx->mutex);
    DeviceBuffer& work = t->add_work;
    const size_t nf = grid_size(t->fine);
    double* w = static_cast<double*>(work.get(std::max<size_t>(1, std::min<size_t>(batch, 8)) * nf * sizeof(double)));
    for (size_t b0 = 0; b0 < batch; b0 += 8) {
      const size_t m = std::min<size_t>(8, batch - b0);
      interpolate_fields_add(t, m, coarse + b0 * grid_size(t->coarse), base + b0 * nf, out + b0 * nf, w);
    }
  });
}

ptb_status ptb_nonfinite_batch(ptb_context* ctx, size_t n, size_t batch, const double* f, int32_t* flags) {
  return guarded([&] {
    DeviceGuard g(ctx->device);
    nonfinite(ctx, n, batch, f, flags);
  });
}

}  // extern "C"

