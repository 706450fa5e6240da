// libgrace C-ABI implementation (include/grace.h): context, validation, device
// memory, the CUDA-graph step loop, errors.  Host code; the arithmetic of the
// path runs in step_kernels.cu and tensor_setup.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/grace.h"
#include "internal.h"

using namespace grace;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_OR(call)                                                                          \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess) return fail(GRACE_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

constexpr double kPI = 3.141592653589793;
constexpr double kMU0 = 4.0 * kPI * 1e-7;  // S:L46, reading Q21
constexpr int kChunk = 16;                 // steps per captured chunk graph

int padded(int n) {
  if (n == 1) return 1;
  int p = 1;
  while (p < 2 * n - 1) p <<= 1;
  return p;
}
long long round_up(long long v, long long m) { return (v + m - 1) / m * m; }
bool finite_pos(double v) { return std::isfinite(v) && v > 0.0; }

}  // namespace

struct grace_ctx {
  Geom g{};
  double dx, dy, dz, Ms, A, Ku, alpha, gamma0;
  double hext[3] = {0, 0, 0};
  long long steps = 0;
  long long nf_step = -1, nf_cell = -1;
  long long N = 0;
  int cur = 0;
  bool fused = false;
  float* M[2] = {nullptr, nullptr};
  float2* X1 = nullptr;
  float2* X2 = nullptr;
  float* KS = nullptr;
  float2* tw = nullptr;
  StepParams* prm = nullptr;
  unsigned long long* flag = nullptr;   // [0] step non-finite, [1] set_m zero cell
  double* red = nullptr;                // mavg partials + 3 outputs
  float* Hbuf = nullptr;
  size_t bytes = 0;
  cudaStream_t own = nullptr, stream = nullptr, cap = nullptr;
  cudaGraphExec_t g1[2] = {nullptr, nullptr}, gc[2] = {nullptr, nullptr};
  bool profiling = false;
  std::vector<double> kms;
  std::vector<long long> klaunch;
  std::vector<cudaEvent_t> ev;
  StepParams hprm{};

  int alloc(void** p, size_t b) {
    cudaError_t e = cudaMalloc(p, b);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(GRACE_ENOMEM, "device allocation of %zu bytes failed (context holds %zu): %s", b, bytes,
                  cudaGetErrorString(e));
    }
    bytes += b;
    return GRACE_OK;
  }

  void fill_params(double dt) {
    const double a2 = 1.0 + alpha * alpha;
    hprm.dt = (float)dt;
    hprm.c_prec = (float)(-gamma0 / a2);
    hprm.c_damp = (float)(-alpha * gamma0 / (a2 * Ms));
    for (int q = 0; q < 3; ++q) hprm.hext[q] = (float)hext[q];
    hprm.step = steps;
  }

  // One step M[c] -> M[1-c] on stream s (bump: advance the device step counter).
  // ev (optional): 2 * kernel_count events, recorded before/after each kernel.
  cudaError_t enqueue_step(int c, cudaStream_t s, cudaEvent_t* ev = nullptr) {
    cudaError_t e;
    int k = 0;
    auto rec = [&](int idx) {
      if (ev) cudaEventRecord(ev[idx], s);
    };
    const int nk = kernel_count(g);
    rec(2 * k);
    if ((e = launch_k1(g, M[c], X1, tw, prm, s)) != cudaSuccess) return e;
    rec(2 * k + 1);
    ++k;
    if (fused) {
      rec(2 * k);
      if ((e = launch_k2f(g, X1, KS, tw, s)) != cudaSuccess) return e;
      rec(2 * k + 1);
      ++k;
    } else {
      rec(2 * k);
      if ((e = launch_k2(g, X1, X2, tw, s)) != cudaSuccess) return e;
      rec(2 * k + 1);
      ++k;
      rec(2 * k);
      if ((e = launch_k3(g, X2, KS, tw, s)) != cudaSuccess) return e;
      rec(2 * k + 1);
      ++k;
      rec(2 * k);
      if ((e = launch_k4(g, X2, X1, tw, s)) != cudaSuccess) return e;
      rec(2 * k + 1);
      ++k;
    }
    rec(2 * k);
    if ((e = launch_k5(g, 0, X1, M[c], M[1 - c], nullptr, tw, prm, flag, s)) != cudaSuccess) return e;
    rec(2 * k + 1);
    (void)nk;
    return cudaSuccess;
  }

  cudaError_t build_graph(int c, int nsteps, cudaGraphExec_t* out) {
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return e;
    for (int i = 0; i < nsteps; ++i) {
      e = enqueue_step((c + i) & 1, cap);
      if (e != cudaSuccess) break;
    }
    cudaError_t e2 = cudaStreamEndCapture(cap, &graph);
    if (e != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      return e;
    }
    if (e2 != cudaSuccess) return e2;
    e = cudaGraphInstantiate(out, graph, 0);
    cudaGraphDestroy(graph);
    return e;
  }

  void release() {
    for (int c = 0; c < 2; ++c) {
      if (g1[c]) cudaGraphExecDestroy(g1[c]);
      if (gc[c]) cudaGraphExecDestroy(gc[c]);
      if (M[c]) cudaFree(M[c]);
    }
    for (auto e : ev) cudaEventDestroy(e);
    void* ptrs[] = {X1, X2, KS, tw, prm, flag, red, Hbuf};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    if (own) cudaStreamDestroy(own);
    if (cap) cudaStreamDestroy(cap);
  }
};

extern "C" {

const char* grace_last_error(void) { return g_err.c_str(); }

int grace_create(int nx, int ny, int nz, double dx, double dy, double dz, double Ms, double A, double Ku, double alpha,
                 double gamma, grace_ctx** out) {
  g_err.clear();
  if (!out) return fail(GRACE_EINVAL, "out is NULL");
  *out = nullptr;
  if (nx < 1 || ny < 1 || nz < 1) return fail(GRACE_EINVAL, "cell counts must be >= 1 (got %d %d %d)", nx, ny, nz);
  if (!finite_pos(dx) || !finite_pos(dy) || !finite_pos(dz))
    return fail(GRACE_EINVAL, "cell sizes must be finite and > 0");
  if (!finite_pos(Ms)) return fail(GRACE_EINVAL, "Ms must be finite and > 0");
  if (!std::isfinite(A) || A < 0) return fail(GRACE_EINVAL, "A must be finite and >= 0");
  if (!std::isfinite(Ku) || Ku < 0) return fail(GRACE_EINVAL, "Ku must be finite and >= 0");
  if (!std::isfinite(alpha) || alpha < 0) return fail(GRACE_EINVAL, "alpha must be finite and >= 0");
  if (!finite_pos(gamma)) return fail(GRACE_EINVAL, "gamma must be finite and > 0");
  if (gamma > 1e9) return fail(GRACE_EINVAL, "pass gamma0 = gamma*mu0 in m/(A s) (e.g. 2.211e5), not gamma in rad/(s T)");
  const long long N = (long long)nx * ny * nz;
  if (N >= (1LL << 36)) return fail(GRACE_EUNSUPPORTED, "grid of %lld cells exceeds 2^36", N);
  Geom g{};
  g.nx = nx;
  g.ny = ny;
  g.nz = nz;
  g.Px = padded(nx);
  g.Py = padded(ny);
  g.Pz = padded(nz);
  if (g.Px > 8192 || g.Py > 4096 || g.Pz > 1024)
    return fail(GRACE_EUNSUPPORTED, "padded FFT %d x %d x %d exceeds the compiled maximum 8192 x 4096 x 1024", g.Px,
                g.Py, g.Pz);
  g.Kx = g.Px == 1 ? 1 : g.Px / 2 + 1;
  g.Kxp = (int)round_up(g.Kx, 16);
  g.Kyh = g.Py == 1 ? 1 : g.Py / 2 + 1;
  g.Kzh = g.Pz == 1 ? 1 : g.Pz / 2 + 1;
  g.KSp = (int)round_up(g.Kx, 32);
  g.Lmax = std::max(g.Px, std::max(g.Py, g.Pz));
  const double ex = 2.0 * A / (kMU0 * Ms * Ms);
  g.cx = nx > 1 ? (float)(ex / (dx * dx)) : 0.f;
  g.cy = ny > 1 ? (float)(ex / (dy * dy)) : 0.f;
  g.cz = nz > 1 ? (float)(ex / (dz * dz)) : 0.f;
  g.ck = (float)(2.0 * Ku / (kMU0 * Ms * Ms));
  g.Ms = (float)Ms;

  grace_ctx* h = new grace_ctx();
  h->g = g;
  h->dx = dx;
  h->dy = dy;
  h->dz = dz;
  h->Ms = Ms;
  h->A = A;
  h->Ku = Ku;
  h->alpha = alpha;
  h->gamma0 = gamma;
  h->N = N;
  h->fused = fused_y_path(g);
  int rc = GRACE_OK;
  auto bail = [&](int code) {
    h->release();
    delete h;
    return code;
  };
  {
    cudaError_t e = cudaStreamCreateWithFlags(&h->own, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking);
    if (e != cudaSuccess) return bail(fail(GRACE_ECUDA, "stream creation: %s", cudaGetErrorString(e)));
  }
  h->stream = h->own;
  const size_t mbytes = sizeof(float) * 3 * (size_t)N;
  const size_t x1 = sizeof(float2) * 3 * (size_t)nz * ny * g.Kxp;
  const size_t x2 = h->fused ? 0 : sizeof(float2) * 3 * (size_t)nz * g.Py * g.Kxp;
  const size_t ks = sizeof(float) * 6 * (size_t)g.Kzh * g.Kyh * g.KSp;
  if ((rc = h->alloc((void**)&h->M[0], mbytes)) || (rc = h->alloc((void**)&h->M[1], mbytes)) ||
      (rc = h->alloc((void**)&h->X1, x1)) || (x2 && (rc = h->alloc((void**)&h->X2, x2))) ||
      (rc = h->alloc((void**)&h->KS, ks)) || (rc = h->alloc((void**)&h->tw, sizeof(float2) * g.Lmax)) ||
      (rc = h->alloc((void**)&h->prm, sizeof(StepParams))) ||
      (rc = h->alloc((void**)&h->flag, 2 * sizeof(unsigned long long))) ||
      (rc = h->alloc((void**)&h->red, sizeof(double) * (kMavgPartials + 3))))
    return bail(rc);
  cudaStream_t s = h->stream;
  // setup: fp64 octant -> fp64 padded spectrum -> fp32 folded KS (S1..S5)
  double* oct = nullptr;
  double2* work = nullptr;
  const size_t octb = sizeof(double) * 6 * (size_t)N;
  const size_t workb = sizeof(double2) * (size_t)g.Px * g.Py * g.Pz;
  if (cudaMalloc(&oct, octb) != cudaSuccess || cudaMalloc(&work, workb) != cudaSuccess) {
    cudaGetLastError();
    if (oct) cudaFree(oct);
    return bail(fail(GRACE_ENOMEM, "setup needs %zu bytes of fp64 scratch", octb + workb));
  }
  cudaError_t e = tensor_octant_device(nx, ny, nz, dx, dy, dz, oct, s);
  if (e == cudaSuccess) e = kernel_spectrum_device(g, oct, work, h->KS, s);
  if (e == cudaSuccess) e = launch_twiddles(h->tw, g.Lmax, s);
  if (e == cudaSuccess) e = launch_fill_uniform_x(h->M[0], N, (float)Ms, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(h->flag, 0xff, 2 * sizeof(unsigned long long), s);
  if (e == cudaSuccess) {
    h->fill_params(1e-15);
    e = cudaMemcpyAsync(h->prm, &h->hprm, sizeof(StepParams), cudaMemcpyHostToDevice, s);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(oct);
  cudaFree(work);
  if (e != cudaSuccess) return bail(fail(GRACE_ECUDA, "tensor setup: %s", cudaGetErrorString(e)));
  // Dry run of one step (M[0] -> M[1], the spare buffer) so every kernel's
  // shared-memory attribute is set before any graph capture; then restore the
  // device step counter and flags.
  e = h->enqueue_step(0, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(h->flag, 0xff, 2 * sizeof(unsigned long long), s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h->prm, &h->hprm, sizeof(StepParams), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return bail(fail(GRACE_ECUDA, "first step: %s", cudaGetErrorString(e)));
  *out = h;
  return GRACE_OK;
}

void grace_destroy(grace_ctx* h) {
  if (!h) return;
  if (h->stream) cudaStreamSynchronize(h->stream);
  h->release();
  delete h;
}

int grace_set_stream(grace_ctx* h, void* stream) {
  if (!h) return fail(GRACE_EINVAL, "NULL context");
  CUDA_OR(cudaStreamSynchronize(h->stream));
  h->stream = stream ? (cudaStream_t)stream : h->own;
  return GRACE_OK;
}

static int finish_set_m(grace_ctx* h, int target) {
  unsigned long long f = kNoFlag;
  CUDA_OR(cudaMemcpyAsync(&f, h->flag + 1, sizeof f, cudaMemcpyDeviceToHost, h->stream));
  CUDA_OR(cudaStreamSynchronize(h->stream));
  if (f != kNoFlag) {
    CUDA_OR(cudaMemsetAsync(h->flag + 1, 0xff, sizeof f, h->stream));
    CUDA_OR(cudaStreamSynchronize(h->stream));
    return fail(GRACE_EZEROCELL, "cell %llu has |M| = 0 or a non-finite component", f);
  }
  h->cur = target;
  return GRACE_OK;
}

int grace_set_m(grace_ctx* h, const double* m) {
  if (!h || !m) return fail(GRACE_EINVAL, "NULL argument");
  // stage the fp64 input in X1 (>= 24 N bytes), normalise into the spare M buffer
  const int target = 1 - h->cur;
  double* stage = reinterpret_cast<double*>(h->X1);
  CUDA_OR(cudaMemcpyAsync(stage, m, sizeof(double) * 3 * (size_t)h->N, cudaMemcpyHostToDevice, h->stream));
  CUDA_OR(launch_set_m_f64(stage, h->M[target], h->N, h->Ms, h->flag + 1, h->stream));
  return finish_set_m(h, target);
}

int grace_set_m_device(grace_ctx* h, const float* d_m) {
  if (!h || !d_m) return fail(GRACE_EINVAL, "NULL argument");
  const int target = 1 - h->cur;
  CUDA_OR(launch_set_m_f32(d_m, h->M[target], h->N, (float)h->Ms, h->flag + 1, h->stream));
  return finish_set_m(h, target);
}

int grace_get_m(grace_ctx* h, double* out) {
  if (!h || !out) return fail(GRACE_EINVAL, "NULL argument");
  double* stage = reinterpret_cast<double*>(h->X1);
  CUDA_OR(launch_widen(h->M[h->cur], stage, 3 * h->N, h->stream));
  CUDA_OR(cudaMemcpyAsync(out, stage, sizeof(double) * 3 * (size_t)h->N, cudaMemcpyDeviceToHost, h->stream));
  CUDA_OR(cudaStreamSynchronize(h->stream));
  return GRACE_OK;
}

int grace_get_m_device(grace_ctx* h, float* d_out) {
  if (!h || !d_out) return fail(GRACE_EINVAL, "NULL argument");
  CUDA_OR(cudaMemcpyAsync(d_out, h->M[h->cur], sizeof(float) * 3 * (size_t)h->N, cudaMemcpyDeviceToDevice, h->stream));
  CUDA_OR(cudaStreamSynchronize(h->stream));
  return GRACE_OK;
}

int grace_set_hext(grace_ctx* h, double hx, double hy, double hz) {
  if (!h) return fail(GRACE_EINVAL, "NULL context");
  if (!std::isfinite(hx) || !std::isfinite(hy) || !std::isfinite(hz)) return fail(GRACE_EINVAL, "H_ext must be finite");
  h->hext[0] = hx;
  h->hext[1] = hy;
  h->hext[2] = hz;
  return GRACE_OK;
}

int grace_set_alpha(grace_ctx* h, double alpha) {
  if (!h) return fail(GRACE_EINVAL, "NULL context");
  if (!std::isfinite(alpha) || alpha < 0) return fail(GRACE_EINVAL, "alpha must be finite and >= 0");
  h->alpha = alpha;
  return GRACE_OK;
}

int grace_heff(grace_ctx* h, double* out) {
  if (!h || !out) return fail(GRACE_EINVAL, "NULL argument");
  const Geom& g = h->g;
  cudaStream_t s = h->stream;
  if (!h->Hbuf) {
    int rc = h->alloc((void**)&h->Hbuf, sizeof(float) * 3 * (size_t)h->N);
    if (rc) return rc;
  }
  h->fill_params(1e-15);
  CUDA_OR(cudaMemcpyAsync(h->prm, &h->hprm, sizeof(StepParams), cudaMemcpyHostToDevice, s));
  CUDA_OR(launch_k1(g, h->M[h->cur], h->X1, h->tw, nullptr, s));
  if (h->fused) {
    CUDA_OR(launch_k2f(g, h->X1, h->KS, h->tw, s));
  } else {
    CUDA_OR(launch_k2(g, h->X1, h->X2, h->tw, s));
    CUDA_OR(launch_k3(g, h->X2, h->KS, h->tw, s));
    CUDA_OR(launch_k4(g, h->X2, h->X1, h->tw, s));
  }
  CUDA_OR(launch_k5(g, 1, h->X1, h->M[h->cur], nullptr, h->Hbuf, h->tw, h->prm, h->flag, s));
  double* stage = reinterpret_cast<double*>(h->X1);
  CUDA_OR(launch_widen(h->Hbuf, stage, 3 * h->N, s));
  CUDA_OR(cudaMemcpyAsync(out, stage, sizeof(double) * 3 * (size_t)h->N, cudaMemcpyDeviceToHost, s));
  CUDA_OR(cudaStreamSynchronize(s));
  return GRACE_OK;
}

int grace_step(grace_ctx* h, int n, double dt) {
  if (!h) return fail(GRACE_EINVAL, "NULL context");
  if (n < 0) return fail(GRACE_EINVAL, "n must be >= 0");
  if (!finite_pos(dt)) return fail(GRACE_EINVAL, "dt must be finite and > 0");
  if (n == 0) return GRACE_OK;
  cudaStream_t s = h->stream;
  h->fill_params(dt);
  CUDA_OR(cudaMemcpyAsync(h->prm, &h->hprm, sizeof(StepParams), cudaMemcpyHostToDevice, s));
  const int nk = kernel_count(h->g);
  if (h->profiling) {
    // eager launches with an event pair around every kernel; events are read in
    // batches of kProfBatch steps so the host never waits inside a batch
    constexpr int kProfBatch = 64;
    if (h->ev.empty()) {
      h->ev.resize((size_t)2 * nk * kProfBatch);
      for (auto& e : h->ev) CUDA_OR(cudaEventCreate(&e));
      h->kms.assign(nk, 0.0);
      h->klaunch.assign(nk, 0);
    }
    for (int i0 = 0; i0 < n; i0 += kProfBatch) {
      const int nb = std::min(kProfBatch, n - i0);
      for (int i = 0; i < nb; ++i) {
        cudaError_t e = h->enqueue_step(h->cur, s, &h->ev[(size_t)2 * nk * i]);
        if (e != cudaSuccess) return fail(GRACE_ECUDA, "step launch: %s", cudaGetErrorString(e));
        h->cur ^= 1;
      }
      CUDA_OR(cudaEventSynchronize(h->ev[(size_t)2 * nk * nb - 1]));
      for (int i = 0; i < nb; ++i)
        for (int k = 0; k < nk; ++k) {
          float ms = 0.f;
          CUDA_OR(cudaEventElapsedTime(&ms, h->ev[(size_t)2 * nk * i + 2 * k], h->ev[(size_t)2 * nk * i + 2 * k + 1]));
          h->kms[k] += ms;
          h->klaunch[k] += 1;
        }
    }
  } else {
    int left = n;
    while (left > 0) {
      const bool chunk = left >= kChunk;
      cudaGraphExec_t* gx = chunk ? &h->gc[h->cur] : &h->g1[h->cur];
      if (!*gx) {
        cudaError_t e = h->build_graph(h->cur, chunk ? kChunk : 1, gx);
        if (e != cudaSuccess) return fail(GRACE_ECUDA, "graph capture: %s", cudaGetErrorString(e));
      }
      CUDA_OR(cudaGraphLaunch(*gx, s));
      const int done = chunk ? kChunk : 1;
      left -= done;
      h->cur ^= (done & 1);
    }
  }
  unsigned long long f = kNoFlag;
  CUDA_OR(cudaMemcpyAsync(&f, h->flag, sizeof f, cudaMemcpyDeviceToHost, s));
  CUDA_OR(cudaStreamSynchronize(s));
  h->steps += n;
  if (f != kNoFlag) {
    h->nf_step = (long long)(f >> 36);
    h->nf_cell = (long long)(f & ((1ULL << 36) - 1));
    CUDA_OR(cudaMemsetAsync(h->flag, 0xff, sizeof f, s));
    CUDA_OR(cudaStreamSynchronize(s));
    return fail(GRACE_ENONFINITE, "non-finite magnetisation at step %lld, cell %lld (dt too large?)", h->nf_step,
                h->nf_cell);
  }
  return GRACE_OK;
}

int grace_mavg(grace_ctx* h, double* out3) {
  if (!h || !out3) return fail(GRACE_EINVAL, "NULL argument");
  CUDA_OR(launch_mavg(h->M[h->cur], h->N, h->Ms, h->red, h->red + kMavgPartials, h->stream));
  CUDA_OR(cudaMemcpyAsync(out3, h->red + kMavgPartials, 3 * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CUDA_OR(cudaStreamSynchronize(h->stream));
  return GRACE_OK;
}

int grace_step_count(grace_ctx* h, long long* steps) {
  if (!h || !steps) return fail(GRACE_EINVAL, "NULL argument");
  *steps = h->steps;
  return GRACE_OK;
}

int grace_last_nonfinite(grace_ctx* h, long long* step, long long* cell) {
  if (!h || !step || !cell) return fail(GRACE_EINVAL, "NULL argument");
  *step = h->nf_step;
  *cell = h->nf_cell;
  return GRACE_OK;
}

int grace_geometry(grace_ctx* h, long long* o) {
  if (!h || !o) return fail(GRACE_EINVAL, "NULL argument");
  const Geom& g = h->g;
  const long long v[12] = {g.nx, g.ny, g.nz, g.Px, g.Py, g.Pz, g.Kx, g.Kxp, g.Kyh, g.Kzh, g.KSp, kernel_count(g)};
  std::memcpy(o, v, sizeof v);
  return GRACE_OK;
}

int grace_device_bytes(grace_ctx* h, size_t* bytes) {
  if (!h || !bytes) return fail(GRACE_EINVAL, "NULL argument");
  *bytes = h->bytes;
  return GRACE_OK;
}

int grace_tensor_octant(int nx, int ny, int nz, double dx, double dy, double dz, double* out) {
  if (!out) return fail(GRACE_EINVAL, "NULL argument");
  if (nx < 1 || ny < 1 || nz < 1) return fail(GRACE_EINVAL, "cell counts must be >= 1");
  if (!finite_pos(dx) || !finite_pos(dy) || !finite_pos(dz)) return fail(GRACE_EINVAL, "cell sizes must be > 0");
  const size_t b = sizeof(double) * 6 * (size_t)nx * ny * nz;
  double* d = nullptr;
  if (cudaMalloc(&d, b) != cudaSuccess) {
    cudaGetLastError();
    return fail(GRACE_ENOMEM, "needs %zu bytes", b);
  }
  cudaError_t e = tensor_octant_device(nx, ny, nz, dx, dy, dz, d, 0);
  if (e == cudaSuccess) e = cudaMemcpy(out, d, b, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(GRACE_ECUDA, "tensor octant: %s", cudaGetErrorString(e));
  return GRACE_OK;
}

int grace_kernel_spectrum(grace_ctx* h, float* out) {
  if (!h || !out) return fail(GRACE_EINVAL, "NULL argument");
  const Geom& g = h->g;
  CUDA_OR(cudaMemcpyAsync(out, h->KS, sizeof(float) * 6 * (size_t)g.Kzh * g.Kyh * g.KSp, cudaMemcpyDeviceToHost,
                          h->stream));
  CUDA_OR(cudaStreamSynchronize(h->stream));
  return GRACE_OK;
}

int grace_set_profiling(grace_ctx* h, int on) {
  if (!h) return fail(GRACE_EINVAL, "NULL context");
  h->profiling = on != 0;
  return GRACE_OK;
}

int grace_kernel_times(grace_ctx* h, double* ms, long long* launches, int* nk, int reset) {
  if (!h || !nk) return fail(GRACE_EINVAL, "NULL argument");
  const int k = kernel_count(h->g);
  const int cap = *nk;
  *nk = k;
  for (int i = 0; i < k && i < cap; ++i) {
    if (ms) ms[i] = h->kms.empty() ? 0.0 : h->kms[i];
    if (launches) launches[i] = h->klaunch.empty() ? 0 : h->klaunch[i];
  }
  if (reset && !h->kms.empty()) {
    std::fill(h->kms.begin(), h->kms.end(), 0.0);
    std::fill(h->klaunch.begin(), h->klaunch.end(), 0);
  }
  return GRACE_OK;
}

}  // extern "C"
