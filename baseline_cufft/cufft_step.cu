// cuFFT comparison baseline of the LLG step (BASELINE.json north_star: "cuFFT is
// timed only as a comparison baseline").  NOT part of libgrace:
// a separate shared library, used only by bench_cufft.py and its GPU test.
//
// The naive library pipeline the hand-written path replaces (the
// paper called its vendor's FFT library):
//   pad      M [3][nz][ny][nx]          -> Mp [3][Pz][Py][Px] (zeros outside)
//   R2C      cufftExecR2C, batch 3       -> Mh [3][Pz][Py][Px/2+1]
//   multiply Hh_a = sum_b Nh_ab Mh_b     (full complex spectrum of the 6 tensor components)
//   C2R      cufftExecC2R, batch 3       -> Hp [3][Pz][Py][Px]
//   LLG      unpad H_demag (1/P folded into Nh) + exchange + anisotropy + Zeeman,
//            Eq. (3), Euler, renormalise (the same arithmetic as libgrace's K6)
// The tensor spectrum comes from libgrace's fp64 real-space octant (setup, not
// timed), embedded circulant and transformed by cufftExecD2Z once.
#include <cuda_runtime.h>
#include <cufft.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

extern "C" int grace_tensor_octant(int nx, int ny, int nz, double dx, double dy, double dz, double* out);

namespace {

constexpr double kPI = 3.141592653589793;
constexpr double kMU0 = 4.0 * kPI * 1e-7;

int padded(int n) {
  if (n == 1) return 1;
  int p = 1;
  while (p < 2 * n - 1) p <<= 1;
  return p;
}

struct Dims {
  int nx, ny, nz, Px, Py, Pz, Kx;
  long long N, P, Ph;  // cells, padded points, half-spectrum points
};

__global__ void k_pad(const float* __restrict__ M, float* __restrict__ Mp, Dims d) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= 3 * d.P) return;
  const int c = (int)(i / d.P);
  const long long p = i - c * d.P;
  const int px = (int)(p % d.Px), py = (int)((p / d.Px) % d.Py), pz = (int)(p / ((long long)d.Px * d.Py));
  float v = 0.f;
  if (px < d.nx && py < d.ny && pz < d.nz) v = M[c * d.N + ((long long)pz * d.ny + py) * d.nx + px];
  Mp[i] = v;
}

// Hh_a = sum_b Nh_ab Mh_b; Nh [6][Ph] complex (xx xy xz yy yz zz), already -1/P scaled
__global__ void k_mul(const cufftComplex* __restrict__ Nh, cufftComplex* __restrict__ Xh, long long Ph) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= Ph) return;
  const cufftComplex mx = Xh[k], my = Xh[Ph + k], mz = Xh[2 * Ph + k];
  cufftComplex n[6];
  for (int q = 0; q < 6; ++q) n[q] = Nh[q * Ph + k];
  auto mac = [](cufftComplex a, cufftComplex b, cufftComplex c, cufftComplex x, cufftComplex y, cufftComplex z) {
    cufftComplex r;
    r.x = a.x * x.x - a.y * x.y + b.x * y.x - b.y * y.y + c.x * z.x - c.y * z.y;
    r.y = a.x * x.y + a.y * x.x + b.x * y.y + b.y * y.x + c.x * z.y + c.y * z.x;
    return r;
  };
  Xh[k] = mac(n[0], n[1], n[2], mx, my, mz);
  Xh[Ph + k] = mac(n[1], n[3], n[4], mx, my, mz);
  Xh[2 * Ph + k] = mac(n[2], n[4], n[5], mx, my, mz);
}

struct Mat {
  float cx, cy, cz, ck, Ms, dt, cprec, cdamp, hx, hy, hz;
};

// one thread per cell: H_eff = H_demag (unpadded) + exchange (Neumann) + x anisotropy
// + Zeeman; Eq. (3); Euler; renormalise.  mode 1 stores H_demag only (parity test).
__global__ void k_llg(const float* __restrict__ Hp, const float* __restrict__ M, float* __restrict__ Mn, Dims d,
                      Mat m, int mode) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= d.N) return;
  const int x = (int)(i % d.nx), y = (int)((i / d.nx) % d.ny), z = (int)(i / ((long long)d.nx * d.ny));
  const long long p = ((long long)z * d.Py + y) * d.Px + x;
  float h[3], a[3];
  for (int c = 0; c < 3; ++c) {
    h[c] = Hp[c * d.P + p];
    a[c] = M[c * d.N + i];
  }
  if (mode == 1) {
    for (int c = 0; c < 3; ++c) Mn[c * d.N + i] = h[c];
    return;
  }
  const long long sx = 1, sy = d.nx, sz = (long long)d.nx * d.ny;
  for (int c = 0; c < 3; ++c) {
    const float* mc = M + c * d.N;
    float e = 0.f;
    e += m.cx * ((x > 0 ? mc[i - sx] : a[c]) - a[c]);
    e += m.cx * ((x + 1 < d.nx ? mc[i + sx] : a[c]) - a[c]);
    e += m.cy * ((y > 0 ? mc[i - sy] : a[c]) - a[c]);
    e += m.cy * ((y + 1 < d.ny ? mc[i + sy] : a[c]) - a[c]);
    e += m.cz * ((z > 0 ? mc[i - sz] : a[c]) - a[c]);
    e += m.cz * ((z + 1 < d.nz ? mc[i + sz] : a[c]) - a[c]);
    h[c] += e;
  }
  h[0] += m.hx + m.ck * a[0];
  h[1] += m.hy;
  h[2] += m.hz;
  const float mx = a[0], my = a[1], mz = a[2];
  const float ax = my * h[2] - mz * h[1], ay = mz * h[0] - mx * h[2], az = mx * h[1] - my * h[0];
  const float bx = my * az - mz * ay, by = mz * ax - mx * az, bz = mx * ay - my * ax;
  const float s0 = mx + m.dt * (m.cprec * ax + m.cdamp * bx);
  const float s1 = my + m.dt * (m.cprec * ay + m.cdamp * by);
  const float s2 = mz + m.dt * (m.cprec * az + m.cdamp * bz);
  const float sc = m.Ms / sqrtf(s0 * s0 + s1 * s1 + s2 * s2);
  Mn[i] = s0 * sc;
  Mn[d.N + i] = s1 * sc;
  Mn[2 * d.N + i] = s2 * sc;
}

// circulant embedding of octant component c (parity signs of the odd components)
__global__ void k_embed64(double* A, const double* oct, int c, Dims d) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= d.P) return;
  const int px = (int)(i % d.Px), py = (int)((i / d.Px) % d.Py), pz = (int)(i / ((long long)d.Px * d.Py));
  auto circ = [](int p, int P, int n, int& s) {
    if (p < n) { s = 1; return p; }
    if (P - p < n) { s = -1; return P - p; }
    return -1;
  };
  int sx, sy, sz;
  const int ix = circ(px, d.Px, d.nx, sx), iy = circ(py, d.Py, d.ny, sy), iz = circ(pz, d.Pz, d.nz, sz);
  double v = 0.0;
  if (ix >= 0 && iy >= 0 && iz >= 0) {
    v = oct[(long long)c * d.N + ((long long)iz * d.ny + iy) * d.nx + ix];
    int s = 1;
    if (c == 1) s = sx * sy;
    else if (c == 2) s = sx * sz;
    else if (c == 4) s = sy * sz;
    if (s < 0) v = -v;
  }
  A[i] = v;
}

__global__ void k_scale_to_c64(const cufftDoubleComplex* A, cufftComplex* Nh, long long Ph, double s) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= Ph) return;
  Nh[k].x = (float)(A[k].x * s);
  Nh[k].y = (float)(A[k].y * s);
}

unsigned grid_of(long long n) { return (unsigned)((n + 255) / 256); }

}  // namespace

extern "C" {

// Runs `warmup` + `steps` Euler steps of the cuFFT pipeline from M0 (host, fp32
// SoA [3][nz][ny][nx], |M| = Ms) and reports the device time per step (CUDA
// events around the timed steps), the final M (host, optional) and, if
// hd_out != NULL, H_demag of M0 (host fp32 SoA) before stepping.
// Returns 0, or a negative code (1-line message in err[256]).
int cufft_baseline_run(int nx, int ny, int nz, double dx, double dy, double dz, double Ms, double A, double Ku,
                       double alpha, double gamma0, const double* hext, double dt, const float* M0, int warmup,
                       int steps, double* ms_per_step, float* m_out, float* hd_out, char* err) {
  Dims d{};
  d.nx = nx; d.ny = ny; d.nz = nz;
  d.Px = padded(nx); d.Py = padded(ny); d.Pz = padded(nz);
  d.Kx = d.Px / 2 + 1;
  d.N = (long long)nx * ny * nz;
  d.P = (long long)d.Px * d.Py * d.Pz;
  d.Ph = (long long)d.Kx * d.Py * d.Pz;
  if (3 * d.P > 0x7fffffffLL) {
    snprintf(err, 256, "grid too large for the 32-bit cuFFT batch strides used here");
    return -4;
  }
  auto fail = [&](const char* what) {
    snprintf(err, 256, "%s: %s", what, cudaGetErrorString(cudaGetLastError()));
    return -1;
  };
  // ---- setup (untimed): tensor spectrum Nh [6][Ph] complex64 = -FFT(N)/P
  std::vector<double> oct(6 * (size_t)d.N);
  if (grace_tensor_octant(nx, ny, nz, dx, dy, dz, oct.data()) != 0) {
    snprintf(err, 256, "grace_tensor_octant failed");
    return -2;
  }
  double *doct = nullptr, *A64 = nullptr;
  cufftDoubleComplex* A64h = nullptr;
  cufftComplex *Nh = nullptr, *Xh = nullptr;
  float *Mp = nullptr, *M = nullptr, *Mn = nullptr;
  if (cudaMalloc(&doct, 8 * oct.size()) || cudaMalloc(&A64, 8 * d.P) || cudaMalloc(&A64h, 16 * d.Ph) ||
      cudaMalloc(&Nh, 8 * 6 * d.Ph))
    return fail("setup alloc");
  cudaMemcpy(doct, oct.data(), 8 * oct.size(), cudaMemcpyHostToDevice);
  cufftHandle p64;
  // transform rank: singleton padded axes (Pz = 1, then Py = 1) are dropped
  int n3[3] = {d.Pz, d.Py, d.Px};
  int rank = 3, off = 0;
  while (rank > 1 && n3[off] == 1) {
    ++off;
    --rank;
  }
  int* nn = n3 + off;
  if (cufftPlanMany(&p64, rank, nn, nullptr, 1, 0, nullptr, 1, 0, CUFFT_D2Z, 1) != CUFFT_SUCCESS) {
    snprintf(err, 256, "cufftPlanMany D2Z failed");
    return -3;
  }
  for (int c = 0; c < 6; ++c) {
    k_embed64<<<grid_of(d.P), 256>>>(A64, doct, c, d);
    cufftExecD2Z(p64, A64, A64h);
    k_scale_to_c64<<<grid_of(d.Ph), 256>>>(A64h, Nh + c * d.Ph, d.Ph, -1.0 / (double)d.P);
  }
  cufftDestroy(p64);
  cudaFree(doct);
  cudaFree(A64);
  cudaFree(A64h);
  if (cudaDeviceSynchronize() != cudaSuccess) return fail("setup");
  // ---- per-step buffers and plans
  if (cudaMalloc(&Mp, 4 * 3 * d.P) || cudaMalloc(&Xh, 8 * 3 * d.Ph) || cudaMalloc(&M, 4 * 3 * d.N) ||
      cudaMalloc(&Mn, 4 * 3 * d.N))
    return fail("step alloc");
  cudaMemcpy(M, M0, 4 * 3 * d.N, cudaMemcpyHostToDevice);
  cufftHandle fwd, inv;
  if (cufftPlanMany(&fwd, rank, nn, nullptr, 1, (int)d.P, nullptr, 1, (int)d.Ph, CUFFT_R2C, 3) != CUFFT_SUCCESS ||
      cufftPlanMany(&inv, rank, nn, nullptr, 1, (int)d.Ph, nullptr, 1, (int)d.P, CUFFT_C2R, 3) != CUFFT_SUCCESS) {
    snprintf(err, 256, "cufftPlanMany R2C/C2R failed");
    return -3;
  }
  const double ex = 2.0 * A / (kMU0 * Ms * Ms);
  const double a2 = 1.0 + alpha * alpha;
  Mat mat{nx > 1 ? (float)(ex / (dx * dx)) : 0.f, ny > 1 ? (float)(ex / (dy * dy)) : 0.f,
          nz > 1 ? (float)(ex / (dz * dz)) : 0.f, (float)(2.0 * Ku / (kMU0 * Ms * Ms)), (float)Ms, (float)dt,
          (float)(-gamma0 / a2), (float)(-alpha * gamma0 / (a2 * Ms)), (float)hext[0], (float)hext[1],
          (float)hext[2]};
  auto demag = [&](const float* Min) {
    k_pad<<<grid_of(3 * d.P), 256>>>(Min, Mp, d);
    cufftExecR2C(fwd, Mp, Xh);
    k_mul<<<grid_of(d.Ph), 256>>>(Nh, Xh, d.Ph);
    cufftExecC2R(inv, Xh, Mp);
  };
  if (hd_out) {
    demag(M);
    k_llg<<<grid_of(d.N), 256>>>(Mp, M, Mn, d, mat, 1);
    cudaMemcpy(hd_out, Mn, 4 * 3 * d.N, cudaMemcpyDeviceToHost);
  }
  auto step = [&]() {
    demag(M);
    k_llg<<<grid_of(d.N), 256>>>(Mp, M, Mn, d, mat, 0);
    std::swap(M, Mn);
  };
  for (int i = 0; i < warmup; ++i) step();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int i = 0; i < steps; ++i) step();
  cudaEventRecord(e1);
  if (cudaEventSynchronize(e1) != cudaSuccess) return fail("steps");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  *ms_per_step = steps > 0 ? ms / steps : 0.0;
  if (m_out) cudaMemcpy(m_out, M, 4 * 3 * d.N, cudaMemcpyDeviceToHost);
  cufftDestroy(fwd);
  cufftDestroy(inv);
  cudaFree(Mp);
  cudaFree(Xh);
  cudaFree(M);
  cudaFree(Mn);
  cudaFree(Nh);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // extern "C"
