// Demag-tensor setup (fp64, once per grace_create): SURVEY §8(a) row a0, S1..S5.
//
// The paper: H_demag is "the convolution of magnetizations and demagnetization
// tensor" whose formula it defers to refs [3],[11].  Readings
// (DESIGN.md §3): Q5 Newell's cell-averaged tensor; Q6 point dipole beyond 30
// cell diagonals; Q7 exact zeros and parity; Q8 a fixed fp64 evaluation order and
// correctly rounded log/atan so the real-space octant is bit-identical to the
// independent CPU oracle (BASELINE.json: "the demag-tensor setup is bit-exact
// between CPU and GPU in fp64").
//
// This file MUST be compiled with -fmad=false: every a*b+c below is two IEEE
// roundings, exactly as the oracle's Python evaluates it.  FMA appears only where
// written explicitly (__fma_rn in the double-double error-free product).
//
//   S1  k_nodes    : Newell f / g at the integer node lattice of each component
//   S2  k_octant   : 27-point second differences (near) or dipole (far), exact zeros
//   S3  k_embed    : circulant embedding of one component in the padded grid (parity signs)
//   S4  k_fft64    : fp64 complex FFT lines along x, y, z
//   S5  k_fold     : KS = -Re / (Px Py Pz) on the folded octant, rounded to fp32
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "internal.h"

namespace grace {
namespace {

constexpr double kPI = 3.141592653589793;

// ---------------------------------------------------------------------------
// double-double arithmetic (error-free transforms)
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  const double e = (a - (s - bb)) + (b - bb);
  return {s, e};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
  const double s = a + b;
  return {s, b - (s - a)};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
  const double p = a * b;
  return {p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  dd t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo;
  p.lo += a.lo * b.hi;
  return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
  dd p = two_prod(a.hi, b);
  p.lo += a.lo * b;
  return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_div(dd a, dd b) {
  const double q1 = a.hi / b.hi;
  dd r = dd_add(a, dd_neg(dd_mul_d(b, q1)));
  const double q2 = r.hi / b.hi;
  r = dd_add(r, dd_neg(dd_mul_d(b, q2)));
  const double q3 = r.hi / b.hi;
  dd q = quick_two_sum(q1, q2);
  return dd_add(q, dd{q3, 0.0});
}
__device__ __forceinline__ dd dd_sqrt(dd a) {
  const double x = sqrt(a.hi);
  const dd x2 = two_prod(x, x);
  const dd r = dd_add(a, dd_neg(x2));
  const double corr = r.hi / (2.0 * x);
  return quick_two_sum(x, corr);
}

// Correctly rounded log: x = m 2^e, m in [1/sqrt2, sqrt2), log m = 2 atanh((m-1)/(m+1))
// summed in double-double (~2^-104 relative), rounded once to double.
__device__ double cr_log(double x) {
  int e;
  double m = frexp(x, &e);  // m in [0.5, 1)
  if (m < 0.70710678118654752) {
    m = m * 2.0;
    e -= 1;
  }
  const dd num{m - 1.0, 0.0};  // exact (Sterbenz)
  const dd den = two_sum(m, 1.0);
  const dd s = dd_div(num, den);
  const dd s2 = dd_mul(s, s);
  dd t{0.0, 0.0};
  for (int k = 28; k >= 0; --k) t = dd_add(dd_div(dd{1.0, 0.0}, dd{2.0 * k + 1.0, 0.0}), dd_mul(s2, t));
  const dd logm = dd_mul_d(dd_mul(s, t), 2.0);
  const dd ln2{0.6931471805599453, 2.3190468138462996e-17};
  const dd r = dd_add(dd_mul_d(ln2, (double)e), logm);
  return r.hi;
}

// Correctly rounded atan: reduce to [0,1] by 1/x, halve the angle three times
// (t <- t/(1+sqrt(1+t^2))), Taylor series in double-double, rounded once.
__device__ double cr_atan(double x) {
  if (x == 0.0) return x;
  const bool neg = x < 0.0;
  double ax = fabs(x);
  const bool inv = ax > 1.0;
  dd t = inv ? dd_div(dd{1.0, 0.0}, dd{ax, 0.0}) : dd{ax, 0.0};
  for (int h = 0; h < 3; ++h) {
    const dd r = dd_sqrt(dd_add(dd{1.0, 0.0}, dd_mul(t, t)));
    t = dd_div(t, dd_add(dd{1.0, 0.0}, r));
  }
  const dd t2 = dd_mul(t, t);
  dd u{0.0, 0.0};
  for (int k = 22; k >= 0; --k) {
    const dd c = dd_div(dd{(k & 1) ? -1.0 : 1.0, 0.0}, dd{2.0 * k + 1.0, 0.0});
    u = dd_add(c, dd_mul(t2, u));
  }
  dd a = dd_mul_d(dd_mul(t, u), 8.0);
  if (inv) a = dd_add(dd{1.5707963267948966, 6.123233995736766e-17}, dd_neg(a));
  return neg ? -a.hi : a.hi;
}

// ---------------------------------------------------------------------------
// Newell f and g (reading Q8 pseudo-code; x, y, z >= 0; g's sign applied by the caller).
__device__ double newell_f(double x, double y, double z) {
  const double x2 = x * x;
  const double y2 = y * y;
  const double z2 = z * z;
  const double R = sqrt((x2 + y2) + z2);
  double t = 0.0;
  if (y > 0.0 && (x2 + z2) > 0.0) t = t + ((0.5 * y) * (z2 - x2)) * cr_log((y + R) / sqrt(x2 + z2));
  if (z > 0.0 && (x2 + y2) > 0.0) t = t + ((0.5 * z) * (y2 - x2)) * cr_log((z + R) / sqrt(x2 + y2));
  if (x > 0.0 && y > 0.0 && z > 0.0) t = t - ((x * y) * z) * cr_atan((y * z) / (x * R));
  t = t + ((((2.0 * x2) - y2) - z2) * R) / 6.0;
  return t;
}

__device__ double newell_g(double x, double y, double z) {
  const double x2 = x * x;
  const double y2 = y * y;
  const double z2 = z * z;
  const double R = sqrt((x2 + y2) + z2);
  double t = 0.0;
  if (x > 0.0 && y > 0.0 && z > 0.0) t = t + ((x * y) * z) * cr_log((z + R) / sqrt(x2 + y2));
  if (x > 0.0 && (y2 + z2) > 0.0) t = t + ((y / 6.0) * ((3.0 * z2) - y2)) * cr_log((x + R) / sqrt(y2 + z2));
  if (y > 0.0 && (x2 + z2) > 0.0) t = t + ((x / 6.0) * ((3.0 * z2) - x2)) * cr_log((y + R) / sqrt(x2 + z2));
  if (x > 0.0 && y > 0.0 && z > 0.0) {
    t = t - ((z2 * z) / 6.0) * cr_atan((x * y) / (z * R));
    t = t - ((z * y2) / 2.0) * cr_atan((x * z) / (y * R));
    t = t - ((z * x2) / 2.0) * cr_atan((y * z) / (x * R));
  }
  t = t - ((x * y) * R) / 3.0;
  return t;
}

// Component c: 0 xx f(X,Y,Z), 1 xy g(X,Y,Z), 2 xz g(X,Z,Y), 3 yy f(Y,X,Z), 4 yz g(Y,Z,X), 5 zz f(Z,Y,X).
__device__ double node_value(int c, int I, int J, int K, double dx, double dy, double dz) {
  const double X = (double)I * dx, Y = (double)J * dy, Z = (double)K * dz;
  switch (c) {
    case 0: return newell_f(X, Y, Z);
    case 1: return newell_g(X, Y, Z);
    case 2: return newell_g(X, Z, Y);
    case 3: return newell_f(Y, X, Z);
    case 4: return newell_g(Y, Z, X);
    default: return newell_f(Z, Y, X);
  }
}

// S1: lat[c][K][J][I] for the node box [0,LI) x [0,LJ) x [0,LK).
__global__ void k_nodes(double* lat, int LI, int LJ, int LK, double dx, double dy, double dz) {
  const long long per = (long long)LI * LJ * LK;
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= 6 * per) return;
  const int c = (int)(idx / per);
  long long r = idx - c * per;
  const int K = (int)(r / ((long long)LI * LJ));
  r -= (long long)K * LI * LJ;
  const int J = (int)(r / LI);
  const int I = (int)(r - (long long)J * LI);
  lat[idx] = node_value(c, I, J, K, dx, dy, dz);
}

__device__ __forceinline__ double sgn(int v) { return (double)((v > 0) - (v < 0)); }

// S2: one octant entry per thread.
// Components c0 .. c0 + nc - 1 into oct[(c - c0) * N + ...].
__global__ void k_octant(double* oct, const double* lat, int LI, int LJ, int LK, int nx, int ny, int nz, double dx,
                         double dy, double dz, int c0, int nc) {
  const long long N = (long long)nx * ny * nz;
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= nc * N) return;
  const int c = c0 + (int)(idx / N);
  long long r = idx - (c - c0) * N;
  const int k = (int)(r / ((long long)nx * ny));
  r -= (long long)k * nx * ny;
  const int j = (int)(r / nx);
  const int i = (int)(r - (long long)j * nx);
  // exact zeros of the odd components (reading Q7)
  if ((c == 1 && (i == 0 || j == 0)) || (c == 2 && (i == 0 || k == 0)) || (c == 4 && (j == 0 || k == 0))) {
    oct[idx] = 0.0;
    return;
  }
  const double X = (double)i * dx, Y = (double)j * dy, Z = (double)k * dz;
  const double r2 = (X * X + Y * Y) + Z * Z;
  const double diag2 = (dx * dx + dy * dy) + dz * dz;
  double v;
  if (r2 <= (30.0 * 30.0) * diag2) {
    const double w3[3] = {-1.0, 2.0, -1.0};
    const double* L = lat + (long long)c * LI * LJ * LK;
    double s = 0.0;
    for (int a = -1; a <= 1; ++a)
      for (int b = -1; b <= 1; ++b)
        for (int cc = -1; cc <= 1; ++cc) {
          const double w = (w3[a + 1] * w3[b + 1]) * w3[cc + 1];
          const int I = abs(i + a), J = abs(j + b), K = abs(k + cc);
          double F = L[((long long)K * LJ + J) * LI + I];
          if (c == 1) F = (sgn(i + a) * sgn(j + b)) * F;
          else if (c == 2) F = (sgn(i + a) * sgn(k + cc)) * F;
          else if (c == 4) F = (sgn(j + b) * sgn(k + cc)) * F;
          s = s + w * F;
        }
    const double inv = 1.0 / ((((4.0 * kPI) * dx) * dy) * dz);
    v = s * inv;
  } else {
    const double rr = sqrt(r2);
    const double r5 = (r2 * r2) * rr;
    const double V = (dx * dy) * dz;
    const double cpre = V / (4.0 * kPI);
    switch (c) {
      case 0: v = -((cpre * ((3.0 * (X * X)) - r2)) / r5); break;
      case 1: v = -((cpre * (3.0 * (X * Y))) / r5); break;
      case 2: v = -((cpre * (3.0 * (X * Z))) / r5); break;
      case 3: v = -((cpre * ((3.0 * (Y * Y)) - r2)) / r5); break;
      case 4: v = -((cpre * (3.0 * (Y * Z))) / r5); break;
      default: v = -((cpre * ((3.0 * (Z * Z)) - r2)) / r5); break;
    }
  }
  oct[idx] = (v == 0.0) ? 0.0 : v;
}

// ---------------------------------------------------------------------------
// S3: circulant embedding of component c: A[p] = sign * N_c(|d|) with d = p (p < n)
// or d = p - P (P - p < n), zeros in the gap (P >= 2n-1, reading Q9).
__device__ __forceinline__ int circ_index(int p, int P, int n, int& s) {
  if (p < n) {
    s = 1;
    return p;
  }
  if (P - p < n) {
    s = -1;
    return P - p;
  }
  return -1;
}
// Padded planes pz0 .. pz0 + npz - 1 into A [npz][Py][Px].
__global__ void k_embed(double2* A, const double* oct_c, int c, int nx, int ny, int nz, int Px, int Py, int Pz,
                        int pz0, int npz) {
  const long long tot = (long long)Px * Py * npz;
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= tot) return;
  const int px = (int)(idx % Px);
  const int py = (int)((idx / Px) % Py);
  const int pz = pz0 + (int)(idx / ((long long)Px * Py));
  int sx, sy, sz;
  const int ix = circ_index(px, Px, nx, sx), iy = circ_index(py, Py, ny, sy), iz = circ_index(pz, Pz, nz, sz);
  double v = 0.0;
  if (ix >= 0 && iy >= 0 && iz >= 0) {
    v = oct_c[((long long)iz * ny + iy) * nx + ix];
    int s = 1;
    if (c == 1) s = sx * sy;
    else if (c == 2) s = sx * sz;
    else if (c == 4) s = sy * sz;
    if (s < 0) v = -v;
  }
  A[idx] = make_double2(v, 0.0);
}

// S4: forward complex fp64 FFT of lines (radix-2, bit-reversed load, one CTA per line).
// line l: base = (l / inner_count) * outer_stride + (l % inner_count); element e at base + e*estride.
__global__ void k_fft64(double2* A, int L, int logL, long long nlines, long long inner_count, long long outer_stride,
                        long long estride) {
  extern __shared__ double2 sh64[];
  for (long long l = blockIdx.x; l < nlines; l += gridDim.x) {
    const long long base = (l / inner_count) * outer_stride + (l % inner_count);
    for (int e = threadIdx.x; e < L; e += blockDim.x) {
      const int rev = (int)(__brev((unsigned)e) >> (32 - logL));
      sh64[rev] = A[base + e * estride];
    }
    __syncthreads();
    for (int len = 2; len <= L; len <<= 1) {
      const int half = len >> 1;
      for (int q = threadIdx.x; q < L / 2; q += blockDim.x) {
        const int grp = q / half, k = q - grp * half;
        const int i0 = grp * len + k, i1 = i0 + half;
        double s, co;
        sincospi(-2.0 * (double)k / (double)len, &s, &co);
        const double2 a = sh64[i0], b = sh64[i1];
        const double2 t = make_double2(b.x * co - b.y * s, b.x * s + b.y * co);
        sh64[i0] = make_double2(a.x + t.x, a.y + t.y);
        sh64[i1] = make_double2(a.x - t.x, a.y - t.y);
      }
      __syncthreads();
    }
    for (int e = threadIdx.x; e < L; e += blockDim.x) A[base + e * estride] = sh64[e];
    __syncthreads();
  }
}

// S5: KS[c][kz'][ky'][kx - kx0] = -Re A[kz'][ky'][kx] / (Px Py Pz), rounded to fp32,
// for the columns kx0 .. kx0 + ncol - 1 (one rank's kx block; pitch KSp, the
// padding columns zero).  A is the compact spectrum [Pz][Py][Kw] of the columns
// kxlo .. kxlo + Kw - 1.
// KS64 (optional): the same values before the fp32 rounding (grace_kernel_spectrum_f64).
__global__ void k_fold(float* KSc, double* KS64c, const double2* A, Geom g, int kx0, int ncol, int KSp, int kxlo,
                       int Kw) {
  const long long tot = (long long)g.Kzh * g.Kyh * KSp;
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= tot) return;
  const int col = (int)(idx % KSp);
  const int ky = (int)((idx / KSp) % g.Kyh);
  const int kz = (int)(idx / ((long long)KSp * g.Kyh));
  const int kx = kx0 + col;
  double v = 0.0;
  if (col < ncol && kx < g.Kx) {
    const double P = (double)g.Px * (double)g.Py * (double)g.Pz;
    v = -A[((long long)kz * g.Py + ky) * Kw + (kx - kxlo)].x / P;
  }
  if (KSc) KSc[idx] = (float)v;
  if (KS64c) KS64c[idx] = v;
}

// Columns kxlo .. kxlo + Kw - 1 of the x-transformed chunk [npz][Py][Px] -> compact [Pz][Py][Kw].
__global__ void k_gather_cols(double2* dst, const double2* chunk, int Px, int Py, int pz0, int npz, int kxlo, int Kw) {
  const long long tot = (long long)npz * Py * Kw;
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= tot) return;
  const int kw = (int)(idx % Kw);
  const long long row = idx / Kw;  // (pz - pz0) * Py + py
  dst[((long long)pz0 * Py + row) * Kw + kw] = chunk[row * Px + kxlo + kw];
}

inline long long cdiv(long long a, long long b) { return (a + b - 1) / b; }

}  // namespace

// Node lattice of f/g values covering every near-field stencil node (S1).
static cudaError_t node_lattice(int nx, int ny, int nz, double dx, double dy, double dz, double** lat, int* L3,
                                cudaStream_t st) {
  // node box: near offsets satisfy |i| dx <= 30 diag, so |i| <= 30 diag/dx; +2 margin, capped by the grid.
  const double diag = std::sqrt((dx * dx + dy * dy) + dz * dz);
  auto ext = [&](int n, double d) {
    const double lim = 30.0 * diag / d + 2.0;
    const long long e = (lim > (double)n) ? (long long)n : (long long)lim;
    return (int)(e + 2);  // nodes 0 .. e+1
  };
  L3[0] = ext(nx, dx);
  L3[1] = ext(ny, dy);
  L3[2] = ext(nz, dz);
  const long long nn = 6LL * L3[0] * L3[1] * L3[2];
  cudaError_t e = cudaMallocAsync(lat, sizeof(double) * nn, st);
  if (e != cudaSuccess) return e;
  k_nodes<<<(unsigned)cdiv(nn, 128), 128, 0, st>>>(*lat, L3[0], L3[1], L3[2], dx, dy, dz);
  return cudaGetLastError();
}

cudaError_t tensor_octant_device(int nx, int ny, int nz, double dx, double dy, double dz, double* oct,
                                 cudaStream_t st) {
  double* lat = nullptr;
  int L3[3];
  cudaError_t e = node_lattice(nx, ny, nz, dx, dy, dz, &lat, L3, st);
  if (e == cudaSuccess) {
    const long long no = 6LL * nx * ny * nz;
    k_octant<<<(unsigned)cdiv(no, 256), 256, 0, st>>>(oct, lat, L3[0], L3[1], L3[2], nx, ny, nz, dx, dy, dz, 0, 6);
    e = cudaGetLastError();
  }
  if (lat) cudaFreeAsync(lat, st);
  return e;
}

static cudaError_t fft64_axis(double2* A, int L, long long nlines, long long inner_count, long long outer_stride,
                              long long estride, cudaStream_t st) {
  if (L == 1) return cudaSuccess;
  int logL = 0;
  while ((1 << logL) < L) ++logL;
  const size_t smem = sizeof(double2) * (size_t)L;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_fft64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const long long grid = nlines < 148 * 64 ? nlines : 148 * 64;
  k_fft64<<<(unsigned)grid, 256, smem, st>>>(A, L, logL, nlines, inner_count, outer_stride, estride);
  return cudaGetLastError();
}

cudaError_t kernel_spectrum_device(const Geom& g, double dx, double dy, double dz, int nout, const KsOut* out,
                                   size_t* scratch_bytes, cudaStream_t st) {
  const long long N = (long long)g.nx * g.ny * g.nz;
  // the union of the requested kx columns: only these survive the x transform
  int kxlo = g.Kx, kxhi = 0;
  for (int o = 0; o < nout; ++o)
    if (out[o].ncol > 0) {
      kxlo = std::min(kxlo, out[o].kx0);
      kxhi = std::max(kxhi, std::min(g.Kx, out[o].kx0 + out[o].ncol));
    }
  if (kxhi <= kxlo) return cudaSuccess;
  const int Kw = kxhi - kxlo;
  const long long plane = (long long)g.Px * g.Py;
  // x transforms in chunks of padded z planes, at most the compact spectrum's size
  int zc = (int)std::max<long long>(1, std::min<long long>(g.Pz, ((long long)g.Py * Kw * g.Pz) / plane));
  const size_t need = sizeof(double) * N + sizeof(double2) * (size_t)plane * zc +
                      sizeof(double2) * (size_t)g.Pz * g.Py * Kw;
  if (scratch_bytes) *scratch_bytes = need;
  double* lat = nullptr;
  double* oct = nullptr;
  double2* chunk = nullptr;
  double2* A = nullptr;
  int L3[3];
  cudaError_t e = node_lattice(g.nx, g.ny, g.nz, dx, dy, dz, &lat, L3, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&oct, sizeof(double) * N, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&chunk, sizeof(double2) * (size_t)plane * zc, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&A, sizeof(double2) * (size_t)g.Pz * g.Py * Kw, st);
  for (int c = 0; c < 6 && e == cudaSuccess; ++c) {
    // S2 (component c), S3 + x lines per z chunk, kept columns -> compact A
    k_octant<<<(unsigned)cdiv(N, 256), 256, 0, st>>>(oct, lat, L3[0], L3[1], L3[2], g.nx, g.ny, g.nz, dx, dy, dz, c,
                                                     1);
    e = cudaGetLastError();
    for (int z0 = 0; z0 < g.Pz && e == cudaSuccess; z0 += zc) {
      const int nz = std::min(zc, g.Pz - z0);
      k_embed<<<(unsigned)cdiv(plane * nz, 256), 256, 0, st>>>(chunk, oct, c, g.nx, g.ny, g.nz, g.Px, g.Py, g.Pz, z0,
                                                                nz);
      e = cudaGetLastError();
      if (e == cudaSuccess) e = fft64_axis(chunk, g.Px, (long long)g.Py * nz, 1, g.Px, 1, st);
      if (e == cudaSuccess) {
        k_gather_cols<<<(unsigned)cdiv((long long)nz * g.Py * Kw, 256), 256, 0, st>>>(A, chunk, g.Px, g.Py, z0, nz,
                                                                                      kxlo, Kw);
        e = cudaGetLastError();
      }
    }
    // S4: y and z lines of the kept columns (the same line transforms as on the full array)
    if (e == cudaSuccess) e = fft64_axis(A, g.Py, (long long)g.Pz * Kw, Kw, (long long)g.Py * Kw, Kw, st);
    if (e == cudaSuccess) e = fft64_axis(A, g.Pz, (long long)g.Py * Kw, (long long)g.Py * Kw, 0, (long long)g.Py * Kw, st);
    for (int o = 0; o < nout && e == cudaSuccess; ++o) {
      const long long kslen = (long long)g.Kzh * g.Kyh * out[o].KSp;
      k_fold<<<(unsigned)cdiv(kslen, 256), 256, 0, st>>>(out[o].KS ? out[o].KS + c * kslen : nullptr,
                                                         out[o].KS64 ? out[o].KS64 + c * kslen : nullptr, A, g,
                                                         out[o].kx0, out[o].ncol, out[o].KSp, kxlo, Kw);
      e = cudaGetLastError();
    }
  }
  if (A) cudaFreeAsync(A, st);
  if (chunk) cudaFreeAsync(chunk, st);
  if (oct) cudaFreeAsync(oct, st);
  if (lat) cudaFreeAsync(lat, st);
  return e;
}

}  // namespace grace
