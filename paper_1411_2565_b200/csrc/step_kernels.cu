// Per-step kernels K1..K5 of the LLG hot path (sm_100a, fp32) and small utilities.
//
// The step for M[3][nz][ny][nx] (x fastest, SoA):
//   K1  x-R2C of the zero-padded rows           M  -> X1 [3][nz][ny][Kxp]       (P:L55 FFT, zero padding)
//   K2  y-FFT (pruned: ny of Py inputs nonzero)  X1 -> X2 [3][nz][Py][Kxp]
//   K3  z-FFT, H~ = KS . M~ (6 real folded comps), inverse z, keep z < nz   X2 -> X2
//   K4  inverse y, keep y < ny                   X2 -> X1
//   K5  inverse x C2R (keep x < nx) = H_demag, + six-neighbour exchange + x anisotropy
//       + Zeeman (Eq. (2)), Eq. (3) LLG, Euler + renormalise   X1, M -> M'
// nz == 1 (thin films, SP4): K2' fuses y-FFT, multiply and inverse y in one
// CTA (the z axis is unpadded), so the step is K1, K2', K5.
// The 1/(Px Py Pz) normalisation and the minus sign of H = -N*M live in KS.
#include <cuda_runtime.h>

#include <cstdint>

#include "fft_engine.cuh"
#include "internal.h"

namespace grace {

// Occupancy target per block size: at most ~64 registers per thread.
#define GRACE_MINB(NT) ((NT) <= 256 ? 4 : ((NT) <= 512 ? 2 : 1))

// ---------------------------------------------------------------------------
// k-space tensor-vector multiply at (kz, ky, kx) from the folded real table.
// KS[c][kz'][ky'][kx], kz' = min(kz, Pz-kz), ky' = min(ky, Py-ky); a folded
// axis flips the sign of the components odd in it (xy, yz odd in y; xz, yz in z).
__device__ __forceinline__ void kmul3(float2& a, float2& b, float2& c, const float* __restrict__ KS, const Geom& g,
                                      int kz, int ky, int kx) {
  const bool fy = ky > (g.Py >> 1), fz = kz > (g.Pz >> 1);
  const int kyf = fy ? g.Py - ky : ky;
  const int kzf = fz ? g.Pz - kz : kz;
  const size_t cs = (size_t)g.Kzh * g.Kyh * g.KSp;
  const float* p = KS + ((size_t)kzf * g.Kyh + kyf) * g.KSp + kx;
  const float nxx = __ldg(p), nyy = __ldg(p + 3 * cs), nzz = __ldg(p + 5 * cs);
  float nxy = __ldg(p + cs);
  if (fy) nxy = -nxy;
  float nxz = 0.f, nyz = 0.f;
  if (g.Pz > 1) {
    nxz = __ldg(p + 2 * cs);
    nyz = __ldg(p + 4 * cs);
    if (fz) nxz = -nxz;
    if (fy != fz) nyz = -nyz;
  }
  const float2 mx = a, my = b, mz = c;
  a = make_float2(nxx * mx.x + nxy * my.x + nxz * mz.x, nxx * mx.y + nxy * my.y + nxz * mz.y);
  b = make_float2(nxy * mx.x + nyy * my.x + nyz * mz.x, nxy * mx.y + nyy * my.y + nyz * mz.y);
  c = make_float2(nxz * mx.x + nyz * my.x + nzz * mz.x, nxz * mx.y + nyz * my.y + nzz * mz.y);
}

// The same multiply with this CTA's KS slice staged in shared memory:
// kss[c][kz'][b] for the CTA's ky' and kx tile (c = 0..5).
__device__ __forceinline__ void kmul3_s(float2& a, float2& b, float2& c, const float* kss, int Kzh, int B,
                                        const Geom& g, int kz, int ky, int bcol) {
  const bool fy = ky > (g.Py >> 1), fz = kz > (g.Pz >> 1);
  const int kzf = fz ? g.Pz - kz : kz;
  const int cs = Kzh * B;
  const float* p = kss + kzf * B + bcol;
  const float nxx = p[0], nyy = p[3 * cs], nzz = p[5 * cs];
  const float nxy = fy ? -p[cs] : p[cs];
  const float nxz = fz ? -p[2 * cs] : p[2 * cs];
  const float nyz = (fy != fz) ? -p[4 * cs] : p[4 * cs];
  const float2 mx = a, my = b, mz = c;
  a = make_float2(nxx * mx.x + nxy * my.x + nxz * mz.x, nxx * mx.y + nxy * my.y + nxz * mz.y);
  b = make_float2(nxy * mx.x + nyy * my.x + nyz * mz.x, nxy * mx.y + nyy * my.y + nyz * mz.y);
  c = make_float2(nxz * mx.x + nyz * my.x + nzz * mz.x, nxz * mx.y + nyz * my.y + nzz * mz.y);
}

__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(gsrc));
}
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// ---------------------------------------------------------------------------
// K1: x R2C.  A real row of Px (nx nonzero) is packed as z[n] = x[2n] + i x[2n+1],
// a length-L = Px/2 complex FFT gives Z, and
//   X[k] = (Z[k] + conj Z[L-k])/2 - (i/2) w^k (Z[k] - conj Z[L-k]),  w = exp(-2 pi i/Px), k = 0..L.
template <int L, int B, int NT, bool DIST>
__global__ void __launch_bounds__(NT, GRACE_MINB(NT)) k1_fwd_x(const float* __restrict__ M, float2* __restrict__ X1,
                                               const float2* __restrict__ tw, Geom g, StepParams* bump) {
  extern __shared__ float2 smem[];
  // The step index lives on the device so captured graphs stay valid: K1 of each
  // step advances it, K5 of the same step reads step - 1.
  if (bump != nullptr && blockIdx.x == 0 && threadIdx.x == 0) bump->step += 1;
  const int nrows = 3 * g.nzl * g.ny;
  const int row0 = blockIdx.x * B;
  if constexpr (L == 0) {  // Px == 1: X[0] = x[0]
    for (int b = threadIdx.x; b < B; b += NT) {
      const int row = row0 + b;
      if (row < nrows) X1[(size_t)row * g.pitch1] = make_float2(__ldg(M + row), 0.f);
    }
  } else {
    struct Ld {
      __device__ static constexpr bool kSmem() { return false; }
      const float* M;
      int row0, nrows, nx;
      __device__ float2 operator()(int b, int ib, int C) const {
        const int i = ib + C;
        float2 v = make_float2(0.f, 0.f);
        const int row = row0 + b;
        if (row < nrows) {
          const float* p = M + (size_t)row * nx;
          const int x0 = 2 * i;
          if (x0 < nx) v.x = __ldg(p + x0);
          if (x0 + 1 < nx) v.y = __ldg(p + x0 + 1);
        }
        return v;
      }
    } ld{M, row0, nrows, g.nx};
    const int twstride = g.Lmax / L;
    fft_tile<L, B, NT, false, false, true>(smem, ld, SmemSt<L, B, false>{smem}, tw, twstride);
    __syncthreads();
    const int twpx = g.Lmax / (2 * L);
    for (int u = threadIdx.x; u < B * (L + 1); u += NT) {
      const int b = u / (L + 1), k = u - b * (L + 1);
      const int row = row0 + b;
      if (row >= nrows) continue;
      const float2 Zk = smem[TileIdx<L, B, false>::at(b, k & (L - 1))];
      const float2 Zn = smem[TileIdx<L, B, false>::at(b, (L - k) & (L - 1))];
      const float2 E = make_float2(0.5f * (Zk.x + Zn.x), 0.5f * (Zk.y - Zn.y));
      const float2 D = make_float2(0.5f * (Zk.x - Zn.x), 0.5f * (Zk.y + Zn.y));
      const float2 wD = cmul(__ldg(tw + k * twpx), D);
      const float2 Xk = make_float2(E.x + wD.y, E.y - wD.x);
      if constexpr (DIST) {  // destination-blocked for the all-to-all: block k / kb
        const int q = k / g.kb;
        X1[q * g.blk1 + (size_t)row * g.pitch1 + (k - q * g.kb)] = Xk;
      } else {
        X1[(size_t)row * g.pitch1 + k] = Xk;
      }
    }
  }
}

// Offset of the (component, global z) slab of an x-row layout: kx block
// z / nzl (the source / destination rank of the all-to-all), plane z % nzl.
__device__ __forceinline__ size_t xrow_slab(const Geom& g, int slab) {
  const int c = slab / g.nz, z = slab - c * g.nz;
  const int q = z / g.nzl, zl = z - q * g.nzl;
  return ((size_t)(q * 3 + c) * g.nzl + zl) * g.ny * g.pitch1;
}

// ---------------------------------------------------------------------------
// K2 / K4: y pencils.  Columns (kx) are contiguous; a CTA owns NCOL columns of one
// (component, z) slab.  Forward: ny of L inputs nonzero.  Inverse: keep y < ny.
template <int L, int NCOL, int NT, bool INV>
__global__ void __launch_bounds__(NT, GRACE_MINB(NT)) k_y(const float2* __restrict__ in, float2* __restrict__ out,
                                          const float2* __restrict__ tw, Geom g, int in_rows, int out_rows,
                                          int n_in, int n_out) {
  extern __shared__ float2 smem[];
  const int kx0 = blockIdx.x * NCOL;
  const size_t slab = blockIdx.y;
  struct Ld {
    __device__ static constexpr bool kSmem() { return false; }
    const float2* p;
    int pitch, n_in, ncol_valid;
    __device__ float2 operator()(int b, int ib, int C) const {
      const int i = ib + C;
      return (i < n_in && b < ncol_valid) ? __ldg(p + (b + i * pitch)) : make_float2(0.f, 0.f);
    }
  } ld{in + (!INV ? xrow_slab(g, (int)slab) : slab * in_rows * g.pitch2) + kx0, !INV ? g.pitch1 : g.pitch2, n_in,
       g.Kc - kx0};
  struct St {
    __device__ static constexpr bool kSmem() { return false; }
    float2* p;
    int pitch, n_out, ncol_valid;
    __device__ void operator()(int b, int ib, int C, float2 v) const {
      const int i = ib + C;
      if (i < n_out && b < ncol_valid) p[b + i * pitch] = v;
    }
  } st{out + (INV ? xrow_slab(g, (int)slab) : slab * out_rows * g.pitch2) + kx0, INV ? g.pitch1 : g.pitch2, n_out,
       g.Kc - kx0};
  fft_tile<L, NCOL, NT, true, INV, !INV && (L > 1), INV && (L > 1)>(smem, ld, st, tw, g.Lmax / L);
}

// ---------------------------------------------------------------------------
// K3: z pencils of the three components for one ky' (and its mirror Py - ky'):
// forward z-FFT (nz of L nonzero), H~ = KS . M~, inverse z-FFT, keep z < nz.
// Processing ky and Py-ky in one CTA reads each folded KS slice once.
template <int L, int B, int NT>
__global__ void __launch_bounds__(NT, GRACE_MINB(NT)) k3_z(float2* __restrict__ X2, const float* __restrict__ KS,
                                           const float2* __restrict__ tw, Geom g) {
  extern __shared__ float2 smem[];
  constexpr int NCOL = 3 * B;
  const int kx0 = blockIdx.x * B;
  const int kyf = blockIdx.y;
  const int zstride = g.Py * g.pitch2;                // between z planes
  const size_t cstride = (size_t)g.nz * zstride;      // between components
  const int nvalid = g.Kc - kx0;
  const int nky = (kyf == 0 || 2 * kyf == g.Py) ? 1 : 2;
  // Stage this CTA's folded KS slice (6 comps x Kzh x B) in smem with cp.async;
  // it lands while the first forward z-FFT runs and serves both ky and Py-ky.
  constexpr int KZH = L / 2 + 1;
  float* kss = reinterpret_cast<float*>(smem + TileIdx<L, NCOL, true>::SMEM_ELEMS);
  {
    const size_t csK = (size_t)g.Kzh * g.Kyh * g.KSp;
    if constexpr (B % 4 == 0) {
      for (int t = threadIdx.x; t < 6 * KZH * (B / 4); t += NT) {
        const int ch = t % (B / 4), r = t / (B / 4);
        const int comp = r / KZH, kz = r - comp * KZH;
        cp_async16(kss + r * B + 4 * ch, KS + comp * csK + ((size_t)kz * g.Kyh + kyf) * g.KSp + kx0 + 4 * ch);
      }
    } else {
      for (int t = threadIdx.x; t < 6 * KZH * B; t += NT) {
        const int bb = t % B, r = t / B;
        const int comp = r / KZH, kz = r - comp * KZH;
        cp_async4(kss + r * B + bb, KS + comp * csK + ((size_t)kz * g.Kyh + kyf) * g.KSp + kx0 + bb);
      }
    }
  }
  for (int rep = 0; rep < nky; ++rep) {
    const int ky = rep == 0 ? kyf : g.Py - kyf;
    float2* base = X2 + (size_t)ky * g.pitch2 + kx0;
    struct Ld {
      __device__ static constexpr bool kSmem() { return false; }
      const float2* p;
      int zs;
      size_t cs;
      int nz, nvalid;
      __device__ float2 operator()(int col, int ib, int C) const {
        const int i = ib + C;
        const int c = col / B, b = col - c * B;
        return (i < nz && b < nvalid) ? __ldg(p + c * cs + (b + i * zs)) : make_float2(0.f, 0.f);
      }
    } ld{base, zstride, cstride, g.nz, nvalid};
    struct St {
      __device__ static constexpr bool kSmem() { return false; }
      float2* p;
      int zs;
      size_t cs;
      int nz, nvalid;
      __device__ void operator()(int col, int ib, int C, float2 v) const {
        const int i = ib + C;
        const int c = col / B, b = col - c * B;
        if (i < nz && b < nvalid) p[c * cs + (b + i * zs)] = v;
      }
    } st{base, zstride, cstride, g.nz, nvalid};
    if (rep) __syncthreads();
    fft_tile<L, NCOL, NT, true, false, (L > 1)>(smem, ld, SmemSt<L, NCOL, true>{smem}, tw, g.Lmax / L);
    if (rep == 0) cp_async_wait_all();
    __syncthreads();
    for (int u = threadIdx.x; u < L * B; u += NT) {
      const int kz = u / B, b = u - kz * B;
      float2* s = smem + TileIdx<L, NCOL, true>::at(b, kz);
      float2 a = s[0], bb = s[B], c = s[2 * B];
      kmul3_s(a, bb, c, kss, KZH, B, g, kz, ky, b);
      s[0] = a;
      s[B] = bb;
      s[2 * B] = c;
    }
    __syncthreads();
    fft_tile<L, NCOL, NT, true, true, false, (L > 1)>(smem, SmemLd<L, NCOL, true>{smem}, st, tw, g.Lmax / L);
  }
}

// Pz == 1 without the fused y path: H~ = KS . M~ on X2 [3][1][Py][Kxp].
__global__ void k_mul_plane(float2* __restrict__ X2, const float* __restrict__ KS, Geom g) {
  const int kx = blockIdx.x * blockDim.x + threadIdx.x;
  const int ky = blockIdx.y;
  if (kx >= g.Kc) return;
  const size_t cs = (size_t)g.Py * g.pitch2;
  float2* p = X2 + (size_t)ky * g.pitch2 + kx;
  float2 a = p[0], b = p[cs], c = p[2 * cs];
  kmul3(a, b, c, KS, g, 0, ky, kx);
  p[0] = a;
  p[cs] = b;
  p[2 * cs] = c;
}

// ---------------------------------------------------------------------------
// K2': nz == 1.  y-FFT (ny of L nonzero), multiply, inverse y (keep y < ny), in place on X1.
template <int L, int B, int NT>
__global__ void __launch_bounds__(NT, GRACE_MINB(NT)) k2f_y_fused(float2* __restrict__ X1, const float* __restrict__ KS,
                                                  const float2* __restrict__ tw, Geom g) {
  extern __shared__ float2 smem[];
  constexpr int NCOL = 3 * B;
  const int kx0 = blockIdx.x * B;
  const int nvalid = g.Kx - kx0;
  const size_t cstride = (size_t)g.ny * g.Kxp;
  float2* base = X1 + kx0;
  struct Ld {
    __device__ static constexpr bool kSmem() { return false; }
    const float2* p;
    size_t cs;
    int pitch, ny, nvalid;
    __device__ float2 operator()(int col, int ib, int C) const {
      const int i = ib + C;
      const int c = col / B, b = col - c * B;
      return (i < ny && b < nvalid) ? __ldg(p + c * cs + (b + i * pitch)) : make_float2(0.f, 0.f);
    }
  } ld{base, cstride, g.Kxp, g.ny, nvalid};
  struct St {
    __device__ static constexpr bool kSmem() { return false; }
    float2* p;
    size_t cs;
    int pitch, ny, nvalid;
    __device__ void operator()(int col, int ib, int C, float2 v) const {
      const int i = ib + C;
      const int c = col / B, b = col - c * B;
      if (i < ny && b < nvalid) p[c * cs + (b + i * pitch)] = v;
    }
  } st{base, cstride, g.Kxp, g.ny, nvalid};
  fft_tile<L, NCOL, NT, true, false, (L > 1)>(smem, ld, SmemSt<L, NCOL, true>{smem}, tw, g.Lmax / L);
  __syncthreads();
  for (int u = threadIdx.x; u < L * B; u += NT) {
    const int ky = u / B, b = u - ky * B;
    if (b >= nvalid) continue;
    float2* s = smem + TileIdx<L, NCOL, true>::at(b, ky);
    float2 a = s[0], bb = s[B], c = s[2 * B];
    kmul3(a, bb, c, KS, g, 0, ky, kx0 + b);
    s[0] = a;
    s[B] = bb;
    s[2 * B] = c;
  }
  __syncthreads();
  fft_tile<L, NCOL, NT, true, true, false, (L > 1)>(smem, SmemLd<L, NCOL, true>{smem}, st, tw, g.Lmax / L);
}

// ---------------------------------------------------------------------------
// K5: inverse x C2R of the three H~ rows, then the local terms and the update.
// C2R of length Px = 2L from the half spectrum X[0..L]:
//   Z[k] = (X[k] + conj X[L-k]) + i w^-k (X[k] - conj X[L-k]),  k < L,
//   z = IFFT_L(Z) (unnormalised; 1/P is in KS),  x[2n] = Re z[n], x[2n+1] = Im z[n].
__device__ __forceinline__ float3 ld3(const float* __restrict__ M, size_t N, size_t i) {
  return make_float3(__ldg(M + i), __ldg(M + N + i), __ldg(M + 2 * N + i));
}

template <int L, int B, int NT, bool DIST>
__global__ void __launch_bounds__(NT, GRACE_MINB(NT)) k5_inv_x_llg(const float2* __restrict__ X1, const float* __restrict__ M,
                                                   float* __restrict__ Mn, float* __restrict__ Hout,
                                                   const float2* __restrict__ tw, Geom g,
                                                   const StepParams* __restrict__ prm,
                                                   unsigned long long* __restrict__ flag, int mode,
                                                   const float* __restrict__ Hlo, const float* __restrict__ Hhi) {
  extern __shared__ float2 smem[];
  constexpr int NCOL = 3 * B;
  const int nrows = g.nzl * g.ny;
  const int row0 = blockIdx.x * B;
  const size_t N = (size_t)nrows * g.nx;
  const size_t cstrideX = (size_t)nrows * g.pitch1;  // X1 component stride
  float* hs = reinterpret_cast<float*>(smem);      // H_demag rows [3B][2L] (reals), aliasing the tile
  if constexpr (L == 0) {
    for (int col = threadIdx.x; col < NCOL; col += NT) {
      const int c = col / B, b = col - c * B;
      const int row = row0 + b;
      hs[col] = row < nrows ? __ldg(X1 + c * cstrideX + (size_t)row * g.pitch1).x : 0.f;
    }
  } else {
    const int twpx = g.Lmax / (2 * L);
    struct Ld {
      __device__ static constexpr bool kSmem() { return false; }
      const float2* X;
      const float2* tw;
      size_t cs;
      int row0, nrows, pitch, twpx, kb;
      long long blk1;
      __device__ float2 operator()(int col, int ib, int C) const {
        const int k = ib + C;
        const int c = col / B, b = col - c * B;
        const int row = row0 + b;
        if (row >= nrows) return make_float2(0.f, 0.f);
        const float2* p = X + c * cs + (size_t)row * pitch;
        float2 a, m;
        if constexpr (DIST) {  // gather from the source kx blocks of the all-to-all
          const int qa = k / kb, qm = (L - k) / kb;
          a = __ldg(p + qa * blk1 + (k - qa * kb));
          m = __ldg(p + qm * blk1 + ((L - k) - qm * kb));
        } else {
          a = __ldg(p + k);
          m = __ldg(p + (L - k));
        }
        const float2 S = make_float2(a.x + m.x, a.y - m.y);  // X[k] + conj X[L-k]
        const float2 D = make_float2(a.x - m.x, a.y + m.y);  // X[k] - conj X[L-k]
        float2 w = __ldg(tw + k * twpx);                       // exp(-2 pi i k/Px)
        w.y = -w.y;                                            // w^-k
        const float2 wD = cmul(w, D);
        return make_float2(S.x - wD.y, S.y + wD.x);            // S + i wD
      }
    } ld{X1, tw, cstrideX, row0, nrows, g.pitch1, twpx, g.kb, g.blk1};
    struct St {
      __device__ static constexpr bool kSmem() { return true; }
      float* hs;
      int nx;
      __device__ void operator()(int col, int ib, int C, float2 v) const {
        const int n = ib + C;
        float* p = hs + col * (2 * L) + 2 * n;
        if (2 * n + 1 < nx) *reinterpret_cast<float2*>(p) = v;
        else if (2 * n < nx) p[0] = v.x;
      }
    } st{hs, g.nx};
    fft_tile<L, NCOL, NT, false, true, false, true>(smem, ld, st, tw, g.Lmax / L);
  }
  __syncthreads();
  constexpr int HP = (L == 0) ? 1 : 2 * L;  // row pitch of hs
  const StepParams p = *prm;
  const size_t plane = (size_t)g.nx * g.ny;
  const int ncell = B * g.nx;
  // Two cells per thread per iteration with all 42 stencil loads issued before
  // any use.  A missing neighbour (Neumann) loads the centre cell instead, so its
  // difference is exactly 0 (reading Q11).
  constexpr int CPI = 2;
  for (int u0 = threadIdx.x; u0 < ncell; u0 += CPI * NT) {
    float3 m[CPI], q[CPI][6];
    size_t ic[CPI];
    int bc[CPI], xc[CPI];
    bool ok[CPI];
#pragma unroll
    for (int c = 0; c < CPI; ++c) {
      const int u = u0 + c * NT;
      const int b = u / g.nx, x = u - b * g.nx;
      const int row = row0 + b;
      ok[c] = u < ncell && row < nrows;
      const int rr = ok[c] ? row : 0;
      const int xx = ok[c] ? x : 0;
      const int z = rr / g.ny, y = rr - z * g.ny;
      const size_t i = (size_t)rr * g.nx + xx;
      ic[c] = i;
      bc[c] = ok[c] ? b : 0;
      xc[c] = xx;
      m[c] = ld3(M, N, i);
      q[c][0] = ld3(M, N, xx > 0 ? i - 1 : i);
      q[c][1] = ld3(M, N, xx + 1 < g.nx ? i + 1 : i);
      q[c][2] = ld3(M, N, y > 0 ? i - g.nx : i);
      q[c][3] = ld3(M, N, y + 1 < g.ny ? i + g.nx : i);
      if (DIST && z == 0 && g.has_lo) q[c][4] = ld3(Hlo, plane, (size_t)y * g.nx + xx);
      else q[c][4] = ld3(M, N, z > 0 ? i - plane : i);
      if (DIST && z + 1 == g.nzl && g.has_hi) q[c][5] = ld3(Hhi, plane, (size_t)y * g.nx + xx);
      else q[c][5] = ld3(M, N, z + 1 < g.nzl ? i + plane : i);
    }
#pragma unroll
    for (int c = 0; c < CPI; ++c) {
      if (!ok[c]) continue;
      const size_t i = ic[c];
      const int b = bc[c], x = xc[c];
      const float3 mm = m[c];
      // Eq. (2): H_eff = H_demag + H_exch + H_anis + H_ext
      float hx = hs[(0 * B + b) * HP + x] + p.hext[0] + g.ck * mm.x;
      float hy = hs[(1 * B + b) * HP + x] + p.hext[1];
      float hz = hs[(2 * B + b) * HP + x] + p.hext[2];
      // six-neighbour exchange (difference form: uniform M gives exactly 0)
      float ex = 0.f, ey = 0.f, ez = 0.f;
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const float ck = k < 2 ? g.cx : (k < 4 ? g.cy : g.cz);
        ex += ck * (q[c][k].x - mm.x);
        ey += ck * (q[c][k].y - mm.y);
        ez += ck * (q[c][k].z - mm.z);
      }
      hx += ex;
      hy += ey;
      hz += ez;
      if (mode == 1) {
        Hout[i] = hx;
        Hout[N + i] = hy;
        Hout[2 * N + i] = hz;
        continue;
      }
      // Eq. (3): dM/dt = c_prec (M x H) + c_damp M x (M x H)
      const float ax = mm.y * hz - mm.z * hy, ay = mm.z * hx - mm.x * hz, az = mm.x * hy - mm.y * hx;
      const float bx = mm.y * az - mm.z * ay, by = mm.z * ax - mm.x * az, bz = mm.x * ay - mm.y * ax;
      const float sx = mm.x + p.dt * (p.c_prec * ax + p.c_damp * bx);
      const float sy = mm.y + p.dt * (p.c_prec * ay + p.c_damp * by);
      const float sz = mm.z + p.dt * (p.c_prec * az + p.c_damp * bz);
      const float sc = g.Ms / sqrtf(sx * sx + sy * sy + sz * sz);  // renormalise to Ms (reading Q16)
      const float ox = sx * sc, oy = sy * sc, oz = sz * sc;
      Mn[i] = ox;
      Mn[N + i] = oy;
      Mn[2 * N + i] = oz;
      if (!(isfinite(ox) && isfinite(oy) && isfinite(oz)))
        atomicMin(flag, ((unsigned long long)(p.step - 1) << 36) | (unsigned long long)i);
    }
  }
}

// ---------------------------------------------------------------------------
// Tile choices and dispatch.  Every engine instance uses TPC = L/16 threads per
// column, i.e. 16 complex values per thread per pass.
// Complex values per thread per Stockham pass (EPT) and tile sizes, per kernel,
// from the sweep in profiles/ (DESIGN.md §6).  TPC = L/EPT threads per column.
#ifndef GRACE_EPT_X1
#define GRACE_EPT_X1 16
#endif
#ifndef GRACE_EPT_X5
#define GRACE_EPT_X5 32
#endif
#ifndef GRACE_EPT_Y
#define GRACE_EPT_Y 16
#endif
#ifndef GRACE_EPT_Z
#define GRACE_EPT_Z 32
#endif
#ifndef GRACE_Y_ELEMS
#define GRACE_Y_ELEMS 16384  // complex values per K2/K4 tile
#endif
__host__ __device__ constexpr int tpc_of(int L, int ept) { return L >= ept ? L / ept : 1; }
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
template <int L>
struct XCfg {  // K1 rows / K5 rows (3 components per row)
  static constexpr int TPC1 = tpc_of(L, GRACE_EPT_X1);
  static constexpr int TPC5 = tpc_of(L, GRACE_EPT_X5);
  static constexpr int B1 = (L == 0) ? 256 : cmax(1, 256 / TPC1);
  static constexpr int NT1 = (L == 0) ? 256 : B1 * TPC1;
  static constexpr int B5 = (L == 0) ? 64 : cmax(1, 128 / TPC5);
  static constexpr int NT5 = (L == 0) ? 256 : 3 * B5 * TPC5;
};
template <int L>
struct YCfg {  // K2/K4 columns
  static constexpr int NCOL = cmax(2, cmin(32, GRACE_Y_ELEMS / L));
  static constexpr int NT = cmin(1024, cmax(32, NCOL * tpc_of(L, GRACE_EPT_Y)));
};
template <int L>
struct ZCfg {  // K3 and K2' (3 components, B kx columns each)
  static constexpr int B = cmax(1, cmin(32, 2048 / L));
  static constexpr int NT = cmax(32, 3 * B * tpc_of(L, GRACE_EPT_Z));
};

template <class K>
static cudaError_t prep(K kern, size_t smem) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e == cudaSuccess && smem > 48 * 1024)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return e;
}

#define GRACE_L_SWITCH(Lval, CASE) \
  switch (Lval) {                   \
    CASE(1) CASE(2) CASE(4) CASE(8) CASE(16) CASE(32) CASE(64) CASE(128) CASE(256) CASE(512) CASE(1024) CASE(2048) CASE(4096) \
    default: return cudaErrorInvalidValue; \
  }

template <int L, bool DIST>
static cudaError_t k1_launch(const Geom& g, const float* M, float2* X1, const float2* tw, StepParams* bump,
                             cudaStream_t st) {
  constexpr int B = XCfg<L>::B1, NT = XCfg<L>::NT1;
  const size_t smem = (L == 0) ? 0 : (size_t)TileIdx<(L > 0 ? L : 1), B, false>::SMEM_ELEMS * sizeof(float2);
  auto kern = k1_fwd_x<L, B, NT, DIST>;
  cudaError_t e = prep(kern, smem);
  if (e != cudaSuccess) return e;
  const int nrows = 3 * g.nzl * g.ny;
  kern<<<(nrows + B - 1) / B, NT, smem, st>>>(M, X1, tw, g, bump);
  return cudaGetLastError();
}

cudaError_t launch_k1(const Geom& g, const float* M, float2* X1, const float2* tw, StepParams* bump,
                      cudaStream_t st) {
  if (g.Px == 1) return g.kb ? k1_launch<0, true>(g, M, X1, tw, bump, st) : k1_launch<0, false>(g, M, X1, tw, bump, st);
  const int L = g.Px / 2;
#define CASE(v)                                                                                         \
  case v:                                                                                               \
    return (v < 2) ? cudaErrorInvalidValue                                                              \
           : g.kb  ? k1_launch<(v >= 2 ? v : 2), true>(g, M, X1, tw, bump, st)                          \
                   : k1_launch<(v >= 2 ? v : 2), false>(g, M, X1, tw, bump, st);
  GRACE_L_SWITCH(L, CASE)
#undef CASE
}

template <int L, bool INV>
static cudaError_t ky_launch(const Geom& g, const float2* in, float2* out, const float2* tw, cudaStream_t st,
                             int in_rows, int out_rows, int n_in, int n_out) {
  constexpr int NCOL = YCfg<L>::NCOL, NT = YCfg<L>::NT;
  const size_t smem = (size_t)TileIdx<L, NCOL, true>::SMEM_ELEMS * sizeof(float2);
  auto kern = k_y<L, NCOL, NT, INV>;
  cudaError_t e = prep(kern, smem);
  if (e != cudaSuccess) return e;
  dim3 grid((g.Kc + NCOL - 1) / NCOL, 3 * g.nz);
  kern<<<grid, NT, smem, st>>>(in, out, tw, g, in_rows, out_rows, n_in, n_out);
  return cudaGetLastError();
}

cudaError_t launch_k2(const Geom& g, const float2* X1, float2* X2, const float2* tw, cudaStream_t st) {
#define CASE(v) case v: return ky_launch<v, false>(g, X1, X2, tw, st, g.ny, g.Py, g.ny, g.Py);
  GRACE_L_SWITCH(g.Py, CASE)
#undef CASE
}

cudaError_t launch_k4(const Geom& g, const float2* X2, float2* X1, const float2* tw, cudaStream_t st) {
#define CASE(v) case v: return ky_launch<v, true>(g, X2, X1, tw, st, g.Py, g.ny, g.Py, g.ny);
  GRACE_L_SWITCH(g.Py, CASE)
#undef CASE
}

template <int L>
static cudaError_t k3_launch(const Geom& g, float2* X2, const float* KS, const float2* tw, cudaStream_t st) {
  constexpr int B = ZCfg<L>::B, NT = ZCfg<L>::NT;
  const size_t smem = (size_t)TileIdx<L, 3 * B, true>::SMEM_ELEMS * sizeof(float2) +
                      (size_t)6 * (L / 2 + 1) * B * sizeof(float);
  auto kern = k3_z<L, B, NT>;
  cudaError_t e = prep(kern, smem);
  if (e != cudaSuccess) return e;
  dim3 grid((g.Kc + B - 1) / B, g.Kyh);
  kern<<<grid, NT, smem, st>>>(X2, KS, tw, g);
  return cudaGetLastError();
}

cudaError_t launch_k3(const Geom& g, float2* X2, const float* KS, const float2* tw, cudaStream_t st) {
  if (g.Pz == 1) {
    dim3 grid((g.Kc + 127) / 128, g.Py);
    k_mul_plane<<<grid, 128, 0, st>>>(X2, KS, g);
    return cudaGetLastError();
  }
#define CASE(v) case v: return (v >= 2 && v <= 1024) ? k3_launch<(v >= 2 && v <= 1024 ? v : 2)>(g, X2, KS, tw, st) : cudaErrorInvalidValue;
  GRACE_L_SWITCH(g.Pz, CASE)
#undef CASE
}

bool fused_y_path(const Geom& g) { return g.Pz == 1 && g.Py <= 512; }
int kernel_count(const Geom& g) { return fused_y_path(g) ? 3 : 5; }

template <int L>
static cudaError_t k2f_launch(const Geom& g, float2* X1, const float* KS, const float2* tw, cudaStream_t st) {
  constexpr int B = ZCfg<L>::B, NT = ZCfg<L>::NT;
  const size_t smem = (size_t)TileIdx<L, 3 * B, true>::SMEM_ELEMS * sizeof(float2);
  auto kern = k2f_y_fused<L, B, NT>;
  cudaError_t e = prep(kern, smem);
  if (e != cudaSuccess) return e;
  k2f_y_fused<L, B, NT><<<(g.Kx + B - 1) / B, NT, smem, st>>>(X1, KS, tw, g);
  return cudaGetLastError();
}

cudaError_t launch_k2f(const Geom& g, float2* X1, const float* KS, const float2* tw, cudaStream_t st) {
#define CASE(v) case v: return (v <= 512) ? k2f_launch<(v <= 512 ? v : 512)>(g, X1, KS, tw, st) : cudaErrorInvalidValue;
  GRACE_L_SWITCH(g.Py, CASE)
#undef CASE
}

template <int L, bool DIST>
static cudaError_t k5_launch(const Geom& g, int mode, const float2* X1, const float* M, float* Mn, float* Hout,
                             const float2* tw, const StepParams* prm, unsigned long long* flag, cudaStream_t st,
                             const float* Hlo, const float* Hhi) {
  constexpr int B = XCfg<L>::B5, NT = XCfg<L>::NT5;
  const size_t smem = (L == 0) ? (size_t)3 * B * sizeof(float)
                               : (size_t)TileIdx<(L > 0 ? L : 1), 3 * B, false>::SMEM_ELEMS * sizeof(float2);
  auto kern = k5_inv_x_llg<L, B, NT, DIST>;
  cudaError_t e = prep(kern, smem);
  if (e != cudaSuccess) return e;
  const int nrows = g.nzl * g.ny;
  kern<<<(nrows + B - 1) / B, NT, smem, st>>>(X1, M, Mn, Hout, tw, g, prm, flag, mode, Hlo, Hhi);
  return cudaGetLastError();
}

cudaError_t launch_k5(const Geom& g, int mode, const float2* X1, const float* M, float* Mn, float* Hout,
                      const float2* tw, const StepParams* prm, unsigned long long* flag, cudaStream_t st,
                      const float* Hlo, const float* Hhi) {
  if (g.Px == 1)
    return g.kb ? k5_launch<0, true>(g, mode, X1, M, Mn, Hout, tw, prm, flag, st, Hlo, Hhi)
                : k5_launch<0, false>(g, mode, X1, M, Mn, Hout, tw, prm, flag, st, Hlo, Hhi);
  const int L = g.Px / 2;
#define CASE(v)                                                                                                 \
  case v:                                                                                                       \
    return (v < 2) ? cudaErrorInvalidValue                                                                      \
           : g.kb  ? k5_launch<(v >= 2 ? v : 2), true>(g, mode, X1, M, Mn, Hout, tw, prm, flag, st, Hlo, Hhi)   \
                   : k5_launch<(v >= 2 ? v : 2), false>(g, mode, X1, M, Mn, Hout, tw, prm, flag, st, Hlo, Hhi);
  GRACE_L_SWITCH(L, CASE)
#undef CASE
}

// ---------------------------------------------------------------------------
// Utilities.
__global__ void k_twiddles(float2* tw, int Lmax) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= Lmax) return;
  double s, c;
  sincospi(-2.0 * (double)k / (double)Lmax, &s, &c);  // fp64, then rounded once to fp32
  tw[k] = make_float2((float)c, (float)s);
}

cudaError_t launch_twiddles(float2* tw, int Lmax, cudaStream_t st) {
  k_twiddles<<<(Lmax + 255) / 256, 256, 0, st>>>(tw, Lmax);
  return cudaGetLastError();
}

// grace_set_m: M <- Ms M/|M| per cell (fp64 input, fp32 output); a zero or
// non-finite cell records its index.
__global__ void k_set_m_f64(const double* __restrict__ src, float* __restrict__ M, long long n, double Ms,
                            unsigned long long* flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double x = src[i], y = src[n + i], z = src[2 * n + i];
    const double r = sqrt(x * x + y * y + z * z);
    if (!(r > 0.0) || !isfinite(r)) {
      atomicMin(flag, (unsigned long long)i);
      continue;
    }
    const double s = Ms / r;
    M[i] = (float)(x * s);
    M[n + i] = (float)(y * s);
    M[2 * n + i] = (float)(z * s);
  }
}

__global__ void k_set_m_f32(const float* __restrict__ src, float* __restrict__ M, long long n, float Ms,
                            unsigned long long* flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float x = src[i], y = src[n + i], z = src[2 * n + i];
    const float r = sqrtf(x * x + y * y + z * z);
    if (!(r > 0.f) || !isfinite(r)) {
      atomicMin(flag, (unsigned long long)i);
      continue;
    }
    const float s = Ms / r;
    M[i] = x * s;
    M[n + i] = y * s;
    M[2 * n + i] = z * s;
  }
}

cudaError_t launch_set_m_f64(const double* src, float* M, long long n, double Ms, unsigned long long* flag,
                             cudaStream_t st) {
  k_set_m_f64<<<148 * 8, 256, 0, st>>>(src, M, n, Ms, flag);
  return cudaGetLastError();
}
cudaError_t launch_set_m_f32(const float* src, float* M, long long n, float Ms, unsigned long long* flag,
                             cudaStream_t st) {
  k_set_m_f32<<<148 * 8, 256, 0, st>>>(src, M, n, Ms, flag);
  return cudaGetLastError();
}

// <M>: deterministic two-stage fixed-order reduction in fp64 (SPEC "fixed-order reduction").
constexpr int kRedBlocks = 296;
constexpr int kRedThreads = 256;
__global__ void k_mavg_partial(const float* __restrict__ M, long long n, double* __restrict__ partial) {
  __shared__ double sh[3][kRedThreads];
  const long long chunk = (n + gridDim.x - 1) / gridDim.x;
  const long long lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
  double a = 0, b = 0, c = 0;
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    a += M[i];
    b += M[n + i];
    c += M[2 * n + i];
  }
  sh[0][threadIdx.x] = a;
  sh[1][threadIdx.x] = b;
  sh[2][threadIdx.x] = c;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int q = 0; q < 3; ++q) sh[q][threadIdx.x] += sh[q][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x < 3) partial[threadIdx.x * gridDim.x + blockIdx.x] = sh[threadIdx.x][0];
}
__global__ void k_mavg_final(const double* __restrict__ partial, int nb, long long n, double Ms, double* out) {
  if (threadIdx.x < 3) {
    double s = 0;
    for (int i = 0; i < nb; ++i) s += partial[threadIdx.x * nb + i];
    out[threadIdx.x] = s / ((double)n * Ms);
  }
}
cudaError_t launch_mavg(const float* M, long long n, double Ms, double* partial, double* out, cudaStream_t st) {
  k_mavg_partial<<<kRedBlocks, kRedThreads, 0, st>>>(M, n, partial);
  k_mavg_final<<<1, 32, 0, st>>>(partial, kRedBlocks, n, Ms, out);
  return cudaGetLastError();
}

__global__ void k_fill_uniform_x(float* M, long long n, float Ms) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    M[i] = Ms;
    M[n + i] = 0.f;
    M[2 * n + i] = 0.f;
  }
}
cudaError_t launch_fill_uniform_x(float* M, long long n, float Ms, cudaStream_t st) {
  k_fill_uniform_x<<<148 * 4, 256, 0, st>>>(M, n, Ms);
  return cudaGetLastError();
}

__global__ void k_widen(const float* __restrict__ src, double* __restrict__ dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = (double)src[i];
}
cudaError_t launch_widen(const float* src, double* dst, long long n, cudaStream_t st) {
  k_widen<<<148 * 4, 256, 0, st>>>(src, dst, n);
  return cudaGetLastError();
}

}  // namespace grace
