// Batched power-of-two FFT building block for the per-step kernels (sm_100a, fp32).
//
// Paper: the demag field is a zero-padded FFT convolution (Sec. 3).  The
// paper called a vendor FFT library; here every transform is this
// hand-written engine, instantiated inside the kernels that need it so the
// zero padding, the k-space multiply and the LLG update fuse into the first and
// last passes instead of separate HBM round trips.
//
// Algorithm: Stockham autosort, mixed radix 2..16.  A CTA transforms NCOL
// independent sequences ("columns") of length L.  Pass p (radix R, Ns = product
// of earlier radices) maps butterfly j in [0, L/R) of column b:
//     v[r] = in[j + r L/R] * w_{Ns R}^{(j mod Ns) r},  v = DFT_R(v),
//     out[(j / Ns) Ns R + (j mod Ns) + r Ns] = v[r]
// and the output is in natural order after the last pass.  The first pass reads
// through a caller functor (global memory, zero padding, pre-processing) and the
// last pass writes through one (global memory, pruned outputs, post-processing);
// intermediate passes run in place in shared memory.  Twiddles come from a
// global fp32 table w_Lmax^k = exp(-2 pi i k / Lmax) computed once in fp64.
//
// Two thread mappings:
//   COLMODE = true : consecutive lanes take consecutive columns (columns are
//                    contiguous in HBM: y and z pencils).  smem (b, i) -> i*NCOL + b.
//   COLMODE = false: consecutive lanes take consecutive butterflies of one column
//                    (the sequence is contiguous in HBM: x rows).  smem (b, i) ->
//                    b*L + swizzle(i), swizzle(i) = i ^ ((i >> 4) & 15).
#pragma once
#include <cuda_runtime.h>

namespace grace {

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }

__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x / 2); }
__host__ __device__ constexpr int fft_npass(int L) { return (ilog2(L) + 3) / 4; }
__host__ __device__ constexpr int fft_pass_bits(int L, int p) {
  return ilog2(L) / fft_npass(L) + (p < ilog2(L) % fft_npass(L) ? 1 : 0);
}

// exp(-2 pi i k / 16) (forward) for compile-time k; INV conjugates.
template <bool INV, int K>
__device__ __forceinline__ float2 tw16_mul(float2 x) {
  constexpr int k = K & 15;
  if constexpr (k == 0) {
    return x;
  } else if constexpr (k == 4) {  // -i (fwd) / +i (inv)
    return INV ? make_float2(-x.y, x.x) : make_float2(x.y, -x.x);
  } else if constexpr (k == 8) {
    return make_float2(-x.x, -x.y);
  } else if constexpr (k == 12) {
    return INV ? make_float2(x.y, -x.x) : make_float2(-x.y, x.x);
  } else {
    constexpr float C[16] = {1.0f, 0.92387953251128674f, 0.70710678118654752f, 0.38268343236508977f,
                             0.0f, -0.38268343236508977f, -0.70710678118654752f, -0.92387953251128674f,
                             -1.0f, -0.92387953251128674f, -0.70710678118654752f, -0.38268343236508977f,
                             0.0f, 0.38268343236508977f, 0.70710678118654752f, 0.92387953251128674f};
    constexpr float c = C[k];
    constexpr float s = INV ? C[(k + 12) & 15] : -C[(k + 12) & 15];  // sin(2 pi k/16), sign per direction
    return make_float2(x.x * c - x.y * s, x.x * s + x.y * c);
  }
}

// In-register DFT of size R (radix-2 decimation in time, natural order in and out).
template <int R, bool INV>
__device__ __forceinline__ void dft_inplace(float2* a);

template <bool INV, int R, int K>
__device__ __forceinline__ void dft_combine(float2* a, const float2* e, const float2* o) {
  if constexpr (K < R / 2) {
    float2 t = tw16_mul<INV, K * (16 / R)>(o[K]);
    a[K] = cadd(e[K], t);
    a[K + R / 2] = csub(e[K], t);
    dft_combine<INV, R, K + 1>(a, e, o);
  }
}

template <int R, bool INV>
__device__ __forceinline__ void dft_inplace(float2* a) {
  if constexpr (R == 1) {
    return;
  } else if constexpr (R == 2) {
    float2 t0 = a[0], t1 = a[1];
    a[0] = cadd(t0, t1);
    a[1] = csub(t0, t1);
  } else {
    float2 e[R / 2], o[R / 2];
#pragma unroll
    for (int q = 0; q < R / 2; ++q) {
      e[q] = a[2 * q];
      o[q] = a[2 * q + 1];
    }
    dft_inplace<R / 2, INV>(e);
    dft_inplace<R / 2, INV>(o);
    dft_combine<INV, R, 0>(a, e, o);
  }
}

// Shared-memory tile addressing.
template <int L, int NCOL, bool COLMODE>
struct TileIdx {
  __device__ __forceinline__ static int at(int b, int i) {
    if constexpr (COLMODE) {
      return i * NCOL + b;
    } else {
      if constexpr (L >= 16) return b * L + (i ^ ((i >> 4) & 15));
      else return b * L + i;
    }
  }
};

// Accessors for the smem tile used by intermediate passes.
template <int L, int NCOL, bool COLMODE>
struct SmemLd {
  __device__ static constexpr bool kSmem() { return true; }
  float2* s;
  __device__ __forceinline__ float2 operator()(int b, int i) const { return s[TileIdx<L, NCOL, COLMODE>::at(b, i)]; }
};
template <int L, int NCOL, bool COLMODE>
struct SmemSt {
  __device__ static constexpr bool kSmem() { return true; }
  float2* s;
  __device__ __forceinline__ void operator()(int b, int i, float2 v) const { s[TileIdx<L, NCOL, COLMODE>::at(b, i)] = v; }
};

// One Stockham pass.
template <int L, int R, int NS, int NCOL, int NT, bool COLMODE, bool INV, class LD, class ST>
__device__ __forceinline__ void fft_pass(const LD& ld, const ST& st, const float2* __restrict__ tw, int twstride) {
  constexpr int JR = L / R;
  constexpr int UNITS = NCOL * JR;
  constexpr int UPT = (UNITS + NT - 1) / NT;
  float2 v[UPT][R];
  int bb[UPT], jj[UPT];
#pragma unroll
  for (int q = 0; q < UPT; ++q) {
    const int u = threadIdx.x + q * NT;
    int b, j;
    if constexpr (COLMODE) {
      b = u % NCOL;
      j = u / NCOL;
    } else {
      j = u % JR;
      b = u / JR;
    }
    bb[q] = b;
    jj[q] = j;
    if (UNITS % NT == 0 || u < UNITS) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[q][r] = ld(b, j + r * JR);
    }
  }
  if constexpr (LD::kSmem() && ST::kSmem()) __syncthreads();  // in-place hazard
#pragma unroll
  for (int q = 0; q < UPT; ++q) {
    const int u = threadIdx.x + q * NT;
    if (UNITS % NT == 0 || u < UNITS) {
      const int b = bb[q], j = jj[q];
      if constexpr (NS > 1) {
        const int k1 = (j % NS) * (L / (NS * R)) * twstride;  // index of w_{Ns R}^{j mod Ns} in the Lmax table
#pragma unroll
        for (int r = 1; r < R; ++r) {
          float2 w = __ldg(tw + k1 * r);
          if constexpr (INV) w.y = -w.y;
          v[q][r] = cmul(v[q][r], w);
        }
      }
      dft_inplace<R, INV>(v[q]);
      const int d0 = (j / NS) * NS * R + (j % NS);
#pragma unroll
      for (int r = 0; r < R; ++r) st(b, d0 + r * NS, v[q][r]);
    }
  }
}

template <int L, int P, int NS, int NCOL, int NT, bool COLMODE, bool INV, class LD, class ST>
__device__ __forceinline__ void fft_passes(float2* s, const LD& ld, const ST& st, const float2* __restrict__ tw,
                                           int twstride) {
  constexpr int NP = fft_npass(L);
  constexpr int R = 1 << fft_pass_bits(L, P);
  constexpr bool first = (P == 0), last = (P == NP - 1);
  using SL = SmemLd<L, NCOL, COLMODE>;
  using SS = SmemSt<L, NCOL, COLMODE>;
  if constexpr (first && last) {
    fft_pass<L, R, NS, NCOL, NT, COLMODE, INV>(ld, st, tw, twstride);
  } else if constexpr (first) {
    fft_pass<L, R, NS, NCOL, NT, COLMODE, INV>(ld, SS{s}, tw, twstride);
    __syncthreads();
    fft_passes<L, P + 1, NS * R, NCOL, NT, COLMODE, INV>(s, ld, st, tw, twstride);
  } else if constexpr (last) {
    fft_pass<L, R, NS, NCOL, NT, COLMODE, INV>(SL{s}, st, tw, twstride);
  } else {
    fft_pass<L, R, NS, NCOL, NT, COLMODE, INV>(SL{s}, SS{s}, tw, twstride);
    __syncthreads();
    fft_passes<L, P + 1, NS * R, NCOL, NT, COLMODE, INV>(s, ld, st, tw, twstride);
  }
}

// Transform NCOL columns of length L.  ld(b, i) supplies input element i of
// column b; st(b, i, v) receives output element i.  s is the smem tile
// (NCOL * L float2); the caller must __syncthreads() before reusing s.
// twstride = Lmax / L.  L == 1 is the identity.
template <int L, int NCOL, int NT, bool COLMODE, bool INV, class LD, class ST>
__device__ __forceinline__ void fft_tile(float2* s, const LD& ld, const ST& st, const float2* __restrict__ tw,
                                         int twstride) {
  if constexpr (L == 1) {
    for (int b = threadIdx.x; b < NCOL; b += NT) st(b, 0, ld(b, 0));
  } else {
    fft_passes<L, 0, 1, NCOL, NT, COLMODE, INV>(s, ld, st, tw, twstride);
  }
}

}  // namespace grace
