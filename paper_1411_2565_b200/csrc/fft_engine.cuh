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
// intermediate passes run in place in shared memory.
//
// Thread mapping is fixed at compile time: each thread owns one column b and the
// butterflies j = jb + q*TPC (TPC = threads per column), so every shared-memory
// offset and twiddle index is a per-thread base plus a compile-time constant.
//   COLMODE = true : consecutive lanes take consecutive columns (columns are
//                    contiguous in HBM: y and z pencils).  smem (b, i) -> (i + pad(i))*NCOL + b,
//                    one pad row per R0 rows when NCOL < 16 (R0 = first radix).
//   COLMODE = false: consecutive lanes take consecutive butterflies of one column
//                    (the sequence is contiguous in HBM: x rows).  smem (b, i) ->
//                    b*LP + i + (i >> 4), LP = L + L/16 (one pad slot per 16).
// Zero-padding pruning: HIN (inputs i >= L/2 are zero) drops the first radix-2
// stage of pass 0; HOUT (only outputs i < L/2 are used) computes half of the
// last pass.  Twiddles w_Lmax^k = exp(-2 pi i k/Lmax) come from a global fp32
// table computed once in fp64; in-register DFT twiddles are constants.
#pragma once
#include <cuda_runtime.h>

#include <type_traits>

namespace grace {

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
  return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}

__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x / 2); }
__host__ __device__ constexpr int fft_npass(int L) { return (ilog2(L) + 3) / 4; }
__host__ __device__ constexpr int fft_pass_bits(int L, int p) {
  return ilog2(L) / fft_npass(L) + (p < ilog2(L) % fft_npass(L) ? 1 : 0);
}
// product of the radices of passes < p
__host__ __device__ constexpr int fft_ns(int L, int p) {
  return p == 0 ? 1 : fft_ns(L, p - 1) << fft_pass_bits(L, p - 1);
}
__host__ __device__ constexpr int fft_rmax(int L) { return L <= 1 ? 1 : 1 << fft_pass_bits(L, 0); }

// x * exp(-+2 pi i K/16) for compile-time K (forward sign -, INV conjugates).
template <bool INV, int K>
__device__ __forceinline__ float2 tw16_mul(float2 x) {
  constexpr int k = K & 15;
  if constexpr (k == 0) {
    return x;
  } else if constexpr (k == 4) {
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
    constexpr float s = INV ? C[(k + 12) & 15] : -C[(k + 12) & 15];
    return make_float2(x.x * c - x.y * s, x.x * s + x.y * c);
  }
}

template <bool INV, int R, int K>
__device__ __forceinline__ void dft_combine(float2* a, const float2* e, const float2* o) {
  if constexpr (K < R / 2) {
    const float2 t = tw16_mul<INV, K * (16 / R)>(o[K]);
    a[K] = cadd(e[K], t);
    a[K + R / 2] = csub(e[K], t);
    dft_combine<INV, R, K + 1>(a, e, o);
  }
}

// In-register DFT of size R (radix-2 decimation in time, natural order in and out).
template <int R, bool INV>
__device__ __forceinline__ void dft_inplace(float2* a) {
  if constexpr (R == 1) {
    return;
  } else if constexpr (R == 2) {
    const float2 t0 = a[0], t1 = a[1];
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

template <bool INV, int R, int K>
__device__ __forceinline__ void tw_range(float2* o) {  // o[K] *= w_R^K for K < R/2
  if constexpr (K < R / 2) {
    o[K] = tw16_mul<INV, K * (16 / R)>(o[K]);
    tw_range<INV, R, K + 1>(o);
  }
}

// DFT_R of a[0..R/2) followed by R/2 zeros (decimation-in-frequency first stage:
// X[2m] = DFT_{R/2}(a)[m], X[2m+1] = DFT_{R/2}(a w_R^r)[m]).
template <int R, bool INV>
__device__ __forceinline__ void dft_halfzero(float2* a) {
  if constexpr (R == 1) {
    return;
  } else {
    float2 e[R / 2], o[R / 2];
#pragma unroll
    for (int q = 0; q < R / 2; ++q) e[q] = o[q] = a[q];
    tw_range<INV, R, 0>(o);
    dft_inplace<R / 2, INV>(e);
    dft_inplace<R / 2, INV>(o);
#pragma unroll
    for (int q = 0; q < R / 2; ++q) {
      a[2 * q] = e[q];
      a[2 * q + 1] = o[q];
    }
  }
}

// First R/2 outputs of DFT_R(a) (the rest are discarded by the caller).
template <int R, bool INV>
__device__ __forceinline__ void dft_halfout(float2* a) {
  if constexpr (R <= 2) {
    dft_inplace<R, INV>(a);
  } else {
    float2 e[R / 2], o[R / 2];
#pragma unroll
    for (int q = 0; q < R / 2; ++q) {
      e[q] = a[2 * q];
      o[q] = a[2 * q + 1];
    }
    dft_inplace<R / 2, INV>(e);
    dft_inplace<R / 2, INV>(o);
    tw_range<INV, R, 0>(o);
#pragma unroll
    for (int q = 0; q < R / 2; ++q) a[q] = cadd(e[q], o[q]);
  }
}

// Shared-memory tile addressing.  A tile holds NCOL columns of ROWS rows; row
// stride RS and column stride CS depend on the mode:
//   COLMODE: element (b, row) at row*NCOL + b   (RS = NCOL, CS = 1)
//   rows   : element (b, row) at b*ROWS + row   (RS = 1,    CS = ROWS)
// The interface written by pass 0 (stride-R0 rows across lanes) is padded with
// one row per R0 rows ("PAD" layout, row(i) = i + i/R0) when that stride would
// hit one bank; every other interface, and the caller-visible layout used by
// SmemLd/SmemSt, is linear, so offsets of the compile-time butterfly pattern
// fold into immediates.
template <int L, int NCOL, bool COLMODE>
struct TileIdx {
  static constexpr int R0 = fft_rmax(L);
  static constexpr int SH = ilog2(R0);
  static constexpr bool PAD = (L >= 16) && (COLMODE ? NCOL < 16 : true);
  static constexpr int ROWS = L + (PAD ? L / R0 : 0);
  static constexpr int SMEM_ELEMS = NCOL * ROWS;
  static constexpr int RS = COLMODE ? NCOL : 1;
  static constexpr int CS = COLMODE ? 1 : ROWS;
  __device__ __forceinline__ static int at(int b, int i) { return b * CS + i * RS; }     // linear
  __device__ __forceinline__ static int padrow(int i) { return PAD ? i + (i >> SH) : i; }
};

// Caller-visible smem accessors (linear layout).  Interface of all accessors:
// element index i = ib + C, ib per thread, C a compile-time constant after unrolling.
template <int L, int NCOL, bool COLMODE>
struct SmemLd {
  __device__ static constexpr bool kSmem() { return true; }
  float2* s;
  __device__ __forceinline__ float2 operator()(int b, int ib, int C) const {
    return s[TileIdx<L, NCOL, COLMODE>::at(b, ib) + C * TileIdx<L, NCOL, COLMODE>::RS];
  }
};
template <int L, int NCOL, bool COLMODE>
struct SmemSt {
  __device__ static constexpr bool kSmem() { return true; }
  float2* s;
  __device__ __forceinline__ void operator()(int b, int ib, int C, float2 v) const {
    s[TileIdx<L, NCOL, COLMODE>::at(b, ib) + C * TileIdx<L, NCOL, COLMODE>::RS] = v;
  }
};

template <int L, int NCOL, int NT, bool COLMODE>
struct ThreadMap {
  static_assert(NT % NCOL == 0, "threads must divide evenly over columns");
  static constexpr int TPC = NT / NCOL;  // threads per column
  int b, jb;
  __device__ __forceinline__ ThreadMap() {
    if constexpr (COLMODE) {
      b = threadIdx.x % NCOL;
      jb = threadIdx.x / NCOL;
    } else {
      jb = threadIdx.x % TPC;
      b = threadIdx.x / TPC;
    }
  }
};

enum { kExt = 0, kLin = 1, kPad = 2 };  // where a pass reads from / writes to

template <class T>
struct IsTileLd : std::false_type {};
template <int L, int N, bool C>
struct IsTileLd<SmemLd<L, N, C>> : std::true_type {};
template <class T>
struct IsTileSt : std::false_type {};
template <int L, int N, bool C>
struct IsTileSt<SmemSt<L, N, C>> : std::true_type {};

// One Stockham pass P of an L-point transform.  SRC/DST: kExt = caller functor,
// kLin = linear smem tile, kPad = padded smem tile (the pass 0 -> 1 interface).
template <int L, int P, int NCOL, int NT, bool COLMODE, bool INV, bool HIN, bool HOUT, int SRC, int DST, class LD,
          class ST>
__device__ __forceinline__ void fft_pass(const ThreadMap<L, NCOL, NT, COLMODE>& tm, const LD& ld, const ST& st,
                                         float2* s, const float2* __restrict__ tw, int twstride) {
  using T = TileIdx<L, NCOL, COLMODE>;
  constexpr int R = 1 << fft_pass_bits(L, P);
  constexpr int NS = fft_ns(L, P);
  constexpr int JR = L / R;
  constexpr int TPC = NT / NCOL;
  static_assert(JR % TPC == 0 || TPC % JR == 0, "pow2 mapping");
  constexpr int UPT = JR >= TPC ? JR / TPC : 1;
  const bool active = (JR >= TPC) || tm.jb < JR;
  constexpr int RIN = HIN ? R / 2 : R;    // inputs loaded
  constexpr int ROUT = HOUT ? R / 2 : R;  // outputs stored
  static_assert(DST != kPad || NS == 1, "only pass 0 writes the padded interface");
  // loads: i = jb + C, C = q TPC + r JR
  constexpr bool SPLIT = ((UPT == 1) || (TPC % T::R0 == 0)) && (JR % T::R0 == 0);
  float2 v[UPT][R];
  if (active) {
    const int lin0 = T::at(tm.b, tm.jb);
    const int pad0 = T::at(tm.b, T::padrow(tm.jb));
#pragma unroll
    for (int q = 0; q < UPT; ++q) {
#pragma unroll
      for (int r = 0; r < RIN; ++r) {
        const int C = q * TPC + r * JR;
        if constexpr (SRC == kExt) {
          v[q][r] = ld(tm.b, tm.jb, C);
        } else if constexpr (SRC == kLin) {
          v[q][r] = s[lin0 + C * T::RS];
        } else if constexpr (SPLIT) {
          v[q][r] = s[pad0 + (C + (C >> T::SH)) * T::RS];
        } else {
          v[q][r] = s[T::at(tm.b, T::padrow(tm.jb + C))];
        }
      }
    }
  }
  constexpr bool SRC_SMEM = (SRC != kExt) || LD::kSmem();
  constexpr bool DST_SMEM = (DST != kExt) || ST::kSmem();
  if constexpr (SRC_SMEM && DST_SMEM) __syncthreads();  // in-place hazard
  if (active) {
    int sb;  // per-thread part of the output row d = sb + C2
    if constexpr (NS <= TPC) sb = (tm.jb / NS) * NS * R + tm.jb % NS;
    else sb = tm.jb;
    const int lin1 = T::at(tm.b, sb);
    const int pad1 = T::at(tm.b, tm.jb * (R + 1));
#pragma unroll
    for (int q = 0; q < UPT; ++q) {
      int jm;  // j mod Ns, j = jb + q TPC
      if constexpr (NS <= TPC) jm = tm.jb % NS;
      else jm = tm.jb + TPC * (q % (NS / TPC));
      if constexpr (NS > 1) {
        const int k1 = jm * ((L / (NS * R)) * twstride);
#pragma unroll
        for (int r = 1; r < RIN; ++r) {
          const float2 w = __ldg(tw + k1 * r);
          v[q][r] = INV ? cmulc(v[q][r], w) : cmul(v[q][r], w);
        }
      }
      if constexpr (HIN) dft_halfzero<R, INV>(v[q]);
      else if constexpr (HOUT) dft_halfout<R, INV>(v[q]);
      else dft_inplace<R, INV>(v[q]);
#pragma unroll
      for (int r = 0; r < ROUT; ++r) {
        int C2;
        if constexpr (NS <= TPC) C2 = q * TPC * R + r * NS;
        else C2 = TPC * (q % (NS / TPC)) + (q / (NS / TPC)) * NS * R + r * NS;
        if constexpr (DST == kExt) {
          st(tm.b, sb, C2, v[q][r]);
        } else if constexpr (DST == kLin) {
          s[lin1 + C2 * T::RS] = v[q][r];
        } else {
          // pass 0 (NS = 1): d = (jb + q TPC) R + r, padded row = (jb + q TPC)(R+1) + r
          s[pad1 + ((q * TPC) * (R + 1) + r) * T::RS] = v[q][r];
        }
      }
    }
  }
}

template <int L, int P, int NCOL, int NT, bool COLMODE, bool INV, bool HIN, bool HOUT, int SRC0, int DSTN, class LD,
          class ST>
__device__ __forceinline__ void fft_passes(const ThreadMap<L, NCOL, NT, COLMODE>& tm, float2* s, const LD& ld,
                                           const ST& st, const float2* __restrict__ tw, int twstride) {
  constexpr int NP = fft_npass(L);
  constexpr bool first = (P == 0), last = (P == NP - 1);
  constexpr int IFACE0 = TileIdx<L, NCOL, COLMODE>::PAD ? kPad : kLin;
  if constexpr (first && last) {
    fft_pass<L, P, NCOL, NT, COLMODE, INV, HIN, HOUT, SRC0, DSTN>(tm, ld, st, s, tw, twstride);
  } else if constexpr (first) {
    fft_pass<L, P, NCOL, NT, COLMODE, INV, HIN, false, SRC0, IFACE0>(tm, ld, st, s, tw, twstride);
    __syncthreads();
    fft_passes<L, P + 1, NCOL, NT, COLMODE, INV, HIN, HOUT, SRC0, DSTN>(tm, s, ld, st, tw, twstride);
  } else {
    constexpr int SRCP = (P == 1) ? IFACE0 : kLin;
    if constexpr (last) {
      fft_pass<L, P, NCOL, NT, COLMODE, INV, false, HOUT, SRCP, DSTN>(tm, ld, st, s, tw, twstride);
    } else {
      fft_pass<L, P, NCOL, NT, COLMODE, INV, false, false, SRCP, kLin>(tm, ld, st, s, tw, twstride);
      __syncthreads();
      fft_passes<L, P + 1, NCOL, NT, COLMODE, INV, HIN, HOUT, SRC0, DSTN>(tm, s, ld, st, tw, twstride);
    }
  }
}

// Transform NCOL columns of length L.  ld(b, ib, C) supplies input element
// i = ib + C of column b (HIN: only i < L/2 is requested, the rest is zero);
// st(b, ib, C, v) receives output i = ib + C (HOUT: only i < L/2 is produced).
// SmemLd/SmemSt as ld/st address the tile s itself (linear layout).  s holds
// TileIdx::SMEM_ELEMS float2; the caller must __syncthreads() before reusing s.
// twstride = Lmax / L.  L == 1 is the identity.
template <int L, int NCOL, int NT, bool COLMODE, bool INV, bool HIN = false, bool HOUT = false, class LD, class ST>
__device__ __forceinline__ void fft_tile(float2* s, const LD& ld, const ST& st, const float2* __restrict__ tw,
                                         int twstride) {
  if constexpr (L == 1) {
    for (int b = threadIdx.x; b < NCOL; b += NT) st(b, 0, 0, ld(b, 0, 0));
  } else {
    const ThreadMap<L, NCOL, NT, COLMODE> tm;
    constexpr int SRC0 = IsTileLd<LD>::value ? kLin : kExt;
    constexpr int DSTN = IsTileSt<ST>::value ? kLin : kExt;
    fft_passes<L, 0, NCOL, NT, COLMODE, INV, HIN, HOUT, SRC0, DSTN>(tm, s, ld, st, tw, twstride);
  }
}

}  // namespace grace
