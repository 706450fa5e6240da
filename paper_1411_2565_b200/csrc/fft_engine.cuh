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
// Radix plan: npass = ceil(log2 L / RB) passes, bits spread as evenly as possible
// (larger radices first); RB = 4 allows radix 16, RB = 3 caps the radix at 8.
__host__ __device__ constexpr int fft_npass(int L, int RB = 4) { return (ilog2(L) + RB - 1) / RB; }
__host__ __device__ constexpr int fft_pass_bits(int L, int p, int RB = 4) {
  return ilog2(L) / fft_npass(L, RB) + (p < ilog2(L) % fft_npass(L, RB) ? 1 : 0);
}
// product of the radices of passes < p
__host__ __device__ constexpr int fft_ns(int L, int p, int RB = 4) {
  return p == 0 ? 1 : fft_ns(L, p - 1, RB) << fft_pass_bits(L, p - 1, RB);
}
__host__ __device__ constexpr int fft_rmax(int L, int RB = 4) { return L <= 1 ? 1 : 1 << fft_pass_bits(L, 0, RB); }
// Radix cap of row-mode kernels that carry the three components per thread.  A
// radix-16 pass leaves half of their threads idle, but capping at 8 (one more
// smem pass) measured slower on the slab (K1 0.431 vs 0.409 ms), so the default
// keeps radix 16; the knob stays for other shapes.
#ifndef GRACE_RB_ROWS3
#define GRACE_RB_ROWS3 4
#endif
// Column-mode three-component 16-point pencils (the film's and 8^3 cubes' z axis):
// radix 4 x 4 (four threads per pencil, 12 complex values each) instead of one
// radix-16 pass (one thread per pencil holding 48: 168 registers, 8 warps/SM).
#ifndef GRACE_RB_Z16
#define GRACE_RB_Z16 2
#endif
#ifndef GRACE_RB_Z64
#define GRACE_RB_Z64 4
#endif
__host__ __device__ constexpr int rb_for(bool colmode, int V, int L = 0) {
  return (!colmode && V == 3) ? GRACE_RB_ROWS3
                              : ((colmode && V == 3 && L == 16) ? GRACE_RB_Z16
                                                                : ((colmode && V == 3 && L == 64) ? GRACE_RB_Z64 : 4));
}

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

// Radix plan of an L-point transform; REV runs the same radices in reverse
// order (an inverse that starts with the forward's last radix keeps every
// thread's elements in place across a fused forward-last / inverse-first pass).
template <int L, bool REV, int RB = 4>
struct Plan {
  static constexpr int NP = fft_npass(L, RB);
  __host__ __device__ static constexpr int bits(int p) { return fft_pass_bits(L, REV ? NP - 1 - p : p, RB); }
  __host__ __device__ static constexpr int R(int p) { return 1 << bits(p); }
  __host__ __device__ static constexpr int NS(int p) { return p == 0 ? 1 : NS(p - 1) * R(p - 1); }
  // per-pass twiddle tables: pass p >= 1 holds w_{NS R}^{jm r} at [r][jm], R(p) NS(p) entries
  __host__ __device__ static constexpr int twoff(int p) { return p <= 1 ? 0 : twoff(p - 1) + R(p - 1) * NS(p - 1); }
  static constexpr int TW_ELEMS = twoff(NP);
};

// Fill the per-pass twiddle tables of Plan PL from the global table w_Lmax^k
// (tw, twstride = Lmax / L) with threads [tid, nt).
template <class PL, int L>
__device__ __forceinline__ void fill_pass_twiddles(float2* dst, const float2* __restrict__ tw, int twstride, int tid,
                                                   int nt) {
#pragma unroll
  for (int p = 1; p < PL::NP; ++p) {
    const int R = PL::R(p), NS = PL::NS(p);
    for (int e = tid; e < R * NS; e += nt) {
      const int r = e / NS, jm = e - r * NS;
      dst[PL::twoff(p) + e] = __ldg(tw + ((jm * r * (L / (NS * R))) % L) * twstride);
    }
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
// fold into immediates.  V components are V consecutive tiles of ELEMS each.
template <int L, int NCOL, bool COLMODE, int R0 = fft_rmax(L)>
struct TileIdx {
  static constexpr int R0v = R0;
  static constexpr int SH = ilog2(R0);
  static constexpr bool PAD = (L >= 16) && (COLMODE ? NCOL < 16 : true);
  static constexpr int RS = COLMODE ? NCOL : 1;
  // rows reserved per column: enough for the padding of either radix order
  // (the smallest radix of the plan pads the most)
  static constexpr int RMIN4 = L <= 1 ? 1 : 1 << fft_pass_bits(L, fft_npass(L, 4) - 1, 4);
  static constexpr int RBR = GRACE_RB_ROWS3;  // row-mode V = 3 plans (see rb_for)
  static constexpr int RMINR = L <= 1 ? 1 : 1 << fft_pass_bits(L, fft_npass(L, RBR) - 1, RBR);
  static constexpr int RMIN = COLMODE ? RMIN4 : (RMINR < RMIN4 ? RMINR : RMIN4);
  static constexpr int ROWS = L + (PAD ? L / RMIN : 0);
  static constexpr int ELEMS = NCOL * ROWS;
  static constexpr int SMEM_ELEMS = ELEMS;
  static constexpr int CS = COLMODE ? 1 : ROWS;
  __device__ __forceinline__ static int at(int b, int i) { return b * CS + i * RS; }  // linear
  __device__ __forceinline__ static int padrow(int i) { return PAD ? i + (i >> SH) : i; }
};

// Caller-visible smem accessors (linear layout, component v in tile v).
// Interface of all accessors: element i = ib + C of component v of column b,
// ib per thread, C a compile-time constant after unrolling.
template <int L, int NCOL, bool COLMODE>
struct SmemLd {
  __device__ static constexpr bool kSmem() { return true; }
  float2* s;
  __device__ __forceinline__ float2 operator()(int b, int v, int ib, int C) const {
    using T = TileIdx<L, NCOL, COLMODE>;
    return s[v * T::ELEMS + T::at(b, ib) + C * T::RS];
  }
};
template <int L, int NCOL, bool COLMODE>
struct SmemSt {
  __device__ static constexpr bool kSmem() { return true; }
  float2* s;
  __device__ __forceinline__ void operator()(int b, int v, int ib, int C, float2 x) const {
    using T = TileIdx<L, NCOL, COLMODE>;
    s[v * T::ELEMS + T::at(b, ib) + C * T::RS] = x;
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

// twiddle read from a shared-memory table
__device__ __forceinline__ float2 tw_lds(const float2* p) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];\n"
               : "=f"(v.x), "=f"(v.y)
               : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}

// One Stockham pass P of an L-point transform (plan REV) over V components per
// thread.  The pieces (load / compute / store) are exposed so kernels can fuse
// work between passes (K3: forward last pass -> k-space multiply -> inverse
// first pass, all in registers).
template <int L, int P, bool REV, int NCOL, int NT, bool COLMODE, int V>
struct Pass {
  static constexpr int RB = rb_for(COLMODE, V, L);
  using PL = Plan<L, REV, RB>;
  using TM = ThreadMap<L, NCOL, NT, COLMODE>;
  using T = TileIdx<L, NCOL, COLMODE, PL::R(0)>;
  static constexpr int R = PL::R(P);
  static constexpr int NS = PL::NS(P);
  static constexpr int JR = L / R;
  static constexpr int TPC = NT / NCOL;
  static_assert(JR % TPC == 0 || TPC % JR == 0, "pow2 mapping");
  static constexpr int UPT = JR >= TPC ? JR / TPC : 1;
  static constexpr bool SPLIT = ((UPT == 1) || (TPC % T::R0v == 0)) && (JR % T::R0v == 0);

  float2 v[UPT][V][R];

  __device__ __forceinline__ static bool active(const TM& tm) { return (JR >= TPC) || tm.jb < JR; }
  // input element of unit (q, r): i = jb + q TPC + r JR
  __device__ __forceinline__ static constexpr int Cin(int q, int r) { return q * TPC + r * JR; }
  // j mod Ns of unit q
  __device__ __forceinline__ static int jm(const TM& tm, int q) {
    if constexpr (NS <= TPC) return tm.jb % NS;
    else return tm.jb + TPC * (q % (NS / TPC));
  }
  // output element of unit (q, r): d = sb + C2
  __device__ __forceinline__ static int sb(const TM& tm) {
    if constexpr (NS <= TPC) return (tm.jb / NS) * NS * R + tm.jb % NS;
    else return tm.jb;
  }
  __device__ __forceinline__ static constexpr int C2(int q, int r) {
    if constexpr (NS <= TPC) return q * TPC * R + r * NS;
    else return TPC * (q % (NS / TPC)) + (q / (NS / TPC)) * NS * R + r * NS;
  }

  template <int RIN, class LD>
  __device__ __forceinline__ void load_ext(const TM& tm, const LD& ld) {
#pragma unroll
    for (int q = 0; q < UPT; ++q)
#pragma unroll
      for (int w = 0; w < V; ++w)
#pragma unroll
        for (int r = 0; r < RIN; ++r) v[q][w][r] = ld(tm.b, w, tm.jb, Cin(q, r));
  }
  template <int RIN, bool PADDED>
  __device__ __forceinline__ void load_smem(const TM& tm, const float2* s) {
    const int lin0 = T::at(tm.b, tm.jb);
    const int pad0 = T::at(tm.b, T::padrow(tm.jb));
#pragma unroll
    for (int q = 0; q < UPT; ++q)
#pragma unroll
      for (int w = 0; w < V; ++w)
#pragma unroll
        for (int r = 0; r < RIN; ++r) {
          const int C = Cin(q, r);
          if constexpr (!PADDED || !T::PAD) v[q][w][r] = s[w * T::ELEMS + lin0 + C * T::RS];
          else if constexpr (SPLIT) v[q][w][r] = s[w * T::ELEMS + pad0 + (C + (C >> T::SH)) * T::RS];
          else v[q][w][r] = s[w * T::ELEMS + T::at(tm.b, T::padrow(tm.jb + C))];
        }
  }
  template <bool INV, bool HIN, bool HOUT, bool TWS = false>
  __device__ __forceinline__ void compute(const TM& tm, const float2* __restrict__ tw, int twstride) {
    constexpr int RIN = HIN ? R / 2 : R;
#pragma unroll
    for (int q = 0; q < UPT; ++q) {
      if constexpr (NS > 1) {
        const int jmq = jm(tm, q);
        const int k1 = jmq * ((L / (NS * R)) * twstride);
#pragma unroll
        for (int r = 1; r < RIN; ++r) {
          // TWS: per-pass shared table [r][jm] (consecutive lanes -> consecutive words)
          const float2 t = TWS ? tw_lds(tw + PL::twoff(P) + r * NS + jmq) : __ldg(tw + k1 * r);
#pragma unroll
          for (int w = 0; w < V; ++w) v[q][w][r] = INV ? cmulc(v[q][w][r], t) : cmul(v[q][w][r], t);
        }
      }
#pragma unroll
      for (int w = 0; w < V; ++w) {
        if constexpr (HIN) dft_halfzero<R, INV>(v[q][w]);
        else if constexpr (HOUT) dft_halfout<R, INV>(v[q][w]);
        else dft_inplace<R, INV>(v[q][w]);
      }
    }
  }
  template <int ROUT, class ST>
  __device__ __forceinline__ void store_ext(const TM& tm, const ST& st) {
    const int b0 = sb(tm);
#pragma unroll
    for (int q = 0; q < UPT; ++q)
#pragma unroll
      for (int w = 0; w < V; ++w)
#pragma unroll
        for (int r = 0; r < ROUT; ++r) st(tm.b, w, b0, C2(q, r), v[q][w][r]);
  }
  template <int ROUT, bool PADDED>
  __device__ __forceinline__ void store_smem(const TM& tm, float2* s) {
    static_assert(!PADDED || NS == 1, "only pass 0 writes the padded interface");
    const int lin1 = T::at(tm.b, sb(tm));
    const int pad1 = T::at(tm.b, tm.jb * (R + 1));
#pragma unroll
    for (int q = 0; q < UPT; ++q)
#pragma unroll
      for (int w = 0; w < V; ++w)
#pragma unroll
        for (int r = 0; r < ROUT; ++r) {
          if constexpr (!PADDED || !T::PAD) s[w * T::ELEMS + lin1 + C2(q, r) * T::RS] = v[q][w][r];
          else s[w * T::ELEMS + pad1 + ((q * TPC) * (R + 1) + r) * T::RS] = v[q][w][r];  // d = (jb+qTPC)R + r
        }
  }
};

// Run pass P with sources/destinations SRC/DST (kExt functor, kLin / kPad smem).
template <int L, int P, bool REV, int NCOL, int NT, bool COLMODE, int V, bool INV, bool HIN, bool HOUT, int SRC,
          int DST, bool TWS = false, class LD, class ST>
__device__ __forceinline__ void fft_pass(const ThreadMap<L, NCOL, NT, COLMODE>& tm, const LD& ld, const ST& st,
                                         float2* s, const float2* __restrict__ tw, int twstride) {
  using PS = Pass<L, P, REV, NCOL, NT, COLMODE, V>;
  constexpr int RIN = HIN ? PS::R / 2 : PS::R;
  constexpr int ROUT = HOUT ? PS::R / 2 : PS::R;
  PS ps;
  const bool act = PS::active(tm);
  if (act) {
    if constexpr (SRC == kExt) ps.template load_ext<RIN>(tm, ld);
    else ps.template load_smem<RIN, SRC == kPad>(tm, s);
  }
  constexpr bool SRC_SMEM = (SRC != kExt) || LD::kSmem();
  constexpr bool DST_SMEM = (DST != kExt) || ST::kSmem();
  if constexpr (SRC_SMEM && DST_SMEM) __syncthreads();  // in-place hazard
  if (act) {
    ps.template compute<INV, HIN, HOUT, TWS>(tm, tw, twstride);
    if constexpr (DST == kExt) ps.template store_ext<ROUT>(tm, st);
    else ps.template store_smem<ROUT, DST == kPad>(tm, s);
  }
}

template <int L, int P, bool REV, int NCOL, int NT, bool COLMODE, int V, bool INV, bool HIN, bool HOUT, int SRC0,
          int DSTN, bool TWS = false, class LD, class ST>
__device__ __forceinline__ void fft_passes(const ThreadMap<L, NCOL, NT, COLMODE>& tm, float2* s, const LD& ld,
                                           const ST& st, const float2* __restrict__ tw, int twstride) {
  constexpr int RB = rb_for(COLMODE, V, L);
  constexpr int NP = fft_npass(L, RB);
  constexpr bool first = (P == 0), last = (P == NP - 1);
  constexpr int IFACE0 = TileIdx<L, NCOL, COLMODE, Plan<L, REV, RB>::R(0)>::PAD ? kPad : kLin;
  if constexpr (first && last) {
    fft_pass<L, P, REV, NCOL, NT, COLMODE, V, INV, HIN, HOUT, SRC0, DSTN, TWS>(tm, ld, st, s, tw, twstride);
  } else if constexpr (first) {
    fft_pass<L, P, REV, NCOL, NT, COLMODE, V, INV, HIN, false, SRC0, IFACE0, TWS>(tm, ld, st, s, tw, twstride);
    __syncthreads();
    fft_passes<L, P + 1, REV, NCOL, NT, COLMODE, V, INV, HIN, HOUT, SRC0, DSTN, TWS>(tm, s, ld, st, tw, twstride);
  } else {
    constexpr int SRCP = (P == 1) ? IFACE0 : kLin;
    if constexpr (last) {
      fft_pass<L, P, REV, NCOL, NT, COLMODE, V, INV, false, HOUT, SRCP, DSTN, TWS>(tm, ld, st, s, tw, twstride);
    } else {
      fft_pass<L, P, REV, NCOL, NT, COLMODE, V, INV, false, false, SRCP, kLin, TWS>(tm, ld, st, s, tw, twstride);
      __syncthreads();
      fft_passes<L, P + 1, REV, NCOL, NT, COLMODE, V, INV, HIN, HOUT, SRC0, DSTN, TWS>(tm, s, ld, st, tw, twstride);
    }
  }
}

// Passes P .. NH-1 of a transform, each writing the smem tile (pass 0 reads `ld`).
template <int L, int P, int NH, bool REV, int NCOL, int NT, bool COLMODE, int V, bool INV, bool HIN, bool TWS,
          class LD, class ST>
__device__ __forceinline__ void fft_head(const ThreadMap<L, NCOL, NT, COLMODE>& tm, float2* s, const LD& ld,
                                         const ST& none, const float2* __restrict__ tw, int twstride) {
  if constexpr (P < NH) {
    constexpr int RB = rb_for(COLMODE, V, L);
    constexpr int IFACE0 = TileIdx<L, NCOL, COLMODE, Plan<L, REV, RB>::R(0)>::PAD ? kPad : kLin;
    if constexpr (P == 0) {
      fft_pass<L, 0, REV, NCOL, NT, COLMODE, V, INV, HIN, false, kExt, IFACE0, TWS>(tm, ld, none, s, tw, twstride);
    } else {
      __syncthreads();
      fft_pass<L, P, REV, NCOL, NT, COLMODE, V, INV, false, false, (P == 1 ? IFACE0 : kLin), kLin, TWS>(
          tm, ld, none, s, tw, twstride);
    }
    fft_head<L, P + 1, NH, REV, NCOL, NT, COLMODE, V, INV, HIN, TWS>(tm, s, ld, none, tw, twstride);
  }
}

// Passes 0 .. NP-2 of a transform (the first from `ld`, writing the smem tile),
// then the last pass is loaded and computed into `ps` and left in registers:
// output element i = PS::sb(tm) + PS::C2(q, r) of component w is ps.v[q][w][r].
// TWS: `tw` is the per-pass shared twiddle table of Plan<L, REV> (fill_pass_twiddles), else the global table.
template <int L, int NCOL, int NT, bool COLMODE, int V, bool INV, bool HIN, bool HOUT, bool REV, bool TWS = false,
          class LD, class PS>
__device__ __forceinline__ void fft_to_regs(const ThreadMap<L, NCOL, NT, COLMODE>& tm, float2* s, const LD& ld,
                                            const float2* __restrict__ tw, int twstride, PS& ps) {
  constexpr int RB = rb_for(COLMODE, V, L);
  constexpr int NP = fft_npass(L, RB);
  constexpr int IFACE0 = TileIdx<L, NCOL, COLMODE, Plan<L, REV, RB>::R(0)>::PAD ? kPad : kLin;
  if constexpr (NP == 1) {
    if (PS::active(tm)) {
      ps.template load_ext<HIN ? PS::R / 2 : PS::R>(tm, ld);
      ps.template compute<INV, HIN, HOUT, TWS>(tm, tw, twstride);
    }
  } else {
    struct None {
      __device__ static constexpr bool kSmem() { return true; }
      __device__ void operator()(int, int, int, int, float2) const {}
    } none;
    fft_head<L, 0, NP - 1, REV, NCOL, NT, COLMODE, V, INV, HIN, TWS>(tm, s, ld, none, tw, twstride);
    __syncthreads();
    if (PS::active(tm)) {
      ps.template load_smem<PS::R, NP == 2 && IFACE0 == kPad>(tm, s);
      ps.template compute<INV, false, HOUT, TWS>(tm, tw, twstride);
    }
  }
}

// The counterpart: `ps` holds pass 0's inputs in registers (element
// i = jb + PS::Cin(q, r)); compute it, then the remaining passes, the last one
// writing through `st`.  The caller must __syncthreads() before if the smem
// tile is still being read.
template <int L, int NCOL, int NT, bool COLMODE, int V, bool INV, bool HOUT, bool REV, bool TWS = false, class ST,
          class PS>
__device__ __forceinline__ void fft_from_regs(const ThreadMap<L, NCOL, NT, COLMODE>& tm, float2* s, const ST& st,
                                              const float2* __restrict__ tw, int twstride, PS& ps) {
  constexpr int RB = rb_for(COLMODE, V, L);
  constexpr int NP = fft_npass(L, RB);
  constexpr int IFACE0 = TileIdx<L, NCOL, COLMODE, Plan<L, REV, RB>::R(0)>::PAD ? kPad : kLin;
  struct None {
    __device__ static constexpr bool kSmem() { return true; }
    __device__ float2 operator()(int, int, int, int) const { return make_float2(0.f, 0.f); }
  } none;
  if constexpr (NP == 1) {
    if (PS::active(tm)) {
      ps.template compute<INV, false, HOUT, TWS>(tm, tw, twstride);
      ps.template store_ext<HOUT ? PS::R / 2 : PS::R>(tm, st);
    }
  } else {
    if (PS::active(tm)) {
      ps.template compute<INV, false, false, TWS>(tm, tw, twstride);
      ps.template store_smem<PS::R, IFACE0 == kPad>(tm, s);
    }
    __syncthreads();
    fft_passes<L, 1, REV, NCOL, NT, COLMODE, V, INV, false, HOUT, kExt, kExt, TWS>(tm, s, none, st, tw, twstride);
  }
}

template <class T>
struct IsTileLd : std::false_type {};
template <int L, int N, bool C>
struct IsTileLd<SmemLd<L, N, C>> : std::true_type {};
template <class T>
struct IsTileSt : std::false_type {};
template <int L, int N, bool C>
struct IsTileSt<SmemSt<L, N, C>> : std::true_type {};

// Transform V components of NCOL columns of length L.  ld(b, v, ib, C) supplies
// input element i = ib + C of component v of column b (HIN: only i < L/2 is
// requested, the rest is zero); st(b, v, ib, C, x) receives output i = ib + C
// (HOUT: only i < L/2 is produced).  SmemLd/SmemSt as ld/st address the tile s
// itself (linear layout).  s holds V * TileIdx::ELEMS float2; the caller must
// __syncthreads() before reusing s.  twstride = Lmax / L.  L == 1 is the identity.
template <int L, int NCOL, int NT, bool COLMODE, bool INV, bool HIN = false, bool HOUT = false, int V = 1,
          bool REV = false, bool TWS = false, class LD, class ST>
__device__ __forceinline__ void fft_tile(float2* s, const LD& ld, const ST& st, const float2* __restrict__ tw,
                                         int twstride) {
  if constexpr (L == 1) {
    for (int b = threadIdx.x; b < NCOL; b += NT)
#pragma unroll
      for (int w = 0; w < V; ++w) st(b, w, 0, 0, ld(b, w, 0, 0));
  } else {
    const ThreadMap<L, NCOL, NT, COLMODE> tm;
    constexpr int SRC0 = IsTileLd<LD>::value ? kLin : kExt;
    constexpr int DSTN = IsTileSt<ST>::value ? kLin : kExt;
    fft_passes<L, 0, REV, NCOL, NT, COLMODE, V, INV, HIN, HOUT, SRC0, DSTN, TWS>(tm, s, ld, st, tw, twstride);
  }
}

}  // namespace grace
