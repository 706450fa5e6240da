// Pencil convolution along one axis (FFT, k-space 3x3 multiply, inverse FFT),
// shared by the step kernels (K3, K2') and the small-grid cluster step.
// (The k-space multiply of P:L55's convolution theorem, with the kernel
// spectrum folded to one octant: DESIGN.md §6.)
#pragma once
#include <cuda_runtime.h>

#include <type_traits>

#include "fft_engine.cuh"

namespace grace {

// k-space multiply with the CTA's folded KS slice staged in smem:
// kss[c][kf][b], c = 0..5 (xx xy xz yy yz zz), kf the folded index of the
// staged axis.  fy / fz: the k index was folded along y / z, which flips the
// sign of the components odd in that axis (xy, yz odd in y; xz, yz odd in z).
__device__ __forceinline__ void kmul_s(float2& a, float2& b, float2& c, const float* kss, int KH, int B, int kf,
                                       int bcol, bool fy, bool fz) {
  const int cs = KH * B;
  const float* p = kss + kf * B + bcol;
  const float nxx = p[0], nyy = p[3 * cs], nzz = p[5 * cs];
  const float nxy = fy ? -p[cs] : p[cs];
  const float nxz = fz ? -p[2 * cs] : p[2 * cs];
  const float nyz = (fy != fz) ? -p[4 * cs] : p[4 * cs];
  const float2 mx = a, my = b, mz = c;
  a = make_float2(nxx * mx.x + nxy * my.x + nxz * mz.x, nxx * mx.y + nxy * my.y + nxz * mz.y);
  b = make_float2(nxy * mx.x + nyy * my.x + nyz * mz.x, nxy * mx.y + nyy * my.y + nyz * mz.y);
  c = make_float2(nxz * mx.x + nyz * my.x + nzz * mz.x, nxz * mx.y + nyz * my.y + nzz * mz.y);
}

// The same multiply with the fold signs known at compile time (the fused
// pencils' last-pass element index decides the pencil-axis fold per register;
// the other axis' fold is uniform per call): the negations fold into the FMAs.
template <bool FY, bool FZ>
__device__ __forceinline__ void kmul_c(float2& a, float2& b, float2& c, const float* kss, int KH, int B, int kf,
                                       int bcol) {
  const int cs = KH * B;
  const float* p = kss + kf * B + bcol;
  const float nxx = p[0], nyy = p[3 * cs], nzz = p[5 * cs];
  const float nxy = FY ? -p[cs] : p[cs];
  const float nxz = FZ ? -p[2 * cs] : p[2 * cs];
  const float nyz = (FY != FZ) ? -p[4 * cs] : p[4 * cs];
  const float2 mx = a, my = b, mz = c;
  a = make_float2(nxx * mx.x + nxy * my.x + nxz * mz.x, nxx * mx.y + nxy * my.y + nxz * mz.y);
  b = make_float2(nxy * mx.x + nyy * my.x + nyz * mz.x, nxy * mx.y + nyy * my.y + nyz * mz.y);
  c = make_float2(nxz * mx.x + nyz * my.x + nzz * mz.x, nxz * mx.y + nyz * my.y + nzz * mz.y);
}

// FFT along one pencil axis of the three components, H~ = KS . M~, inverse FFT.
// The forward input has n nonzero of L (HIN), the inverse keeps n outputs (HOUT).
// FUSE (L <= 64): the forward last pass, the multiply and the inverse first pass
// (reversed radix plan) run in registers without a shared-memory round trip.
#ifndef GRACE_ZB
#define GRACE_ZB 16  // kx columns per K3 / K2' CTA (at most, except short pencils)
#endif
#ifndef GRACE_Z_MINNT
#define GRACE_Z_MINNT 128
#endif
#ifndef GRACE_ZB_128
#define GRACE_ZB_128 16
#endif
#ifndef GRACE_ZB_256
#define GRACE_ZB_256 4
#endif
#ifndef GRACE_ZB_512
#define GRACE_ZB_512 8
#endif
template <int L>
struct ZPlan {
  static constexpr bool FUSE = L >= 2 && L <= 64;
  static constexpr int RB = rb_for(true, 3, L);  // radix bits of the three-component pencil plans
  static constexpr int RLAST = L <= 1 ? 1 : 1 << fft_pass_bits(L, fft_npass(L, RB) - 1, RB);
  // threads per column, unfused: L / R for the plan's largest radix R up to
  // L = 512, so no pass leaves threads idle (L / 8 idled half of them in the
  // radix-16 passes: 128^3 cube K3 0.32 -> 0.17 ms, block 17.9 -> 12.1 ms);
  // L / 8 for L = 1024 (16.8.8: more threads beat the idle pass, 20.7 vs 23.0 ms)
  static constexpr int R0 = L <= 1 ? 1 : 1 << fft_pass_bits(L, 0, RB);
  static constexpr int TPC = L <= 1 ? 1 : (FUSE ? L / RLAST : (L <= 512 ? L / R0 : L / 8));
  // fused (short) pencils: at least GRACE_Z_MINNT threads per CTA; unfused:
  // GRACE_Z_ELEMS values per component per CTA (smem: 3 components resident)
  static constexpr int BF = (GRACE_Z_MINNT / TPC > GRACE_ZB ? GRACE_Z_MINNT / TPC : GRACE_ZB);
  // unfused columns per CTA by length, measured (K3 ms): L = 128 16 (block
  // 2048x2048x64: 12.1 vs 15.9 at 8; the 64^3 cube prefers 8, 0.021 vs 0.025);
  // L = 256 (128^3) 4 (0.17, same at 8); L = 512 (256^3) 8 (1.45 vs 1.50 at 4,
  // 2.17 at 2); L = 1024 (512^3) 4 (20.7 vs 26.9 at 2)
  static constexpr int BN = L <= 128 ? GRACE_ZB_128 : (L == 256 ? GRACE_ZB_256 : (L == 512 ? GRACE_ZB_512 : (L == 1024 ? 4 : (2048 / L > 1 ? 2048 / L : 1))));
  static constexpr int B = L <= 1 ? GRACE_ZB : (FUSE ? (BF < 2048 / L ? BF : 2048 / L) : BN);
  static constexpr int NT = B * TPC < 32 ? 32 : B * TPC;
};

template <int L>
__host__ __device__ constexpr int pencil_tw_elems() {
  constexpr int RB = ZPlan<L>::RB;
  return ZPlan<L>::FUSE ? Plan<L, false, RB>::TW_ELEMS + Plan<L, true, RB>::TW_ELEMS : Plan<L, false, RB>::TW_ELEMS;
}
// Fill the shared table pencil_conv<..., TWS = true> reads (threads [tid, nt)).
template <int L>
__device__ __forceinline__ void fill_pencil_twiddles(float2* dst, const float2* __restrict__ tw, int twstride, int tid,
                                                     int nt) {
  constexpr int RB = ZPlan<L>::RB;
  fill_pass_twiddles<Plan<L, false, RB>, L>(dst, tw, twstride, tid, nt);
  if constexpr (ZPlan<L>::FUSE)
    fill_pass_twiddles<Plan<L, true, RB>, L>(dst + Plan<L, false, RB>::TW_ELEMS, tw, twstride, tid, nt);
}

// kw(): called before the multiply's barrier -- waits for this thread's part of
// the KS slice (cp.async group or TMA mbarrier).
// TWS: tw is a shared table of per-pass twiddles (fill_pass_twiddles): for fused
// plans the forward plan's followed by the reversed (inverse) plan's (Plan<L, false>
// then Plan<L, true>), for unfused ones the forward plan's alone (both directions
// run it); else tw is the global table.  pencil_tw_elems<L>() sizes it.
template <int L, int B, int NT, bool TWS = false, class LD, class ST, class KW>
__device__ __forceinline__ void pencil_conv(float2* smem, const LD& ld, const ST& st, const float* kss, int KH,
                                            const float2* __restrict__ tw, int twstride, int P_other, int k_other,
                                            bool fold_is_y, const KW& kw) {
  // k along the pencil axis (length L = P_axis); the other folded axis index is
  // fixed for the CTA.  fold_is_y: the pencil axis is y (K2'), else z (K3).
  auto flags = [&](int k, bool& fy, bool& fz, int& kf) {
    const bool fa = k > (L >> 1);
    kf = fa ? L - k : k;
    const bool fo = k_other > (P_other >> 1);
    if (fold_is_y) {
      fy = fa;
      fz = false;
    } else {
      fy = fo;
      fz = fa;
    }
  };
  const ThreadMap<L, B, NT, true> tm;
  if constexpr (ZPlan<L>::FUSE) {
    using PF = Pass<L, fft_npass(L, ZPlan<L>::RB) - 1, false, B, NT, true, 3>;
    using PI = Pass<L, 0, true, B, NT, true, 3>;
    static_assert(PF::R == PI::R && PF::UPT == 1 && PI::UPT == 1, "fused plan");
    PF pf;
    const float2* twi = TWS ? tw + Plan<L, false, ZPlan<L>::RB>::TW_ELEMS : tw;
    fft_to_regs<L, B, NT, true, 3, false, true, false, false, TWS>(tm, smem, ld, tw, twstride, pf);
    kw();
    __syncthreads();
    PI pi;
    // The last forward pass leaves element k = jb + r NS in register r (jb < NS =
    // L / R), so k > L/2 exactly for r > R/2, and for r = R/2 except at k = L/2,
    // the Nyquist index, where folding maps kf to itself and the odd components
    // of the spectrum vanish (their circulant sequences are odd): the fold of the
    // pencil axis is r >= R/2, known at compile time once the loop is unrolled.
    static_assert(PF::NS == PF::TPC || PF::NS == 1, "fused last pass: one element per register and NS");
    auto mul = [&](auto fo_tag) {
      constexpr bool FO = decltype(fo_tag)::value;
#pragma unroll
      for (int r = 0; r < PF::R; ++r) {
        const int k = PF::sb(tm) + PF::C2(0, r);
        const bool fa = r >= PF::R / 2;
        const int kf = fa ? L - k : k;
        float2 a = pf.v[0][0][r], b = pf.v[0][1][r], c = pf.v[0][2][r];
        if (fold_is_y) {
          if (fa) kmul_c<true, false>(a, b, c, kss, KH, B, kf, tm.b);
          else kmul_c<false, false>(a, b, c, kss, KH, B, kf, tm.b);
        } else {
          if (fa) kmul_c<FO, true>(a, b, c, kss, KH, B, kf, tm.b);
          else kmul_c<FO, false>(a, b, c, kss, KH, B, kf, tm.b);
        }
        pi.v[0][0][r] = a;
        pi.v[0][1][r] = b;
        pi.v[0][2][r] = c;
      }
    };
    if (!fold_is_y && k_other > (P_other >> 1)) mul(std::true_type{});
    else mul(std::false_type{});
    fft_from_regs<L, B, NT, true, 3, true, true, true, TWS>(tm, smem, st, twi, twstride, pi);
  } else {
    using T = TileIdx<L, B, true>;
    fft_tile<L, B, NT, true, false, (L > 1), false, 3, false, TWS>(smem, ld, SmemSt<L, B, true>{smem}, tw, twstride);
    kw();
    __syncthreads();
    for (int u = threadIdx.x; u < L * B; u += NT) {
      const int k = u / B, b = u - k * B;
      bool fy, fz;
      int kf;
      flags(k, fy, fz, kf);
      float2* s0 = smem + T::at(b, k);
      float2 a = s0[0], bb = s0[T::ELEMS], c = s0[2 * T::ELEMS];
      kmul_s(a, bb, c, kss, KH, B, kf, b, fy, fz);
      s0[0] = a;
      s0[T::ELEMS] = bb;
      s0[2 * T::ELEMS] = c;
    }
    __syncthreads();
    fft_tile<L, B, NT, true, true, false, (L > 1), 3, false, TWS>(smem, SmemLd<L, B, true>{smem}, st, tw, twstride);
  }
}

}  // namespace grace
