// Per-step kernels K1..K5 of the LLG hot path (sm_100a, fp32) and small utilities.
//
// The step for M[3][nz][ny][nx] (x fastest, SoA):
//   K1  x-R2C of the zero-padded rows           M  -> X1 [3][nz][ny][Kxp]       (P:L55 FFT, zero padding)
//   K2  y-FFT (pruned: ny of Py inputs nonzero)  X1 -> X2 [3][nz][Py][Kxp]
//   K3  z-FFT, H~ = KS . M~ (6 real folded comps), inverse z, keep z < nz   X2 -> X2
//   K4  inverse y, keep y < ny                   X2 -> X1
//   K5  inverse x C2R (keep x < nx) = H_demag                X1 -> Hd
//   K6  six-neighbour exchange + x anisotropy + Zeeman (Eq. (2)), Eq. (3) LLG,
//       Euler + renormalise                                 Hd, M -> M'
// nz == 1 (thin films, SP4): K2' fuses y-FFT, multiply and inverse y in one
// CTA (the z axis is unpadded), so the step is K1, K2', K5, K6.
// The 1/(Px Py Pz) normalisation and the minus sign of H = -N*M live in KS.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>
#include <utility>
#include <cstring>
#include <type_traits>

#include "fft_engine.cuh"
#include "internal.h"
#include "pencil.cuh"

namespace grace {

// Occupancy target per block size: at most ~64 registers per thread.
#define GRACE_MINB(NT) ((NT) <= 256 ? 4 : ((NT) <= 512 ? 2 : 1))

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

// ---- TMA + mbarrier (sm_90+ async proxy) ----
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// Programmatic dependent launch (PDL): each step kernel lets the next one be
// scheduled as soon as all of its own CTAs are resident; the next kernel runs
// its input-independent prologue (twiddle tables, barriers, the KS slice) and
// then waits here for this grid's completion and memory flush.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], "
      "[%2];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// expect tx bytes on the barrier's current phase without arriving
__device__ __forceinline__ void mbar_expect_tx_only(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// TMA tensor store from shared memory (bulk async-group completion) and its waits
__device__ __forceinline__ void tma_store_5d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3,
                                             int c4) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];\n" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
               : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];\n" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// ---------------------------------------------------------------------------
// K1: x R2C.  A real row of Px (nx nonzero) is packed as z[n] = x[2n] + i x[2n+1],
// a length-L = Px/2 complex FFT gives Z, and
//   X[k] = (Z[k] + conj Z[L-k])/2 - (i/2) w^k (Z[k] - conj Z[L-k]),  w = exp(-2 pi i/Px), k = 0..L.
// The three components of a spatial row are transformed by the same thread
// (V = 3: shared twiddles and indexing).
template <int L, int B, int NT, int MINB, bool DIST>
__global__ void __launch_bounds__(NT, MINB) k1_fwd_x(const float* __restrict__ M, float2* __restrict__ X1,
                                                     const float2* __restrict__ tw, Geom g, StepParams* bump) {
  extern __shared__ float2 smem[];
  pdl_trigger();
  pdl_wait();
  // The step index lives on the device so captured graphs stay valid: K1 of each
  // step advances it, K5 of the same step reads step - 1.
  if (bump != nullptr && blockIdx.x == 0 && threadIdx.x == 0) bump->step += 1;
  const int nrows = g.nzl * g.ny;  // spatial rows of this slab
  const int row0 = blockIdx.x * B;
  const size_t N = (size_t)nrows * g.nx;
  auto out = [&](int c, int row, int k) -> size_t {
    if constexpr (DIST) {  // destination-blocked for the all-to-all: block k / kb
      const int q = k / g.kb;
      return q * g.blk1 + ((size_t)c * nrows + row) * g.pitch1 + (k - q * g.kb);
    } else {
      return ((size_t)c * nrows + row) * g.pitch1 + k;
    }
  };
  if constexpr (L == 0) {  // Px == 1: X[0] = x[0]
    for (int t = threadIdx.x; t < 3 * B; t += NT) {
      const int c = t / B, row = row0 + (t - c * B);
      if (row < nrows) X1[out(c, row, 0)] = make_float2(__ldg(M + c * N + row), 0.f);
    }
  } else {
    struct Ld {
      __device__ static constexpr bool kSmem() { return false; }
      const float* M;
      size_t N;
      int row0, nrows, nx;
      __device__ float2 operator()(int b, int c, int ib, int C) const {
        const int i = ib + C;
        float2 v = make_float2(0.f, 0.f);
        const int row = row0 + b;
        if (row < nrows) {
          const float* p = M + c * N + (size_t)row * nx;
          const int x0 = 2 * i;
          if ((nx & 1) == 0) {
            if (x0 < nx) v = __ldg(reinterpret_cast<const float2*>(p + x0));
          } else {
            if (x0 < nx) v.x = __ldg(p + x0);
            if (x0 + 1 < nx) v.y = __ldg(p + x0 + 1);
          }
        }
        return v;
      }
    } ld{M, N, row0, nrows, g.nx};
    fft_tile<L, B, NT, false, false, true, false, 3>(smem, ld, SmemSt<L, B, false>{smem}, tw, g.Lmax / L);
    __syncthreads();
    using T = TileIdx<L, B, false>;
    const int twpx = g.Lmax / (2 * L);
    for (int u = threadIdx.x; u < B * (L + 1); u += NT) {
      const int b = u / (L + 1), k = u - b * (L + 1);
      const int row = row0 + b;
      if (row >= nrows) continue;
      const float2 w = __ldg(tw + k * twpx);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float2 Zk = smem[c * T::ELEMS + T::at(b, k & (L - 1))];
        const float2 Zn = smem[c * T::ELEMS + T::at(b, (L - k) & (L - 1))];
        const float2 E = make_float2(0.5f * (Zk.x + Zn.x), 0.5f * (Zk.y - Zn.y));
        const float2 D = make_float2(0.5f * (Zk.x - Zn.x), 0.5f * (Zk.y + Zn.y));
        const float2 wD = cmul(w, D);
        X1[out(c, row, k)] = make_float2(E.x + wD.y, E.y - wD.x);
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
// K4's destination for that slab: its own buffer (then the C2 transpose), or with
// fused transposes block `rank` of the owning rank q's buffer (peer memory).
__device__ __forceinline__ float2* xrow_dst(const Geom& g, float2* out, int slab) {
  if (!g.p2p) return out + xrow_slab(g, slab);
  const int c = slab / g.nz, z = slab - c * g.nz;
  const int q = z / g.nzl, zl = z - q * g.nzl;
  return g.peer[q] + ((size_t)(g.rank * 3 + c) * g.nzl + zl) * g.ny * g.pitch1;
}

// ---------------------------------------------------------------------------
// K2 / K4: y pencils.  Columns (kx) are contiguous; a CTA owns NCOL columns of one
// (component, z) slab.  Forward: ny of L inputs nonzero.  Inverse: keep y < ny.
template <int L, int NCOL, int NT, int MINB, bool INV>
__global__ void __launch_bounds__(NT, MINB) k_y(const float2* __restrict__ in, float2* __restrict__ out,
                                                const float2* __restrict__ tw, Geom g, int in_rows, int out_rows,
                                                int n_in, int n_out) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float2 smem[];
  const int kx0 = blockIdx.x * NCOL;
  const size_t slab = blockIdx.y + (size_t)g.c0 * g.nz;  // components c0 .. c0 + nc - 1
  struct Ld {
    __device__ static constexpr bool kSmem() { return false; }
    const float2* p;
    int pitch, n_in, ncol_valid;
    __device__ float2 operator()(int b, int, int ib, int C) const {
      const int i = ib + C;
      return (i < n_in && b < ncol_valid) ? __ldg(p + (b + i * pitch)) : make_float2(0.f, 0.f);
    }
  } ld{in + (!INV ? xrow_slab(g, (int)slab) : slab * in_rows * g.pitch2) + kx0, !INV ? g.pitch1 : g.pitch2, n_in,
       g.Kc - kx0};
  struct St {
    __device__ static constexpr bool kSmem() { return false; }
    float2* p;
    int pitch, n_out, ncol_valid;
    __device__ void operator()(int b, int, int ib, int C, float2 v) const {
      const int i = ib + C;
      if (i < n_out && b < ncol_valid) p[b + i * pitch] = v;
    }
  } st{out + (INV ? xrow_slab(g, (int)slab) : slab * out_rows * g.pitch2) + kx0, INV ? g.pitch1 : g.pitch2, n_out,
       g.Kc - kx0};
  fft_tile<L, NCOL, NT, true, INV, !INV && (L > 1), INV && (L > 1)>(smem, ld, st, tw, g.Lmax / L);
}

// Persistent, TMA-fed variant of K2/K4 (L >= 64): each CTA loops over tiles;
// while the FFT of tile t runs in place in one smem buffer, the tensor-map load
// of the CTA's next tile lands in the other (mbarrier completion), so HBM reads
// overlap the radix passes.  Box = {NCOL columns, <= 256 rows}; rows beyond ny
// (forward) and columns beyond Kc are zero-filled by the TMA unit.
template <int L, int NCOL, int NB = 2>
struct YTma {
  using T = TileIdx<L, NCOL, true>;
  static constexpr int TB = ((T::ELEMS * 8 + 1023) / 1024) * 1024;  // bytes per tile buffer
  using PL = Plan<L, false, 4>;
  static constexpr int TWE = PL::TW_ELEMS > 1 ? PL::TW_ELEMS : 1;
  // NB tile buffers (2: double-buffered; 1: single, latency hidden by 2 CTAs/SM),
  // per-pass twiddles, barriers
  static constexpr size_t SMEM = NB * (size_t)TB + (size_t)TWE * 8 + 64;
  static constexpr int NT = NCOL * (L / 16);
  __host__ __device__ static constexpr int rows_in(bool inv) { return inv ? L : L / 2; }
  __host__ __device__ static constexpr int br(bool inv) { return rows_in(inv) < 256 ? rows_in(inv) : 256; }
};

#ifndef GRACE_YT_MINB
#define GRACE_YT_MINB 1
#endif
#ifndef GRACE_YT_NB_INV
#define GRACE_YT_NB_INV 1  // K4 tile buffers per CTA (1: two single-buffered CTAs per SM, 0.596 -> 0.585 ms; 2: double-buffered)
#endif
// TST (K4, single GPU): the inverse's last pass writes the tile's linear layout in
// place and one thread stores rows y < n_out with TMA boxes (tout), overlapping
// the next tile's load and passes; the buffer is reloaded once the store has read it.
template <int L, int NCOL, bool INV, int NB = 2, bool TST = false>
__global__ void __launch_bounds__(YTma<L, NCOL>::NT, NB == 1 ? (YTma<L, NCOL>::NT <= 512 ? 2 : 1) : GRACE_YT_MINB)
    k_y_tma(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
            float2* __restrict__ out, const float2* __restrict__ tw, Geom g, int n_out) {
  static_assert(!TST || INV, "TMA stores on the inverse (K4) only");
  using Y = YTma<L, NCOL, NB>;
  constexpr int NT = Y::NT;
  constexpr int ROWS = Y::rows_in(INV);
  constexpr int BR = Y::br(INV);
  constexpr int NBOX = ROWS / BR;
  constexpr unsigned TX = NCOL * ROWS * 8;
  extern __shared__ __align__(1024) unsigned char smraw[];
  // tile buffer k & 1 at smraw + (k & 1) * TB (pointer arithmetic on the shared
  // array keeps every access in the shared address space: LDS/STS, not LD/ST)
  float2* tws = reinterpret_cast<float2*>(smraw + NB * Y::TB);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smraw + NB * Y::TB + Y::TWE * 8);
#ifdef GRACE_PDL_EARLY
  pdl_trigger();
#endif
  fill_pass_twiddles<typename Y::PL, L>(tws, tw, g.Lmax / L, threadIdx.x, NT);
  const int ntx = (g.Kc + NCOL - 1) / NCOL;
  const int ntiles = ntx * g.nc * g.nz;  // components c0 .. c0 + nc - 1
  const int slab0 = g.c0 * g.nz;
  auto issue = [&](int t, float2* dst, uint64_t* b) {
    const int slab = slab0 + t / ntx, xt = t - (t / ntx) * ntx;
    const int c = slab / g.nz, z = slab - c * g.nz;
    int c2 = z, c4 = 0;
    if (!INV) {  // x-row layout [q][c][zl][y][kx]
      c4 = z / g.nzl;
      c2 = z - c4 * g.nzl;
    }
    mbar_expect_tx(b, TX);
#pragma unroll
    for (int nb = 0; nb < NBOX; ++nb) tma_load_5d(dst + nb * BR * NCOL, &tin, b, xt * NCOL, nb * BR, c2, c, c4);
  };
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    mbar_fence_init();
  }
  __syncthreads();
  pdl_wait();
  int t = blockIdx.x;
  if (NB == 2 && threadIdx.x == 0 && t < ntiles) issue(t, reinterpret_cast<float2*>(smraw), bar);
  struct St {
    __device__ static constexpr bool kSmem() { return false; }
    float2* p;
    int pitch, n_out, ncol_valid;
    __device__ void operator()(int b, int, int ib, int C, float2 v) const {
      const int i = ib + C;
      if (i < n_out && b < ncol_valid) p[b + i * pitch] = v;
    }
  };
  struct StFull {  // every column valid and every produced row kept: no per-element guard
    __device__ static constexpr bool kSmem() { return false; }
    float2* p;
    int pitch;
    __device__ void operator()(int b, int, int ib, int C, float2 v) const { p[b + (ib + C) * pitch] = v; }
  };
  if (t + (int)gridDim.x >= ntiles) pdl_trigger();  // no tile or one tile left
  for (int k = 0; t < ntiles; ++k, t += gridDim.x) {
    float2* cur = reinterpret_cast<float2*>(smraw + (NB == 2 ? (k & 1) * Y::TB : 0));
    if (t + (int)gridDim.x < ntiles && t + 2 * (int)gridDim.x >= ntiles) pdl_trigger();  // last tile next
    if constexpr (NB == 2) {
      if (threadIdx.x == 0 && t + (int)gridDim.x < ntiles) {
        if constexpr (TST) bulk_wait_read0();  // the other buffer's store has read it
        fence_proxy_async();
        issue(t + gridDim.x, reinterpret_cast<float2*>(smraw + ((k + 1) & 1) * Y::TB), bar + ((k + 1) & 1));
      }
      mbar_wait(bar + (k & 1), (k >> 1) & 1);
    } else {
      if (threadIdx.x == 0) {
        if constexpr (TST) bulk_wait_read0();  // the previous tile's store has read the buffer
        fence_proxy_async();
        issue(t, cur, bar);
      }
      mbar_wait(bar, k & 1);
    }
    const int slab = slab0 + t / ntx, xt = t - (t / ntx) * ntx;
    const int kx0 = xt * NCOL;
    float2* o = (INV ? xrow_dst(g, out, slab) : out + (size_t)slab * g.Py * g.pitch2) + kx0;
    const int pitch = INV ? g.pitch1 : g.pitch2;
    if constexpr (TST) {
      fft_tile<L, NCOL, NT, true, INV, !INV, INV, 1, false, true>(cur, SmemLd<L, NCOL, true>{cur},
                                                                   SmemSt<L, NCOL, true>{cur}, tws, 1);
      fence_proxy_async();  // this thread's tile writes -> the async proxy
      __syncthreads();
      if (threadIdx.x == 0) {
        const int c = slab / g.nz, z = slab - c * g.nz;
        for (int y0 = 0; y0 < n_out; y0 += BR) tma_store_5d(&tout, cur + y0 * NCOL, kx0, y0, z, c, 0);
        bulk_commit();
      }
      continue;
    }
    if (g.Kc - kx0 >= NCOL && n_out >= (INV ? L / 2 : L))
      fft_tile<L, NCOL, NT, true, INV, !INV, INV, 1, false, true>(cur, SmemLd<L, NCOL, true>{cur}, StFull{o, pitch},
                                                                   tws, 1);
    else
      fft_tile<L, NCOL, NT, true, INV, !INV, INV, 1, false, true>(cur, SmemLd<L, NCOL, true>{cur},
                                                                   St{o, pitch, n_out, g.Kc - kx0}, tws, 1);
    __syncthreads();
  }
  if constexpr (TST) {
    if (threadIdx.x == 0) bulk_wait0();  // the stores land before the grid completes (K5 waits on it)
  }
}

// K2 for long pencils (L >= 4096), where two TMA tiles of >= 4 columns do not fit:
// one work tile of 4 columns (full 32-byte row sectors on the store side) plus
// one staging buffer for the forward input (rows < L/2).  Pass 0 reads the
// staged rows into registers and writes the work tile; as soon as every thread
// is past it, the next tile's TMA load goes into the staging buffer and overlaps
// the remaining passes.  Twiddles from the global table (no room for smem ones).
#ifndef GRACE_YSTAGE_1024
#define GRACE_YSTAGE_1024 8  // columns of the staged K2 at L = 1024 (0: the double-buffered TMA kernel; 8: film -0.5 %, 512^3 23.36 -> 22.83 ms)
#endif
#ifndef GRACE_YSTAGE_2048
#define GRACE_YSTAGE_2048 8  // columns of the staged K2 at L = 2048 (0: the double-buffered TMA kernel; 0.68 -> 0.61 ms)
#endif
#ifndef GRACE_YSTAGE_MINB
#define GRACE_YSTAGE_MINB 1
#endif
#ifndef GRACE_YSTAGE_TWS
#define GRACE_YSTAGE_TWS 1  // per-pass twiddle tables in smem when they fit beside the tiles
#endif
template <int L>
struct YStage {
  static constexpr int NCOL = (L == 2048 && GRACE_YSTAGE_2048) ? GRACE_YSTAGE_2048
                             : ((L == 1024 && GRACE_YSTAGE_1024) ? GRACE_YSTAGE_1024 : 4);
  using T = TileIdx<L, NCOL, true>;
  using PL = Plan<L, false, 4>;
  static constexpr int WB = ((T::ELEMS * 8 + 1023) / 1024) * 1024;  // work tile bytes
  static constexpr int SB = NCOL * (L / 2) * 8;                       // staging bytes
  static constexpr int TWB = PL::TW_ELEMS * 8;                        // per-pass twiddle tables
  static constexpr bool TWS = GRACE_YSTAGE_TWS && (size_t)WB + SB + TWB + 64 <= 232448;
  static constexpr size_t SMEM = (size_t)WB + SB + (TWS ? TWB : 0) + 64;
  static constexpr int NT = NCOL * (L / 16);
  static constexpr int BR = 256;
};

#ifndef GRACE_K2_TMA_STORE
#define GRACE_K2_TMA_STORE 0  // 1: X2 rows by TMA stores from the work tile (measured slower: slab K2 0.627 vs 0.549 ms)
#endif
template <int L>
__global__ void __launch_bounds__(YStage<L>::NT, (L == 2048 ? GRACE_YSTAGE_MINB : 1))
    k_y_stage(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout,
              float2* __restrict__ out, const float2* __restrict__ tw, Geom g, int n_out) {
  using Y = YStage<L>;
  constexpr int NCOL = Y::NCOL, NT = Y::NT, ROWS = L / 2, NBOX = ROWS / Y::BR;
  constexpr unsigned TX = NCOL * ROWS * 8;
  extern __shared__ __align__(1024) unsigned char smraw[];
  float2* work = reinterpret_cast<float2*>(smraw);
  float2* stage = reinterpret_cast<float2*>(smraw + Y::WB);
  float2* tws = reinterpret_cast<float2*>(smraw + Y::WB + Y::SB);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smraw + Y::WB + Y::SB + (Y::TWS ? Y::TWB : 0));
  pdl_trigger();
  if constexpr (Y::TWS) fill_pass_twiddles<typename Y::PL, L>(tws, tw, g.Lmax / L, threadIdx.x, NT);
  const float2* twp = Y::TWS ? tws : tw;  // the passes' twiddle source
  const int tws_stride = Y::TWS ? 1 : g.Lmax / L;
  const int ntx = (g.Kc + NCOL - 1) / NCOL;
  const int ntiles = ntx * g.nc * g.nz;  // components c0 .. c0 + nc - 1
  const int slab0 = g.c0 * g.nz;
  auto issue = [&](int t) {
    const int slab = slab0 + t / ntx, xt = t - (t / ntx) * ntx;
    const int c = slab / g.nz, z = slab - c * g.nz;
    const int c4 = z / g.nzl, c2 = z - c4 * g.nzl;  // x-row layout [q][c][zl][y][kx]
    mbar_expect_tx(bar, TX);
#pragma unroll
    for (int nb = 0; nb < NBOX; ++nb) tma_load_5d(stage + nb * Y::BR * NCOL, &tin, bar, xt * NCOL, nb * Y::BR, c2, c, c4);
  };
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  pdl_wait();
  int t = blockIdx.x;
  if (threadIdx.x == 0 && t < ntiles) issue(t);
  struct StageLd {
    __device__ static constexpr bool kSmem() { return false; }  // not the work tile: no in-place hazard
    const float2* s;
    __device__ float2 operator()(int b, int, int ib, int C) const { return s[(ib + C) * NCOL + b]; }
  };
  struct St {
    __device__ static constexpr bool kSmem() { return false; }
    float2* p;
    int pitch, ncol_valid;
    __device__ void operator()(int b, int, int ib, int C, float2 v) const {
      if (b < ncol_valid) p[b + (ib + C) * pitch] = v;
    }
  };
  using PL = Plan<L, false, 4>;
  constexpr int IFACE0 = TileIdx<L, NCOL, true, PL::R(0)>::PAD ? kPad : kLin;
  const ThreadMap<L, NCOL, NT, true> tm;
  constexpr bool TST = GRACE_K2_TMA_STORE;  // X2 rows from the work tile by TMA stores
  for (int k = 0; t < ntiles; ++k, t += gridDim.x) {
    mbar_wait(bar, k & 1);
    if constexpr (TST) {
      if (threadIdx.x == 0) bulk_wait_read0();  // the previous tile's store has read the work tile
      __syncthreads();
    }
    const int slab = slab0 + t / ntx, xt = t - (t / ntx) * ntx;
    const int kx0 = xt * NCOL;
    const St st{out + (size_t)slab * g.Py * g.pitch2 + kx0, g.pitch2, g.Kc - kx0};
    // pass 0: staged rows (< L/2, the rest is the zero padding) -> work tile
    fft_pass<L, 0, false, NCOL, NT, true, 1, false, true, false, kExt, IFACE0, Y::TWS>(tm, StageLd{stage}, st, work,
                                                                                       twp, tws_stride);
    __syncthreads();  // the staging buffer is free
    if (threadIdx.x == 0 && t + (int)gridDim.x < ntiles) {
      fence_proxy_async();
      issue(t + gridDim.x);
    }
    if constexpr (TST) {
      fft_passes<L, 1, false, NCOL, NT, true, 1, false, true, false, kExt, kExt, Y::TWS>(
          tm, work, StageLd{stage}, SmemSt<L, NCOL, true>{work}, twp, tws_stride);
      fence_proxy_async();
      __syncthreads();
      if (threadIdx.x == 0) {
        const int c = slab / g.nz, z = slab - c * g.nz;
#pragma unroll 1
        for (int y0 = 0; y0 < L; y0 += Y::BR) tma_store_5d(&tout, work + y0 * NCOL, kx0, y0, z, c, 0);
        bulk_commit();
      }
    } else {
      fft_passes<L, 1, false, NCOL, NT, true, 1, false, true, false, kExt, kExt, Y::TWS>(tm, work, StageLd{stage}, st,
                                                                                           twp, tws_stride);
      __syncthreads();
    }
  }
  if constexpr (TST) {
    if (threadIdx.x == 0) bulk_wait0();
  }
  (void)n_out;
}

// ---------------------------------------------------------------------------
// Stage KS[c][k1][k2][kx0 .. kx0+B) for c = 0..5 into kss[c][k][b] with cp.async,
// where the staged axis k runs over KH entries at stride kstride (floats) from `base`.
// Columns at or beyond `avail` (= KSp - kx0: past the end of the KS row) are
// zero-filled instead of read, so the last CTA never reads past the table.
template <int B, int NT>
__device__ __forceinline__ void stage_ks(float* kss, const float* __restrict__ base, size_t cstride, size_t kstride,
                                         int KH, int avail) {
  if constexpr (B % 4 == 0) {
    for (int t = threadIdx.x; t < 6 * KH * (B / 4); t += NT) {
      const int ch = t % (B / 4), r = t / (B / 4);
      const int comp = r / KH, k = r - comp * KH;
      if (4 * ch < avail)  // KSp is a multiple of 32: a 4-float chunk is all in or all out
        cp_async16(kss + r * B + 4 * ch, base + comp * cstride + k * kstride + 4 * ch);
      else
        *reinterpret_cast<float4*>(kss + r * B + 4 * ch) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  } else {
    for (int t = threadIdx.x; t < 6 * KH * B; t += NT) {
      const int bb = t % B, r = t / B;
      const int comp = r / KH, k = r - comp * KH;
      if (bb < avail) cp_async4(kss + r * B + bb, base + comp * cstride + k * kstride + bb);
      else kss[r * B + bb] = 0.f;
    }
  }
}

#ifndef GRACE_PENCIL_TWS
#define GRACE_PENCIL_TWS 0  // K3 (LDG) and K2': per-pass twiddles in smem (off: the block's Pz = 128 K3 drops to 2 CTAs/SM, 11.9 -> 12.6 ms; SP4 unchanged)
#endif
constexpr bool PENCIL_TWS = GRACE_PENCIL_TWS;

// K3: z pencils of the three components for one ky' (and its mirror Py - ky'):
// forward z-FFT (nz of L nonzero), H~ = KS . M~, inverse z-FFT, keep z < nz.
// Processing ky and Py-ky in one CTA reads each folded KS slice once; the slice
// is staged by cp.async while the first forward FFT runs.
template <int L, int B, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k3_z(float2* __restrict__ X2, const float* __restrict__ KS,
                                                 const float2* __restrict__ tw, Geom g) {
  extern __shared__ float2 smem[];
  constexpr int KZH = L / 2 + 1;
  const int kx0 = blockIdx.x * B;
  const int kyf = blockIdx.y;
  const int zstride = g.Py * g.pitch2;            // between z planes
  const size_t cstride = (size_t)g.nz * zstride;  // between components
  const int nvalid = g.Kc - kx0;
  const int nky = (kyf == 0 || 2 * kyf == g.Py) ? 1 : 2;
  float* kss = reinterpret_cast<float*>(smem + 3 * TileIdx<L, B, true>::ELEMS);
  float2* tws = reinterpret_cast<float2*>(kss + 6 * KZH * B);  // per-pass twiddles (GRACE_PENCIL_TWS)
  pdl_trigger();
  stage_ks<B, NT>(kss, KS + (size_t)kyf * g.KSp + kx0, (size_t)g.Kzh * g.Kyh * g.KSp, (size_t)g.Kyh * g.KSp, KZH,
                  g.KSp - kx0);
  if constexpr (PENCIL_TWS) {
    fill_pencil_twiddles<L>(tws, tw, g.Lmax / L, threadIdx.x, NT);
    __syncthreads();
  }
  pdl_wait();  // the KS slice is constant; X2 comes from K2
  for (int rep = 0; rep < nky; ++rep) {
    const int ky = rep == 0 ? kyf : g.Py - kyf;
    float2* base = X2 + (size_t)ky * g.pitch2 + kx0;
    struct Ld {
      __device__ static constexpr bool kSmem() { return false; }
      const float2* p;
      int zs;
      size_t cs;
      int nz, nvalid;
      __device__ float2 operator()(int b, int c, int ib, int C) const {
        const int i = ib + C;
        return (i < nz && b < nvalid) ? __ldg(p + c * cs + (b + i * zs)) : make_float2(0.f, 0.f);
      }
    } ld{base, zstride, cstride, g.nz, nvalid};
    struct St {
      __device__ static constexpr bool kSmem() { return false; }
      float2* p;
      int zs;
      size_t cs;
      int nz, nvalid;
      __device__ void operator()(int b, int c, int ib, int C, float2 v) const {
        const int i = ib + C;
        if (i < nz && b < nvalid) p[c * cs + (b + i * zs)] = v;
      }
    } st{base, zstride, cstride, g.nz, nvalid};
    if (rep) __syncthreads();
    pencil_conv<L, B, NT, PENCIL_TWS>(smem, ld, st, kss, KZH, PENCIL_TWS ? tws : tw, PENCIL_TWS ? 1 : g.Lmax / L,
                                      g.Py, ky, false, [&] {
                                        if (rep == 0) cp_async_wait_all();
                                      });
  }
}

// K3 fed by TMA (fused short pencils, L <= 64).  The same pencil convolution as
// k3_z, but every global read is a tensor-map copy issued by one thread, so the
// HBM latency overlaps this and the other resident CTAs' work and no thread
// spends instructions on address arithmetic, bounds checks or LDGs:
//   * the KS slice [6][Kzh][B] (box {B, 1, Kzh, 6} of KS) before the PDL wait
//     (it is constant), landing in the kss layout kmul_s reads;
//   * the ky pencils of the three components (boxes {B, 1, L/2, 1} of X2, rows
//     z >= nz and columns kx >= Kc zero-filled by the TMA unit) straight into
//     the work tile, where the forward first pass runs in place;
//   * with PRE, the mirror ky' = Py - ky pencils at the same time into a staging
//     buffer, so the second pencil set never waits on HBM.
// Outputs (z < nz) are stored from the inverse last pass as in k3_z.
template <int L>
struct Z3Tma {
  static constexpr int B = ZPlan<L>::B;
  static constexpr int NT = ZPlan<L>::NT;
  using T = TileIdx<L, B, true>;
  static_assert(!T::PAD, "TMA boxes land in the linear tile layout");
  static constexpr int H = L / 2;  // rows per pencil box (nz <= L/2)
  static constexpr int KZH = L / 2 + 1;
  static constexpr size_t WORK = 3 * (size_t)T::ELEMS * 8;
  static constexpr size_t STAGE = 3 * (size_t)H * B * 8;
  static constexpr size_t KSB = 6 * (size_t)KZH * B * 4;
  static constexpr size_t KSB16 = (KSB + 15) / 16 * 16;
  // per-pass twiddles in smem, forward then inverse plan (fused plans; unfused
  // long pencils keep the global table so the CTA count per SM is unchanged)
  static constexpr bool TWS = ZPlan<L>::FUSE;
  static constexpr int TWF = TWS ? Plan<L, false, ZPlan<L>::RB>::TW_ELEMS : 0;
  static constexpr int TWI = TWS ? Plan<L, true, ZPlan<L>::RB>::TW_ELEMS : 0;
  static constexpr size_t TWB = (size_t)(TWF + TWI) * 8;
#ifndef GRACE_K3_PRE
#define GRACE_K3_PRE 1  // prefetch the mirror pencils where 4 CTAs/SM still fit
#endif
  static constexpr bool PRE = GRACE_K3_PRE && (WORK + STAGE + KSB16 + TWB + 64) * 4 <= 220 * 1024;
  static constexpr size_t KSOFF = WORK + (PRE ? STAGE : 0);
  static constexpr size_t TWOFF = KSOFF + KSB16;
  static constexpr size_t SMEM = TWOFF + TWB + 64;
};

#ifndef GRACE_K3_TMA_STORE
#define GRACE_K3_TMA_STORE 0  // 1: K3 pencils stored by TMA from the work tile (measured slower: slab K3 0.933 vs 0.905 ms; profiles/r02_sweeps.md)
#endif
template <int L, int MINB>
__global__ void __launch_bounds__(Z3Tma<L>::NT, MINB)
    k3_z_tma(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap kmap,
             float2* __restrict__ X2, const float2* __restrict__ tw, const float2* __restrict__ tw3, Geom g) {
  using Z = Z3Tma<L>;
  constexpr int B = Z::B, NT = Z::NT, H = Z::H;
  constexpr unsigned TXP = 3u * H * B * 8;  // bytes of one pencil set
  extern __shared__ __align__(128) unsigned char smraw[];
  float2* work = reinterpret_cast<float2*>(smraw);
  float2* stage = reinterpret_cast<float2*>(smraw + Z::WORK);
  float* kss = reinterpret_cast<float*>(smraw + Z::KSOFF);
  float2* tws = reinterpret_cast<float2*>(smraw + Z::TWOFF);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smraw + Z::TWOFF + Z::TWB);  // KS, work, stage
  const int kx0 = blockIdx.x * B;
  const int kyf = blockIdx.y;
  const int nky = (kyf == 0 || 2 * kyf == g.Py) ? 1 : 2;
  const size_t zstride = (size_t)g.Py * g.pitch2;
  const size_t cstride = (size_t)g.nz * zstride;
  const int nvalid = g.Kc - kx0;
  pdl_trigger();
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    mbar_init(bar + 2, 1);
    mbar_fence_init();
    mbar_expect_tx(bar, (unsigned)Z::KSB);
    tma_load_4d(kss, &kmap, bar, kx0, kyf, 0, 0);
  }
  // per-pass twiddle tables in smem (the global table's lines would miss the
  // minimal L1 of a shared-memory-carveout kernel)
  if constexpr (Z::TWS) {
    if (tw3 != nullptr) {  // the tables precomputed in this layout (k3_twiddle_tables): one bulk copy
      if (threadIdx.x == 0) {
        mbar_expect_tx_only(bar + 1, (unsigned)Z::TWB);
        bulk_load(tws, tw3, (unsigned)Z::TWB, bar + 1);
      }
    } else {
      fill_pass_twiddles<Plan<L, false, ZPlan<L>::RB>, L>(tws, tw, g.Lmax / L, threadIdx.x, NT);
      fill_pass_twiddles<Plan<L, true, ZPlan<L>::RB>, L>(tws + Z::TWF, tw, g.Lmax / L, threadIdx.x, NT);
    }
  }
  const float2* twp = Z::TWS ? tws : tw;  // the passes' twiddle source and stride
  const int twstr = Z::TWS ? 1 : g.Lmax / L;
  __syncthreads();
  pdl_wait();  // X2 comes from K2
  auto issue = [&](float2* dst, int ky, uint64_t* b, int cstep) {
    mbar_expect_tx(b, TXP);
#pragma unroll
    for (int c = 0; c < 3; ++c) tma_load_4d(dst + c * cstep, &xmap, b, kx0, ky, 0, c);
  };
  if (threadIdx.x == 0) {
    issue(work, kyf, bar + 1, Z::T::ELEMS);
    if (Z::PRE && nky == 2) issue(stage, g.Py - kyf, bar + 2, H * B);
  }
  struct StageLd {  // staged mirror pencils [c][z][b] (a different buffer: no in-place hazard)
    __device__ static constexpr bool kSmem() { return false; }
    const float2* s;
    __device__ float2 operator()(int b, int c, int ib, int C) const { return s[(c * H + ib + C) * B + b]; }
  };
  struct St {
    __device__ static constexpr bool kSmem() { return false; }
    float2* p;
    size_t zs, cs;
    int nz, nvalid;
    __device__ void operator()(int b, int c, int ib, int C, float2 v) const {
      const int i = ib + C;
      if (i < nz && b < nvalid) p[c * cs + (b + i * zs)] = v;
    }
  };
  // TST: the inverse's last pass writes the work tile (linear [c][z][b]) and one
  // thread stores the pencils with TMA boxes of the same map (z >= nz and
  // kx >= Kc clipped by the unit); the tile is reused once the store has read it
  constexpr bool TST = GRACE_K3_TMA_STORE;
  auto store = [&](int ky) {
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
      for (int c = 0; c < 3; ++c) tma_store_4d(&xmap, work + c * Z::T::ELEMS, kx0, ky, 0, c);
      bulk_commit();
    }
  };
  const SmemSt<L, B, true> sst{work};
  for (int rep = 0; rep < nky; ++rep) {
    const int ky = rep == 0 ? kyf : g.Py - kyf;
    const St st{X2 + (size_t)ky * g.pitch2 + kx0, zstride, cstride, g.nz, nvalid};
    auto kw = [&] {
      if (rep == 0) mbar_wait(bar, 0);
    };
    if (rep == 0) {
      mbar_wait(bar + 1, 0);
      if constexpr (TST)
        pencil_conv<L, B, NT, Z::TWS>(work, SmemLd<L, B, true>{work}, sst, kss, Z::KZH, twp, twstr, g.Py, ky, false, kw);
      else
        pencil_conv<L, B, NT, Z::TWS>(work, SmemLd<L, B, true>{work}, st, kss, Z::KZH, twp, twstr, g.Py, ky, false, kw);
    } else if constexpr (Z::PRE) {
      if (TST && threadIdx.x == 0) bulk_wait_read0();
      __syncthreads();  // the work tile is free
      mbar_wait(bar + 2, 0);
      if constexpr (TST)
        pencil_conv<L, B, NT, Z::TWS>(work, StageLd{stage}, sst, kss, Z::KZH, twp, twstr, g.Py, ky, false, kw);
      else
        pencil_conv<L, B, NT, Z::TWS>(work, StageLd{stage}, st, kss, Z::KZH, twp, twstr, g.Py, ky, false, kw);
    } else {
      __syncthreads();
      if (threadIdx.x == 0) {
        if constexpr (TST) bulk_wait_read0();
        fence_proxy_async();
        issue(work, ky, bar + 1, Z::T::ELEMS);
      }
      mbar_wait(bar + 1, 1);
      if constexpr (TST)
        pencil_conv<L, B, NT, Z::TWS>(work, SmemLd<L, B, true>{work}, sst, kss, Z::KZH, twp, twstr, g.Py, ky, false, kw);
      else
        pencil_conv<L, B, NT, Z::TWS>(work, SmemLd<L, B, true>{work}, st, kss, Z::KZH, twp, twstr, g.Py, ky, false, kw);
    }
    if constexpr (TST) store(ky);
  }
  if constexpr (TST) {
    if (threadIdx.x == 0) bulk_wait0();  // the stores land before the grid completes (K4 waits on it)
  }
}

// Pz == 1 without the fused y path: H~ = KS . M~ on X2 [3][1][Py][pitch2].
__device__ __forceinline__ void kmul3(float2& a, float2& b, float2& c, const float* __restrict__ KS, const Geom& g,
                                      int ky, int kx) {
  const bool fy = ky > (g.Py >> 1);
  const int kyf = fy ? g.Py - ky : ky;
  const size_t cs = (size_t)g.Kzh * g.Kyh * g.KSp;
  const float* p = KS + (size_t)kyf * g.KSp + kx;
  const float nxx = __ldg(p), nyy = __ldg(p + 3 * cs), nzz = __ldg(p + 5 * cs);
  const float nxy = fy ? -__ldg(p + cs) : __ldg(p + cs);
  const float2 mx = a, my = b, mz = c;
  a = make_float2(nxx * mx.x + nxy * my.x, nxx * mx.y + nxy * my.y);
  b = make_float2(nxy * mx.x + nyy * my.x, nxy * mx.y + nyy * my.y);
  c = make_float2(nzz * mz.x, nzz * mz.y);
}

__global__ void k_mul_plane(float2* __restrict__ X2, const float* __restrict__ KS, Geom g) {
  pdl_trigger();
  pdl_wait();
  const int kx = blockIdx.x * blockDim.x + threadIdx.x;
  const int ky = blockIdx.y;
  if (kx >= g.Kc) return;
  const size_t cs = (size_t)g.Py * g.pitch2;
  float2* p = X2 + (size_t)ky * g.pitch2 + kx;
  float2 a = p[0], b = p[cs], c = p[2 * cs];
  kmul3(a, b, c, KS, g, ky, kx);
  p[0] = a;
  p[cs] = b;
  p[2 * cs] = c;
}

// ---------------------------------------------------------------------------
// K2': nz == 1.  y-FFT (ny of L nonzero), multiply, inverse y (keep y < ny), in place on X1.
template <int L, int B, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k2f_y_fused(float2* __restrict__ X1, const float* __restrict__ KS,
                                                        const float2* __restrict__ tw, Geom g) {
  pdl_trigger();
  extern __shared__ float2 smem[];
  constexpr int KYH = L / 2 + 1;
  const int kx0 = blockIdx.x * B;
  const int nvalid = g.Kx - kx0;
  const size_t cstride = (size_t)g.ny * g.pitch1;
  float2* base = X1 + kx0;
  float* kss = reinterpret_cast<float*>(smem + 3 * TileIdx<L, B, true>::ELEMS);
  float2* tws = reinterpret_cast<float2*>(kss + 6 * KYH * B);
  if constexpr (PENCIL_TWS) {
    fill_pencil_twiddles<L>(tws, tw, g.Lmax / L, threadIdx.x, NT);
    __syncthreads();
  }
  stage_ks<B, NT>(kss, KS + kx0, (size_t)g.Kzh * g.Kyh * g.KSp, (size_t)g.KSp, KYH, g.KSp - kx0);
  pdl_wait();
  struct Ld {
    __device__ static constexpr bool kSmem() { return false; }
    const float2* p;
    size_t cs;
    int pitch, ny, nvalid;
    __device__ float2 operator()(int b, int c, int ib, int C) const {
      const int i = ib + C;
      return (i < ny && b < nvalid) ? __ldg(p + c * cs + (b + i * pitch)) : make_float2(0.f, 0.f);
    }
  } ld{base, cstride, g.pitch1, g.ny, nvalid};
  struct St {
    __device__ static constexpr bool kSmem() { return false; }
    float2* p;
    size_t cs;
    int pitch, ny, nvalid;
    __device__ void operator()(int b, int c, int ib, int C, float2 v) const {
      const int i = ib + C;
      if (i < ny && b < nvalid) p[c * cs + (b + i * pitch)] = v;
    }
  } st{base, cstride, g.pitch1, g.ny, nvalid};
  pencil_conv<L, B, NT, PENCIL_TWS>(smem, ld, st, kss, KYH, PENCIL_TWS ? tws : tw, PENCIL_TWS ? 1 : g.Lmax / L, 1, 0,
                                    true, [] { cp_async_wait_all(); });
}

// ---------------------------------------------------------------------------
// KP: plane-fused y.z.y pass for thin films.  One CTA holds a
// whole kx plane of the three components in shared memory and runs, between one
// read and one write of its X1 column, the forward y-FFT, the z-FFT, H~ = KS.M~
// (P:L55's convolution theorem), the inverse z-FFT and the inverse y-FFT, so
// K2, K3 and K4 (and X2) drop out of the step: 24 + 24 B/cell of X1 plus the
// plane's KS slice instead of K2..K4's ~267 B/cell.  The plane of the y spectra
// is Py x 3 HZ complex (HZ = Pz/2 >= nz z rows, the rows z >= nz zero), which
// fits the 227 KB of one CTA for Pz <= 16 (thin films; Py <= 1024 at Pz = 16).
//   y stage : rows-mode tile, column b = c HZ + z (component c, z row), LY = Py
//             points with the ny < LY/2 nonzero inputs read straight from X1
//             (HIN); outputs in the tile's linear layout (b, ky) at b ROWS + ky.
//   z stage : pencil ky, two adjacent lanes per pencil, lane h = the kz = 2m + h
//             half of the pruned Pz-point transform: with a[n] = 0 for n >= Pz/2,
//             M~[2m + h] = DFT_{Pz/2}(a[n] w_Pz^{hn})[m], and the inverse
//             keeping n < nz is the sum over h of w_Pz^{-hn} IDFT_{Pz/2}(H~_h)[n]
//             (one shuffle).  In registers, no shared-memory passes; consecutive
//             pencils on consecutive lanes read consecutive words.
//   KS      : the plane-ordered copy KSP [kx][6][Kzh][Kyh] (contiguous per kx,
//             prefetched into L2 by one bulk prefetch before the PDL wait).
// largest divisor d of ncol with d <= cap and d * tpc a multiple of 32
__host__ __device__ constexpr int plane_ncolg(int ncol, int cap, int tpc, int d = 0) {
  return d == 0 ? plane_ncolg(ncol, cap, tpc, ncol)
                : (d == 1 || (ncol % d == 0 && d <= cap && (d * tpc) % 32 == 0) ? d : plane_ncolg(ncol, cap, tpc, d - 1));
}
template <int LY, int PZ>
struct PlaneCfg {
  static_assert(PZ == 4 || PZ == 8 || PZ == 16, "plane path: Pz in {4, 8, 16}");
  static constexpr int HZ = PZ / 2;
  static constexpr int NCOL = 3 * HZ;
  // the y stage runs in G column groups of NCOLG columns, LY/16 threads per
  // column (at most 16 complex values per thread in any pass) and at most 512
  // threads (128 registers: the z stage holds 3 x HZ complex values per thread)
  static constexpr int NCOLG = plane_ncolg(NCOL, 8192 / LY, LY / 16);
  static constexpr int G = NCOL / NCOLG;
  static constexpr int TPC = LY / 16;
  static constexpr int NT = NCOLG * TPC;
  using T = TileIdx<LY, NCOLG, false>;
  static constexpr int ROWS = T::ROWS;  // rows-mode tiles: per-column region, the same for every group size
  static constexpr int TILE = NCOL * ROWS;  // float2
  static constexpr int BY = 256;            // TMA box rows (y)
  using PL = Plan<LY, false, rb_for(false, 1, LY)>;  // the y transforms' radix plan (rows mode, V = 1)
  static constexpr int TWE = PL::TW_ELEMS;               // per-pass twiddle tables (fill_pass_twiddles)
  static constexpr size_t SMEM = (size_t)(TILE + TWE) * sizeof(float2) + 16;
  static_assert(NT % 32 == 0 && (2 * LY) % 32 == 0, "whole warps in the z stage");
  static_assert((ROWS * 8) % 128 == 0, "128-byte aligned column regions (TMA destinations)");
};
__host__ __device__ constexpr long long plane_ks_stride(int Kzh, int Kyh) { return ((6LL * Kzh * Kyh + 31) / 32) * 32; }
// a[N] *= w_PZ^{+-N} for N < HZ (compile-time twiddles)
template <bool INV, int PZ, int HZ, int N = 0>
__device__ __forceinline__ void tw_rows(float2* a) {
  if constexpr (N < HZ) {
    a[N] = tw16_mul<INV, N * (16 / PZ)>(a[N]);
    tw_rows<INV, PZ, HZ, N + 1>(a);
  }
}

template <int LY, int PZ>
__global__ void __launch_bounds__(PlaneCfg<LY, PZ>::NT, 1)
    k_plane(const __grid_constant__ CUtensorMap xmap, float2* __restrict__ X1, const float* __restrict__ KSP,
            const float2* __restrict__ tw, Geom g) {
  using C = PlaneCfg<LY, PZ>;
  using T = typename C::T;
  constexpr int HZ = C::HZ, NCOLG = C::NCOLG, NT = C::NT, ROWS = C::ROWS, BY = C::BY;
  extern __shared__ __align__(1024) unsigned char kp_raw[];
  float2* smem = reinterpret_cast<float2*>(kp_raw);
  float2* tws = smem + C::TILE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::TILE + C::TWE);
  const int kx = blockIdx.x;
  const long long kss = plane_ks_stride(g.Kzh, g.Kyh);
  const float* ks = KSP + kx * kss;
  const int nz = g.nz, ny = g.ny;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  pdl_trigger();
  pdl_wait();
  // X1 column pairs (kx & ~1, kx | 1) x BY rows of every (c, z < nz) land in the
  // upper part of their own column region of the tile (rows >= ny zero-filled by
  // the TMA unit); pass 0 of the y-FFT reads them from there
  const int by = ny < BY ? ny : BY;  // the map's box rows (make_plane_tmap)
  const int nb = (ny + by - 1) / by;
  if (threadIdx.x == 0) {
    mbar_expect_tx(bar, (unsigned)(3 * nz * nb * by * 16));
    for (int c = 0; c < 3; ++c)
      for (int z = 0; z < nz; ++z)
        for (int j = 0; j < nb; ++j)
          tma_load_3d(smem + (size_t)(c * HZ + z) * ROWS + j * by * 2, &xmap, bar, kx & ~1, j * by, c * nz + z);
    // the KS slice into L2 while the y stage runs (after the PDL wait: issued
    // before it, the graph-replayed step read garbage -- measured, non-finite M)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(ks), "r"((unsigned)(kss * 4)) : "memory");
  }
  // per-pass twiddles of the y plan in smem (the global table's scattered 8-byte
  // reads were the kernel's largest L2 sector traffic)
  fill_pass_twiddles<typename C::PL, LY>(tws, tw, g.Lmax / LY, threadIdx.x, NT);
  __syncthreads();
  mbar_wait(bar, 0);
  const int odd = kx & 1;
#pragma unroll 1
  for (int grp = 0; grp < C::G; ++grp) {
    float2* tile = smem + (size_t)grp * NCOLG * ROWS;
    struct Ld {  // column b of the group: y row i of (c, z), from the staged pair
      __device__ static constexpr bool kSmem() { return true; }
      const float2* s;
      int b0, odd, nz, ny;
      __device__ float2 operator()(int b, int, int ib, int Cc) const {
        const int y = ib + Cc, bb = b0 + b, c = bb / HZ, z = bb - c * HZ;
        return (y < ny && z < nz) ? s[b * ROWS + 2 * y + odd] : make_float2(0.f, 0.f);
      }
    } ld{tile, grp * NCOLG, odd, nz, ny};
    if (grp) __syncthreads();
    fft_tile<LY, NCOLG, NT, false, false, true, false, 1, false, true>(tile, ld, SmemSt<LY, NCOLG, false>{tile}, tws, 1);
  }
  __syncthreads();
  // z stage: unit u = (pencil ky = u / 2, half h = u % 2)
  const int Kyh = g.Kyh, Kzh = g.Kzh;
  const size_t kcs = (size_t)Kzh * Kyh;
  for (int u = threadIdx.x; u < 2 * LY; u += NT) {
    const int ky = u >> 1, h = u & 1;
    const bool fy = ky > (LY >> 1);
    const int kyf = fy ? LY - ky : ky;
    float2 a[3][HZ];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int n = 0; n < HZ; ++n) a[c][n] = smem[(c * HZ + n) * ROWS + ky];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      if (h) tw_rows<false, PZ, HZ>(a[c]);  // a[n] w_Pz^n
      dft_inplace<HZ, false>(a[c]);
    }
#pragma unroll
    for (int m = 0; m < HZ; ++m) {
      const int kz = 2 * m + h;
      const bool fz = kz > (PZ >> 1);
      const int kzf = fz ? PZ - kz : kz;
      const float* q = ks + (size_t)kzf * Kyh + kyf;
      const float nxx = __ldg(q), nyy = __ldg(q + 3 * kcs), nzz = __ldg(q + 5 * kcs);
      const float nxy = fy ? -__ldg(q + kcs) : __ldg(q + kcs);
      const float nxz = fz ? -__ldg(q + 2 * kcs) : __ldg(q + 2 * kcs);
      const float nyz = (fy != fz) ? -__ldg(q + 4 * kcs) : __ldg(q + 4 * kcs);
      const float2 mx = a[0][m], my = a[1][m], mz = a[2][m];
      a[0][m] = make_float2(nxx * mx.x + nxy * my.x + nxz * mz.x, nxx * mx.y + nxy * my.y + nxz * mz.y);
      a[1][m] = make_float2(nxy * mx.x + nyy * my.x + nyz * mz.x, nxy * mx.y + nyy * my.y + nyz * mz.y);
      a[2][m] = make_float2(nxz * mx.x + nyz * my.x + nzz * mz.x, nxz * mx.y + nyz * my.y + nzz * mz.y);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      dft_inplace<HZ, true>(a[c]);
      if (h) tw_rows<true, PZ, HZ>(a[c]);  // w_Pz^-n IDFT(H~_odd)[n]
    }
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int n = 0; n < HZ; ++n) {
        const float2 v = a[c][n];
        const float2 o = make_float2(__shfl_xor_sync(0xffffffffu, v.x, 1), __shfl_xor_sync(0xffffffffu, v.y, 1));
        if ((n & 1) == h) smem[(c * HZ + n) * ROWS + ky] = cadd(v, o);  // rows n >= nz are never stored to X1
      }
  }
  __syncthreads();
  const size_t ps = g.pitch1;
#pragma unroll 1
  for (int grp = 0; grp < C::G; ++grp) {
    float2* tile = smem + (size_t)grp * NCOLG * ROWS;
    struct St {
      __device__ static constexpr bool kSmem() { return false; }
      float2* p;
      size_t ps;
      int b0, nz, ny;
      __device__ void operator()(int b, int, int ib, int Cc, float2 v) const {
        const int y = ib + Cc, bb = b0 + b, c = bb / HZ, z = bb - c * HZ;
        if (y < ny && z < nz) p[((size_t)(c * nz + z) * ny + y) * ps] = v;
      }
    } st{X1 + kx, ps, grp * NCOLG, nz, ny};
    if (grp) __syncthreads();
    fft_tile<LY, NCOLG, NT, false, true, false, true, 1, false, true>(tile, SmemLd<LY, NCOLG, false>{tile}, st, tws, 1);
  }
}

// KSP [kx][6][Kzh][Kyh] (stride plane_ks_stride per kx) from KS [6][Kzh][Kyh][KSp].
__global__ void k_plane_ks(float* __restrict__ KSP, const float* __restrict__ KS, Geom g) {
  const long long per = 6LL * g.Kzh * g.Kyh;
  const long long kss = plane_ks_stride(g.Kzh, g.Kyh);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < per * g.Kx;
       i += (long long)gridDim.x * blockDim.x) {
    const int kx = (int)(i % g.Kx);
    const long long r = i / g.Kx;  // (c, kzf, kyf) row of KS
    KSP[kx * kss + r] = KS[r * g.KSp + kx];
  }
}

// ---------------------------------------------------------------------------
// K5: inverse x C2R of the three H~ rows -> H_demag (K6 then applies the local
// terms and the update).  C2R of length Px = 2L from the half spectrum X[0..L]:
//   Z[k] = (X[k] + conj X[L-k]) + i w^-k (X[k] - conj X[L-k]),  k < L,
//   z = IFFT_L(Z) (unnormalised; 1/P is in KS),  x[2n] = Re z[n], x[2n+1] = Im z[n].
// This non-persistent kernel covers the rows the bulk-copy kernel (k_x_bulk)
// does not take: nx % 4 != 0, L < 64, nx == 1.
template <int L, int B, int NT, int MINB, bool DIST>
__global__ void __launch_bounds__(NT, MINB) k5_inv_x(const float2* __restrict__ X1, float* __restrict__ Hout,
                                                     const float2* __restrict__ tw, Geom g) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ float2 smem[];
  const int nrows = g.nzl * g.ny;
  const int row0 = blockIdx.x * B;
  const size_t N = (size_t)nrows * g.nx;
  const size_t cstrideX = (size_t)nrows * g.pitch1;  // X1 component stride
  if constexpr (L == 0) {  // nx == 1: H_demag = Re X[0]
    for (int b = threadIdx.x; b < B; b += NT) {
      const int row = row0 + b;
      if (row >= nrows) continue;
#pragma unroll
      for (int c = 0; c < 3; ++c) Hout[c * N + row] = __ldg(X1 + c * cstrideX + (size_t)row * g.pitch1).x;
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
      __device__ float2 operator()(int b, int c, int ib, int C) const {
        const int k = ib + C;
        const int row = row0 + b;
        if (row >= nrows) return make_float2(0.f, 0.f);
        const float2* q = X + c * cs + (size_t)row * pitch;
        float2 a, m;
        if constexpr (DIST) {  // gather from the source kx blocks of the all-to-all
          const int qa = k / kb, qm = (L - k) / kb;
          a = __ldg(q + qa * blk1 + (k - qa * kb));
          m = __ldg(q + qm * blk1 + ((L - k) - qm * kb));
        } else {
          a = __ldg(q + k);
          m = __ldg(q + (L - k));
        }
        const float2 S = make_float2(a.x + m.x, a.y - m.y);  // X[k] + conj X[L-k]
        const float2 D = make_float2(a.x - m.x, a.y + m.y);  // X[k] - conj X[L-k]
        const float2 w = __ldg(tw + k * twpx);                 // exp(-2 pi i k/Px)
        const float2 wD = cmulc(D, w);                         // w^-k D
        return make_float2(S.x - wD.y, S.y + wD.x);            // S + i w^-k D
      }
    } ld{X1, tw, cstrideX, row0, nrows, g.pitch1, twpx, g.kb, g.blk1};
    using PS = Pass<L, fft_npass(L, rb_for(false, 3, L)) - 1, false, B, NT, false, 3>;
    const ThreadMap<L, B, NT, false> tm;
    PS ps;
    fft_to_regs<L, B, NT, false, 3, true, false, true, false>(tm, smem, ld, tw, g.Lmax / L, ps);
    const int row = row0 + tm.b;
    if (PS::active(tm) && row < nrows) {
      const bool vec = (g.nx & 1) == 0;
#pragma unroll
      for (int q = 0; q < PS::UPT; ++q)
#pragma unroll
        for (int r = 0; r < PS::R / 2; ++r) {
          const int x0 = 2 * (PS::sb(tm) + PS::C2(q, r));
          if (x0 >= g.nx) continue;
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            float* h = Hout + c * N + (size_t)row * g.nx + x0;
            if (vec) *reinterpret_cast<float2*>(h) = ps.v[q][c][r];
            else {
              h[0] = ps.v[q][c][r].x;
              if (x0 + 1 < g.nx) h[1] = ps.v[q][c][r].y;
            }
          }
        }
    }
  }
}

// ---------------------------------------------------------------------------
// K1 / K5 as persistent bulk-copy kernels.  One tile = RB rows of
// the flattened (component, z, y) row index (each row transformed on its own,
// V = 1), 512 threads, two tile buffers: while the FFT of tile t runs in place
// in one buffer, one-dimensional bulk copies (cp.async.bulk, mbarrier
// completion) bring the CTA's next tile into the other, so the row reads of
// HBM overlap the radix passes instead of stalling the first one.
//   FWD (K1): rows of M (nx floats) -> R2C post-process -> X1 rows
//   !FWD (K5): X1 rows (Kx = L + 1 complex; DIST: P blocks of kb)
//              -> C2R pre-process -> H_demag rows (nx floats)
// Requires nx % 4 == 0 (16-byte row copies); the launchers fall back to the
// non-persistent kernels otherwise.

// K1 loader: packed pairs z[i] = (x[2i], x[2i+1]) of raw row b (nh = nx/2 of them).
template <int ROWS, bool GUARD>
struct XbLd {
  __device__ static constexpr bool kSmem() { return true; }
  const float2* s;
  int nh;
  __device__ float2 operator()(int b, int, int ib, int C) const {
    const int i = ib + C;
    if (GUARD && i >= nh) return make_float2(0.f, 0.f);
    return s[b * ROWS + i];
  }
};
// K5 store: output pair n -> H_demag x = 2n, 2n+1 of row b (nv valid rows).
template <bool GUARD>
struct XbSt {
  __device__ static constexpr bool kSmem() { return false; }
  float* H;
  int nx, nv;
  __device__ void operator()(int b, int, int ib, int C, float2 v) const {
    const int x0 = 2 * (ib + C);
    if (!GUARD || (b < nv && x0 < nx)) *reinterpret_cast<float2*>(H + (size_t)b * nx + x0) = v;
  }
};

#ifndef GRACE_XB_ELEMS
#define GRACE_XB_ELEMS 2048  // complex values per x tile (L = 1024: 2 rows, 128 threads at 16 elements each)
#endif
#ifndef GRACE_XB_MINB
#define GRACE_XB_MINB 6  // resident x-kernel CTAs per SM (8192 x 1 -> 2048 x 4: slab K1 0.348 -> 0.288, K5 0.296 -> 0.275 ms, SP4 19.3 -> 11.3 us/step; 4 -> 6: film 0.204 -> 0.199, 128^3 0.291 -> 0.285 ms/step in the graph, where the early-launched K5 co-resides with K4, slab neutral)
#endif
#ifndef GRACE_XB_ELEMS_TINY
#define GRACE_XB_ELEMS_TINY 512  // tiles of tiny grids (fewer default tiles than half the SMs): SP4 9.1 -> 8.2 us/step
#endif
template <int L, int E = GRACE_XB_ELEMS>
struct XBulk {
  static constexpr int RB = E / L > 0 ? E / L : 1;  // rows per tile
  static constexpr int NT = RB * (L / 16);
  using T = TileIdx<L, RB, false>;
  static constexpr int TB = ((T::ELEMS * 8 + 1023) / 1024) * 1024;
  using PL = Plan<L, false, 4>;
  static constexpr int TWE = PL::TW_ELEMS > 1 ? PL::TW_ELEMS : 1;
  static constexpr int PPE = L / 2 + 1;  // R2C post-process twiddles w^k, k = 0..L/2
  static constexpr size_t SMEM = 2 * (size_t)TB + (size_t)(TWE + PPE) * 8 + 64;
};
constexpr int kXBulkMinL = 64, kXBulkMaxL = 4096;

template <int L, bool FWD, bool DIST, int E = GRACE_XB_ELEMS>
__global__ void __launch_bounds__(XBulk<L, E>::NT, GRACE_XB_MINB)
    k_x_bulk(const void* __restrict__ in, void* __restrict__ out, const float2* __restrict__ tw, Geom g,
             StepParams* bump) {
  using X = XBulk<L, E>;
  using T = typename X::T;
  constexpr int RB = X::RB, NT = X::NT;
  extern __shared__ __align__(1024) unsigned char smraw[];
  float2* tws = reinterpret_cast<float2*>(smraw + 2 * X::TB);
  float2* twp = tws + X::TWE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smraw + 2 * X::TB + (X::TWE + X::PPE) * 8);
#ifdef GRACE_PDL_EARLY
  pdl_trigger();
#endif
  fill_pass_twiddles<typename X::PL, L>(tws, tw, g.Lmax / L, threadIdx.x, NT);
  // w^k = exp(-2 pi i k / Px), k = 0 .. L/2 (K1's post-process; K5's pre-process
  // takes k > L/2 as w^k = -conj w^(L-k))
  for (int kk = threadIdx.x; kk < X::PPE; kk += NT) twp[kk] = __ldg(tw + kk * (g.Lmax / (2 * L)));
  const int nrows = g.nzl * g.ny;
  const int total = g.nc * nrows;  // rows of components c0 .. c0 + nc - 1
  const size_t rowoff = (size_t)g.c0 * nrows;
  const int ntiles = (total + RB - 1) / RB;
  const int nseg = (!FWD && DIST) ? g.nz / g.nzl : 1;
  const unsigned seg = FWD ? 4u * g.nx : (DIST ? 8u * g.kb : 8u * (L + 2));
  const int lane = threadIdx.x & 31;
  const bool issuer = threadIdx.x < 32;
  auto issue = [&](int t, unsigned char* dst, uint64_t* b) {  // warp 0
    const int r0 = t * RB;
    const int nv = total - r0 < RB ? total - r0 : RB;
    if (lane == 0) mbar_expect_tx(b, (unsigned)(nv * nseg) * seg);
    __syncwarp();
    for (int u = lane; u < nv * nseg; u += 32) {
      const int bb = u / nseg, q = u - bb * nseg;
      const size_t gr = rowoff + (size_t)(r0 + bb);
      const void* src;
      if constexpr (FWD) src = static_cast<const float*>(in) + gr * g.nx;
      else if constexpr (DIST) src = static_cast<const float2*>(in) + q * g.blk1 + gr * g.pitch1;
      else src = static_cast<const float2*>(in) + gr * g.pitch1;
      bulk_load(dst + ((size_t)bb * T::ROWS + (size_t)q * g.kb) * 8, src, seg, b);
    }
  };
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    mbar_fence_init();
  }
  __syncthreads();
  pdl_wait();
  // K1 advances the device step counter (K5 / K6 of the previous step read it)
  if (FWD && bump != nullptr && blockIdx.x == 0 && threadIdx.x == 0) bump->step += 1;
  int t = blockIdx.x;
  if (issuer && t < ntiles) issue(t, smraw, bar);
  if (t + (int)gridDim.x >= ntiles) pdl_trigger();
  for (int k = 0; t < ntiles; ++k, t += gridDim.x) {
    float2* cur = reinterpret_cast<float2*>(smraw + (k & 1) * X::TB);
    if (t + (int)gridDim.x < ntiles && t + 2 * (int)gridDim.x >= ntiles) pdl_trigger();
    if (issuer && t + (int)gridDim.x < ntiles) {
      if (lane == 0) fence_proxy_async();
      __syncwarp();
      issue(t + gridDim.x, smraw + ((k + 1) & 1) * X::TB, bar + ((k + 1) & 1));
    }
    mbar_wait(bar + (k & 1), (k >> 1) & 1);
    const int r0 = t * RB;
    const int nv = total - r0 < RB ? total - r0 : RB;
    if constexpr (FWD) {
      if (g.nx == L)  // the pruned first pass reads exactly the nx/2 packed inputs
        fft_tile<L, RB, NT, false, false, true, false, 1, false, true>(cur, XbLd<T::ROWS, false>{cur, g.nx >> 1},
                                                                       SmemSt<L, RB, false>{cur}, tws, 1);
      else
        fft_tile<L, RB, NT, false, false, true, false, 1, false, true>(cur, XbLd<T::ROWS, true>{cur, g.nx >> 1},
                                                                       SmemSt<L, RB, false>{cur}, tws, 1);
      __syncthreads();
      // X[k] and X[L-k] from the same pair Z[k], Z[L-k] (w^(L-k) = -conj w^k);
      // a thread keeps the row the FFT mapped to it.
      constexpr int TPC = NT / RB;
      const int b = threadIdx.x / TPC, jb = threadIdx.x - b * TPC;
      if (b < nv) {
        float2* X1 = static_cast<float2*>(out);
        const size_t gr = rowoff + (size_t)(r0 + b);
        auto at = [&](int kk) -> float2* {
          if constexpr (DIST) {  // destination-blocked: kx block q goes to rank q
            const int q = kk / g.kb;
            if (g.p2p) return g.peer[q] + g.rank * g.blk1 + gr * g.pitch1 + (kk - q * g.kb);  // fused transpose
            return X1 + q * g.blk1 + gr * g.pitch1 + (kk - q * g.kb);
          } else {
            return X1 + gr * g.pitch1 + kk;
          }
        };
        const float2* z = cur + b * T::ROWS;
        auto post = [](float2 Zk, float2 Zn, float2 w) {
          const float2 E = make_float2(0.5f * (Zk.x + Zn.x), 0.5f * (Zk.y - Zn.y));
          const float2 D = make_float2(0.5f * (Zk.x - Zn.x), 0.5f * (Zk.y + Zn.y));
          const float2 wD = cmul(w, D);
          return make_float2(E.x + wD.y, E.y - wD.x);
        };
#pragma unroll
        for (int i = 0; i < (L / 2) / TPC; ++i) {
          const int kk = jb + i * TPC;
          const float2 w = twp[kk];
          const float2 Zk = z[kk], Zn = z[(L - kk) & (L - 1)];
          *at(kk) = post(Zk, Zn, w);
          *at(L - kk) = post(Zn, Zk, make_float2(-w.x, w.y));
        }
        if (jb == 0) {  // k = L/2 pairs with itself
          const float2 Zk = z[L / 2];
          *at(L / 2) = post(Zk, Zk, twp[L / 2]);
        }
      }
    } else {
      struct Ld {
        __device__ static constexpr bool kSmem() { return true; }
        const float2* s;
        const float2* twp;  // w^k, k <= L/2, in smem
        __device__ float2 operator()(int b, int, int ib, int C) const {
          const int kk = ib + C;
          const float2 a = s[b * T::ROWS + kk];
          const float2 m = s[b * T::ROWS + (L - kk)];
          const float2 S = make_float2(a.x + m.x, a.y - m.y);  // X[k] + conj X[L-k]
          const float2 D = make_float2(a.x - m.x, a.y + m.y);  // X[k] - conj X[L-k]
          float2 w;                                              // exp(-2 pi i k/Px)
          if (kk <= L / 2) {
            w = twp[kk];
          } else {
            const float2 u = twp[L - kk];
            w = make_float2(-u.x, u.y);
          }
          const float2 wD = cmulc(D, w);
          return make_float2(S.x - wD.y, S.y + wD.x);  // S + i w^-k D
        }
      } ld{cur, twp};
      float* H = static_cast<float*>(out) + (rowoff + (size_t)r0) * g.nx;
      if (nv == RB && g.nx == L)  // the pruned last pass produces exactly the nx outputs
        fft_tile<L, RB, NT, false, true, false, true, 1, false, true>(cur, ld, XbSt<false>{H, g.nx, nv}, tws, 1);
      else
        fft_tile<L, RB, NT, false, true, false, true, 1, false, true>(cur, ld, XbSt<true>{H, g.nx, nv}, tws, 1);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K6: Eq. (2) local terms + Eq. (3) + Euler from H_demag in HBM.
// A streaming stencil: each thread owns 4 consecutive cells of a row (16-byte
// loads), components are processed one after another to keep registers low.
// mode 0: M -> Mn; mode 1: store H_eff into Hout.
#ifndef GRACE_K6_MINB
#define GRACE_K6_MINB 4
#endif
// HEUN = 3: predictor (also stores f = dM/dt into Hout); HEUN = 4: corrector,
// M' = renorm(M0 + dt (f0 + f(M*)) / 2) with M0 = Mn (updated in place), f0 = Hout,
// M* = M; the applied field of the next timestep.  HEUN = 5: the adaptive-step
// corrector (grace_step_adaptive): the same M' written over f0 in Hout (M0 kept
// for a rejected attempt), and max over cells |M' - M*| / Ms -- the Euler step's
// local error estimate -- into *aerr (float bits, atomic max).  HEUN = 0: modes 0 / 1.
// MASK (geometry mask, reading Q26): a cell with M = 0 is empty; an empty
// neighbour is a free surface (replaced by the centre, like a missing one), an
// empty centre stays 0 (H_eff 0, f 0).
template <bool VEC, bool DIST, int HEUN = 0, bool MASK = false>
__global__ void __launch_bounds__(256, GRACE_K6_MINB) k6_llg(const float* __restrict__ Hd, const float* __restrict__ M,
                                              float* __restrict__ Mn, float* __restrict__ Hout, Geom g,
                                              const StepParams* __restrict__ prm, unsigned long long* __restrict__ flag,
                                              int mode, const float* __restrict__ Hlo, const float* __restrict__ Hhi,
                                              unsigned* __restrict__ aerr) {
  pdl_trigger();
  pdl_wait();
  constexpr int W = VEC ? 4 : 1;
  const int nrows = g.nzl * g.ny;
  const size_t N = (size_t)nrows * g.nx;
  const size_t plane = (size_t)g.nx * g.ny;
  const size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * W;
  if (i >= N) return;
  const StepParams p = *prm;
  const int row = (int)(i / g.nx), x = (int)(i - (size_t)row * g.nx);
  const int zl = row / g.ny, y = row - zl * g.ny;
  auto ldw = [&](const float* q, float* o) {
    if constexpr (VEC) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(q));
      o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    } else {
      o[0] = __ldg(q);
    }
  };
  const float cxyz[3] = {g.cx, g.cy, g.cz};
  float ha[3];
  {
    StepParams pf = p;
    if (HEUN >= 4) pf.step += 1;  // the corrector's field: timestep k + 1
    applied_field(pf, ha);
  }
  // all 24 loads (3 components x centre, Hd, 4 neighbour rows, 2 row ends) first
  float a[3][W], t[3][W], ym[3][W], yp[3][W], zm[3][W], zp[3][W], xl[3], xr[3];
  const size_t iym = y > 0 ? i - g.nx : i, iyp = y + 1 < g.ny ? i + g.nx : i;
  const float* zlo = zl > 0 ? M + (i - plane) : ((DIST && g.has_lo) ? Hlo + (size_t)y * g.nx + x : M + i);
  const float* zhi = zl + 1 < g.nzl ? M + (i + plane) : ((DIST && g.has_hi) ? Hhi + (size_t)y * g.nx + x : M + i);
  const size_t czlo = (zl > 0 || !(DIST && g.has_lo)) ? N : plane;
  const size_t czhi = (zl + 1 < g.nzl || !(DIST && g.has_hi)) ? N : plane;
  const size_t ixl = x > 0 ? i - 1 : i, ixr = x + W < g.nx ? i + W : i + W - 1;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const float* mc = M + c * N;
    ldw(mc + i, a[c]);
    ldw(Hd + c * N + i, t[c]);
    ldw(mc + iym, ym[c]);
    ldw(mc + iyp, yp[c]);
    ldw(zlo + c * czlo, zm[c]);
    ldw(zhi + c * czhi, zp[c]);
    xl[c] = __ldg(mc + ixl);
    xr[c] = __ldg(mc + ixr);
  }
  bool ea[W], exl = false, exr = false;
  if constexpr (MASK) {
    auto empty = [](float u, float v, float w) { return u == 0.f && v == 0.f && w == 0.f; };
    exl = empty(xl[0], xl[1], xl[2]);
    exr = empty(xr[0], xr[1], xr[2]);
#pragma unroll
    for (int s = 0; s < W; ++s) {
      ea[s] = empty(a[0][s], a[1][s], a[2][s]);
      const bool e0 = empty(ym[0][s], ym[1][s], ym[2][s]), e1 = empty(yp[0][s], yp[1][s], yp[2][s]);
      const bool e2 = empty(zm[0][s], zm[1][s], zm[2][s]), e3 = empty(zp[0][s], zp[1][s], zp[2][s]);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if (e0) ym[c][s] = a[c][s];
        if (e1) yp[c][s] = a[c][s];
        if (e2) zm[c][s] = a[c][s];
        if (e3) zp[c][s] = a[c][s];
      }
    }
  }
  float m[3][W], h[3][W];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
#pragma unroll
    for (int s = 0; s < W; ++s) {
      float l = s > 0 ? a[c][s - 1] : xl[c], r = s + 1 < W ? a[c][s + 1] : xr[c];
      if constexpr (MASK) {
        if (s > 0 ? ea[s - 1] : exl) l = a[c][s];
        if (s + 1 < W ? ea[s + 1] : exr) r = a[c][s];
      }
      // Eq. (2): H_demag + six-neighbour exchange (difference form, Q11) + Zeeman (+ x anisotropy)
      float e = 0.f;
      e += cxyz[0] * (l - a[c][s]);
      e += cxyz[0] * (r - a[c][s]);
      e += cxyz[1] * (ym[c][s] - a[c][s]);
      e += cxyz[1] * (yp[c][s] - a[c][s]);
      e += cxyz[2] * (zm[c][s] - a[c][s]);
      e += cxyz[2] * (zp[c][s] - a[c][s]);
      float hv = t[c][s] + ha[c];
      if (c == 0) hv += g.ck * a[c][s];
      h[c][s] = hv + e;
      m[c][s] = a[c][s];
    }
  }
  float o[3][W], f[3][W], m0[3][W];
  if constexpr (HEUN >= 4) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      ldw(Hout + c * N + i, f[c]);
      ldw(Mn + c * N + i, m0[c]);
    }
  }
#pragma unroll
  for (int s = 0; s < W; ++s) {
    if constexpr (MASK) {
      if (ea[s]) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          o[c][s] = 0.f;
          if constexpr (HEUN == 3) f[c][s] = 0.f;
        }
        continue;
      }
    }
    if (HEUN == 0 && mode == 1) {
      for (int c = 0; c < 3; ++c) o[c][s] = h[c][s];
      continue;
    }
    const float mx = m[0][s], my = m[1][s], mz = m[2][s];
    const float hx = h[0][s], hy = h[1][s], hz = h[2][s];
    // Eq. (3): dM/dt = c_prec (M x H) + c_damp M x (M x H); Euler; renormalise (Q16)
    const float ax = my * hz - mz * hy, ay = mz * hx - mx * hz, az = mx * hy - my * hx;
    const float bx = my * az - mz * ay, by = mz * ax - mx * az, bz = mx * ay - my * ax;
    float sx, sy, sz;
    if constexpr (HEUN >= 4) {
      const float dx = p.c_prec * ax + p.c_damp * bx, dy = p.c_prec * ay + p.c_damp * by,
                  dz = p.c_prec * az + p.c_damp * bz;
      const float hdt = 0.5f * p.dt;
      sx = m0[0][s] + hdt * (f[0][s] + dx);
      sy = m0[1][s] + hdt * (f[1][s] + dy);
      sz = m0[2][s] + hdt * (f[2][s] + dz);
    } else {
      if constexpr (HEUN == 3) {
        f[0][s] = p.c_prec * ax + p.c_damp * bx;
        f[1][s] = p.c_prec * ay + p.c_damp * by;
        f[2][s] = p.c_prec * az + p.c_damp * bz;
      }
      sx = mx + p.dt * (p.c_prec * ax + p.c_damp * bx);
      sy = my + p.dt * (p.c_prec * ay + p.c_damp * by);
      sz = mz + p.dt * (p.c_prec * az + p.c_damp * bz);
    }
    const float sc = g.Ms / sqrtf(sx * sx + sy * sy + sz * sz);
    o[0][s] = sx * sc;
    o[1][s] = sy * sc;
    o[2][s] = sz * sc;
    if (!(isfinite(o[0][s]) && isfinite(o[1][s]) && isfinite(o[2][s])))
      atomicMin(flag, ((unsigned long long)(p.step - 1) << 36) | (unsigned long long)(i + s));
  }
  if constexpr (HEUN == 5) {  // local error estimate |M_Heun - M_Euler| / Ms, max over cells
    float e2 = 0.f;
#pragma unroll
    for (int s = 0; s < W; ++s) {
      const float d0 = o[0][s] - m[0][s], d1 = o[1][s] - m[1][s], d2 = o[2][s] - m[2][s];
      e2 = fmaxf(e2, d0 * d0 + d1 * d1 + d2 * d2);
    }
    const float ev = sqrtf(e2) / g.Ms;
    // non-negative floats order like their bit patterns; NaN (all bits set past inf) wins the max
    const unsigned bits = __reduce_max_sync(__activemask(), isnan(ev) ? 0x7fffffffu : __float_as_uint(ev));
    if ((threadIdx.x & 31) == __ffs(__activemask()) - 1 && bits != 0u) atomicMax(aerr, bits);
  }
  float* dst = (HEUN == 0 && mode == 1) || HEUN == 5 ? Hout : Mn;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    if constexpr (VEC) *reinterpret_cast<float4*>(dst + c * N + i) = make_float4(o[c][0], o[c][1], o[c][2], o[c][3]);
    else dst[c * N + i] = o[c][0];
    if constexpr (HEUN == 3) {
      if constexpr (VEC) *reinterpret_cast<float4*>(Hout + c * N + i) = make_float4(f[c][0], f[c][1], f[c][2], f[c][3]);
      else Hout[c * N + i] = f[c][0];
    }
  }
}

// ---------------------------------------------------------------------------
// Tile choices and dispatch.  EPT = complex values per thread
// per pass and component.
#ifndef GRACE_EPT_K1
#define GRACE_EPT_K1 8
#endif
#ifndef GRACE_MINB_K1
#define GRACE_MINB_K1 3  // CTAs/SM the register budget of K1 (256 threads) is sized for
#endif
#ifndef GRACE_MINB_Z
#define GRACE_MINB_Z 4
#endif
#ifndef GRACE_MINB_Z128
#define GRACE_MINB_Z128 3  // scripts/sweep_z128.sh: block K3 12.15 -> 11.76 ms (4: 128 registers; 2: 15.1 ms)
#endif
#ifndef GRACE_MINB_Z256
#define GRACE_MINB_Z256 8  // scripts/sweep_zlong.sh: 256^3 K3 1.46 -> 1.34 ms
#endif
#ifndef GRACE_MINB_Z512
#define GRACE_MINB_Z512 1  // 2: 64 registers with spills
#endif
#ifndef GRACE_MINB_Z1024
#define GRACE_MINB_Z1024 1  // 512^3 K3 20.7 -> 15.6 ms (2: 648 B of spills)
#endif
#ifndef GRACE_MINB_Z16
#define GRACE_MINB_Z16 8  // radix-4x4 plan (GRACE_RB_Z16): film K3 0.0765 -> 0.064 ms at 8 CTAs/SM (6: 0.0686; radix 16 at 3: 0.0765)
#endif
#ifndef GRACE_EPT_Y
#define GRACE_EPT_Y 16
#endif
#ifndef GRACE_Y_ELEMS
#define GRACE_Y_ELEMS 16384  // complex values per K2/K4 tile
#endif
__host__ __device__ constexpr int tpc_of(int L, int ept) { return L >= ept ? L / ept : 1; }
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }
template <int L, int EPT, int MINB256, int NTT = 256>
struct XCfgT {  // K1 / K5: B spatial rows x 3 components per CTA
  static constexpr int TPC = tpc_of(L, EPT);
  static constexpr int B = (L == 0) ? 64 : cmax(1, NTT / TPC);
  static constexpr int NT = (L == 0) ? 64 : B * TPC;
  static constexpr int MINB = NT <= 256 ? MINB256 : (NT <= 512 ? 2 : 1);
};
// Short rows (L <= 32: cubes up to 32^3, 8^3 .. 32^3 of Table 1) have few rows
// in all: fewer elements per thread and smaller CTAs spread them over more SMs
// (16^3: K5 was one 256-thread CTA).  GRACE_EPT_SMALL = 0 keeps the large-row
// configuration everywhere.
#ifndef GRACE_EPT_SMALL
#define GRACE_EPT_SMALL 4
#endif
#ifndef GRACE_NT_SMALL
#define GRACE_NT_SMALL 64
#endif
template <int L>
constexpr bool x_small() { return GRACE_EPT_SMALL > 0 && L > 0 && L <= 32; }
template <int L>
using X1Cfg = XCfgT<L, x_small<L>() ? GRACE_EPT_SMALL : GRACE_EPT_K1, GRACE_MINB_K1,
                    x_small<L>() ? GRACE_NT_SMALL : 256>;
#ifndef GRACE_EPT_K5S
#define GRACE_EPT_K5S 16
#endif
#ifndef GRACE_MINB_K5S
#define GRACE_MINB_K5S 2
#endif
template <int L>
using X5SCfg = XCfgT<L, x_small<L>() ? GRACE_EPT_SMALL : GRACE_EPT_K5S, GRACE_MINB_K5S,
                     x_small<L>() ? GRACE_NT_SMALL : 256>;  // K5 (C2R -> H_demag)
template <int L>
struct YCfg {  // K2/K4 columns
  static constexpr int NCOL = cmax(2, cmin(32, GRACE_Y_ELEMS / L));
  static constexpr int NT = cmin(1024, cmax(32, NCOL * tpc_of(L, GRACE_EPT_Y)));
  static constexpr int MINB = NT <= 256 ? 4 : (NT <= 512 ? 2 : 1);
};
template <int L>
struct ZCfg {  // K3 and K2'
  static constexpr int B = ZPlan<L>::B;
  static constexpr int NT = ZPlan<L>::NT;
  // L = 16 (film Pz, 8^3 cubes): one thread holds a radix-16 pencil of 3 components
  static constexpr int MINB = (L == 16 ? GRACE_MINB_Z16
                                : L == 128 ? GRACE_MINB_Z128
                                : L == 256 ? GRACE_MINB_Z256
                                : L == 512 ? GRACE_MINB_Z512
                                : L == 1024 ? GRACE_MINB_Z1024
                                : (NT <= 256 ? GRACE_MINB_Z : (NT <= 512 ? 2 : 1)));
  static constexpr size_t SMEM = (size_t)3 * TileIdx<L, B, true>::ELEMS * 8 + (size_t)6 * (L / 2 + 1) * B * 4 +
                                 (PENCIL_TWS ? (size_t)pencil_tw_elems<L>() * 8 : 0);
};

#define GRACE_TRY(x)                       \
  do {                                     \
    const cudaError_t le_ = (x);           \
    if (le_ != cudaSuccess) return le_;    \
  } while (0)

// PDL per step kernel (bit: K1 1, K2 2, K3 4, K4 8, K5 16, K6 32).  Default 23:
// an early-launched persistent K4 behind K3, or K6 behind K5, measured slower on
// the slab (+0.14 / +0.08 ms); the rest gain 4-10% on small grids (SP4, film).
// GRACE_PDL_MASK overrides, GRACE_NO_PDL turns it off.
// A kernel that follows a wait on another stream's event (the pipelined
// distributed step: K2 after its C1 transpose, K5 after its C2) is launched
// without PDL: the programmatic edge would tie it to the preceding kernel only.
static thread_local bool t_no_pdl = false;
void set_pdl_blocked(bool b) { t_no_pdl = b; }
// kid | 64: a kernel of the nz = 1 (K2') step, where every boundary is latency:
// there K6 behind K5 gains too (SP4 10.4 -> 10.0 us/step, refined 13.2 -> 12.7;
// profiles/r02_sweeps.md), so the default mask for those launches is 63.
static bool pdl_on(int kid) {
  static const char* env = getenv("GRACE_PDL_MASK");
  static const int mask = getenv("GRACE_NO_PDL") ? 0 : (env ? atoi(env) : 23);
  static const int mask1 = getenv("GRACE_NO_PDL") ? 0 : (env ? atoi(env) : 63);
  return !t_no_pdl && (((kid & 64) ? mask1 : mask) & kid & 63) != 0;
}
// Step-kernel launch with programmatic stream serialization (PDL, see pdl_wait).
template <class... E, class... A>
static cudaError_t launch_k(int kid, void (*kern)(E...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on(kid) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...);
}

template <class K>
static cudaError_t prep(K kern, size_t smem) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e == cudaSuccess && smem > 48 * 1024)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return e;
}

// Persistent bulk-copy x kernels: 16-byte row copies and the raw X1 row
// (P blocks of kb on the distributed path) inside one tile row.
template <int L>
static bool xbulk_ok(const Geom& g, bool fwd) {
#ifdef GRACE_NO_XBULK
  return false;
#endif
#ifdef GRACE_NO_XBULK_FWD
  if (fwd) return false;
#endif
  constexpr int ROWS = XBulk<L>::T::ROWS;
  if (g.nx % 4 != 0) return false;
  if (fwd) return true;
  if (g.kb) return (g.kb % 2 == 0) && (g.blk1 % 2 == 0) && (long long)(g.nz / g.nzl) * g.kb <= ROWS;
  return g.pitch1 % 2 == 0 && g.pitch1 >= L + 2 && ROWS >= L + 2;
}

template <int L, bool FWD, bool DIST, int E = GRACE_XB_ELEMS>
static cudaError_t xbulk_launch(const Geom& g, const void* in, void* out, const float2* tw, StepParams* bump,
                                cudaStream_t st) {
  using X = XBulk<L, E>;
  if constexpr (E == GRACE_XB_ELEMS && GRACE_XB_ELEMS_TINY < GRACE_XB_ELEMS && L <= GRACE_XB_ELEMS_TINY / 2) {
    // tiny grids: shorter tiles, more CTAs (each CTA's chain is one tile either way)
    if ((g.nc * g.nzl * g.ny + X::RB - 1) / X::RB < g.nsm / 2)
      return xbulk_launch<L, FWD, DIST, GRACE_XB_ELEMS_TINY>(g, in, out, tw, bump, st);
  }
  auto kern = k_x_bulk<L, FWD, DIST, E>;
  cudaError_t e = prep(kern, X::SMEM);
  if (e != cudaSuccess) return e;
  const int ntiles = (g.nc * g.nzl * g.ny + X::RB - 1) / X::RB;
  int per_sm = 0;  // resident CTAs per SM (shared memory may allow fewer than GRACE_XB_MINB)
  GRACE_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, X::NT, X::SMEM));
  const int cap = g.nsm * (per_sm < 1 ? 1 : (per_sm < GRACE_XB_MINB ? per_sm : GRACE_XB_MINB));
  const int grid = ntiles < cap ? ntiles : cap;
  GRACE_TRY(launch_k(FWD ? 1 : 16, kern, grid, X::NT, X::SMEM, st, in, out, tw, g, bump));
  return cudaGetLastError();
}

#define GRACE_L_SWITCH(Lval, CASE) \
  switch (Lval) {                   \
    CASE(1) CASE(2) CASE(4) CASE(8) CASE(16) CASE(32) CASE(64) CASE(128) CASE(256) CASE(512) CASE(1024) CASE(2048) CASE(4096) \
    default: return cudaErrorInvalidValue; \
  }

template <int L, bool DIST>
static cudaError_t k1_launch(const Geom& g, const float* M, float2* X1, const float2* tw, StepParams* bump,
                             cudaStream_t st) {
  using C = X1Cfg<L>;
  const size_t smem = (L == 0) ? 0 : (size_t)3 * TileIdx<(L > 0 ? L : 1), C::B, false>::ELEMS * sizeof(float2);
  if constexpr (L >= kXBulkMinL && L <= kXBulkMaxL) {
    if (xbulk_ok<L>(g, true)) return xbulk_launch<L, true, DIST>(g, M, X1, tw, bump, st);
  }
  auto kern = k1_fwd_x<L, C::B, C::NT, C::MINB, DIST>;
  cudaError_t e = prep(kern, smem);
  if (e != cudaSuccess) return e;
  const int nrows = g.nzl * g.ny;
  GRACE_TRY(launch_k(1, kern, (nrows + C::B - 1) / C::B, C::NT, smem, st, M, X1, tw, g, bump));
  return cudaGetLastError();
}

cudaError_t launch_k1(const Geom& g, const float* M, float2* X1, const float2* tw, StepParams* bump,
                      cudaStream_t st) {
  if (g.Px == 1) return g.kb ? k1_launch<0, true>(g, M, X1, tw, bump, st) : k1_launch<0, false>(g, M, X1, tw, bump, st);
  const int L = g.Px / 2;
#define CASE(v)                                                                \
  case v:                                                                      \
    return (v < 2) ? cudaErrorInvalidValue                                     \
           : g.kb  ? k1_launch<(v >= 2 ? v : 2), true>(g, M, X1, tw, bump, st) \
                   : k1_launch<(v >= 2 ? v : 2), false>(g, M, X1, tw, bump, st);
  GRACE_L_SWITCH(L, CASE)
#undef CASE
}

template <int L, bool INV>
static cudaError_t ky_launch(const Geom& g, const float2* in, float2* out, const float2* tw, cudaStream_t st,
                             int in_rows, int out_rows, int n_in, int n_out) {
  using C = YCfg<L>;
  const size_t smem = (size_t)TileIdx<L, C::NCOL, true>::ELEMS * sizeof(float2);
  auto kern = k_y<L, C::NCOL, C::NT, C::MINB, INV>;
  cudaError_t e = prep(kern, smem);
  if (e != cudaSuccess) return e;
  dim3 grid((g.Kc + C::NCOL - 1) / C::NCOL, g.nc * g.nz);
  GRACE_TRY(launch_k(INV ? 8 : 2, kern, grid, C::NT, smem, st, in, out, tw, g, in_rows, out_rows, n_in, n_out));
  return cudaGetLastError();
}

#ifndef GRACE_YT_ELEMS
#define GRACE_YT_ELEMS 8192  // complex values per TMA y-pencil tile buffer
#endif
template <int L>
__host__ __device__ constexpr int ytma_ncol() {
  return GRACE_YT_ELEMS / L > 32 ? 32 : (GRACE_YT_ELEMS / L < 2 ? 2 : GRACE_YT_ELEMS / L);
}
constexpr int kTmaMinL = 64;

template <int L, bool INV>
static cudaError_t ky_tma_launch(const Geom& g, float2* out, const float2* tw, cudaStream_t st, int n_out,
                                 const TmapBlob* tmap, const TmapBlob* tout = nullptr) {
  constexpr int NCOL = ytma_ncol<L>();
#ifndef GRACE_YT_NB1_1024
#define GRACE_YT_NB1_1024 0  // K4 at L = 1024 single-buffered (two CTAs per SM) as at 2048
#endif
  constexpr int NB = (INV && (L == 2048 || (L == 1024 && GRACE_YT_NB1_1024))) ? GRACE_YT_NB_INV
                                                                            : 2;  // single-buffered slower elsewhere (block K4 27.6 vs 8.0 ms)
  using Y = YTma<L, NCOL, NB>;
  // TMA stores where they measured faster: the single-buffered K4 (slab: 0.63 -> 0.59 ms);
  // the double-buffered one (film, L = 1024) lost 5 % to the read-wait before each reload
  const bool tst = INV && NB == 1 && tout != nullptr && g.kb == 0 && !g.p2p;
  auto kern = tst ? k_y_tma<L, NCOL, INV, NB, INV && NB == 1> : k_y_tma<L, NCOL, INV, NB, false>;
  cudaError_t e = prep(kern, Y::SMEM);
  if (e != cudaSuccess) return e;
  const int ntiles = ((g.Kc + NCOL - 1) / NCOL) * g.nc * g.nz;
  const int want = NB == 1 ? (Y::NT <= 512 ? 2 : 1) : GRACE_YT_MINB;
  const int per_sm = (int)(220 * 1024 / Y::SMEM) < want ? (int)(220 * 1024 / Y::SMEM) : want;
  const int cap = g.nsm * (per_sm > 0 ? per_sm : 1);
  const int grid = ntiles < cap ? ntiles : cap;
  CUtensorMap map, omap;
  static_assert(sizeof(CUtensorMap) == sizeof(TmapBlob), "tensor map size");
  memcpy(&map, tmap->b, sizeof map);
  memcpy(&omap, (tst ? tout : tmap)->b, sizeof omap);
  GRACE_TRY(launch_k(INV ? 8 : 2, kern, grid, Y::NT, Y::SMEM, st, map, omap, out, tw, g, n_out));
  return cudaGetLastError();
}

static cudaError_t encode5(TmapBlob* out, const void* base, const unsigned long long dims[5],
                           const unsigned long long strides[4], unsigned box_cols, unsigned box_rows);
template <int L>
static cudaError_t ky_stage_launch(const Geom& g, float2* out, const float2* tw, cudaStream_t st,
                                   const TmapBlob* tmap) {
  using Y = YStage<L>;
  auto kern = k_y_stage<L>;
  cudaError_t e = prep(kern, Y::SMEM);
  if (e != cudaSuccess) return e;
  const int ntiles = ((g.Kc + Y::NCOL - 1) / Y::NCOL) * g.nc * g.nz;
  const int cap = g.nsm * (L == 2048 ? GRACE_YSTAGE_MINB : 1);
  const int grid = ntiles < cap ? ntiles : cap;
  CUtensorMap map;
  memcpy(&map, tmap->b, sizeof map);
  CUtensorMap omap = map;
  if constexpr (GRACE_K2_TMA_STORE) {  // X2 [3][nz][Py][pitch2]: boxes of the tile's columns x BR rows
    const unsigned long long p2 = 8ull * g.pitch2;
    const unsigned long long d[5] = {(unsigned long long)g.Kc, (unsigned long long)g.Py, (unsigned long long)g.nz, 3, 1};
    const unsigned long long sd[4] = {p2, p2 * g.Py, p2 * g.Py * g.nz, p2 * g.Py * g.nz * 3};
    TmapBlob ob;
    GRACE_TRY(encode5(&ob, out, d, sd, Y::NCOL, Y::BR));
    memcpy(&omap, ob.b, sizeof omap);
  }
  GRACE_TRY(launch_k(2, kern, grid, Y::NT, Y::SMEM, st, map, omap, out, tw, g, g.Py));
  return cudaGetLastError();
}

cudaError_t launch_k2(const Geom& g, const float2* X1, float2* X2, const float2* tw, cudaStream_t st,
                      const TmapBlob* tmap) {
#ifndef GRACE_NO_YSTAGE
  if (tmap != nullptr && g.Py == 4096) return ky_stage_launch<4096>(g, X2, tw, st, tmap);
  if (GRACE_YSTAGE_2048 && tmap != nullptr && g.Py == 2048) return ky_stage_launch<2048>(g, X2, tw, st, tmap);
  if (GRACE_YSTAGE_1024 && tmap != nullptr && g.Py == 1024) return ky_stage_launch<1024>(g, X2, tw, st, tmap);
#endif
  // The TMA tiles hold GRACE_YT_ELEMS / L columns; below 4 (L >= 4096) K2's row
  // stores are 16-byte half sectors and cost L2 read-modify-writes (block
  // 2048x2048x64: 22.3 ms, 4.6x the input read from DRAM), so K2 takes the
  // 4-column non-TMA kernel there (11.4 ms); K4 keeps TMA (7.9 vs 13.6 ms).
  if (tmap != nullptr && g.Py >= kTmaMinL && GRACE_YT_ELEMS / g.Py >= 4) {
#define CASE(v) case v: return (v >= kTmaMinL) ? ky_tma_launch<(v >= kTmaMinL ? v : kTmaMinL), false>(g, X2, tw, st, g.Py, tmap) : cudaErrorInvalidValue;
    GRACE_L_SWITCH(g.Py, CASE)
#undef CASE
  }
#define CASE(v) case v: return ky_launch<v, false>(g, X1, X2, tw, st, g.ny, g.Py, g.ny, g.Py);
  GRACE_L_SWITCH(g.Py, CASE)
#undef CASE
}

cudaError_t launch_k4(const Geom& g, const float2* X2, float2* X1, const float2* tw, cudaStream_t st,
                      const TmapBlob* tmap, const TmapBlob* tout) {
  if (tmap != nullptr && g.Py >= kTmaMinL) {
#define CASE(v) case v: return (v >= kTmaMinL) ? ky_tma_launch<(v >= kTmaMinL ? v : kTmaMinL), true>(g, X1, tw, st, g.ny, tmap, tout) : cudaErrorInvalidValue;
    GRACE_L_SWITCH(g.Py, CASE)
#undef CASE
  }
#define CASE(v) case v: return ky_launch<v, true>(g, X2, X1, tw, st, g.Py, g.ny, g.Py, g.ny);
  GRACE_L_SWITCH(g.Py, CASE)
#undef CASE
}

// Host: 5-D tensor maps {kx, rows, z, component, block} over 8-byte elements.
#ifndef GRACE_TMA_PROMO
#define GRACE_TMA_PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_128B
#endif
static cudaError_t encode5(TmapBlob* out, const void* base, const unsigned long long dims[5],
                           const unsigned long long strides[4], unsigned box_cols, unsigned box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
    enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  cuuint64_t gd[5], gs[4];
  for (int i = 0; i < 5; ++i) gd[i] = dims[i];
  for (int i = 0; i < 4; ++i) gs[i] = strides[i];
  const cuuint32_t box[5] = {box_cols, box_rows, 1, 1, 1};
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(reinterpret_cast<CUtensorMap*>(out->b), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5,
                   const_cast<void*>(base), gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   GRACE_TMA_PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Host: N-D tensor map (rank 1..5) over `dtype` elements, box `box`, no swizzle.
static cudaError_t encode_map(TmapBlob* out, CUtensorMapDataType dtype, int rank, const void* base,
                              const unsigned long long* dims, const unsigned long long* strides,
                              const unsigned* box) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
    enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  cuuint64_t gd[5], gs[4];
  cuuint32_t bx[5], es[5];
  for (int i = 0; i < rank; ++i) {
    gd[i] = dims[i];
    bx[i] = box[i];
    es[i] = 1;
  }
  for (int i = 0; i + 1 < rank; ++i) gs[i] = strides[i];
  CUresult r = enc(reinterpret_cast<CUtensorMap*>(out->b), dtype, rank, const_cast<void*>(base), gd, gs, bx, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, GRACE_TMA_PROMO,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// KP's input: X1 [3 nz][ny][pitch1] complex (8-byte elements), boxes of one column
// pair x BY rows x one (c, z) row set.
cudaError_t make_plane_tmap(const Geom& g, const float2* X1, TmapBlob* map) {
  const unsigned long long p1 = 8ull * g.pitch1;
  const unsigned long long d[3] = {(unsigned long long)g.Kx, (unsigned long long)g.ny, 3ull * g.nz};
  const unsigned long long str[2] = {p1, p1 * g.ny};
  const unsigned by = (unsigned)(g.ny < 256 ? g.ny : 256);
  const unsigned box[3] = {2, by, 1};
  return encode_map(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, X1, d, str, box);
}

template <int L>
static cudaError_t ky_maps(const Geom& g, const float2* k2_in, const float2* x2, TmapBlob* k2map, TmapBlob* k4map,
                           TmapBlob* k4out) {
  constexpr int NCOL = ytma_ncol<L>();
  using Y = YTma<L, NCOL>;
  const int nq = g.kb ? (g.nz / g.nzl) : 1;
  const unsigned long long p1 = 8ull * g.pitch1, p2 = 8ull * g.pitch2;
  const unsigned long long d2[5] = {(unsigned long long)g.Kc, (unsigned long long)g.ny, (unsigned long long)g.nzl, 3,
                                    (unsigned long long)nq};
  const unsigned long long s2[4] = {p1, p1 * g.ny, p1 * g.ny * g.nzl, p1 * g.ny * g.nzl * 3};
  // K2's map: 4-column boxes for the staged long-pencil kernel (k_y_stage)
#ifndef GRACE_NO_YSTAGE
  constexpr int NCOL2 = (L == 4096 || (L == 2048 && GRACE_YSTAGE_2048) || (L == 1024 && GRACE_YSTAGE_1024))
                            ? YStage<(L >= 1024 ? L : 1024)>::NCOL
                            : NCOL;
#else
  constexpr int NCOL2 = NCOL;
#endif
  cudaError_t e = encode5(k2map, k2_in, d2, s2, NCOL2, Y::br(false));
  if (e != cudaSuccess) return e;
  // K4's TMA stores into X1 (single GPU: one block): boxes of the K4 tile's columns
  if (k4out != nullptr && g.kb == 0) {
    e = encode5(k4out, k2_in, d2, s2, NCOL, Y::br(true));
    if (e != cudaSuccess) return e;
  }
  const unsigned long long d4[5] = {(unsigned long long)g.Kc, (unsigned long long)g.Py, (unsigned long long)g.nz, 3, 1};
  const unsigned long long s4[4] = {p2, p2 * g.Py, p2 * g.Py * g.nz, p2 * g.Py * g.nz * 3};
  return encode5(k4map, x2, d4, s4, NCOL, Y::br(true));
}

cudaError_t make_ky_tmaps(const Geom& g, const float2* k2_in, const float2* x2, TmapBlob* k2map, TmapBlob* k4map,
                          TmapBlob* k4out) {
  if (g.Py < kTmaMinL || g.Kc < 1) return cudaErrorNotSupported;
#define CASE(v) case v: return (v >= kTmaMinL) ? ky_maps<(v >= kTmaMinL ? v : kTmaMinL)>(g, k2_in, x2, k2map, k4map, k4out) : cudaErrorNotSupported;
  GRACE_L_SWITCH(g.Py, CASE)
#undef CASE
}

#ifndef GRACE_MINB_Z3T64
#define GRACE_MINB_Z3T64 4  // CTAs/SM the TMA K3's register budget is sized for at Pz = 64
#endif
#ifndef GRACE_K3_TMA_MINL
#define GRACE_K3_TMA_MINL 16  // shortest z pencil fed by TMA (film Pz = 16: K3 0.064 -> 0.054 ms, step 0.216 -> 0.205)
#endif
template <int L>
#ifndef GRACE_K3_TMA_MAXL
#define GRACE_K3_TMA_MAXL 128  // longest z pencil fed by TMA (block Pz = 128: K3 11.4 -> 10.5 ms; 256 neutral)
#endif
constexpr bool k3_tma_ok() {
  return L >= GRACE_K3_TMA_MINL && L >= 16 && L <= GRACE_K3_TMA_MAXL && !TileIdx<L, ZPlan<L>::B, true>::PAD &&
         ZPlan<L>::B * 8 >= 16;
}

// K3 tensor maps: X2 [3][nz][Py][pitch2] complex as 4-D {kx < Kc, ky, z, c}, box
// {B, 1, Pz/2, 1}; KS [6][Kzh][Kyh][KSp] fp32 as 4-D {kx, ky', kz', c}, box
// {B, 1, Kzh, 6}.
template <int L>
static cudaError_t k3_maps(const Geom& g, const float2* X2, const float* KS, TmapBlob* xmap, TmapBlob* kmap) {
  if constexpr (!k3_tma_ok<L>()) {
    return cudaErrorNotSupported;
  } else {
    using Z = Z3Tma<L>;
    const unsigned long long p2 = 8ull * g.pitch2;
    const unsigned long long xd[4] = {(unsigned long long)g.Kc, (unsigned long long)g.Py, (unsigned long long)g.nz, 3};
    const unsigned long long xs[3] = {p2, p2 * g.Py, p2 * g.Py * g.nz};
    const unsigned xb[4] = {(unsigned)Z::B, 1, (unsigned)Z::H, 1};
    cudaError_t e = encode_map(xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, X2, xd, xs, xb);
    if (e != cudaSuccess) return e;
    const unsigned long long pk = 4ull * g.KSp;
    const unsigned long long kd[4] = {(unsigned long long)g.KSp, (unsigned long long)g.Kyh, (unsigned long long)g.Kzh,
                                      6};
    const unsigned long long ks[3] = {pk, pk * g.Kyh, pk * g.Kyh * g.Kzh};
    const unsigned kbx[4] = {(unsigned)Z::B, 1, (unsigned)Z::KZH, 6};
    return encode_map(kmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, KS, kd, ks, kbx);
  }
}

cudaError_t make_k3_tmaps(const Geom& g, const float2* X2, const float* KS, TmapBlob* xmap, TmapBlob* kmap) {
  if (g.Pz < 2 || g.Kc < 1 || fused_y_path(g)) return cudaErrorNotSupported;
#define CASE(v) case v: return (v >= 2 && v <= 1024) ? k3_maps<(v >= 2 && v <= 1024 ? v : 2)>(g, X2, KS, xmap, kmap) : cudaErrorNotSupported;
  GRACE_L_SWITCH(g.Pz, CASE)
#undef CASE
}

// The TMA K3's per-pass twiddle tables in its shared-memory layout, built once
// per context so each CTA brings them in with one bulk copy.
template <int L>
__global__ void k_k3_twiddles(float2* dst, const float2* tw, int twstride) {
  constexpr int RB = ZPlan<L>::RB;
  fill_pass_twiddles<Plan<L, false, RB>, L>(dst, tw, twstride, threadIdx.x, blockDim.x);
  fill_pass_twiddles<Plan<L, true, RB>, L>(dst + Plan<L, false, RB>::TW_ELEMS, tw, twstride, threadIdx.x, blockDim.x);
}

template <int L>
static cudaError_t k3_tables(const Geom& g, const float2* tw, float2** out, cudaStream_t st) {
  *out = nullptr;
  if constexpr (k3_tma_ok<L>()) {
    if constexpr (Z3Tma<L>::TWS && Z3Tma<L>::TWB > 0) {
      GRACE_TRY(cudaMalloc(out, Z3Tma<L>::TWB));
      k_k3_twiddles<L><<<1, 256, 0, st>>>(*out, tw, g.Lmax / L);
      return cudaGetLastError();
    }
  }
  return cudaSuccess;
}

cudaError_t make_k3_twiddles(const Geom& g, const float2* tw, float2** out, cudaStream_t st) {
  *out = nullptr;
  if (g.Pz < 2 || fused_y_path(g)) return cudaSuccess;
#define CASE(v) case v: return (v >= 2 && v <= 1024) ? k3_tables<(v >= 2 && v <= 1024 ? v : 2)>(g, tw, out, st) : cudaSuccess;
  GRACE_L_SWITCH(g.Pz, CASE)
#undef CASE
}

template <int L>
static cudaError_t k3_launch(const Geom& g, float2* X2, const float* KS, const float2* tw, cudaStream_t st,
                             const TmapBlob* xmap, const TmapBlob* kmap, const float2* tw3) {
  using C = ZCfg<L>;
  if constexpr (k3_tma_ok<L>()) {
    if (xmap != nullptr && kmap != nullptr && !getenv("GRACE_NO_K3_TMA")) {
      using Z = Z3Tma<L>;
      CUtensorMap xm, km;
      memcpy(&xm, xmap->b, sizeof xm);
      memcpy(&km, kmap->b, sizeof km);
      auto kern = k3_z_tma<L, (L == 64 ? GRACE_MINB_Z3T64 : C::MINB)>;
      cudaError_t e = prep(kern, Z::SMEM);
      if (e != cudaSuccess) return e;
      dim3 grid((g.Kc + Z::B - 1) / Z::B, g.Kyh);
      GRACE_TRY(launch_k(4, kern, grid, Z::NT, Z::SMEM, st, xm, km, X2, tw, tw3, g));
      return cudaGetLastError();
    }
  }
  auto kern = k3_z<L, C::B, C::NT, C::MINB>;
  cudaError_t e = prep(kern, C::SMEM);
  if (e != cudaSuccess) return e;
  dim3 grid((g.Kc + C::B - 1) / C::B, g.Kyh);
  GRACE_TRY(launch_k(4, kern, grid, C::NT, C::SMEM, st, X2, KS, tw, g));
  return cudaGetLastError();
}

cudaError_t launch_k3(const Geom& g, float2* X2, const float* KS, const float2* tw, cudaStream_t st,
                      const TmapBlob* xmap, const TmapBlob* kmap, const float2* tw3) {
  if (g.Pz == 1) {
    dim3 grid((g.Kc + 127) / 128, g.Py);
    GRACE_TRY(launch_k(4, k_mul_plane, grid, 128, 0, st, X2, KS, g));
    return cudaGetLastError();
  }
#define CASE(v) case v: return (v >= 2 && v <= 1024) ? k3_launch<(v >= 2 && v <= 1024 ? v : 2)>(g, X2, KS, tw, st, xmap, kmap, tw3) : cudaErrorInvalidValue;
  GRACE_L_SWITCH(g.Pz, CASE)
#undef CASE
}

bool fused_y_path(const Geom& g) { return g.Pz == 1 && g.Py <= 512; }

// K1 and K5 take the persistent bulk-copy kernels (which, like K2 and K4, can run
// on a range of components): the distributed step may then pipeline the
// transposes per component.
bool p2p_ok(const Geom& g) { return comp_split_ok(g) && g.Py >= kTmaMinL; }

bool comp_split_ok(const Geom& g) {
  if (g.Px < 2 || fused_y_path(g)) return false;
#define CASE(v) case v: return (v >= kXBulkMinL && v <= kXBulkMaxL) && xbulk_ok<(v >= kXBulkMinL && v <= kXBulkMaxL ? v : kXBulkMinL)>(g, true) && xbulk_ok<(v >= kXBulkMinL && v <= kXBulkMaxL ? v : kXBulkMinL)>(g, false);
  switch (g.Px / 2) {
    CASE(1) CASE(2) CASE(4) CASE(8) CASE(16) CASE(32) CASE(64) CASE(128) CASE(256) CASE(512) CASE(1024) CASE(2048) CASE(4096)
    default: return false;
  }
#undef CASE
}
int kernel_count(const Geom& g) { return (fused_y_path(g) || g.plane ? 3 : 5) + 1; }

template <int HEUN, bool MASK>
static cudaError_t k6_launch(const Geom& g, int mode, const float* Hd, const float* M, float* Mn, float* Hout,
                             const StepParams* prm, unsigned long long* flag, cudaStream_t st, const float* Hlo,
                             const float* Hhi, unsigned* aerr) {
  const long long N = (long long)g.nzl * g.ny * g.nx;
#ifndef GRACE_K6_VEC_MIN
#define GRACE_K6_VEC_MIN 16384  // cells below which K6 runs one cell per thread: 4x the CTAs on tiny grids (SP4 10.5 -> 9.1 us/step; 32^3 is 4 % slower scalar)
#endif
  const bool vec = g.nx % 4 == 0 && N >= GRACE_K6_VEC_MIN;
  const long long threads = vec ? N / 4 : N;
  const unsigned grid = (unsigned)((threads + 255) / 256);
  const int k6kid = fused_y_path(g) ? 32 | 64 : 32;
  if (vec) {
    if (g.kb) GRACE_TRY(launch_k(k6kid, k6_llg<true, true, HEUN, MASK>, grid, 256, 0, st, Hd, M, Mn, Hout, g, prm, flag, mode, Hlo, Hhi, aerr));
    else GRACE_TRY(launch_k(k6kid, k6_llg<true, false, HEUN, MASK>, grid, 256, 0, st, Hd, M, Mn, Hout, g, prm, flag, mode, Hlo, Hhi, aerr));
  } else {
    if (g.kb) GRACE_TRY(launch_k(k6kid, k6_llg<false, true, HEUN, MASK>, grid, 256, 0, st, Hd, M, Mn, Hout, g, prm, flag, mode, Hlo, Hhi, aerr));
    else GRACE_TRY(launch_k(k6kid, k6_llg<false, false, HEUN, MASK>, grid, 256, 0, st, Hd, M, Mn, Hout, g, prm, flag, mode, Hlo, Hhi, aerr));
  }
  return cudaGetLastError();
}

// mode 0: Euler step M -> Mn; 1: H_eff -> Hout; 3: Heun predictor (M* -> Mn,
// dM/dt -> Hout); 4: Heun corrector (M = M*, Mn = M_k updated in place, Hout = f0);
// 5: adaptive corrector (M = M*, Mn = M_k kept, Hout = f0 -> M', error into aerr).
cudaError_t launch_k6(const Geom& g, int mode, const float* Hd, const float* M, float* Mn, float* Hout,
                      const StepParams* prm, unsigned long long* flag, cudaStream_t st, const float* Hlo,
                      const float* Hhi, unsigned* aerr) {
  if (g.masked) {  // geometry mask (reading Q26)
    if (mode == 3) return k6_launch<3, true>(g, mode, Hd, M, Mn, Hout, prm, flag, st, Hlo, Hhi, aerr);
    if (mode == 4) return k6_launch<4, true>(g, mode, Hd, M, Mn, Hout, prm, flag, st, Hlo, Hhi, aerr);
    if (mode == 5) return k6_launch<5, true>(g, mode, Hd, M, Mn, Hout, prm, flag, st, Hlo, Hhi, aerr);
    return k6_launch<0, true>(g, mode, Hd, M, Mn, Hout, prm, flag, st, Hlo, Hhi, aerr);
  }
  if (mode == 3) return k6_launch<3, false>(g, mode, Hd, M, Mn, Hout, prm, flag, st, Hlo, Hhi, aerr);
  if (mode == 4) return k6_launch<4, false>(g, mode, Hd, M, Mn, Hout, prm, flag, st, Hlo, Hhi, aerr);
  if (mode == 5) return k6_launch<5, false>(g, mode, Hd, M, Mn, Hout, prm, flag, st, Hlo, Hhi, aerr);
  return k6_launch<0, false>(g, mode, Hd, M, Mn, Hout, prm, flag, st, Hlo, Hhi, aerr);
}

template <int L>
static cudaError_t k2f_launch(const Geom& g, float2* X1, const float* KS, const float2* tw, cudaStream_t st) {
  using C = ZCfg<L>;
  auto kern = k2f_y_fused<L, C::B, C::NT, C::MINB>;
  cudaError_t e = prep(kern, C::SMEM);
  if (e != cudaSuccess) return e;
  GRACE_TRY(launch_k(2, kern, (g.Kx + C::B - 1) / C::B, C::NT, C::SMEM, st, X1, KS, tw, g));
  return cudaGetLastError();
}

cudaError_t launch_k2f(const Geom& g, float2* X1, const float* KS, const float2* tw, cudaStream_t st) {
#define CASE(v) case v: return (v <= 512) ? k2f_launch<(v <= 512 ? v : 512)>(g, X1, KS, tw, st) : cudaErrorInvalidValue;
  GRACE_L_SWITCH(g.Py, CASE)
#undef CASE
}

// KP eligibility: GRACE_PLANE=1, single GPU (unblocked kx), 2 <= nz with
// Pz <= 16, Py an instantiated length whose plane fits one CTA.
template <int LY, int PZ>
static constexpr bool plane_fits() {
  return LY >= 256 && LY <= 4096 && PlaneCfg<LY, PZ>::SMEM <= 227 * 1024;
}
template <int PZ>
static bool plane_fits_rt(int LY) {
  switch (LY) {
    case 256: return plane_fits<256, PZ>();
    case 512: return plane_fits<512, PZ>();
    case 1024: return plane_fits<1024, PZ>();
    case 2048: return plane_fits<2048, PZ>();
    case 4096: return plane_fits<4096, PZ>();
    default: return false;
  }
}
bool plane_ok(const Geom& g) {
  const char* on = getenv("GRACE_PLANE");  // opt-in: measured slower than K2..K4 on B200
  if (!on || on[0] != '1' || g.kb != 0 || g.Kc != g.Kx || g.nz < 2 || g.Px < 2) return false;
  if (g.Pz == 4) return plane_fits_rt<4>(g.Py);
  if (g.Pz == 8) return plane_fits_rt<8>(g.Py);
  if (g.Pz == 16) return plane_fits_rt<16>(g.Py);
  return false;
}
size_t plane_ks_floats(const Geom& g) { return (size_t)plane_ks_stride(g.Kzh, g.Kyh) * g.Kx; }
cudaError_t launch_plane_ks(const Geom& g, float* KSP, const float* KS, cudaStream_t st) {
  k_plane_ks<<<4 * g.nsm, 256, 0, st>>>(KSP, KS, g);
  return cudaGetLastError();
}
template <int LY, int PZ>
static cudaError_t kplane_launch(const Geom& g, float2* X1, const float* KSP, const float2* tw, cudaStream_t st,
                                 const TmapBlob* map) {
  if constexpr (plane_fits<LY, PZ>()) {
    using C = PlaneCfg<LY, PZ>;
    auto kern = k_plane<LY, PZ>;
    cudaError_t e = prep(kern, C::SMEM);
    if (e != cudaSuccess) return e;
    CUtensorMap xm;
    std::memcpy(&xm, map->b, sizeof xm);
    GRACE_TRY(launch_k(2, kern, g.Kx, C::NT, C::SMEM, st, xm, X1, KSP, tw, g));
    return cudaGetLastError();
  } else {
    return cudaErrorInvalidValue;
  }
}
template <int PZ>
static cudaError_t kplane_launch_z(const Geom& g, float2* X1, const float* KSP, const float2* tw, cudaStream_t st,
                                   const TmapBlob* map) {
  switch (g.Py) {
    case 256: return kplane_launch<256, PZ>(g, X1, KSP, tw, st, map);
    case 512: return kplane_launch<512, PZ>(g, X1, KSP, tw, st, map);
    case 1024: return kplane_launch<1024, PZ>(g, X1, KSP, tw, st, map);
    case 2048: return kplane_launch<2048, PZ>(g, X1, KSP, tw, st, map);
    case 4096: return kplane_launch<4096, PZ>(g, X1, KSP, tw, st, map);
    default: return cudaErrorInvalidValue;
  }
}
cudaError_t launch_kplane(const Geom& g, float2* X1, const float* KSP, const float2* tw, cudaStream_t st,
                          const TmapBlob* map) {
  if (!map) return cudaErrorInvalidValue;
  if (g.Pz == 4) return kplane_launch_z<4>(g, X1, KSP, tw, st, map);
  if (g.Pz == 8) return kplane_launch_z<8>(g, X1, KSP, tw, st, map);
  if (g.Pz == 16) return kplane_launch_z<16>(g, X1, KSP, tw, st, map);
  return cudaErrorInvalidValue;
}

template <int L, bool DIST>
static cudaError_t k5_launch(const Geom& g, const float2* X1, float* Hd, const float2* tw, cudaStream_t st) {
  if constexpr (L >= kXBulkMinL && L <= kXBulkMaxL) {
    if (xbulk_ok<L>(g, false)) return xbulk_launch<L, false, DIST>(g, X1, Hd, tw, nullptr, st);
  }
  using C = X5SCfg<L>;
  const size_t smem = (L == 0) ? 0 : (size_t)3 * TileIdx<(L > 0 ? L : 1), C::B, false>::ELEMS * sizeof(float2);
  auto kern = k5_inv_x<L, C::B, C::NT, C::MINB, DIST>;
  cudaError_t e = prep(kern, smem);
  if (e != cudaSuccess) return e;
  const int nrows = g.nzl * g.ny;
  GRACE_TRY(launch_k(16, kern, (nrows + C::B - 1) / C::B, C::NT, smem, st, X1, Hd, tw, g));
  return cudaGetLastError();
}

cudaError_t launch_k5(const Geom& g, const float2* X1, float* Hd, const float2* tw, cudaStream_t st) {
  if (g.Px == 1) return g.kb ? k5_launch<0, true>(g, X1, Hd, tw, st) : k5_launch<0, false>(g, X1, Hd, tw, st);
  const int L = g.Px / 2;
#define CASE(v)                                                          \
  case v:                                                                \
    return (v < 2) ? cudaErrorInvalidValue                               \
           : g.kb  ? k5_launch<(v >= 2 ? v : 2), true>(g, X1, Hd, tw, st) \
                   : k5_launch<(v >= 2 ? v : 2), false>(g, X1, Hd, tw, st);
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
// non-finite cell records its index.  With a geometry mask, empty
// cells (mask 0) get M = 0 whatever the input (reading Q26).
__global__ void k_set_m_f64(const double* __restrict__ src, float* __restrict__ M, long long n, double Ms,
                            const unsigned char* __restrict__ mask, unsigned long long* flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    if (mask && !mask[i]) {
      M[i] = M[n + i] = M[2 * n + i] = 0.f;
      continue;
    }
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
                            const unsigned char* __restrict__ mask, unsigned long long* flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    if (mask && !mask[i]) {
      M[i] = M[n + i] = M[2 * n + i] = 0.f;
      continue;
    }
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

cudaError_t launch_set_m_f64(const double* src, float* M, long long n, double Ms, const unsigned char* mask,
                             unsigned long long* flag, cudaStream_t st) {
  k_set_m_f64<<<148 * 8, 256, 0, st>>>(src, M, n, Ms, mask, flag);
  return cudaGetLastError();
}
cudaError_t launch_set_m_f32(const float* src, float* M, long long n, float Ms, const unsigned char* mask,
                             unsigned long long* flag, cudaStream_t st) {
  k_set_m_f32<<<148 * 8, 256, 0, st>>>(src, M, n, Ms, mask, flag);
  return cudaGetLastError();
}

// grace_set_geometry: M <- 0 in the empty cells of the mask (reading Q26).
__global__ void k_apply_mask(float* __restrict__ M, long long n, const unsigned char* __restrict__ mask) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (!mask[i]) M[i] = M[n + i] = M[2 * n + i] = 0.f;
}
cudaError_t launch_apply_mask(float* M, long long n, const unsigned char* mask, cudaStream_t st) {
  k_apply_mask<<<148 * 8, 256, 0, st>>>(M, n, mask);
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

// Diagnostics: the discrete Eq. (1) energy terms
// (per bond to the +x/+y/+z neighbour, per cell otherwise) and the
// SPEC relax torque max_c |M x H_eff| / (Ms |H_eff| + eps),
// per cell in fp64, fixed-order two-stage reduction.  Sums out[0..3] =
// sum |M_nb - M|^2 / Delta^2, sum (Ms^2 - Mx^2), sum H_d.M, sum H_ext.M (the host
// applies V, A/Ms^2, Ku/Ms^2, -mu0/2, -mu0); out[4] = max torque.
template <bool DIST>
__global__ void k_diag_partial(const float* __restrict__ M, const float* __restrict__ Hd, Geom g,
                               const StepParams* __restrict__ prm, const float* __restrict__ Hlo,
                               const float* __restrict__ Hhi, double idx2, double idy2, double idz2,
                               double* __restrict__ partial) {
  __shared__ double sh[5][kRedThreads];
  const long long n = (long long)g.nzl * g.ny * g.nx;
  const long long plane = (long long)g.ny * g.nx;
  const long long chunk = (n + gridDim.x - 1) / gridDim.x;
  const long long lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
  const StepParams p = *prm;
  float ha[3];
  applied_field(p, ha);
  double acc[4] = {0, 0, 0, 0}, tmax = 0;
  for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const long long row = i / g.nx;
    const int x = (int)(i - row * g.nx);
    const int zl = (int)(row / g.ny), y = (int)(row - (long long)zl * g.ny);
    const long long ip = i - (long long)zl * plane;  // in-plane index (halo buffers)
    float a[3], nb[6][3];
    for (int c = 0; c < 3; ++c) a[c] = M[c * n + i];
    for (int c = 0; c < 3; ++c) {
      nb[0][c] = x > 0 ? M[c * n + i - 1] : a[c];
      nb[1][c] = x + 1 < g.nx ? M[c * n + i + 1] : a[c];
      nb[2][c] = y > 0 ? M[c * n + i - g.nx] : a[c];
      nb[3][c] = y + 1 < g.ny ? M[c * n + i + g.nx] : a[c];
      nb[4][c] = zl > 0 ? M[c * n + i - plane] : ((DIST && g.has_lo) ? Hlo[c * plane + ip] : a[c]);
      nb[5][c] = zl + 1 < g.nzl ? M[c * n + i + plane] : ((DIST && g.has_hi) ? Hhi[c * plane + ip] : a[c]);
    }
    if (g.masked) {  // reading Q26: skip empty cells; an empty neighbour is a free surface
      if (a[0] == 0.f && a[1] == 0.f && a[2] == 0.f) continue;
      for (int k = 0; k < 6; ++k)
        if (nb[k][0] == 0.f && nb[k][1] == 0.f && nb[k][2] == 0.f)
          for (int c = 0; c < 3; ++c) nb[k][c] = a[c];
    }
    // bonds to the +x, +y, +z neighbours (a missing neighbour adds nothing)
    const double w[3] = {idx2, idy2, idz2};
    for (int ax = 0; ax < 3; ++ax)
      for (int c = 0; c < 3; ++c) {
        const double d = (double)nb[2 * ax + 1][c] - (double)a[c];
        acc[0] += w[ax] * d * d;
      }
    acc[1] += (double)g.Ms * g.Ms - (double)a[0] * a[0];
    float h[3];
    for (int c = 0; c < 3; ++c) {
      acc[2] += (double)Hd[c * n + i] * a[c];
      acc[3] += (double)ha[c] * a[c];
      // H_eff as the step kernels form it (Eq. (2), six-neighbour difference form)
      float e = 0.f;
      e += g.cx * (nb[0][c] - a[c]);
      e += g.cx * (nb[1][c] - a[c]);
      e += g.cy * (nb[2][c] - a[c]);
      e += g.cy * (nb[3][c] - a[c]);
      e += g.cz * (nb[4][c] - a[c]);
      e += g.cz * (nb[5][c] - a[c]);
      h[c] = Hd[c * n + i] + ha[c] + (c == 0 ? g.ck * a[0] : 0.f) + e;
    }
    const double tx = (double)a[1] * h[2] - (double)a[2] * h[1];
    const double ty = (double)a[2] * h[0] - (double)a[0] * h[2];
    const double tz = (double)a[0] * h[1] - (double)a[1] * h[0];
    const double hn = sqrt((double)h[0] * h[0] + (double)h[1] * h[1] + (double)h[2] * h[2]);
    const double t = sqrt(tx * tx + ty * ty + tz * tz) / ((double)g.Ms * hn + 1e-30);
    tmax = t > tmax ? t : tmax;
  }
  for (int q = 0; q < 4; ++q) sh[q][threadIdx.x] = acc[q];
  sh[4][threadIdx.x] = tmax;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      for (int q = 0; q < 4; ++q) sh[q][threadIdx.x] += sh[q][threadIdx.x + st];
      sh[4][threadIdx.x] = fmax(sh[4][threadIdx.x], sh[4][threadIdx.x + st]);
    }
    __syncthreads();
  }
  if (threadIdx.x < 5) partial[threadIdx.x * gridDim.x + blockIdx.x] = sh[threadIdx.x][0];
}
__global__ void k_diag_final(const double* __restrict__ partial, int nb, double* out) {
  if (threadIdx.x < 5) {
    double s = 0;
    for (int i = 0; i < nb; ++i)
      s = threadIdx.x < 4 ? s + partial[threadIdx.x * nb + i] : fmax(s, partial[threadIdx.x * nb + i]);
    out[threadIdx.x] = s;
  }
}
cudaError_t launch_diag(const Geom& g, const float* M, const float* Hd, const StepParams* prm, const float* Hlo,
                        const float* Hhi, double dx, double dy, double dz, double* partial, double* out,
                        cudaStream_t st) {
  const double ix = 1.0 / (dx * dx), iy = 1.0 / (dy * dy), iz = 1.0 / (dz * dz);
  if (g.kb) k_diag_partial<true><<<kRedBlocks, kRedThreads, 0, st>>>(M, Hd, g, prm, Hlo, Hhi, ix, iy, iz, partial);
  else k_diag_partial<false><<<kRedBlocks, kRedThreads, 0, st>>>(M, Hd, g, prm, Hlo, Hhi, ix, iy, iz, partial);
  k_diag_final<<<1, 32, 0, st>>>(partial, kRedBlocks, out);
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
