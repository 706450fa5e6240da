// Small-grid latency path: the whole LLG step of a thin
// single-layer grid (nz = 1: muMAG SP4) in ONE thread-block cluster that
// stays resident for all n steps of a grace_step(n) call.
//
// The paper explains its small-N times by constant launch overhead and idle
// processors.  At SP4 sizes the graph-replayed step (K1, K2', K5, K6)
// is bound by four kernel boundaries per step; here every intermediate lives in
// the cluster's distributed shared memory (DSMEM) and the stage boundaries are
// cluster barriers:
//   A  x-R2C of this CTA's rows of M (smem), the half spectra scattered by kx
//      chunk to the owning CTA's y tiles (DSMEM stores)          [cluster barrier]
//   B  per owned kx chunk: y-FFT, H~ = KS . M~ (KS slice resident), inverse y
//      (pencil_conv, in place in the chunk's tile)               [cluster barrier]
//   C  x-C2R of this CTA's rows, the spectra gathered from the owners' tiles
//      (DSMEM loads) -> H_demag (smem)                           [cluster barrier]
//   D  Eq. (2) local terms (exchange y+-1 rows from the neighbouring CTAs'
//      M over DSMEM) + Eq. (3) + Euler + renormalise -> the other M buffer
// The arithmetic is the same as the pencil path's (same engine, same KS
// table, same stencil and update expressions), so the result matches it to
// fp32 rounding order.  M is read from HBM once at the start and written once
// at the end of the call.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "fft_engine.cuh"
#include "internal.h"
#include "pencil.cuh"

namespace cg = cooperative_groups;

namespace grace {

template <int LX, int PY, int C>
struct Small {
  static constexpr int NT = ZPlan<PY>::NT;  // the chunk tiles' pencil plan sets the CTA size
  static constexpr int B = 16;   // kx columns per chunk
  static constexpr int RT = 16;  // component rows per x tile
  static constexpr int KX = LX + 1;
  static constexpr int NCH = (KX + B - 1) / B;    // kx chunks
  static constexpr int CPC = (NCH + C - 1) / C;   // chunk slots per CTA (chunk j -> CTA j % C, slot j / C)
  static constexpr int KYH = PY / 2 + 1;
  using TX = TileIdx<LX, RT, false>;
  using TY = TileIdx<PY, B, true>;
  static_assert(!TY::PAD, "chunk tiles in the linear column layout");
  static_assert(ZPlan<PY>::B == B && NT % RT == 0, "pencil_conv plan of the chunk tiles");
  static constexpr int YT = 3 * TY::ELEMS;   // float2 per chunk tile
  static constexpr int KSS = 6 * KYH * B;    // floats per chunk KS slice
  // dynamic smem for rmax rows per CTA (bytes)
  __host__ __device__ static size_t smem(int rmax) {
    return (size_t)CPC * YT * 8 + (size_t)TX::ELEMS * 8 + (size_t)CPC * KSS * 4 + (size_t)9 * rmax * LX * 4;
  }
};

struct SmallArgs {
  const float* Min;   // M[cur] [3][ny][nx]
  float* Mout;        // M[cur ^ (n & 1)]
  const float* KS;    // [6][1][Kyh][KSp]
  const float2* tw;
  StepParams* prm;
  unsigned long long* flag;
  int nsteps, rmax;
};

template <int LX, int PY, int C>
__global__ void __launch_bounds__(Small<LX, PY, C>::NT, 1) k_small_step(Geom g, SmallArgs a) {
  using S = Small<LX, PY, C>;
  constexpr int NT = S::NT, B = S::B, RT = S::RT;
  using TX = typename S::TX;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* yt = reinterpret_cast<float2*>(smraw);                       // [CPC][3][PY][B]
  float2* xt = yt + S::CPC * S::YT;                                    // x tile
  float* kss = reinterpret_cast<float*>(xt + TX::ELEMS);              // [CPC][6][KYH][B]
  float* mb = kss + S::CPC * S::KSS;                                   // [2][3][rmax][LX]
  float* hd = mb + 6 * a.rmax * LX;                                    // [3][rmax][LX]
  const int nx = g.nx, ny = g.ny, rmax = a.rmax;
  const int y0 = rank * rmax;
  const int nr = max(0, min(rmax, ny - y0));
  const size_t N = (size_t)nx * ny;
  const size_t cplane = (size_t)rmax * LX;  // component stride of the smem M / Hd rows
  const int twx = g.Lmax / LX, twpx = g.Lmax / (2 * LX), twy = g.Lmax / PY;

  // ---- prologue: zero the chunk tiles, stage the KS slices, load M
  for (int i = threadIdx.x; i < S::CPC * S::YT; i += NT) yt[i] = make_float2(0.f, 0.f);
  for (int s = 0; s < S::CPC; ++s) {
    const int kx0 = (rank + s * C) * B;
    for (int t = threadIdx.x; t < S::KSS; t += NT) {
      const int b = t % B, r = t / B;  // r = comp * KYH + ky
      const int comp = r / S::KYH, ky = r - comp * S::KYH;
      const int kx = kx0 + b;
      kss[s * S::KSS + t] =
          kx < g.KSp ? __ldg(a.KS + ((size_t)comp * g.Kyh + ky) * g.KSp + kx) : 0.f;  // Kzh = 1
    }
  }
  for (int t = threadIdx.x; t < 3 * nr * nx; t += NT) {
    const int c = t / (nr * nx), r = t - c * nr * nx, yl = r / nx, x = r - yl * nx;
    mb[c * cplane + yl * LX + x] = __ldg(a.Min + c * N + (size_t)(y0 + yl) * nx + x);
  }
  const StepParams p0 = *a.prm;
  cl.sync();

  // remote chunk tile of kx (owner CTA, slot, column)
  auto chunk_of = [&](int k, int& owner, int& off) {
    const int j = k / B;
    owner = j % C;
    off = (j / C) * S::YT + (k - j * B);
  };
  const int ntile = (3 * nr + RT - 1) / RT;

  for (int step = 0; step < a.nsteps; ++step) {
    float* mc = mb + (step & 1) * 3 * cplane;        // M of this step
    float* mn = mb + ((step + 1) & 1) * 3 * cplane;  // M of the next
    // ---- A: x-R2C of the own rows -> owners' chunk tiles
    for (int tile = 0; tile < ntile; ++tile) {
      struct Ld {
        __device__ static constexpr bool kSmem() { return false; }
        const float* m;
        size_t cp;
        int q0, nr, nx, nq;
        __device__ float2 operator()(int b, int, int ib, int Cc) const {
          const int q = q0 + b, i = ib + Cc;
          if (q >= nq) return make_float2(0.f, 0.f);
          const int c = q / nr, yl = q - c * nr;
          const float* row = m + c * cp + yl * LX;
          const int x0 = 2 * i;
          return make_float2(x0 < nx ? row[x0] : 0.f, x0 + 1 < nx ? row[x0 + 1] : 0.f);
        }
      } ld{mc, cplane, tile * RT, nr, nx, 3 * nr};
      fft_tile<LX, RT, NT, false, false, true, false, 1>(xt, ld, SmemSt<LX, RT, false>{xt}, a.tw, twx);
      __syncthreads();
      // X[k] = (Z[k] + conj Z[L-k])/2 - (i/2) w^k (Z[k] - conj Z[L-k]), k = 0..L
      for (int u = threadIdx.x; u < RT * (LX + 1); u += NT) {
        const int b = u / (LX + 1), k = u - b * (LX + 1);
        const int q = tile * RT + b;
        if (q >= 3 * nr) continue;
        const int c = q / nr, yl = q - c * nr;
        const float2 Zk = xt[TX::at(b, k & (LX - 1))];
        const float2 Zn = xt[TX::at(b, (LX - k) & (LX - 1))];
        const float2 w = __ldg(a.tw + k * twpx);
        const float2 E = make_float2(0.5f * (Zk.x + Zn.x), 0.5f * (Zk.y - Zn.y));
        const float2 D = make_float2(0.5f * (Zk.x - Zn.x), 0.5f * (Zk.y + Zn.y));
        const float2 wD = cmul(w, D);
        int owner, off;
        chunk_of(k, owner, off);
        float2* dst = cl.map_shared_rank(yt, owner);
        dst[off + c * S::TY::ELEMS + (y0 + yl) * B] = make_float2(E.x + wD.y, E.y - wD.x);
      }
      __syncthreads();
    }
    cl.sync();
    // ---- B: y-FFT . KS . y-iFFT of the own chunks, in place
    for (int s = 0; s < S::CPC; ++s) {
      if (rank + s * C >= S::NCH) break;
      float2* tile = yt + s * S::YT;
      struct LdY {  // rows y >= ny of the tile are zero padding (stale after a step)
        __device__ static constexpr bool kSmem() { return true; }
        const float2* t;
        int ny;
        __device__ float2 operator()(int b, int c, int ib, int Cc) const {
          const int i = ib + Cc;
          return i < ny ? t[c * S::TY::ELEMS + i * B + b] : make_float2(0.f, 0.f);
        }
      };
      pencil_conv<PY, B, NT>(tile, LdY{tile, ny}, SmemSt<PY, B, true>{tile}, kss + s * S::KSS, S::KYH, a.tw, twy, 1,
                             0, true, [] {});
      __syncthreads();
    }
    cl.sync();
    // ---- C: x-C2R of the own rows from the owners' tiles -> H_demag
    for (int tile = 0; tile < ntile; ++tile) {
      struct LdC {
        __device__ static constexpr bool kSmem() { return false; }
        const float2* ytl;
        const float2* tw;
        int q0, nr, nq, y0, twpx;
        __device__ float2 operator()(int b, int, int ib, int Cc) const {
          const int q = q0 + b, k = ib + Cc;
          if (q >= nq) return make_float2(0.f, 0.f);
          const int c = q / nr, y = y0 + (q - c * nr);
          cg::cluster_group cl = cg::this_cluster();
          const int ja = k / B, jm = (LX - k) / B;
          const float2* ta = cl.map_shared_rank(ytl, ja % C);
          const float2* tm = cl.map_shared_rank(ytl, jm % C);
          const float2 av = ta[(ja / C) * S::YT + c * S::TY::ELEMS + y * B + (k - ja * B)];
          const float2 mv = tm[(jm / C) * S::YT + c * S::TY::ELEMS + y * B + ((LX - k) - jm * B)];
          const float2 Sv = make_float2(av.x + mv.x, av.y - mv.y);  // X[k] + conj X[L-k]
          const float2 Dv = make_float2(av.x - mv.x, av.y + mv.y);  // X[k] - conj X[L-k]
          const float2 w = __ldg(tw + k * twpx);
          const float2 wD = cmulc(Dv, w);                        // w^-k D
          return make_float2(Sv.x - wD.y, Sv.y + wD.x);          // S + i w^-k D
        }
      } ld{yt, a.tw, tile * RT, nr, 3 * nr, y0, twpx};
      struct StC {
        __device__ static constexpr bool kSmem() { return false; }
        float* h;
        size_t cp;
        int q0, nr, nq, nx;
        __device__ void operator()(int b, int, int ib, int Cc, float2 v) const {
          const int q = q0 + b, x0 = 2 * (ib + Cc);
          if (q >= nq) return;
          const int c = q / nr, yl = q - c * nr;
          float* row = h + c * cp + yl * LX;
          if (x0 < nx) row[x0] = v.x;
          if (x0 + 1 < nx) row[x0 + 1] = v.y;
        }
      } st{hd, cplane, tile * RT, nr, 3 * nr, nx};
      fft_tile<LX, RT, NT, false, true, false, true, 1>(xt, ld, st, a.tw, twx);
      __syncthreads();
    }
    cl.sync();
    // ---- D: local terms + LLG + Euler + renormalise (the arithmetic of K6)
    StepParams p = p0;
    p.step = p0.step + step + 1;  // what K1 would have advanced it to
    float ha[3];
    applied_field(p, ha);
    const float* mup = y0 > 0 ? cl.map_shared_rank(mc, rank - 1) : nullptr;  // rank - 1 holds rmax rows
    const float* mdn = cl.map_shared_rank(mc, rank + 1 < C ? rank + 1 : rank);
    for (int t = threadIdx.x; t < nr * nx; t += NT) {
      const int yl = t / nx, x = t - yl * nx, y = y0 + yl;
      float m[3], h[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) m[c] = mc[c * cplane + yl * LX + x];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float* row = mc + c * cplane + yl * LX;
        const float xl = x > 0 ? row[x - 1] : m[c];
        const float xr = x + 1 < nx ? row[x + 1] : m[c];
        float ym = m[c], yp = m[c];
        if (y > 0) ym = yl > 0 ? row[x - LX] : mup[c * cplane + (rmax - 1) * LX + x];
        if (y + 1 < ny) yp = yl + 1 < nr ? row[x + LX] : mdn[c * cplane + x];
        // Eq. (2): H_demag + six-neighbour exchange (difference form, Q11) + Zeeman (+ x anisotropy)
        float e = 0.f;
        e += g.cx * (xl - m[c]);
        e += g.cx * (xr - m[c]);
        e += g.cy * (ym - m[c]);
        e += g.cy * (yp - m[c]);
        e += g.cz * (m[c] - m[c]);
        e += g.cz * (m[c] - m[c]);
        float hv = hd[c * cplane + yl * LX + x] + ha[c];
        if (c == 0) hv += g.ck * m[c];
        h[c] = hv + e;
      }
      const float mx = m[0], my = m[1], mz = m[2];
      const float hx = h[0], hy = h[1], hz = h[2];
      // Eq. (3): dM/dt = c_prec (M x H) + c_damp M x (M x H); Euler; renormalise (Q16)
      const float ax = my * hz - mz * hy, ay = mz * hx - mx * hz, az = mx * hy - my * hx;
      const float bx = my * az - mz * ay, by = mz * ax - mx * az, bz = mx * ay - my * ax;
      const float sx = mx + p.dt * (p.c_prec * ax + p.c_damp * bx);
      const float sy = my + p.dt * (p.c_prec * ay + p.c_damp * by);
      const float sz = mz + p.dt * (p.c_prec * az + p.c_damp * bz);
      const float sc = g.Ms / sqrtf(sx * sx + sy * sy + sz * sz);
      const float o0 = sx * sc, o1 = sy * sc, o2 = sz * sc;
      mn[yl * LX + x] = o0;
      mn[cplane + yl * LX + x] = o1;
      mn[2 * cplane + yl * LX + x] = o2;
      if (!(isfinite(o0) && isfinite(o1) && isfinite(o2)))
        atomicMin(a.flag, ((unsigned long long)(p.step - 1) << 36) | (unsigned long long)((size_t)y * nx + x));
    }
    __syncthreads();
  }
  // ---- epilogue: the final M to HBM, the device step counter
  const float* mf = mb + (a.nsteps & 1) * 3 * cplane;
  for (int t = threadIdx.x; t < 3 * nr * nx; t += NT) {
    const int c = t / (nr * nx), r = t - c * nr * nx, yl = r / nx, x = r - yl * nx;
    a.Mout[c * N + (size_t)(y0 + yl) * nx + x] = mf[c * cplane + yl * LX + x];
  }
  if (rank == 0 && threadIdx.x == 0) a.prm->step = p0.step + a.nsteps;
  cl.sync();  // no CTA leaves while others may still read its shared memory
}

template <int LX, int PY, int C>
static cudaError_t small_launch(const Geom& g, const SmallArgs& a0, cudaStream_t st) {
  using S = Small<LX, PY, C>;
  SmallArgs a = a0;
  a.rmax = (g.ny + C - 1) / C;
  const size_t smem = S::smem(a.rmax);
  auto kern = k_small_step<LX, PY, C>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess && C > 8) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(S::NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, g, a);
  return e == cudaSuccess ? cudaGetLastError() : e;
}

// Which (LX, PY, C) instantiation serves this grid (0: none -> the pencil path).
// Opt-in (GRACE_SMALL=1): measured slower than the graph-replayed pencil path on
// one B200 (SP4 coarse 13.8 vs 10.9 us/step, refined 29.3 vs 14.1):
// one cluster of 8-16 SMs at 4 warps each is compute-starved, while the pencil
// path's four kernels spread each stage over the whole GPU.
static int small_kind(const Geom& g) {
  const char* on = getenv("GRACE_SMALL");
  if (!on || on[0] != '1') return 0;
  if (g.nz != 1 || g.Pz != 1 || g.kb != 0 || g.masked) return 0;
  const int LX = g.Px / 2;
  if (LX == 128 && g.Py == 64) return 1;   // SP4 coarse 100x25x1
  if (LX == 256 && g.Py == 128) return 2;  // SP4 refined 200x50x1
  return 0;
}

bool small_path_ok(const Geom& g) {
  const int k = small_kind(g);
  if (k == 0) return false;
  int dev = 0, maxsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t need = k == 1 ? Small<128, 64, 8>::smem((g.ny + 7) / 8) : Small<256, 128, 16>::smem((g.ny + 15) / 16);
  return need <= (size_t)maxsm;
}

cudaError_t launch_small_step(const Geom& g, const float* Min, float* Mout, const float* KS, const float2* tw,
                              StepParams* prm, unsigned long long* flag, int nsteps, cudaStream_t st) {
  SmallArgs a{Min, Mout, KS, tw, prm, flag, nsteps, 0};
  switch (small_kind(g)) {
    case 1: return small_launch<128, 64, 8>(g, a, st);
    case 2: return small_launch<256, 128, 16>(g, a, st);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace grace
