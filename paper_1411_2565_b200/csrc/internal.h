// Internal declarations shared by the libgrace translation units (not part of the C-ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace grace {

// Device-resident per-step parameters.  Kernel arguments are frozen into the
// captured CUDA graphs, so everything that may change between grace_step calls
// (dt, alpha, H_ext, the step index) is read from here; one cudaMemcpyAsync of
// this block per call updates it.
struct StepParams {
  float dt;       // s
  float c_prec;   // -gamma0/(1+alpha^2)                  (Eq. (3) precession prefactor)
  float c_damp;   // -alpha gamma0/((1+alpha^2) Ms)       (Eq. (3) damping prefactor)
  float hext[3];  // A/m
  long long step; // steps started so far; K1 increments it, K5 reports step - 1
  // SPEC FieldSchedule: at timestep k = step - 1 the applied field is
  // hext + a(k) h0, a = 1 on [t0, t1), 1 - (k - t1)/(t2 - t1) on [t1, t2), else 0
  float h0[3];
  int sched;
  long long t0, t1, t2;
};

// Applied field of the step being computed (constant part + scheduled part).
__host__ __device__ inline void applied_field(const StepParams& p, float h[3]) {
  float a = 0.f;
  if (p.sched) {
    const long long k = p.step - 1;
    if (k >= p.t0 && k < p.t2) a = k < p.t1 ? 1.f : 1.f - (float)(k - p.t1) / (float)(p.t2 - p.t1);
  }
  for (int q = 0; q < 3; ++q) h[q] = p.hext[q] + a * p.h0[q];
}

// Geometry and the constant material coefficients (fp32, rounded once from fp64 on the host).
struct Geom {
  int nx, ny, nz;   // global grid
  int Px, Py, Pz;   // padded FFT sizes (power of two >= 2n-1, 1 for a singleton axis)
  int Kx;           // Px/2 + 1 complex outputs of the x R2C (1 when Px == 1)
  int Kxp;          // complex row pitch of X1/X2 on a single GPU
  int Kyh, Kzh;     // Py/2 + 1, Pz/2 + 1 (1 for a singleton axis): folded spectrum extents
  int KSp;          // float row pitch of this rank's spectral table KS
  int Lmax;         // length of the twiddle table
  // z-slab partition.  Single GPU: nzl = nz, pitch1 = pitch2 = Kxp,
  // kb = 0 (no kx blocks), Kc = Kx, no halos.
  int nzl;          // z planes owned by this rank (K1 / K5 rows)
  int pitch1;       // row pitch of the x-row layouts (K1 out, K2 in, K4 out, K5 in)
  int kb;           // kx block of the all-to-all (0: unblocked)
  long long blk1;   // complex elements per kx block of an x-row layout (3 nzl ny pitch1)
  int Kc;           // kx columns handled by K2..K4 on this rank
  int pitch2;       // row pitch of X2
  int has_lo, has_hi;  // z-1 / z+1 halo planes present
  int nsm;             // SMs of the device (persistent grids)
  int masked;          // geometry mask set (grace_set_geometry): M = 0 marks an empty cell (reading Q26)
  int c0, nc;          // components c0 .. c0 + nc - 1 handled by K1, K2, K4, K5 (default 0, 3; the
                       // distributed step runs them per component to pipeline the transposes)
  // Fused transposes (GRACE_P2P, distributed path): K1 / K4 store x-row block q
  // straight into rank q's receive buffer peer[q] (block `rank` of it) instead of
  // their own send buffer -- peer memory over NVLink (CUDA IPC) on the NCCL path,
  // the other ranks' buffers on the virtual path.  0: off.
  int p2p, rank;
  float2* peer[8];
  int plane;           // KP plane-fused y.z.y pass replaces K2..K4 (single GPU, thin films)
  float cx, cy, cz; // exchange 2A/(mu0 Ms^2 d^2) per axis (0 for a singleton axis)
  float ck;         // anisotropy 2Ku/(mu0 Ms^2)
  float Ms;
};

constexpr unsigned long long kNoFlag = ~0ull;

// Per-step kernel launchers (step_kernels.cu).  All enqueue on `st`.
// K1 also advances bump->step (nullptr: no step, e.g. grace_heff).
cudaError_t launch_k1(const Geom& g, const float* M, float2* X1, const float2* tw, StepParams* bump,
                      cudaStream_t st);
// K2 in / K4 out use the x-row layout (pitch1, slabs of nzl planes per kx block);
// X2 is [3][nz][Py][pitch2] over this rank's Kc columns.
// 128-byte CUtensorMap storage (TMA descriptor built on the host, passed by value).
struct alignas(64) TmapBlob {
  unsigned char b[128];
};
// Tensor maps of the K2 input (x-row layout) and the K4 input (X2) for TMA loads.
// k4out (nullable, single GPU): the K4 output map for TMA stores into X1.
cudaError_t make_ky_tmaps(const Geom& g, const float2* k2_in, const float2* x2, TmapBlob* k2map, TmapBlob* k4map,
                          TmapBlob* k4out = nullptr);
cudaError_t launch_k2(const Geom& g, const float2* X1, float2* X2, const float2* tw, cudaStream_t st,
                      const TmapBlob* tmap = nullptr);
// K3 tensor maps (X2 pencils, KS slices) for the TMA-fed kernel; cudaErrorNotSupported
// where K3 takes the LDG kernel (unfused long pencils, short L, nz == 1).
cudaError_t make_k3_tmaps(const Geom& g, const float2* X2, const float* KS, TmapBlob* xmap, TmapBlob* kmap);
// tw3: the TMA K3's twiddle tables in their smem layout (make_k3_twiddles; nullptr:
// each CTA builds them from tw).
cudaError_t launch_k3(const Geom& g, float2* X2, const float* KS, const float2* tw, cudaStream_t st,
                      const TmapBlob* xmap = nullptr, const TmapBlob* kmap = nullptr, const float2* tw3 = nullptr);
cudaError_t make_k3_twiddles(const Geom& g, const float2* tw, float2** out, cudaStream_t st);
cudaError_t launch_k4(const Geom& g, const float2* X2, float2* X1, const float2* tw, cudaStream_t st,
                      const TmapBlob* tmap = nullptr, const TmapBlob* tout = nullptr);
cudaError_t launch_k2f(const Geom& g, float2* X1, const float* KS, const float2* tw, cudaStream_t st);
// K5: inverse x C2R of X1 -> H_demag Hd [3][nzl][ny][nx].
cudaError_t launch_k5(const Geom& g, const float2* X1, float* Hd, const float2* tw, cudaStream_t st);
// K6: local terms + LLG + Euler from H_demag (mode 0: M -> Mn; mode 1: H_eff -> Hout).
// Hlo / Hhi: halo planes [3][ny][nx] of z-1 / z+1 (used when g.has_lo / g.has_hi).
// mode 3 / 4: Heun predictor / corrector; mode 5: adaptive-step corrector (error into *aerr).
cudaError_t launch_k6(const Geom& g, int mode, const float* Hd, const float* M, float* Mn, float* Hout,
                      const StepParams* prm, unsigned long long* flag, cudaStream_t st, const float* Hlo,
                      const float* Hhi, unsigned* aerr = nullptr);
bool fused_y_path(const Geom& g);
// KP (plane-fused y.z.y, nz >= 2 with Pz <= 16, single GPU): in place on X1 [3][nz][ny][pitch1]
// with KSP, the plane-ordered spectrum [kx][6][Kzh][Kyh] (plane_ks_floats floats, filled
// from KS by launch_plane_ks).
bool plane_ok(const Geom& g);
size_t plane_ks_floats(const Geom& g);
cudaError_t launch_plane_ks(const Geom& g, float* KSP, const float* KS, cudaStream_t st);
cudaError_t make_plane_tmap(const Geom& g, const float2* X1, TmapBlob* map);
cudaError_t launch_kplane(const Geom& g, float2* X1, const float* KSP, const float2* tw, cudaStream_t st,
                          const TmapBlob* map);  // nz == 1 and the y-pencils of 3 components fit one CTA
bool comp_split_ok(const Geom& g); // K1 .. K5 can run per component (bulk-copy x kernels)
bool p2p_ok(const Geom& g);        // K1 / K4 can store into peers' buffers (bulk-copy K1, TMA K4)
void set_pdl_blocked(bool b);      // this thread's next launches without programmatic dependent launch
int kernel_count(const Geom& g);   // kernels per step

// Small-grid latency path (small_step.cu): n Euler steps of an nz = 1
// grid in one thread-block cluster, all intermediates in distributed shared memory.
bool small_path_ok(const Geom& g);
cudaError_t launch_small_step(const Geom& g, const float* Min, float* Mout, const float* KS, const float2* tw,
                              StepParams* prm, unsigned long long* flag, int nsteps, cudaStream_t st);

// Utilities (step_kernels.cu).
cudaError_t launch_twiddles(float2* tw, int Lmax, cudaStream_t st);
cudaError_t launch_set_m_f64(const double* src, float* M, long long n, double Ms, const unsigned char* mask,
                             unsigned long long* flag,
                             cudaStream_t st);
cudaError_t launch_apply_mask(float* M, long long n, const unsigned char* mask, cudaStream_t st);
cudaError_t launch_set_m_f32(const float* src, float* M, long long n, float Ms, const unsigned char* mask,
                             unsigned long long* flag,
                             cudaStream_t st);
cudaError_t launch_mavg(const float* M, long long n, double Ms, double* partial, double* out, cudaStream_t st);
constexpr int kMavgPartials = 3 * 296;
// Eq. (1) energy sums and the relax torque of the current state (out[5], see step_kernels.cu);
// partial holds kDiagPartials doubles.
cudaError_t launch_diag(const Geom& g, const float* M, const float* Hd, const StepParams* prm, const float* Hlo,
                        const float* Hhi, double dx, double dy, double dz, double* partial, double* out,
                        cudaStream_t st);
constexpr int kDiagPartials = 5 * 296;
cudaError_t launch_fill_uniform_x(float* M, long long n, float Ms, cudaStream_t st);
cudaError_t launch_widen(const float* src, double* dst, long long n, cudaStream_t st);

// Demag-tensor setup (tensor_setup.cu), fp64.
// Real-space octant [6][nz][ny][nx] into device memory `oct` (bit-exact with the oracle).
cudaError_t tensor_octant_device(int nx, int ny, int nz, double dx, double dy, double dz, double* oct,
                                 cudaStream_t st);
// Spectral table KS [6][Kzh][Kyh][KSp] fp32 = -Re(FFT(circulant N))/(Px Py Pz), written for
// each output's kx columns [kx0, kx0 + ncol) (a rank's kx block; the single-GPU table is
// kx0 = 0, ncol = Kx).  Lean: one octant component at a time (8 B/cell), the x lines
// in chunks of padded z planes, and only the union of the requested kx columns kept
// for the y and z lines; the transient device memory is reported in *scratch_bytes.
struct KsOut {
  float* KS;
  int kx0, ncol, KSp;
  double* KS64 = nullptr;  // optional: the fp64 values before rounding (same layout)
};
cudaError_t kernel_spectrum_device(const Geom& g, double dx, double dy, double dz, int nout, const KsOut* out,
                                   size_t* scratch_bytes, cudaStream_t st);

}  // namespace grace
