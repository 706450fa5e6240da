/* grace.h -- C-ABI of libgrace: the B200 hot path of Grace (Zhu, arXiv 1411.2565).
 *
 * One finite-difference micromagnetic LLG step on a regular nx x ny x nz grid:
 *   H_eff = H_demag + H_exch + H_anis + H_ext                      (Eq. (2))
 *   H_demag = -N * M, zero-padded FFT convolution with the
 *             precomputed cell-averaged demag tensor                 (Sec. 3)
 *   H_exch  = six-neighbour scheme, Neumann boundaries               (reading Q11)
 *   H_anis  = (2Ku/(mu0 Ms^2)) Mx x, uniaxial along x                (reading Q4)
 *   dM/dt   = -g0/(1+a^2) M x H - a g0/((1+a^2) Ms) M x (M x H)      (Eq. (3); reading Q1)
 *   M      <- Ms (M + dt dM/dt)/|M + dt dM/dt|                       (Euler; reading Q16)
 * "Qnn" are the readings of DESIGN.md §3 where the paper is silent or garbled.
 *
 * Conventions (all functions):
 *  - Units are SI: metres, A/m, J/m, J/m^3, seconds.  `gamma` is gamma0 = gamma*mu0
 *    in m/(A s) (muMAG SP4 value 2.211e5), never gamma in rad/(s T) (reading Q1).
 *  - Host arrays are structure-of-arrays [3][nz][ny][nx] doubles, x fastest: element
 *    (c, k, j, i) at ((c*nz + k)*ny + j)*nx + i.  They belong to the caller; calls
 *    copy synchronously and return after the copy completed.
 *  - The context owns all device memory (allocated in grace_create, freed in
 *    grace_destroy).  Device state is fp32 except the fp64 tensor setup.
 *  - Every int-returning call returns GRACE_OK or a negative status; on error the
 *    outputs are untouched, the context stays usable and grace_last_error()
 *    describes the failure.  Calls on one context must not run concurrently;
 *    distinct contexts are independent.
 *  - Device work is queued on the context's CUDA stream (grace_set_stream);
 *    calls that return host data synchronise that stream.
 */
#ifndef GRACE_H
#define GRACE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct grace_ctx grace_ctx;

enum {
  GRACE_OK = 0,
  GRACE_EINVAL = -1,       /* bad argument (count < 1, non-positive/non-finite length, Ms <= 0, A < 0,
                              Ku < 0, alpha < 0, gamma <= 0 or > 1e9, dt <= 0, n < 0, NULL pointer) */
  GRACE_ENOMEM = -2,       /* device allocation failed; message carries the bytes required */
  GRACE_EZEROCELL = -3,    /* grace_set_m: a cell with |M| = 0 or non-finite; message names the cell */
  GRACE_ENONFINITE = -4,   /* grace_step: non-finite M; grace_last_nonfinite gives step and cell */
  GRACE_ECUDA = -5,        /* CUDA runtime error (message has the CUDA error string) */
  GRACE_EUNSUPPORTED = -6  /* padded FFT length above the compiled maximum (x 8192, y 4096, z 1024) */
};

/* Create a context and build the demag tensor:
 * the fp64 real-space octant of the six N_ab (Newell near field within 30 cell
 * diagonals, point dipole beyond; readings Q5-Q8) and its spectrum
 * KS = -Re FFT(N)/(Px Py Pz) on the padded grid Pa = smallest power of two
 * >= 2 na - 1 (Pa = 1 when na = 1; reading Q9), folded to one octant in fp32.
 * nx, ny, nz >= 1 cells; dx, dy, dz > 0 metres; Ms > 0 A/m; A >= 0 J/m;
 * Ku >= 0 J/m^3 (easy axis x); alpha >= 0; gamma = gamma0 > 0 m/(A s).
 * Initial M is uniform Ms along x, H_ext = 0, the step counter 0.
 * On error *out = NULL. */
int grace_create(int nx, int ny, int nz, double dx, double dy, double dz, double Ms, double A, double Ku,
                 double alpha, double gamma, grace_ctx **out);

/* Free all device memory of the context.  NULL-safe. */
void grace_destroy(grace_ctx *h);

/* Set M from a host array (3 N doubles, A/m).  Each cell is renormalised to |M| = Ms
 * on the device.  A zero or non-finite cell fails with GRACE_EZEROCELL and
 * leaves M unchanged.  Does not reset the step counter. */
int grace_set_m(grace_ctx *h, const double *m);

/* Copy M to a host array (3 N doubles, A/m; fp32 values widened exactly). */
int grace_get_m(grace_ctx *h, double *m_out);

/* Uniform external (Zeeman) field in A/m, used by every later step / heff. */
int grace_set_hext(grace_ctx *h, double hx, double hy, double hz);

/* H_eff(current M, H_ext) per Eq. (2) into a host array (3 N doubles, A/m). */
int grace_heff(grace_ctx *h, double *h_out);

/* Advance n >= 0 explicit Euler steps of size dt > 0 seconds, entirely on the
 * device (replay of CUDA graphs instantiated in grace_create: 16-step chunks, then
 * single steps; no host round trip inside).  After the n steps one 8-byte flag is
 * read back: a non-finite M returns GRACE_ENONFINITE (the first failing step and
 * cell are kept for grace_last_nonfinite; M then holds non-finite values).  With
 * GRACE_SMALL=1 an SP4-sized nz = 1 grid runs the whole call in one cluster kernel
 * (small_step.cu; measured slower, opt-in). */
int grace_step(grace_ctx *h, int n, double dt);

/* Thread-local text of the last failure on this thread ("" if none). */
const char *grace_last_error(void);

/* ---- extensions (not in the paper's call list) -------------------------------- */

/* Change the damping constant without rebuilding the tensor (SP4: relax at alpha = 1,
 * then reverse at 0.02). */
int grace_set_alpha(grace_ctx *h, double alpha);

/* Queue all device work on `cuda_stream` (a cudaStream_t, e.g. torch's current
 * stream); NULL restores the context's own stream. */
int grace_set_stream(grace_ctx *h, void *cuda_stream);

/* Device-pointer variants: fp32 SoA [3][nz][ny][nx] in device memory, no host hop.
 * set_m_device renormalises like grace_set_m. */
int grace_set_m_device(grace_ctx *h, const float *d_m);
int grace_get_m_device(grace_ctx *h, float *d_m_out);

/* Host fp32 variants of grace_set_m / grace_get_m (SoA [3][nz][ny][nx], A/m;
 * the rank-local slab on the NCCL path): the device state is fp32, so these move
 * 12 bytes per cell each way instead of 24 (pinned host memory gives full PCIe
 * bandwidth).  set renormalises like grace_set_m (GRACE_EZEROCELL likewise);
 * both return after the copy has completed. */
int grace_set_m_f32(grace_ctx *h, const float *m);
int grace_get_m_f32(grace_ctx *h, float *m_out);

/* <M>/Ms (3 doubles) by a fixed-order two-stage reduction (deterministic). */
int grace_mavg(grace_ctx *h, double *out3);

/* Diagnostics; both evaluate H_demag of the current M with the
 * step's own kernels, then reduce in fp64 in a fixed order.
 * grace_energy: the discrete Eq. (1) energy, joules,
 *   out5 = {total, exchange, anisotropy, demag, Zeeman}: exchange
 *   V A sum over +x/+y/+z bonds |m_nb - m|^2 / Delta^2, anisotropy V Ku sum (1 - m_x^2),
 *   demag -mu0/2 V sum H_demag.M, Zeeman -mu0 V sum H_ext.M (m = M/Ms).
 * grace_max_torque: max over cells |M x H_eff| / (Ms |H_eff| + 1e-30), the SPEC
 *   relaxation criterion (eps S:L331), H_eff as the step forms it. */
int grace_energy(grace_ctx *h, double *out5);
int grace_max_torque(grace_ctx *h, double *out);

/* SPEC relax: Euler steps of dt at damping alpha_relax until the max
 * torque is below tol (checked every check_every steps) or max_steps are taken;
 * alpha is restored afterwards.  steps_taken / torque receive the outcome
 * (torque < tol: converged).  Errors as grace_step. */
int grace_relax(grace_ctx *h, double alpha_relax, double dt, long long max_steps, double tol, int check_every,
                long long *steps_taken, double *torque);

/* Time-scheduled applied field, the paper's "Hx Hy Hz startTime decayTime stopTime"
 * input (paper Sec. 5; SPEC FieldSchedule S:L182-187).  At timestep index k (the
 * step computing M_{k+1} from M_k; grace_heff / grace_energy evaluate k = steps
 * taken) the applied field is H_ext + a(k) H0 (A/m, added to grace_set_hext's
 * constant field): a = 1 on [start, decay), a linear ramp 1 - (k - decay)/(stop - decay)
 * on [decay, stop), 0 otherwise.  Requires 0 <= start <= decay <= stop (else
 * GRACE_EINVAL); H0 = 0 or stop == start disables it.  Indices count
 * grace_step_count, which grace_set_m does not reset. */
int grace_set_field_schedule(grace_ctx *h, double h0x, double h0y, double h0z, long long start, long long decay,
                             long long stop);

/* Time integrator of grace_step: 0 = explicit Euler +
 * renormalisation (the paper's; default), 1 = Heun (explicit trapezoid,
 * second order) with the same renormalisation: f0 = dM/dt(M_k, t_k),
 * M* = renorm(M_k + dt f0), M_{k+1} = renorm(M_k + dt (f0 + dM/dt(M*, t_{k+1}))/2);
 * two H_eff evaluations per step.  GRACE_EINVAL for another kind; grace_step
 * returns GRACE_EUNSUPPORTED for Heun in profiling mode. */
int grace_set_integrator(grace_ctx *h, int kind);

/* Adaptive time steps ("adaptive time steps" -- the paper's future work;
 * SURVEY 8(f) #4(iv); the oracle twin is oracle.llg.Sim.adaptive_run).  Advances
 * the state by t_span seconds with the embedded Euler / Heun pair: an attempt
 * of step dt computes the Euler step M_E = renorm(M + dt f0) and the Heun step
 * M_H = renorm(M + dt (f0 + f(M_E))/2); err = max over cells |M_H - M_E| / Ms
 * (the Euler step's local error estimate).  err <= tol accepts M_H, else the
 * attempt is discarded; the next dt = dt * min(5, max(0.2, 0.9 sqrt(tol/err))),
 * and the last step is shortened to end on t_span.  *dt_io: first trial step in,
 * suggested next step out.  Eager launches and one device-to-host read per
 * attempt.  accepted / rejected: attempts of each kind (accepted ones advance
 * grace_step_count).  GRACE_EINVAL for t_span < 0, dt <= 0, tol <= 0,
 * max_attempts < 1; GRACE_EUNSUPPORTED with a field schedule; GRACE_ENONFINITE
 * as grace_step.  Collective on the NCCL path (the error is max-reduced). */
int grace_step_adaptive(grace_ctx *h, double t_span, double *dt_io, double tol, long long max_attempts,
                        long long *accepted, long long *rejected);

/* Geometry mask (the paper's "non-regular geometry", P:L121;
 * DESIGN.md reading Q26).  mask: host uint8 [nz][ny][nx] (the rank-local slab
 * [nz/P][ny][nx] for grace_create_dist), nonzero = magnetic cell, copied before
 * return; NULL removes the mask.  Empty cells hold M = 0 (they carry no magnetic
 * charge in the demag sum); an exchange bond exists only between two magnetic
 * cells (an empty neighbour is a free surface, like the outer boundary);
 * grace_heff reports 0 in empty cells; grace_step leaves them at 0; grace_mavg and
 * grace_energy sum over magnetic cells.  The current M is zeroed in empty cells;
 * grace_set_m afterwards ignores the input there (cells newly made magnetic need
 * a grace_set_m).  GRACE_EINVAL if no cell is magnetic.  Costs Nl bytes of
 * device memory per rank. */
int grace_set_geometry(grace_ctx *h, const unsigned char *mask);

/* Steps taken so far (t = steps * dt). */
int grace_step_count(grace_ctx *h, long long *steps);

/* Step index and linear cell index of the first non-finite value of the last failing
 * grace_step (-1, -1 if none). */
int grace_last_nonfinite(grace_ctx *h, long long *step, long long *cell);

/* Geometry: out[0..11] = nx ny nz Px Py Pz Kx Kxp Kyh Kzh KSp kernels_per_step. */
int grace_geometry(grace_ctx *h, long long *out12);

/* Bytes of device memory the context holds. */
int grace_device_bytes(grace_ctx *h, size_t *bytes);

/* The real-space demag-tensor octant [6][nz][ny][nx] (components xx xy xz yy yz zz,
 * entry (c,k,j,i) = N_c at offset (i dx, j dy, k dz)), computed on the device exactly
 * as grace_create does (S1+S2, fp64) and copied to the host array `out` (6 N doubles).
 * Standalone: needs no context. */
int grace_tensor_octant(int nx, int ny, int nz, double dx, double dy, double dz, double *out);

/* Copy the fp32 spectral table KS [6][Kzh][Kyh][KSp] to the host (6*Kzh*Kyh*KSp floats). */
int grace_kernel_spectrum(grace_ctx *h, float *out);

/* The same table before its fp32 rounding: -Re FFT(circulant N) / (Px Py Pz) in fp64
 * (S4-S5 of the setup, exactly as grace_create computes it), [6][Kzh][Kyh][KSp]
 * doubles with Kzh, Kyh, KSp as grace_geometry reports them.  Standalone (no context);
 * for checking the fp64 spectrum against the oracle at 1e-12. */
int grace_kernel_spectrum_f64(int nx, int ny, int nz, double dx, double dy, double dz, double *out);

/* Per-kernel timing.  grace_set_profiling(h, 1) makes grace_step launch the kernels
 * eagerly with a CUDA event pair around each; grace_kernel_times returns, per kernel
 * of the step (order K1, K2, K3, K4, K5, K6; K1, K2', K5, K6 for nz = 1; K1, KP, K5, K6 on the
 * opt-in plane-fused thin-film path, GRACE_PLANE=1), the summed milliseconds and
 * the launch count since the last reset (reset = 1 clears after reading).  nk in:
 * capacity of ms[]/launches[]; out: number of kernels per step. */
int grace_set_profiling(grace_ctx *h, int on);
int grace_kernel_times(grace_ctx *h, double *ms, long long *launches, int *nk, int reset);

/* ---- distributed z-slab path ------------------------------------
 * The grid is split into P slabs of nz/P planes (nz % P == 0).  One step: K1 on
 * each slab, all-to-all to kx blocks of ceil(Kx/P) columns (C1), K2..K4 on the
 * block (all z), all-to-all back (C2), one-plane halo exchange of M (C3), K5 + K6
 * on each slab.  When K1 and K5 run as the bulk-copy kernels (nx % 4 == 0,
 * 128 <= Px <= 8192) the transposes are pipelined per magnetisation component:
 * C1 of component q runs on a communication stream while K1 computes q + 1 and
 * K2 starts on q once it has landed; likewise C2 against K4 / K5 (GRACE_NO_PIPE
 * turns this off).  C3 runs on its own stream and, on the NCCL path, its own
 * communicator (ncclCommSplit).  The step is captured into CUDA graphs like the
 * single-GPU step (GRACE_DIST_EAGER: eager launches).  Opt-in fused transposes
 * (GRACE_P2P=1 on every rank, P <= 8): K1 and K4 store their destination blocks
 * straight into the peers' receive buffers over NVLink (CUDA IPC handles exchanged
 * at create), and each all-to-all shrinks to a one-float all-reduce barrier.
 * Results are identical to the single-GPU path (same per-pencil arithmetic).
 *
 * Collective calls on the NCCL path (call them on every rank, in the same order):
 * grace_create_dist, grace_step, grace_heff, grace_mavg, grace_energy,
 * grace_max_torque, grace_relax, grace_step_adaptive, grace_set_geometry, grace_set_m,
 * grace_set_m_device (their status is agreed over the ranks: a non-finite value
 * or zero cell anywhere is reported by every rank, with the global cell index). */

/* P ranks of one grid in this context on the current GPU; the exchanges are
 * device-to-device copies.  Same interface as grace_create (whole-grid arrays);
 * used to test the partition logic on one GPU.  nranks = 1 is grace_create. */
int grace_create_virtual(int nx, int ny, int nz, double dx, double dy, double dz, double Ms, double A, double Ku,
                         double alpha, double gamma, int nranks, grace_ctx **out);

/* Write a fresh NCCL unique id (128 bytes) into out128 (rank 0; broadcast it to the
 * other ranks, e.g. with torch.distributed). */
int grace_nccl_unique_id(void *out128);

/* This process's rank of an nranks-way NCCL partition on the current GPU.
 * set_m/get_m/heff then address the local slab [3][nz/nranks][ny][nx] (z offset
 * rank*nz/nranks); see the collective calls above. */
int grace_create_dist(int nx, int ny, int nz, double dx, double dy, double dz, double Ms, double A, double Ku,
                      double alpha, double gamma, int rank, int nranks, const void *nccl_id, grace_ctx **out);

/* out[0..11] = P, rank, nz_local, z_offset, kx_block, kx_columns_here, pitch1, pitch2,
 * transposes pipelined per component (0/1), step captured into graphs (0/1), halo on
 * its own NCCL communicator (0/1), fused P2P transposes (0/1). */
int grace_partition(grace_ctx *h, long long *out12);

#ifdef __cplusplus
}
#endif
#endif /* GRACE_H */
