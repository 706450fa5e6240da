// libgrace C-ABI implementation (include/grace.h): contexts, validation, device
// memory, the CUDA-graph step loop, the z-slab distributed step and errors.
// Host code; the arithmetic of the path runs in step_kernels.cu and
// tensor_setup.cu.
//
// A context holds one or more "ranks" (z slabs):
//   single  - one rank, the whole grid; step = CUDA-graph replay.
//   virtual - P ranks of one grid on one GPU in one process; the all-to-all and
//             halo exchanges are cudaMemcpyAsync between the ranks' buffers
//             (exercises the partition logic against the single path).
//   nccl    - this process's rank of P (one GPU per process); the exchanges are
//             grouped ncclSend/ncclRecv over NVLink (the all-to-all transposes,
//             pipelined per component; the halos on a split communicator).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/grace.h"
#include "internal.h"

using namespace grace;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_OR(call)                                                                          \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess) return fail(GRACE_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)
#define CE(call)                      \
  do {                                \
    cudaError_t e_ = (call);          \
    if (e_ != cudaSuccess) return e_; \
  } while (0)

constexpr double kPI = 3.141592653589793;
constexpr double kMU0 = 4.0 * kPI * 1e-7;  // S:L46, reading Q21
constexpr int kChunk = 16;                 // steps per captured chunk graph

int padded(int n) {
  if (n == 1) return 1;
  int p = 1;
  while (p < 2 * n - 1) p <<= 1;
  return p;
}
long long round_up(long long v, long long m) { return (v + m - 1) / m * m; }
bool finite_pos(double v) { return std::isfinite(v) && v > 0.0; }

// ---- NCCL, loaded at run time (torch has normally loaded libnccl.so.2 already) ----
typedef struct ncclComm* ncclComm_t;
typedef int ncclResult_t;
struct ncclUniqueId {
  char internal[128];
};
enum { kNcclUint8 = 1, kNcclUint32 = 3, kNcclUint64 = 5, kNcclFloat32 = 7, kNcclFloat64 = 8, kNcclSum = 0, kNcclMax = 2, kNcclMin = 3 };
struct Nccl {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*commSplit)(ncclComm_t, int, int, ncclComm_t*, void*) = nullptr;  // optional (NCCL >= 2.18)
  ncclResult_t (*allReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
  // The process's NCCL: GRACE_NCCL_LIB (the Python binding points it at torch's
  // bundled libnccl), else an already-loaded or system libnccl.so.2.  Only calls
  // present in every NCCL >= 2.7 are required (the transposes are grouped
  // send/recv); ncclCommSplit, when present, gives the halo exchange its own
  // communicator.
  bool load() {
    if (h) return true;
    const char* env = getenv("GRACE_NCCL_LIB");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      if (!n) continue;
      h = dlopen(n, RTLD_NOW | RTLD_NOLOAD);
      if (!h) h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (h && bind()) return true;
      h = nullptr;
    }
    return false;
  }
  bool bind() {
    getUniqueId = (decltype(getUniqueId))dlsym(h, "ncclGetUniqueId");
    commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
    commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
    commSplit = (decltype(commSplit))dlsym(h, "ncclCommSplit");
    allReduce = (decltype(allReduce))dlsym(h, "ncclAllReduce");
    allGather = (decltype(allGather))dlsym(h, "ncclAllGather");
    send = (decltype(send))dlsym(h, "ncclSend");
    recv = (decltype(recv))dlsym(h, "ncclRecv");
    groupStart = (decltype(groupStart))dlsym(h, "ncclGroupStart");
    groupEnd = (decltype(groupEnd))dlsym(h, "ncclGroupEnd");
    errStr = (decltype(errStr))dlsym(h, "ncclGetErrorString");
    return getUniqueId && commInitRank && commDestroy && allReduce && allGather && send && recv && groupStart &&
           groupEnd && errStr;
  }
};
Nccl g_nccl;

}  // namespace

// ---------------------------------------------------------------------------------
// One z slab with its device state.
struct Rank {
  Geom g{};
  int r = 0;
  long long Nl = 0;  // cells in the slab
  float* M[2] = {nullptr, nullptr};
  float2* A = nullptr;   // single: X1 [3][nz][ny][Kxp]; dist: S1 / R2 [P][3][nzl][ny][Kb]
  float2* B = nullptr;   // dist: R1 / S2 [P][3][nzl][ny][Kb]
  float2* X2 = nullptr;  // [3][nz][Py][pitch2] (absent on the fused nz = 1 path)
  float* KS = nullptr;
  float* KSP = nullptr;  // plane-ordered KS [kx][6][Kzh][Kyh] (KP path only)
  TmapBlob kpmap{};      // KP's TMA map of X1
  float* Hlo = nullptr;  // halo planes [3][ny][nx]
  float* Hhi = nullptr;
  StepParams* prm = nullptr;
  unsigned long long* flag = nullptr;  // [0] step non-finite, [1] set_m zero cell, [2] NCCL reduction slot
  double* red = nullptr;               // mavg partials + 3 outputs
  double* dred = nullptr;              // diagnostics partials + 5 outputs (allocated on first use)
  float* Hbuf = nullptr;
  float* Hd = nullptr;                 // H_demag [3][nzl][ny][nx] (split K5/K6 step)
  float* F = nullptr;                  // Heun: dM/dt of the predictor stage
  unsigned* aerr = nullptr;            // grace_step_adaptive: error estimate (float bits), allocated on first use
  unsigned char* mask = nullptr;       // geometry mask [nzl][ny][nx] (grace_set_geometry; null: none)
  bool tma = false;                    // TMA descriptors of the K2 / K4 inputs built
  TmapBlob k2map{}, k4map{};
  bool tma4s = false;  // K4's TMA-store map of X1 built (single GPU)
  TmapBlob k4out{};
  bool tma3 = false;                   // TMA descriptors of the K3 pencils and KS slices built
  TmapBlob k3x{}, k3k{};
  float2* tw3 = nullptr;               // K3's twiddle tables in their smem layout
};

struct grace_ctx {
  enum Mode { kSingle, kVirtual, kNccl } mode = kSingle;
  int P = 1;       // ranks in the partition
  int myrank = 0;  // nccl mode: this process's rank
  double dx, dy, dz, Ms, A, Ku, alpha, gamma0;
  double hext[3] = {0, 0, 0};
  double h0[3] = {0, 0, 0};       // field schedule (grace_set_field_schedule)
  long long sched[3] = {0, 0, 0};
  bool has_sched = false;
  int integrator = 0;             // 0 Euler (the paper's), 1 Heun (grace_set_integrator)
  long long steps = 0;
  long long nf_step = -1, nf_cell = -1;
  long long N = 0;  // cells addressed by set_m/get_m/heff (whole grid, or the local slab in nccl mode)
  double nmag = 0;  // magnetic cells of the whole grid under the geometry mask (0: no mask)
  int cur = 0;
  bool fused = false;
  bool plane = false;  // KP replaces K2..K4 (thin films, single GPU)
  Geom g0{};  // global geometry
  std::vector<Rank> ranks;
  float2* tw = nullptr;
  size_t bytes = 0;
  cudaStream_t own = nullptr, stream = nullptr, cap = nullptr;
  cudaStream_t hs = nullptr;                  // distributed: halo exchange (C3) side stream
  cudaEvent_t evM = nullptr, evH = nullptr;   // fork (M[c] ready) / join (halos landed)
  // Per-component pipelining of the transposes: K1, K2, K4
  // and K5 run per magnetisation component, and the all-to-all of component q
  // (C1 after K1, C2 after K4) runs on the comm stream `cs` while the step
  // stream computes component q + 1 (K1 / K4) or consumes component q - 1 (K2 / K5).
  bool pipe = false;
  cudaStream_t cs = nullptr;
  cudaEvent_t evk[3] = {nullptr, nullptr, nullptr};  // component q computed (K1 / K4)
  cudaEvent_t evc[3] = {nullptr, nullptr, nullptr};  // component q transposed (C1 / C2)
  bool dist_graphs = true;                    // distributed step captured into graphs (else eager)
  // Fused transposes (GRACE_P2P=1): K1 / K4 store into the peers' receive
  // buffers directly (CUDA IPC over NVLink on the NCCL path); the exchanges
  // shrink to a barrier (a one-float ncclAllReduce) after each.
  bool p2p = false;
  float2* peerA[8] = {};  // rank q's A (K4's destination) and B (K1's destination)
  float2* peerB[8] = {};
  std::vector<void*> ipc_open;  // handles opened with cudaIpcOpenMemHandle
  float* p2p_bar = nullptr;     // device float of the barrier all-reduce
  cudaGraphExec_t g1[2] = {nullptr, nullptr}, gc[2] = {nullptr, nullptr};
  ncclComm_t comm = nullptr;
  ncclComm_t comm_halo = nullptr;  // C3's own communicator (NCCL orders work per communicator)
  bool profiling = false;
  std::vector<double> kms;
  std::vector<long long> klaunch;
  std::vector<cudaEvent_t> ev;
  StepParams hprm{};
  // pinned staging for the small per-call transfers (params up; flag, <M> and
  // diagnostics down): truly asynchronous copies instead of pageable staging
  struct Pinned {
    StepParams prm;
    unsigned long long flag;
    double red[8];
  };
  Pinned* pin = nullptr;

  int alloc(void** p, size_t b) {
    if (b == 0) b = 16;
    cudaError_t e = cudaMalloc(p, b);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(GRACE_ENOMEM, "device allocation of %zu bytes failed (context holds %zu): %s", b, bytes,
                  cudaGetErrorString(e));
    }
    bytes += b;
    return GRACE_OK;
  }

  void fill_params(double dt) {
    const double a2 = 1.0 + alpha * alpha;
    hprm.dt = (float)dt;
    hprm.c_prec = (float)(-gamma0 / a2);
    hprm.c_damp = (float)(-alpha * gamma0 / (a2 * Ms));
    for (int q = 0; q < 3; ++q) hprm.hext[q] = (float)hext[q];
    for (int q = 0; q < 3; ++q) hprm.h0[q] = (float)h0[q];
    hprm.sched = has_sched ? 1 : 0;
    hprm.t0 = sched[0];
    hprm.t1 = sched[1];
    hprm.t2 = sched[2];
    hprm.step = steps;
  }
  // eval: H_eff of the current state (grace_heff / diagnostics), i.e. at timestep
  // index `steps` -- the value the step counter has once K1 has advanced it
  cudaError_t upload_params(double dt, bool eval = false) {
    fill_params(dt);
    if (eval) hprm.step = steps + 1;
    pin->prm = hprm;  // every caller synchronises the stream before the next upload
    for (auto& rk : ranks) CE(cudaMemcpyAsync(rk.prm, &pin->prm, sizeof(StepParams), cudaMemcpyHostToDevice, stream));
    return cudaSuccess;
  }

  // ---- exchanges (distributed modes) ----
  // all-to-all of [P][blk1] complex blocks: block q of rank s's send buffer goes to
  // block s of rank q's receive buffer.
  // comp < 0: all three components (whole blocks); else only component comp's
  // sub-block [nzl][ny][Kb] of every block ([P][3][nzl][ny][Kb] layout).
  cudaError_t alltoall(float2* Rank::*src, float2* Rank::*dst, cudaStream_t s, int comp = -1) {
    const long long blk = ranks[0].g.blk1;
    const long long sub = blk / 3;
    const long long off = comp < 0 ? 0 : comp * sub, cnt = comp < 0 ? blk : sub;
    if (mode == kVirtual) {
      for (int a = 0; a < P; ++a)
        for (int b = 0; b < P; ++b)
          CE(cudaMemcpyAsync(ranks[b].*dst + (size_t)a * blk + off, ranks[a].*src + (size_t)b * blk + off,
                             sizeof(float2) * cnt, cudaMemcpyDeviceToDevice, s));
      return cudaSuccess;
    }
    // grouped point-to-point: block q of the send buffer to rank q, block q of the
    // receive buffer from rank q (what ncclAlltoAll does, without needing NCCL >= 2.28)
    Rank& rk = ranks[0];
    bool bad = g_nccl.groupStart() != 0;
    for (int q = 0; q < P && !bad; ++q) {
      bad |= g_nccl.send(rk.*src + (size_t)q * blk + off, (size_t)cnt * 2, kNcclFloat32, q, comm, s) != 0;
      bad |= g_nccl.recv(rk.*dst + (size_t)q * blk + off, (size_t)cnt * 2, kNcclFloat32, q, comm, s) != 0;
    }
    bad |= g_nccl.groupEnd() != 0;
    return bad ? cudaErrorUnknown : cudaSuccess;
  }
  // rank rk's geometry with the fused-transpose destinations
  Geom p2p_geom(const Rank& rk, float2* const* peers) const {
    Geom g = rk.g;
    g.p2p = 1;
    g.rank = rk.r;
    for (int q = 0; q < P; ++q) g.peer[q] = peers[q];
    return g;
  }
  // every rank's K1 (or K4) stores have landed: stream order on the virtual path,
  // a one-float all-reduce (all ranks reach it after their kernel) on the NCCL path
  cudaError_t p2p_barrier(cudaStream_t s) {
    if (mode != kNccl) return cudaSuccess;
    return g_nccl.allReduce(p2p_bar, p2p_bar, 1, kNcclFloat32, kNcclSum, comm, s) == 0 ? cudaSuccess
                                                                                      : cudaErrorUnknown;
  }
  // Set up the fused transposes: peer buffer tables (IPC handles exchanged with
  // ncclAllGather on the NCCL path).  The ranks agree on the outcome (min-reduce).
  cudaError_t setup_p2p() {
    if (mode == kSingle || P > 8) return cudaSuccess;
    bool ok = true;
    for (auto& rk : ranks) ok = ok && p2p_ok(rk.g) && (rk.g.Kc == 0 || rk.tma);
    if (mode == kVirtual) {
      if (!ok) return cudaSuccess;
      for (int q = 0; q < P; ++q) {
        peerA[q] = ranks[q].A;
        peerB[q] = ranks[q].B;
      }
      p2p = true;
      return cudaSuccess;
    }
    Rank& rk = ranks[0];
    const size_t hb = 2 * sizeof(cudaIpcMemHandle_t);  // this rank's (A, B) handles
    // [barrier float | pad to 64 B | own handles | every rank's handles]
    CE(cudaMalloc(&p2p_bar, 64 + hb * (P + 1)));
    unsigned char* dev = reinterpret_cast<unsigned char*>(p2p_bar) + 64;
    std::vector<unsigned char> hs(hb * P, 0), mine(hb, 0);
    if (ok) {
      cudaIpcMemHandle_t h2[2];
      ok = cudaIpcGetMemHandle(&h2[0], rk.A) == cudaSuccess && cudaIpcGetMemHandle(&h2[1], rk.B) == cudaSuccess;
      if (ok) std::memcpy(mine.data(), h2, hb);
    }
    cudaGetLastError();
    CE(cudaMemcpy(dev, mine.data(), hb, cudaMemcpyHostToDevice));
    if (g_nccl.allGather(dev, dev + hb, hb, kNcclUint8, comm, stream) != 0) return cudaErrorUnknown;
    CE(cudaMemcpyAsync(hs.data(), dev + hb, hb * P, cudaMemcpyDeviceToHost, stream));
    CE(cudaStreamSynchronize(stream));
    for (int q = 0; q < P && ok; ++q) {
      if (q == myrank) {
        peerA[q] = rk.A;
        peerB[q] = rk.B;
        continue;
      }
      cudaIpcMemHandle_t h2[2];
      std::memcpy(h2, hs.data() + hb * q, hb);
      void* pa = nullptr;
      void* pb = nullptr;
      ok = cudaIpcOpenMemHandle(&pa, h2[0], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
      if (ok) ipc_open.push_back(pa);
      ok = ok && cudaIpcOpenMemHandle(&pb, h2[1], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
      if (ok) ipc_open.push_back(pb);
      peerA[q] = static_cast<float2*>(pa);
      peerB[q] = static_cast<float2*>(pb);
    }
    cudaGetLastError();
    // agree: every rank uses the fused transposes or none does
    float v = ok ? 0.f : 1.f;
    CE(cudaMemcpy(p2p_bar, &v, sizeof v, cudaMemcpyHostToDevice));
    if (g_nccl.allReduce(p2p_bar, p2p_bar, 1, kNcclFloat32, kNcclSum, comm, stream) != 0) return cudaErrorUnknown;
    CE(cudaMemcpyAsync(&v, p2p_bar, sizeof v, cudaMemcpyDeviceToHost, stream));
    CE(cudaStreamSynchronize(stream));
    p2p = v == 0.f;
    return cudaSuccess;
  }

  // component q of rank rk's geometry (K1, K2, K4, K5 on one component)
  static Geom comp_geom(const Rank& rk, int q) {
    Geom g = rk.g;
    g.c0 = q;
    g.nc = 1;
    return g;
  }
  // halo: plane nzl-1 of rank r-1 -> Hlo of rank r; plane 0 of rank r+1 -> Hhi of rank r.
  cudaError_t halo(int c, cudaStream_t s) {
    const size_t plane = (size_t)g0.ny * g0.nx;
    const int nzl = ranks[0].g.nzl;
    const long long Nl = ranks[0].Nl;
    if (mode == kVirtual) {
      for (int r = 0; r < P; ++r)
        for (int q = 0; q < 3; ++q) {
          if (r > 0)
            CE(cudaMemcpyAsync(ranks[r].Hlo + q * plane, ranks[r - 1].M[c] + q * Nl + (size_t)(nzl - 1) * plane,
                               sizeof(float) * plane, cudaMemcpyDeviceToDevice, s));
          if (r + 1 < P)
            CE(cudaMemcpyAsync(ranks[r].Hhi + q * plane, ranks[r + 1].M[c] + q * Nl, sizeof(float) * plane,
                               cudaMemcpyDeviceToDevice, s));
        }
      return cudaSuccess;
    }
    Rank& rk = ranks[0];
    const int r = myrank;
    ncclComm_t hc = comm_halo ? comm_halo : comm;
    bool bad = g_nccl.groupStart() != 0;
    for (int q = 0; q < 3 && !bad; ++q) {
      if (r > 0) {
        bad |= g_nccl.send(rk.M[c] + q * Nl, plane, kNcclFloat32, r - 1, hc, s) != 0;
        bad |= g_nccl.recv(rk.Hlo + q * plane, plane, kNcclFloat32, r - 1, hc, s) != 0;
      }
      if (r + 1 < P) {
        bad |= g_nccl.send(rk.M[c] + q * Nl + (size_t)(nzl - 1) * plane, plane, kNcclFloat32, r + 1, hc, s) != 0;
        bad |= g_nccl.recv(rk.Hhi + q * plane, plane, kNcclFloat32, r + 1, hc, s) != 0;
      }
    }
    bad |= g_nccl.groupEnd() != 0;
    return bad ? cudaErrorUnknown : cudaSuccess;
  }

  // C3 on the side stream: it needs only M[c], so it runs under K1..K4 and the
  // transposes; the stencil kernel joins it (halo_join) before reading Hlo/Hhi.
  // On the NCCL path the side stream is used only with the halo's own
  // communicator (ncclCommSplit): on the transposes' communicator NCCL would
  // run it in issue order anyway, so it then goes on the step stream.
  cudaError_t halo_start(int c, cudaStream_t s) {
    if (mode == kNccl && !comm_halo) return halo(c, s);
    CE(cudaEventRecord(evM, s));
    CE(cudaStreamWaitEvent(hs, evM, 0));
    CE(halo(c, hs));
    return cudaEventRecord(evH, hs);
  }
  cudaError_t halo_join(cudaStream_t s) {
    return (mode == kSingle || (mode == kNccl && !comm_halo)) ? cudaSuccess : cudaStreamWaitEvent(s, evH, 0);
  }

  // H~ for every rank: K1 .. K4 plus the transposes.  M[c] is the input.  Always
  // follow it with k5_stage (on the pipelined path the C2 transposes are still in
  // flight on the comm stream when this returns; k5_stage joins them).
  cudaError_t demag_stages(int c, cudaStream_t s, bool bump, cudaEvent_t* ev = nullptr) {
    auto rec = [&](int idx) {
      if (ev) cudaEventRecord(ev[idx], s);
    };
    if (mode == kSingle) {
      Rank& rk = ranks[0];
      rec(0);
      CE(launch_k1(rk.g, rk.M[c], rk.A, tw, bump ? rk.prm : nullptr, s));
      rec(1);
      if (fused) {
        rec(2);
        CE(launch_k2f(rk.g, rk.A, rk.KS, tw, s));
        rec(3);
      } else if (plane) {
        rec(2);
        CE(launch_kplane(rk.g, rk.A, rk.KSP, tw, s, &rk.kpmap));
        rec(3);
      } else {
        rec(2);
        CE(launch_k2(rk.g, rk.A, rk.X2, tw, s, rk.tma ? &rk.k2map : nullptr));
        rec(3);
        rec(4);
        CE(launch_k3(rk.g, rk.X2, rk.KS, tw, s, rk.tma3 ? &rk.k3x : nullptr, rk.tma3 ? &rk.k3k : nullptr, rk.tw3));
        rec(5);
        rec(6);
        CE(launch_k4(rk.g, rk.X2, rk.A, tw, s, rk.tma ? &rk.k4map : nullptr, rk.tma4s ? &rk.k4out : nullptr));
        rec(7);
      }
      return cudaSuccess;
    }
    CE(halo_start(c, s));  // C3: one M plane to each neighbour, overlapped
    if (p2p) {  // fused transposes: K1 / K4 store into the peers' buffers
      for (auto& rk : ranks) CE(launch_k1(p2p_geom(rk, peerB), rk.M[c], rk.A, tw, bump ? rk.prm : nullptr, s));
      CE(p2p_barrier(s));
      for (auto& rk : ranks) {
        if (rk.g.Kc > 0) {
          CE(launch_k2(rk.g, rk.B, rk.X2, tw, s, rk.tma ? &rk.k2map : nullptr));
          CE(launch_k3(rk.g, rk.X2, rk.KS, tw, s, rk.tma3 ? &rk.k3x : nullptr, rk.tma3 ? &rk.k3k : nullptr, rk.tw3));
          CE(launch_k4(p2p_geom(rk, peerA), rk.X2, rk.B, tw, s, rk.tma ? &rk.k4map : nullptr));
        }
      }
      return p2p_barrier(s);
    }
    if (!pipe) {
      for (auto& rk : ranks) CE(launch_k1(rk.g, rk.M[c], rk.A, tw, bump ? rk.prm : nullptr, s));
      CE(alltoall(&Rank::A, &Rank::B, s));  // C1: z slabs -> kx blocks
      for (auto& rk : ranks) {
        if (rk.g.Kc > 0) {
          CE(launch_k2(rk.g, rk.B, rk.X2, tw, s, rk.tma ? &rk.k2map : nullptr));
          CE(launch_k3(rk.g, rk.X2, rk.KS, tw, s, rk.tma3 ? &rk.k3x : nullptr, rk.tma3 ? &rk.k3k : nullptr, rk.tw3));
          CE(launch_k4(rk.g, rk.X2, rk.B, tw, s, rk.tma ? &rk.k4map : nullptr));
        }
      }
      return alltoall(&Rank::B, &Rank::A, s);  // C2: kx blocks -> z slabs
    }
    // pipelined: K1(q) | C1(q) on cs while K1(q+1); K2(q) once C1(q) has landed
    for (int q = 0; q < 3; ++q) {
      for (auto& rk : ranks) CE(launch_k1(comp_geom(rk, q), rk.M[c], rk.A, tw, (bump && q == 0) ? rk.prm : nullptr, s));
      CE(cudaEventRecord(evk[q], s));
      CE(cudaStreamWaitEvent(cs, evk[q], 0));
      CE(alltoall(&Rank::A, &Rank::B, cs, q));
      CE(cudaEventRecord(evc[q], cs));
    }
    set_pdl_blocked(true);  // K2(q) waits on the comm stream: no programmatic edge
    for (int q = 0; q < 3; ++q) {
      CE(cudaStreamWaitEvent(s, evc[q], 0));
      for (auto& rk : ranks) {
        if (rk.g.Kc == 0) continue;
        const cudaError_t e = launch_k2(comp_geom(rk, q), rk.B, rk.X2, tw, s, rk.tma ? &rk.k2map : nullptr);
        if (e != cudaSuccess) {
          set_pdl_blocked(false);
          return e;
        }
      }
    }
    set_pdl_blocked(false);
    for (auto& rk : ranks)
      if (rk.g.Kc > 0)
        CE(launch_k3(rk.g, rk.X2, rk.KS, tw, s, rk.tma3 ? &rk.k3x : nullptr, rk.tma3 ? &rk.k3k : nullptr, rk.tw3));
    // K4(q) | C2(q) on cs while K4(q+1); k5_stage consumes component q once C2(q) landed
    for (int q = 0; q < 3; ++q) {
      for (auto& rk : ranks)
        if (rk.g.Kc > 0) CE(launch_k4(comp_geom(rk, q), rk.X2, rk.B, tw, s, rk.tma ? &rk.k4map : nullptr));
      CE(cudaEventRecord(evk[q], s));
      CE(cudaStreamWaitEvent(cs, evk[q], 0));
      CE(alltoall(&Rank::B, &Rank::A, cs, q));
      CE(cudaEventRecord(evc[q], cs));
    }
    return cudaSuccess;
  }

  // K5 (C2R -> H_demag) of every rank after demag_stages; pipelined: component q
  // as soon as its C2 transpose has landed.
  cudaError_t k5_stage(cudaStream_t s) {
    if (!pipe) {
      for (auto& rk : ranks) CE(launch_k5(rk.g, rk.A, rk.Hd, tw, s));
      return cudaSuccess;
    }
    set_pdl_blocked(true);  // K5(q) waits on the comm stream: no programmatic edge
    cudaError_t e = cudaSuccess;
    for (int q = 0; q < 3 && e == cudaSuccess; ++q) {
      e = cudaStreamWaitEvent(s, evc[q], 0);
      for (auto& rk : ranks)
        if (e == cudaSuccess) e = launch_k5(comp_geom(rk, q), rk.A, rk.Hd, tw, s);
    }
    set_pdl_blocked(false);
    return e;
  }

  // One Heun step, M[c] -> M[c]: predictor M* = renorm(M + dt f0) into M[1-c]
  // (f0 kept in F), then H(M*) and the corrector updates M[c] in place.
  cudaError_t enqueue_heun(int c, cudaStream_t s) {
    CE(demag_stages(c, s, true));
    CE(k5_stage(s));
    CE(halo_join(s));
    for (auto& rk : ranks)
      CE(launch_k6(rk.g, 3, rk.Hd, rk.M[c], rk.M[1 - c], rk.F, rk.prm, rk.flag, s, rk.Hlo, rk.Hhi));
    CE(demag_stages(1 - c, s, false));
    CE(k5_stage(s));
    CE(halo_join(s));
    for (auto& rk : ranks)
      CE(launch_k6(rk.g, 4, rk.Hd, rk.M[1 - c], rk.M[c], rk.F, rk.prm, rk.flag, s, rk.Hlo, rk.Hhi));
    return cudaSuccess;
  }
  // buffer index after one step from c
  int next(int c) const { return integrator == 1 ? c : 1 - c; }

  // One step M[c] -> M[1-c] (ev: optional 2 events per kernel, single mode).
  cudaError_t enqueue_step(int c, cudaStream_t s, cudaEvent_t* ev = nullptr) {
    if (integrator == 1) return enqueue_heun(c, s);
    CE(demag_stages(c, s, true, ev));
    const int nk = kernel_count(g0);
    const int k5 = 2 * (nk - 2);
    if (ev) cudaEventRecord(ev[k5], s);
    CE(k5_stage(s));
    CE(halo_join(s));
    if (ev) cudaEventRecord(ev[k5 + 1], s);
    if (ev) cudaEventRecord(ev[k5 + 2], s);
    for (auto& rk : ranks)
      CE(launch_k6(rk.g, 0, rk.Hd, rk.M[c], rk.M[1 - c], nullptr, rk.prm, rk.flag, s, rk.Hlo, rk.Hhi));
    if (ev) cudaEventRecord(ev[k5 + 3], s);
    return cudaSuccess;
  }

  cudaError_t build_graph(int c, int nsteps, cudaGraphExec_t* out) {
    cudaGraph_t graph = nullptr;
    CE(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    cudaError_t e = cudaSuccess;
    for (int i = 0, cc = c; i < nsteps && e == cudaSuccess; ++i, cc = next(cc)) e = enqueue_step(cc, cap);
    cudaError_t e2 = cudaStreamEndCapture(cap, &graph);
    if (e != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      return e;
    }
    if (e2 != cudaSuccess) return e2;
    e = cudaGraphInstantiate(out, graph, 0);
    cudaGraphDestroy(graph);
    return e;
  }

  // Capture and instantiate every single-GPU step graph the loop can use (16-step
  // chunks and single steps, from either M buffer) ahead of time, so no
  // grace_step call pays a capture: done at create and after anything that
  // invalidates them (integrator, geometry mask).
  // The distributed step is captured too (NCCL calls, the comm and halo streams
  // forked and joined by events); if capture fails there (e.g. an NCCL build
  // without graph support) it runs eagerly instead.
  cudaError_t prepare_graphs() {
    if (mode != kSingle && (!dist_graphs || getenv("GRACE_DIST_EAGER"))) {
      dist_graphs = false;
      return cudaSuccess;
    }
    for (int c = 0; c < 2; ++c) {
      cudaError_t e = cudaSuccess;
      if (!gc[c]) e = build_graph(c, kChunk, &gc[c]);
      if (e == cudaSuccess && !g1[c]) e = build_graph(c, 1, &g1[c]);
      if (e != cudaSuccess) {
        if (mode == kSingle) return e;
        cudaGetLastError();
        drop_graphs();
        dist_graphs = false;
        return cudaSuccess;
      }
    }
    return cudaSuccess;
  }
  void drop_graphs() {
    for (int c = 0; c < 2; ++c) {
      if (g1[c]) cudaGraphExecDestroy(g1[c]);
      if (gc[c]) cudaGraphExecDestroy(gc[c]);
      g1[c] = gc[c] = nullptr;
    }
  }

  void release() {
    for (int c = 0; c < 2; ++c) {
      if (g1[c]) cudaGraphExecDestroy(g1[c]);
      if (gc[c]) cudaGraphExecDestroy(gc[c]);
    }
    for (auto e : ev) cudaEventDestroy(e);
    for (auto& rk : ranks) {
      void* ptrs[] = {rk.M[0], rk.M[1], rk.A,   rk.B,    rk.X2,  rk.KS,   rk.Hlo, rk.Hhi,
                      rk.prm,  rk.flag, rk.red, rk.Hbuf, rk.Hd,  rk.dred, rk.F,   rk.mask, rk.aerr, rk.tw3, rk.KSP};
      for (void* p : ptrs)
        if (p) cudaFree(p);
    }
    if (tw) cudaFree(tw);
    if (comm_halo) g_nccl.commDestroy(comm_halo);
    if (comm) g_nccl.commDestroy(comm);
    if (own) cudaStreamDestroy(own);
    if (cap) cudaStreamDestroy(cap);
    if (pin) cudaFreeHost(pin);
    if (hs) cudaStreamDestroy(hs);
    if (evM) cudaEventDestroy(evM);
    if (evH) cudaEventDestroy(evH);
    if (cs) cudaStreamDestroy(cs);
    for (void* p : ipc_open) cudaIpcCloseMemHandle(p);
    if (p2p_bar) cudaFree(p2p_bar);
    for (int q = 0; q < 3; ++q) {
      if (evk[q]) cudaEventDestroy(evk[q]);
      if (evc[q]) cudaEventDestroy(evc[q]);
    }
  }
};

namespace {

// Global geometry and material coefficients.
int make_geom(int nx, int ny, int nz, double dx, double dy, double dz, double Ms, double A, double Ku, Geom* out) {
  Geom g{};
  g.nx = nx;
  g.ny = ny;
  g.nz = nz;
  g.Px = padded(nx);
  g.Py = padded(ny);
  g.Pz = padded(nz);
  if (g.Px > 8192 || g.Py > 4096 || g.Pz > 1024)
    return fail(GRACE_EUNSUPPORTED, "padded FFT %d x %d x %d exceeds the compiled maximum 8192 x 4096 x 1024", g.Px,
                g.Py, g.Pz);
  g.Kx = g.Px == 1 ? 1 : g.Px / 2 + 1;
  g.Kxp = (int)round_up(g.Kx, 16);
  g.Kyh = g.Py == 1 ? 1 : g.Py / 2 + 1;
  g.Kzh = g.Pz == 1 ? 1 : g.Pz / 2 + 1;
  g.KSp = (int)round_up(g.Kx, 32);
  g.Lmax = std::max(g.Px, std::max(g.Py, g.Pz));
  const double ex = 2.0 * A / (kMU0 * Ms * Ms);
  g.cx = nx > 1 ? (float)(ex / (dx * dx)) : 0.f;
  g.cy = ny > 1 ? (float)(ex / (dy * dy)) : 0.f;
  g.cz = nz > 1 ? (float)(ex / (dz * dz)) : 0.f;
  g.ck = (float)(2.0 * Ku / (kMU0 * Ms * Ms));
  g.Ms = (float)Ms;
  g.nzl = nz;
  g.pitch1 = g.Kxp;
  g.kb = 0;
  g.blk1 = 0;
  g.Kc = g.Kx;
  g.pitch2 = g.Kxp;
  g.has_lo = g.has_hi = 0;
  g.c0 = 0;
  g.nc = 3;
  int dev = 0, nsm = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaGetLastError();
  g.nsm = nsm > 0 ? nsm : 148;
  *out = g;
  return GRACE_OK;
}

// The slab of rank r of P.
// dist: the distributed layouts (also with P = 1, GRACE_FORCE_NCCL)
Geom rank_geom(const Geom& g0, int r, int P, bool dist) {
  Geom g = g0;
  if (!dist) return g;
  const int Kb = (int)round_up((g0.Kx + P - 1) / P, 2);  // even: 16-byte TMA row strides
  g.nzl = g0.nz / P;
  g.kb = Kb;
  g.pitch1 = Kb;
  g.blk1 = 3LL * g.nzl * g0.ny * Kb;
  g.Kc = std::max(0, std::min(g0.Kx, (r + 1) * Kb) - r * Kb);
  g.pitch2 = (int)round_up(std::max(g.Kc, 1), 16);
  g.KSp = (int)round_up(std::max(g.Kc, 1), 32);
  g.has_lo = r > 0;
  g.has_hi = r + 1 < P;
  return g;
}

int validate(int nx, int ny, int nz, double dx, double dy, double dz, double Ms, double A, double Ku, double alpha,
             double gamma) {
  if (nx < 1 || ny < 1 || nz < 1) return fail(GRACE_EINVAL, "cell counts must be >= 1 (got %d %d %d)", nx, ny, nz);
  if (!finite_pos(dx) || !finite_pos(dy) || !finite_pos(dz))
    return fail(GRACE_EINVAL, "cell sizes must be finite and > 0");
  if (!finite_pos(Ms)) return fail(GRACE_EINVAL, "Ms must be finite and > 0");
  if (!std::isfinite(A) || A < 0) return fail(GRACE_EINVAL, "A must be finite and >= 0");
  if (!std::isfinite(Ku) || Ku < 0) return fail(GRACE_EINVAL, "Ku must be finite and >= 0");
  if (!std::isfinite(alpha) || alpha < 0) return fail(GRACE_EINVAL, "alpha must be finite and >= 0");
  if (!finite_pos(gamma)) return fail(GRACE_EINVAL, "gamma must be finite and > 0");
  if (gamma > 1e9)
    return fail(GRACE_EINVAL, "pass gamma0 = gamma*mu0 in m/(A s) (e.g. 2.211e5), not gamma in rad/(s T)");
  if ((long long)nx * ny * nz >= (1LL << 36)) return fail(GRACE_EUNSUPPORTED, "grid exceeds 2^36 cells");
  return GRACE_OK;
}

// Build a context with `nranks_here` rank slabs (ranks first_rank ...) of a P-way partition.
int create_impl(int nx, int ny, int nz, double dx, double dy, double dz, double Ms, double A, double Ku,
                double alpha, double gamma, grace_ctx::Mode mode, int P, int first_rank, int nranks_here,
                const void* nccl_id, grace_ctx** out) {
  g_err.clear();
  if (!out) return fail(GRACE_EINVAL, "out is NULL");
  *out = nullptr;
  int rc = validate(nx, ny, nz, dx, dy, dz, Ms, A, Ku, alpha, gamma);
  if (rc) return rc;
  if (P < 1 || nz % P != 0) return fail(GRACE_EINVAL, "nz = %d must be a multiple of the rank count %d", nz, P);
  Geom g0{};
  if ((rc = make_geom(nx, ny, nz, dx, dy, dz, Ms, A, Ku, &g0))) return rc;
  grace_ctx* h = new grace_ctx();
  h->mode = mode;
  h->P = P;
  h->myrank = first_rank;
  h->g0 = g0;
  h->g0.plane = mode == grace_ctx::kSingle && !fused_y_path(g0) && plane_ok(g0);
  h->plane = h->g0.plane;
  h->dx = dx;
  h->dy = dy;
  h->dz = dz;
  h->Ms = Ms;
  h->A = A;
  h->Ku = Ku;
  h->alpha = alpha;
  h->gamma0 = gamma;
  const bool dlay = mode != grace_ctx::kSingle;  // distributed layouts and transposes
  h->fused = !dlay && fused_y_path(g0);
  auto bail = [&](int code) {
    h->release();
    delete h;
    return code;
  };
  {
    cudaError_t e = cudaStreamCreateWithFlags(&h->own, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMallocHost((void**)&h->pin, sizeof(grace_ctx::Pinned));
    if (e == cudaSuccess && mode != grace_ctx::kSingle) e = cudaStreamCreateWithFlags(&h->hs, cudaStreamNonBlocking);
    if (e == cudaSuccess && mode != grace_ctx::kSingle) e = cudaEventCreateWithFlags(&h->evM, cudaEventDisableTiming);
    if (e == cudaSuccess && mode != grace_ctx::kSingle) e = cudaEventCreateWithFlags(&h->evH, cudaEventDisableTiming);
    if (e == cudaSuccess && mode != grace_ctx::kSingle) e = cudaStreamCreateWithFlags(&h->cs, cudaStreamNonBlocking);
    for (int q = 0; q < 3 && e == cudaSuccess && mode != grace_ctx::kSingle; ++q) {
      e = cudaEventCreateWithFlags(&h->evk[q], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->evc[q], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) return bail(fail(GRACE_ECUDA, "stream creation: %s", cudaGetErrorString(e)));
  }
  h->stream = h->own;
  cudaStream_t s = h->stream;
  if (mode == grace_ctx::kNccl) {
    if (!g_nccl.load()) return bail(fail(GRACE_EUNSUPPORTED, "libnccl.so.2 not found (set GRACE_NCCL_LIB)"));
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof id);
    const ncclResult_t r = g_nccl.commInitRank(&h->comm, P, id, first_rank);
    if (r != 0) return bail(fail(GRACE_ECUDA, "ncclCommInitRank: %s", g_nccl.errStr(r)));
    if (g_nccl.commSplit && !getenv("GRACE_NO_HALO_COMM")) {  // collective over the ranks: all or none
      if (g_nccl.commSplit(h->comm, 0, first_rank, &h->comm_halo, nullptr) != 0) h->comm_halo = nullptr;
    }
  }
  h->ranks.resize(nranks_here);
  for (int i = 0; i < nranks_here; ++i) {
    Rank& rk = h->ranks[i];
    rk.r = first_rank + i;
    rk.g = rank_geom(h->g0, rk.r, P, dlay);
    const Geom& g = rk.g;
    rk.Nl = (long long)g.nzl * ny * nx;
    const size_t mb = sizeof(float) * 3 * (size_t)rk.Nl;
    const size_t ab = !dlay ? sizeof(float2) * 3 * (size_t)nz * ny * g.Kxp : sizeof(float2) * (size_t)P * g.blk1;
    const size_t x2 = (h->fused || h->plane) ? 0 : sizeof(float2) * 3 * (size_t)nz * g.Py * g.pitch2;
    const size_t ks = sizeof(float) * 6 * (size_t)g.Kzh * g.Kyh * g.KSp;
    const size_t hb = sizeof(float) * 3 * (size_t)ny * nx;
    if ((rc = h->alloc((void**)&rk.M[0], mb)) || (rc = h->alloc((void**)&rk.M[1], mb)) ||
        (rc = h->alloc((void**)&rk.A, ab)) || (dlay && (rc = h->alloc((void**)&rk.B, ab))) ||
        (x2 && (rc = h->alloc((void**)&rk.X2, x2))) || (rc = h->alloc((void**)&rk.KS, ks)) ||
        (h->plane && (rc = h->alloc((void**)&rk.KSP, sizeof(float) * plane_ks_floats(g)))) ||
        (g.has_lo && (rc = h->alloc((void**)&rk.Hlo, hb))) || (g.has_hi && (rc = h->alloc((void**)&rk.Hhi, hb))) ||
        (rc = h->alloc((void**)&rk.prm, sizeof(StepParams))) ||
        (rc = h->alloc((void**)&rk.flag, 3 * sizeof(unsigned long long))) ||
        (rc = h->alloc((void**)&rk.red, sizeof(double) * (kMavgPartials + 3))) ||
        (rc = h->alloc((void**)&rk.Hd, mb)))
      return bail(rc);
  }
  if ((rc = h->alloc((void**)&h->tw, sizeof(float2) * g0.Lmax))) return bail(rc);
  if (dlay && !getenv("GRACE_NO_PIPE")) {
    h->pipe = true;
    for (auto& rk : h->ranks) h->pipe = h->pipe && comp_split_ok(rk.g);
  }
  // TMA descriptors for the y-pencil kernels (K2 reads the x-row layout, K4 reads X2)
  for (auto& rk : h->ranks)
    if (h->plane && make_plane_tmap(rk.g, rk.A, &rk.kpmap) != cudaSuccess)
      return bail(fail(GRACE_ECUDA, "plane path: TMA descriptor of X1 failed"));
  if (!h->fused && !h->plane && !getenv("GRACE_NO_TMA"))
    for (auto& rk : h->ranks) {
      rk.tma = make_ky_tmaps(rk.g, dlay ? rk.B : rk.A, rk.X2, &rk.k2map, &rk.k4map,
                             (dlay || getenv("GRACE_NO_TMA_STORE")) ? nullptr : &rk.k4out) == cudaSuccess;
      rk.tma4s = rk.tma && !dlay && !getenv("GRACE_NO_TMA_STORE");
      rk.tma3 = rk.X2 && make_k3_tmaps(rk.g, rk.X2, rk.KS, &rk.k3x, &rk.k3k) == cudaSuccess;
    }
  cudaGetLastError();
  h->N = (mode == grace_ctx::kNccl) ? h->ranks[0].Nl : (long long)nx * ny * nz;
  if (dlay) {  // fused transposes (opt-in; collective on the NCCL path: set GRACE_P2P on every rank)
    const char* pe = getenv("GRACE_P2P");
    if (pe && pe[0] == '1') {
      if (h->setup_p2p() != cudaSuccess) return bail(fail(GRACE_ECUDA, "fused-transpose (P2P) setup failed"));
      if (h->p2p) h->pipe = false;
    }
  }

  // setup: fp64 octant -> fp64 padded spectrum -> fp32 folded KS (S1..S5), once,
  // one tensor component at a time; each rank's table receives only its kx
  // columns and only those columns are carried through the y and z transforms.
  std::vector<KsOut> kso;
  for (auto& rk : h->ranks)
    if (rk.g.Kc > 0 || !dlay) kso.push_back(KsOut{rk.KS, dlay ? rk.r * rk.g.kb : 0, rk.g.Kc, rk.g.KSp});
  size_t scratch = 0;
  cudaError_t e = kernel_spectrum_device(g0, dx, dy, dz, (int)kso.size(), kso.data(), &scratch, s);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    return bail(fail(GRACE_ENOMEM, "tensor setup needs %zu bytes of fp64 scratch", scratch));
  }
  if (e == cudaSuccess) e = launch_twiddles(h->tw, g0.Lmax, s);
  for (auto& rk : h->ranks)
    if (e == cudaSuccess && rk.KSP) e = launch_plane_ks(rk.g, rk.KSP, rk.KS, s);
  for (auto& rk : h->ranks)
    if (e == cudaSuccess && rk.tma3) e = make_k3_twiddles(rk.g, h->tw, &rk.tw3, s);
  for (auto& rk : h->ranks) {
    if (e == cudaSuccess) e = launch_fill_uniform_x(rk.M[0], rk.Nl, (float)Ms, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(rk.flag, 0xff, 2 * sizeof(unsigned long long), s);
  }
  if (e == cudaSuccess) e = h->upload_params(1e-15);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return bail(fail(GRACE_ECUDA, "tensor setup: %s", cudaGetErrorString(e)));
  // Dry run of one step (M[0] -> M[1], the spare buffer) so every kernel's
  // shared-memory attribute is set before any graph capture; then restore the
  // device step counters and flags.
  e = h->enqueue_step(0, s);
  for (auto& rk : h->ranks)
    if (e == cudaSuccess) e = cudaMemsetAsync(rk.flag, 0xff, 2 * sizeof(unsigned long long), s);
  if (e == cudaSuccess) e = h->upload_params(1e-15);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = h->prepare_graphs();
  if (e != cudaSuccess) return bail(fail(GRACE_ECUDA, "first step: %s", cudaGetErrorString(e)));
  *out = h;
  return GRACE_OK;
}

// First set flag over the ranks (0: step non-finite, packed step<<36|cell; 1: set_m
// zero cell), translated to the global cell numbering (z-slab offset added), and
// reset on the device.  On the NCCL path the ranks agree: the translated flags
// are min-reduced over the communicator, so every rank returns the same status
// (a rank that alone returned an error would leave the others waiting in the
// next collective).
int check_flags(grace_ctx* h, int which, unsigned long long* first) {
  *first = kNoFlag;
  const unsigned long long mask = (1ULL << 36) - 1;
  for (auto& rk : h->ranks) {
    unsigned long long f = kNoFlag;
    CUDA_OR(cudaMemcpyAsync(&h->pin->flag, rk.flag + which, sizeof f, cudaMemcpyDeviceToHost, h->stream));
    CUDA_OR(cudaStreamSynchronize(h->stream));
    f = h->pin->flag;
    if (f != kNoFlag) {
      CUDA_OR(cudaMemsetAsync(rk.flag + which, 0xff, sizeof f, h->stream));
      const unsigned long long off = (unsigned long long)rk.r * rk.g.nzl * h->g0.ny * h->g0.nx;
      f = (which == 0) ? ((f & ~mask) | ((f & mask) + off)) : f + off;
    }
    if (h->mode == grace_ctx::kNccl) {
      h->pin->flag = f;
      CUDA_OR(cudaMemcpyAsync(rk.flag + 2, &h->pin->flag, sizeof f, cudaMemcpyHostToDevice, h->stream));
      const ncclResult_t r = g_nccl.allReduce(rk.flag + 2, rk.flag + 2, 1, kNcclUint64, kNcclMin, h->comm, h->stream);
      if (r != 0) return fail(GRACE_ECUDA, "ncclAllReduce: %s", g_nccl.errStr(r));
      CUDA_OR(cudaMemcpyAsync(&h->pin->flag, rk.flag + 2, sizeof f, cudaMemcpyDeviceToHost, h->stream));
      CUDA_OR(cudaStreamSynchronize(h->stream));
      f = h->pin->flag;
    }
    if (f < *first) *first = f;
  }
  CUDA_OR(cudaStreamSynchronize(h->stream));
  return GRACE_OK;
}

// Offset of rank rk's slab inside the caller's component array (virtual mode).
size_t slab_offset(const grace_ctx* h, const Rank& rk) {
  return (h->mode == grace_ctx::kVirtual) ? (size_t)rk.r * rk.Nl : 0;
}

}  // namespace

extern "C" {

const char* grace_last_error(void) { return g_err.c_str(); }

int grace_create(int nx, int ny, int nz, double dx, double dy, double dz, double Ms, double A, double Ku, double alpha,
                 double gamma, grace_ctx** out) {
  return create_impl(nx, ny, nz, dx, dy, dz, Ms, A, Ku, alpha, gamma, grace_ctx::kSingle, 1, 0, 1, nullptr, out);
}

int grace_create_virtual(int nx, int ny, int nz, double dx, double dy, double dz, double Ms, double A, double Ku,
                         double alpha, double gamma, int nranks, grace_ctx** out) {
  if (nranks < 1) return fail(GRACE_EINVAL, "nranks must be >= 1");
  const auto mode = nranks == 1 ? grace_ctx::kSingle : grace_ctx::kVirtual;
  return create_impl(nx, ny, nz, dx, dy, dz, Ms, A, Ku, alpha, gamma, mode, nranks, 0, nranks, nullptr, out);
}

int grace_nccl_unique_id(void* out128) {
  if (!out128) return fail(GRACE_EINVAL, "NULL argument");
  if (!g_nccl.load()) return fail(GRACE_EUNSUPPORTED, "libnccl.so.2 not found (set GRACE_NCCL_LIB)");
  ncclUniqueId id;
  const ncclResult_t r = g_nccl.getUniqueId(&id);
  if (r != 0) return fail(GRACE_ECUDA, "ncclGetUniqueId: %s", g_nccl.errStr(r));
  std::memcpy(out128, &id, sizeof id);
  return GRACE_OK;
}

int grace_create_dist(int nx, int ny, int nz, double dx, double dy, double dz, double Ms, double A, double Ku,
                      double alpha, double gamma, int rank, int nranks, const void* nccl_id, grace_ctx** out) {
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(GRACE_EINVAL, "bad rank %d of %d", rank, nranks);
  // One rank is the single-GPU context, unless GRACE_FORCE_NCCL is set: then the
  // NCCL path runs with P = 1 (distributed layouts, grouped send/recv / ncclAllReduce on
  // a one-rank communicator) -- how its host and device plumbing is exercised on a
  // one-GPU machine (tests/test_gpu_dist.py).
  if (nranks == 1 && !getenv("GRACE_FORCE_NCCL")) return grace_create(nx, ny, nz, dx, dy, dz, Ms, A, Ku, alpha, gamma, out);
  if (!nccl_id) return fail(GRACE_EINVAL, "NULL nccl id");
  return create_impl(nx, ny, nz, dx, dy, dz, Ms, A, Ku, alpha, gamma, grace_ctx::kNccl, nranks, rank, 1, nccl_id,
                     out);
}

void grace_destroy(grace_ctx* h) {
  if (!h) return;
  if (h->stream) cudaStreamSynchronize(h->stream);
  h->release();
  delete h;
}

int grace_set_stream(grace_ctx* h, void* stream) {
  if (!h) return fail(GRACE_EINVAL, "NULL context");
  CUDA_OR(cudaStreamSynchronize(h->stream));
  h->stream = stream ? (cudaStream_t)stream : h->own;
  return GRACE_OK;
}

static int finish_set_m(grace_ctx* h, int target) {
  unsigned long long f;
  int rc = check_flags(h, 1, &f);
  if (rc) return rc;
  if (f != kNoFlag) return fail(GRACE_EZEROCELL, "cell %llu has |M| = 0 or a non-finite component", f);
  h->cur = target;
  return GRACE_OK;
}

int grace_set_m(grace_ctx* h, const double* m) {
  if (!h || !m) return fail(GRACE_EINVAL, "NULL argument");
  // stage the fp64 input (24 bytes/cell fits in the A buffer), normalise into the spare M buffer
  const int target = 1 - h->cur;
  for (auto& rk : h->ranks) {
    double* stage = reinterpret_cast<double*>(rk.A);
    const size_t off = slab_offset(h, rk);
    for (int c = 0; c < 3; ++c)
      CUDA_OR(cudaMemcpyAsync(stage + c * rk.Nl, m + c * h->N + off, sizeof(double) * rk.Nl, cudaMemcpyHostToDevice,
                              h->stream));
    CUDA_OR(launch_set_m_f64(stage, rk.M[target], rk.Nl, h->Ms, rk.mask, rk.flag + 1, h->stream));
  }
  return finish_set_m(h, target);
}

int grace_set_m_device(grace_ctx* h, const float* d_m) {
  if (!h || !d_m) return fail(GRACE_EINVAL, "NULL argument");
  const int target = 1 - h->cur;
  for (auto& rk : h->ranks) {
    if (h->mode != grace_ctx::kVirtual) {
      CUDA_OR(launch_set_m_f32(d_m, rk.M[target], rk.Nl, (float)h->Ms, rk.mask, rk.flag + 1, h->stream));
    } else {
      float* stage = reinterpret_cast<float*>(rk.A);
      const size_t off = slab_offset(h, rk);
      for (int c = 0; c < 3; ++c)
        CUDA_OR(cudaMemcpyAsync(stage + c * rk.Nl, d_m + c * h->N + off, sizeof(float) * rk.Nl,
                                cudaMemcpyDeviceToDevice, h->stream));
      CUDA_OR(launch_set_m_f32(stage, rk.M[target], rk.Nl, (float)h->Ms, rk.mask, rk.flag + 1, h->stream));
    }
  }
  return finish_set_m(h, target);
}

int grace_get_m(grace_ctx* h, double* out) {
  if (!h || !out) return fail(GRACE_EINVAL, "NULL argument");
  for (auto& rk : h->ranks) {
    double* stage = reinterpret_cast<double*>(rk.A);
    const size_t off = slab_offset(h, rk);
    CUDA_OR(launch_widen(rk.M[h->cur], stage, 3 * rk.Nl, h->stream));
    for (int c = 0; c < 3; ++c)
      CUDA_OR(cudaMemcpyAsync(out + c * h->N + off, stage + c * rk.Nl, sizeof(double) * rk.Nl,
                              cudaMemcpyDeviceToHost, h->stream));
    CUDA_OR(cudaStreamSynchronize(h->stream));
  }
  return GRACE_OK;
}

int grace_set_m_f32(grace_ctx* h, const float* m) {
  if (!h || !m) return fail(GRACE_EINVAL, "NULL argument");
  // stage the fp32 input in the A buffer, normalise into the spare M buffer
  const int target = 1 - h->cur;
  for (auto& rk : h->ranks) {
    float* stage = reinterpret_cast<float*>(rk.A);
    const size_t off = slab_offset(h, rk);
    for (int c = 0; c < 3; ++c)
      CUDA_OR(cudaMemcpyAsync(stage + c * rk.Nl, m + c * h->N + off, sizeof(float) * rk.Nl, cudaMemcpyHostToDevice,
                              h->stream));
    CUDA_OR(launch_set_m_f32(stage, rk.M[target], rk.Nl, (float)h->Ms, rk.mask, rk.flag + 1, h->stream));
  }
  return finish_set_m(h, target);
}

int grace_get_m_f32(grace_ctx* h, float* out) {
  if (!h || !out) return fail(GRACE_EINVAL, "NULL argument");
  for (auto& rk : h->ranks) {
    const size_t off = slab_offset(h, rk);
    for (int c = 0; c < 3; ++c)
      CUDA_OR(cudaMemcpyAsync(out + c * h->N + off, rk.M[h->cur] + c * rk.Nl, sizeof(float) * rk.Nl,
                              cudaMemcpyDeviceToHost, h->stream));
  }
  CUDA_OR(cudaStreamSynchronize(h->stream));
  return GRACE_OK;
}

int grace_get_m_device(grace_ctx* h, float* d_out) {
  if (!h || !d_out) return fail(GRACE_EINVAL, "NULL argument");
  for (auto& rk : h->ranks) {
    const size_t off = slab_offset(h, rk);
    for (int c = 0; c < 3; ++c)
      CUDA_OR(cudaMemcpyAsync(d_out + c * h->N + off, rk.M[h->cur] + c * rk.Nl, sizeof(float) * rk.Nl,
                              cudaMemcpyDeviceToDevice, h->stream));
  }
  CUDA_OR(cudaStreamSynchronize(h->stream));
  return GRACE_OK;
}

int grace_set_hext(grace_ctx* h, double hx, double hy, double hz) {
  if (!h) return fail(GRACE_EINVAL, "NULL context");
  if (!std::isfinite(hx) || !std::isfinite(hy) || !std::isfinite(hz)) return fail(GRACE_EINVAL, "H_ext must be finite");
  h->hext[0] = hx;
  h->hext[1] = hy;
  h->hext[2] = hz;
  return GRACE_OK;
}

int grace_set_field_schedule(grace_ctx* h, double h0x, double h0y, double h0z, long long start, long long decay,
                             long long stop) {
  if (!h) return fail(GRACE_EINVAL, "NULL context");
  if (!std::isfinite(h0x) || !std::isfinite(h0y) || !std::isfinite(h0z))
    return fail(GRACE_EINVAL, "scheduled field must be finite");
  if (!(0 <= start && start <= decay && decay <= stop))
    return fail(GRACE_EINVAL, "schedule needs 0 <= start <= decay <= stop (got %lld, %lld, %lld)", start, decay, stop);
  h->h0[0] = h0x;
  h->h0[1] = h0y;
  h->h0[2] = h0z;
  h->sched[0] = start;
  h->sched[1] = decay;
  h->sched[2] = stop;
  h->has_sched = (h0x != 0 || h0y != 0 || h0z != 0) && stop > start;
  return GRACE_OK;
}

int grace_set_integrator(grace_ctx* h, int kind) {
  if (!h) return fail(GRACE_EINVAL, "NULL context");
  if (kind != 0 && kind != 1) return fail(GRACE_EINVAL, "integrator must be 0 (Euler) or 1 (Heun)");
  if (kind == h->integrator) return GRACE_OK;
  if (kind == 1) {
    for (auto& rk : h->ranks)
      if (!rk.F) {
        int rc = h->alloc((void**)&rk.F, sizeof(float) * 3 * (size_t)rk.Nl);
        if (rc) return rc;
      }
  }
  h->drop_graphs();  // captured step graphs belong to the old integrator
  h->integrator = kind;
  CUDA_OR(h->prepare_graphs());
  return GRACE_OK;
}

int grace_set_geometry(grace_ctx* h, const unsigned char* mask) {
  if (!h) return fail(GRACE_EINVAL, "NULL context");
  double local = 0;
  if (mask) {
    for (auto& rk : h->ranks) {
      const size_t off = slab_offset(h, rk);
      for (long long i = 0; i < rk.Nl; ++i) local += mask[off + i] ? 1.0 : 0.0;
    }
    double total = local;
    if (h->mode == grace_ctx::kNccl) {  // magnetic cells of the whole grid
      Rank& rk = h->ranks[0];
      double* d = rk.red + kMavgPartials;
      CUDA_OR(cudaMemcpyAsync(d, &local, sizeof(double), cudaMemcpyHostToDevice, h->stream));
      const ncclResult_t r = g_nccl.allReduce(d, d, 1, kNcclFloat64, kNcclSum, h->comm, h->stream);
      if (r != 0) return fail(GRACE_ECUDA, "ncclAllReduce: %s", g_nccl.errStr(r));
      CUDA_OR(cudaMemcpyAsync(&total, d, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
      CUDA_OR(cudaStreamSynchronize(h->stream));
    }
    if (!(total > 0)) return fail(GRACE_EINVAL, "geometry mask selects no cell");
    for (auto& rk : h->ranks) {
      if (!rk.mask) {
        int rc = h->alloc((void**)&rk.mask, (size_t)rk.Nl);
        if (rc) return rc;
      }
      CUDA_OR(cudaMemcpyAsync(rk.mask, mask + slab_offset(h, rk), (size_t)rk.Nl, cudaMemcpyHostToDevice, h->stream));
      // empty cells of the current M become 0 (magnetic cells keep their value)
      CUDA_OR(launch_apply_mask(rk.M[h->cur], rk.Nl, rk.mask, h->stream));
      rk.g.masked = 1;
    }
    h->nmag = total;
  } else {
    for (auto& rk : h->ranks) {
      if (rk.mask) {
        cudaFree(rk.mask);
        h->bytes -= (size_t)rk.Nl;
      }
      rk.mask = nullptr;
      rk.g.masked = 0;
    }
    h->nmag = 0;
  }
  CUDA_OR(cudaStreamSynchronize(h->stream));
  h->g0.masked = mask ? 1 : 0;
  h->drop_graphs();  // captured step graphs carry the old K6 instantiation
  CUDA_OR(h->prepare_graphs());
  return GRACE_OK;
}

int grace_set_alpha(grace_ctx* h, double alpha) {
  if (!h) return fail(GRACE_EINVAL, "NULL context");
  if (!std::isfinite(alpha) || alpha < 0) return fail(GRACE_EINVAL, "alpha must be finite and >= 0");
  h->alpha = alpha;
  return GRACE_OK;
}

int grace_heff(grace_ctx* h, double* out) {
  if (!h || !out) return fail(GRACE_EINVAL, "NULL argument");
  cudaStream_t s = h->stream;
  for (auto& rk : h->ranks)
    if (!rk.Hbuf) {
      int rc = h->alloc((void**)&rk.Hbuf, sizeof(float) * 3 * (size_t)rk.Nl);
      if (rc) return rc;
    }
  CUDA_OR(h->upload_params(1e-15, true));
  CUDA_OR(h->demag_stages(h->cur, s, false));
  CUDA_OR(h->k5_stage(s));
  CUDA_OR(h->halo_join(s));
  for (auto& rk : h->ranks)
    CUDA_OR(launch_k6(rk.g, 1, rk.Hd, rk.M[h->cur], nullptr, rk.Hbuf, rk.prm, rk.flag, s, rk.Hlo, rk.Hhi));
  for (auto& rk : h->ranks) {
    double* stage = reinterpret_cast<double*>(rk.A);
    const size_t off = slab_offset(h, rk);
    CUDA_OR(launch_widen(rk.Hbuf, stage, 3 * rk.Nl, s));
    for (int c = 0; c < 3; ++c)
      CUDA_OR(cudaMemcpyAsync(out + c * h->N + off, stage + c * rk.Nl, sizeof(double) * rk.Nl,
                              cudaMemcpyDeviceToHost, s));
    CUDA_OR(cudaStreamSynchronize(s));
  }
  return GRACE_OK;
}

int grace_step(grace_ctx* h, int n, double dt) {
  if (!h) return fail(GRACE_EINVAL, "NULL context");
  if (n < 0) return fail(GRACE_EINVAL, "n must be >= 0");
  if (!finite_pos(dt)) return fail(GRACE_EINVAL, "dt must be finite and > 0");
  if (n == 0) return GRACE_OK;
  cudaStream_t s = h->stream;
  CUDA_OR(h->upload_params(dt));
  const int nk = kernel_count(h->g0);
  if (h->mode != grace_ctx::kSingle && !h->dist_graphs) {
    for (int i = 0; i < n; ++i) {
      cudaError_t e = h->enqueue_step(h->cur, s);
      if (e != cudaSuccess) return fail(GRACE_ECUDA, "distributed step: %s", cudaGetErrorString(e));
      h->cur = h->next(h->cur);
    }
  } else if (h->mode == grace_ctx::kSingle && !h->profiling && h->integrator == 0 && small_path_ok(h->ranks[0].g)) {
    // small nz = 1 grids: the whole call in one cluster-resident kernel (small_step.cu)
    Rank& rk = h->ranks[0];
    const int dst = h->cur ^ (n & 1);
    CUDA_OR(launch_small_step(rk.g, rk.M[h->cur], rk.M[dst], rk.KS, h->tw, rk.prm, rk.flag, n, s));
    h->cur = dst;
  } else if (h->profiling && h->integrator != 0) {
    return fail(GRACE_EUNSUPPORTED, "profiling mode times the Euler step only");
  } else if (h->profiling) {
    // eager launches with an event pair around every kernel; events are read in
    // batches of kProfBatch steps so the host never waits inside a batch
    constexpr int kProfBatch = 64;
    if (h->ev.empty()) {
      h->ev.resize((size_t)2 * nk * kProfBatch);
      for (auto& e : h->ev) CUDA_OR(cudaEventCreate(&e));
      h->kms.assign(nk, 0.0);
      h->klaunch.assign(nk, 0);
    }
    for (int i0 = 0; i0 < n; i0 += kProfBatch) {
      const int nb = std::min(kProfBatch, n - i0);
      for (int i = 0; i < nb; ++i) {
        cudaError_t e = h->enqueue_step(h->cur, s, &h->ev[(size_t)2 * nk * i]);
        if (e != cudaSuccess) return fail(GRACE_ECUDA, "step launch: %s", cudaGetErrorString(e));
        h->cur ^= 1;
      }
      CUDA_OR(cudaEventSynchronize(h->ev[(size_t)2 * nk * nb - 1]));
      for (int i = 0; i < nb; ++i)
        for (int k = 0; k < nk; ++k) {
          float ms = 0.f;
          CUDA_OR(cudaEventElapsedTime(&ms, h->ev[(size_t)2 * nk * i + 2 * k], h->ev[(size_t)2 * nk * i + 2 * k + 1]));
          h->kms[k] += ms;
          h->klaunch[k] += 1;
        }
    }
  } else {
    int left = n;
    while (left > 0) {
      const bool chunk = left >= kChunk;
      cudaGraphExec_t* gx = chunk ? &h->gc[h->cur] : &h->g1[h->cur];
      if (!*gx) {
        cudaError_t e = h->build_graph(h->cur, chunk ? kChunk : 1, gx);
        if (e != cudaSuccess) return fail(GRACE_ECUDA, "graph capture: %s", cudaGetErrorString(e));
      }
      CUDA_OR(cudaGraphLaunch(*gx, s));
      const int done = chunk ? kChunk : 1;
      left -= done;
      if (h->integrator == 0) h->cur ^= (done & 1);
    }
  }
  unsigned long long f;
  int rc = check_flags(h, 0, &f);
  if (rc) return rc;
  h->steps += n;
  if (f != kNoFlag) {
    h->nf_step = (long long)(f >> 36);
    h->nf_cell = (long long)(f & ((1ULL << 36) - 1));
    return fail(GRACE_ENONFINITE, "non-finite magnetisation at step %lld, cell %lld (dt too large?)", h->nf_step,
                h->nf_cell);
  }
  return GRACE_OK;
}

int grace_step_adaptive(grace_ctx* h, double t_span, double* dt_io, double tol, long long max_attempts,
                        long long* accepted, long long* rejected) {
  if (!h || !dt_io || !accepted || !rejected) return fail(GRACE_EINVAL, "NULL argument");
  if (!std::isfinite(t_span) || t_span < 0 || !finite_pos(*dt_io) || !finite_pos(tol) || max_attempts < 1)
    return fail(GRACE_EINVAL, "adaptive steps need t_span >= 0, dt > 0, tol > 0, max_attempts >= 1");
  if (h->has_sched) return fail(GRACE_EUNSUPPORTED, "adaptive steps take a constant applied field (no schedule)");
  cudaStream_t s = h->stream;
  for (auto& rk : h->ranks) {
    if (!rk.F) {
      int rc = h->alloc((void**)&rk.F, sizeof(float) * 3 * (size_t)rk.Nl);
      if (rc) return rc;
    }
    if (!rk.aerr) {
      int rc = h->alloc((void**)&rk.aerr, sizeof(unsigned));
      if (rc) return rc;
    }
  }
  // controller constants (the oracle's Sim.adaptive_run)
  const double safety = 0.9, fac_min = 0.2, fac_max = 5.0;
  const int c = h->cur;
  double t = 0.0, dt = *dt_io;
  long long acc = 0, rej = 0;
  int rc = GRACE_OK;
  while (t < t_span && acc + rej < max_attempts) {
    const bool last = t + dt >= t_span;
    const double hs = last ? t_span - t : dt;
    if (!(hs > 0)) break;
    CUDA_OR(h->upload_params(hs));
    for (auto& rk : h->ranks) CUDA_OR(cudaMemsetAsync(rk.aerr, 0, sizeof(unsigned), s));
    // Euler attempt M_E = renorm(M + dt f0) into M[1-c] (f0 kept in F) ...
    CUDA_OR(h->demag_stages(c, s, false));
    CUDA_OR(h->k5_stage(s));
    CUDA_OR(h->halo_join(s));
    for (auto& rk : h->ranks)
      CUDA_OR(launch_k6(rk.g, 3, rk.Hd, rk.M[c], rk.M[1 - c], rk.F, rk.prm, rk.flag, s, rk.Hlo, rk.Hhi));
    // ... and the Heun step M_H = renorm(M + dt (f0 + f(M_E))/2) over F, with max |M_H - M_E| / Ms
    CUDA_OR(h->demag_stages(1 - c, s, false));
    CUDA_OR(h->k5_stage(s));
    CUDA_OR(h->halo_join(s));
    for (auto& rk : h->ranks)
      CUDA_OR(launch_k6(rk.g, 5, rk.Hd, rk.M[1 - c], rk.M[c], rk.F, rk.prm, rk.flag, s, rk.Hlo, rk.Hhi, rk.aerr));
    unsigned bits = 0;
    for (auto& rk : h->ranks) {
      if (h->mode == grace_ctx::kNccl) {
        const ncclResult_t r = g_nccl.allReduce(rk.aerr, rk.aerr, 1, kNcclUint32, kNcclMax, h->comm, s);
        if (r != 0) return fail(GRACE_ECUDA, "ncclAllReduce: %s", g_nccl.errStr(r));
      }
      CUDA_OR(cudaMemcpyAsync(&h->pin->flag, rk.aerr, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
      CUDA_OR(cudaStreamSynchronize(s));
      unsigned b;
      std::memcpy(&b, &h->pin->flag, sizeof b);
      bits = std::max(bits, b);
    }
    float errf;
    std::memcpy(&errf, &bits, sizeof errf);
    const double err = errf;
    if (!std::isfinite(err)) {
      rc = fail(GRACE_ENONFINITE, "non-finite magnetisation in an adaptive attempt (dt %g s)", hs);
      break;
    }
    const double fac = err == 0.0 ? fac_max : std::min(fac_max, std::max(fac_min, safety * std::sqrt(tol / err)));
    if (err <= tol) {  // accept: M[c] <- M_H
      for (auto& rk : h->ranks)
        CUDA_OR(cudaMemcpyAsync(rk.M[c], rk.F, sizeof(float) * 3 * (size_t)rk.Nl, cudaMemcpyDeviceToDevice, s));
      t = last ? t_span : t + hs;
      ++acc;
      ++h->steps;
    } else {
      ++rej;
    }
    dt = hs * fac;
  }
  unsigned long long f;
  int rc2 = check_flags(h, 0, &f);
  *dt_io = dt;
  *accepted = acc;
  *rejected = rej;
  if (rc) return rc;
  if (rc2) return rc2;
  if (f != kNoFlag) {
    h->nf_step = (long long)(f >> 36);
    h->nf_cell = (long long)(f & ((1ULL << 36) - 1));
    return fail(GRACE_ENONFINITE, "non-finite magnetisation at cell %lld", h->nf_cell);
  }
  return GRACE_OK;
}

int grace_mavg(grace_ctx* h, double* out3) {
  if (!h || !out3) return fail(GRACE_EINVAL, "NULL argument");
  double acc[3] = {0, 0, 0};
  for (auto& rk : h->ranks) {
    double part[3];
    CUDA_OR(launch_mavg(rk.M[h->cur], rk.Nl, h->Ms, rk.red, rk.red + kMavgPartials, h->stream));
    if (h->mode == grace_ctx::kNccl) {
      const ncclResult_t r = g_nccl.allReduce(rk.red + kMavgPartials, rk.red + kMavgPartials, 3, kNcclFloat64,
                                              kNcclSum, h->comm, h->stream);
      if (r != 0) return fail(GRACE_ECUDA, "ncclAllReduce: %s", g_nccl.errStr(r));
    }
    CUDA_OR(cudaMemcpyAsync(h->pin->red, rk.red + kMavgPartials, 3 * sizeof(double), cudaMemcpyDeviceToHost,
                            h->stream));
    CUDA_OR(cudaStreamSynchronize(h->stream));
    std::memcpy(part, h->pin->red, sizeof part);
    for (int q = 0; q < 3; ++q) acc[q] += part[q];
  }
  // equal slabs: mean of the slab means; with a geometry mask, over magnetic cells (reading Q26)
  const double scale = h->nmag > 0 ? (double)h->g0.nx * h->g0.ny * h->g0.nz / h->nmag : 1.0;
  for (int q = 0; q < 3; ++q) out3[q] = acc[q] / h->P * scale;
  return GRACE_OK;
}

// Energy sums and max torque over the whole grid (all ranks): S[0..3] sums, S[4] max.
static int diagnostics(grace_ctx* h, double S[5]) {
  cudaStream_t s = h->stream;
  for (auto& rk : h->ranks) {
    if (!rk.Hd) {
      int rc = h->alloc((void**)&rk.Hd, sizeof(float) * 3 * (size_t)rk.Nl);
      if (rc) return rc;
    }
    if (!rk.dred) {
      int rc = h->alloc((void**)&rk.dred, sizeof(double) * (kDiagPartials + 8));
      if (rc) return rc;
    }
  }
  CUDA_OR(h->upload_params(1e-15, true));
  CUDA_OR(h->demag_stages(h->cur, s, false));
  CUDA_OR(h->k5_stage(s));
  CUDA_OR(h->halo_join(s));
  for (int q = 0; q < 4; ++q) S[q] = 0.0;
  S[4] = 0.0;
  for (auto& rk : h->ranks) {
    double* out = rk.dred + kDiagPartials;
    CUDA_OR(launch_diag(rk.g, rk.M[h->cur], rk.Hd, rk.prm, rk.Hlo, rk.Hhi, h->dx, h->dy, h->dz, rk.dred, out, s));
    if (h->mode == grace_ctx::kNccl) {
      ncclResult_t r = g_nccl.allReduce(out, out, 4, kNcclFloat64, kNcclSum, h->comm, s);
      if (r == 0) r = g_nccl.allReduce(out + 4, out + 4, 1, kNcclFloat64, kNcclMax, h->comm, s);
      if (r != 0) return fail(GRACE_ECUDA, "ncclAllReduce: %s", g_nccl.errStr(r));
    }
    double v[5];
    CUDA_OR(cudaMemcpyAsync(h->pin->red, out, sizeof v, cudaMemcpyDeviceToHost, s));
    CUDA_OR(cudaStreamSynchronize(s));
    std::memcpy(v, h->pin->red, sizeof v);
    for (int q = 0; q < 4; ++q) S[q] += v[q];
    S[4] = std::max(S[4], v[4]);
  }
  return GRACE_OK;
}

int grace_energy(grace_ctx* h, double* out5) {
  if (!h || !out5) return fail(GRACE_EINVAL, "NULL argument");
  double S[5];
  int rc = diagnostics(h, S);
  if (rc) return rc;
  const double V = (h->dx * h->dy) * h->dz, Ms2 = h->Ms * h->Ms, mu0 = 4e-7 * 3.14159265358979323846;
  out5[1] = V * h->A * S[0] / Ms2;      // exchange
  out5[2] = V * h->Ku * S[1] / Ms2;     // anisotropy Ku (1 - m_x^2)
  out5[3] = -0.5 * mu0 * V * S[2];      // demag
  out5[4] = -mu0 * V * S[3];            // Zeeman
  out5[0] = out5[1] + out5[2] + out5[3] + out5[4];
  return GRACE_OK;
}

int grace_max_torque(grace_ctx* h, double* out) {
  if (!h || !out) return fail(GRACE_EINVAL, "NULL argument");
  double S[5];
  int rc = diagnostics(h, S);
  if (rc) return rc;
  *out = S[4];
  return GRACE_OK;
}

int grace_relax(grace_ctx* h, double alpha_relax, double dt, long long max_steps, double tol, int check_every,
                long long* steps_taken, double* torque) {
  if (!h || !steps_taken || !torque) return fail(GRACE_EINVAL, "NULL argument");
  if (!(alpha_relax > 0) || !finite_pos(tol) || max_steps < 0 || check_every < 1)
    return fail(GRACE_EINVAL, "relax needs alpha_relax > 0, tol > 0, max_steps >= 0, check_every >= 1");
  const double alpha0 = h->alpha;
  h->alpha = alpha_relax;
  long long done = 0;
  double t = 0.0;
  int rc = grace_max_torque(h, &t);
  while (rc == GRACE_OK && t >= tol && done < max_steps) {
    const int k = (int)std::min<long long>(check_every, max_steps - done);
    rc = grace_step(h, k, dt);
    if (rc == GRACE_OK) {
      done += k;
      rc = grace_max_torque(h, &t);
    }
  }
  h->alpha = alpha0;
  *steps_taken = done;
  *torque = t;
  return rc;
}

int grace_step_count(grace_ctx* h, long long* steps) {
  if (!h || !steps) return fail(GRACE_EINVAL, "NULL argument");
  *steps = h->steps;
  return GRACE_OK;
}

int grace_last_nonfinite(grace_ctx* h, long long* step, long long* cell) {
  if (!h || !step || !cell) return fail(GRACE_EINVAL, "NULL argument");
  *step = h->nf_step;
  *cell = h->nf_cell;
  return GRACE_OK;
}

int grace_geometry(grace_ctx* h, long long* o) {
  if (!h || !o) return fail(GRACE_EINVAL, "NULL argument");
  const Geom& g = h->g0;
  const long long v[12] = {g.nx, g.ny, g.nz, g.Px, g.Py, g.Pz, g.Kx, g.Kxp, g.Kyh, g.Kzh, g.KSp, kernel_count(g)};
  std::memcpy(o, v, sizeof v);
  return GRACE_OK;
}

int grace_partition(grace_ctx* h, long long* o) {
  if (!h || !o) return fail(GRACE_EINVAL, "NULL argument");
  const Geom& g = h->ranks[0].g;
  const long long v[12] = {h->P,      h->ranks[0].r, g.nzl,    (long long)h->ranks[0].r * g.nzl,
                           g.kb,      g.Kc,          g.pitch1, g.pitch2,
                           h->pipe,   (h->mode == grace_ctx::kSingle || h->dist_graphs) ? 1 : 0,
                           h->comm_halo != nullptr, h->p2p};
  std::memcpy(o, v, sizeof v);
  return GRACE_OK;
}

int grace_device_bytes(grace_ctx* h, size_t* bytes) {
  if (!h || !bytes) return fail(GRACE_EINVAL, "NULL argument");
  *bytes = h->bytes;
  return GRACE_OK;
}

int grace_tensor_octant(int nx, int ny, int nz, double dx, double dy, double dz, double* out) {
  if (!out) return fail(GRACE_EINVAL, "NULL argument");
  if (nx < 1 || ny < 1 || nz < 1) return fail(GRACE_EINVAL, "cell counts must be >= 1");
  if (!finite_pos(dx) || !finite_pos(dy) || !finite_pos(dz)) return fail(GRACE_EINVAL, "cell sizes must be > 0");
  const size_t b = sizeof(double) * 6 * (size_t)nx * ny * nz;
  double* d = nullptr;
  if (cudaMalloc(&d, b) != cudaSuccess) {
    cudaGetLastError();
    return fail(GRACE_ENOMEM, "needs %zu bytes", b);
  }
  cudaError_t e = tensor_octant_device(nx, ny, nz, dx, dy, dz, d, 0);
  if (e == cudaSuccess) e = cudaMemcpy(out, d, b, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(GRACE_ECUDA, "tensor octant: %s", cudaGetErrorString(e));
  return GRACE_OK;
}

int grace_kernel_spectrum(grace_ctx* h, float* out) {
  if (!h || !out) return fail(GRACE_EINVAL, "NULL argument");
  if (h->P != 1) return fail(GRACE_EUNSUPPORTED, "kernel spectrum copy is single-rank only");
  const Geom& g = h->g0;
  CUDA_OR(cudaMemcpyAsync(out, h->ranks[0].KS, sizeof(float) * 6 * (size_t)g.Kzh * g.Kyh * g.KSp,
                          cudaMemcpyDeviceToHost, h->stream));
  CUDA_OR(cudaStreamSynchronize(h->stream));
  return GRACE_OK;
}

int grace_kernel_spectrum_f64(int nx, int ny, int nz, double dx, double dy, double dz, double* out) {
  if (!out) return fail(GRACE_EINVAL, "NULL argument");
  if (nx < 1 || ny < 1 || nz < 1) return fail(GRACE_EINVAL, "cell counts must be >= 1");
  if (!finite_pos(dx) || !finite_pos(dy) || !finite_pos(dz)) return fail(GRACE_EINVAL, "cell sizes must be > 0");
  Geom g{};
  int rc = make_geom(nx, ny, nz, dx, dy, dz, 1.0, 0.0, 0.0, &g);
  if (rc) return rc;
  const size_t n = (size_t)6 * g.Kzh * g.Kyh * g.KSp;
  double* d = nullptr;
  if (cudaMalloc(&d, sizeof(double) * n) != cudaSuccess) {
    cudaGetLastError();
    return fail(GRACE_ENOMEM, "needs %zu bytes", sizeof(double) * n);
  }
  KsOut o{nullptr, 0, g.Kx, g.KSp, d};
  size_t scratch = 0;
  cudaError_t e = kernel_spectrum_device(g, dx, dy, dz, 1, &o, &scratch, 0);
  if (e == cudaSuccess) e = cudaMemcpy(out, d, sizeof(double) * n, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return fail(GRACE_ECUDA, "kernel spectrum: %s", cudaGetErrorString(e));
  return GRACE_OK;
}

int grace_set_profiling(grace_ctx* h, int on) {
  if (!h) return fail(GRACE_EINVAL, "NULL context");
  h->profiling = on != 0;
  return GRACE_OK;
}

int grace_kernel_times(grace_ctx* h, double* ms, long long* launches, int* nk, int reset) {
  if (!h || !nk) return fail(GRACE_EINVAL, "NULL argument");
  const int k = kernel_count(h->g0);
  const int cap = *nk;
  *nk = k;
  for (int i = 0; i < k && i < cap; ++i) {
    if (ms) ms[i] = h->kms.empty() ? 0.0 : h->kms[i];
    if (launches) launches[i] = h->klaunch.empty() ? 0 : h->klaunch[i];
  }
  if (reset && !h->kms.empty()) {
    std::fill(h->kms.begin(), h->kms.end(), 0.0);
    std::fill(h->klaunch.begin(), h->klaunch.end(), 0);
  }
  return GRACE_OK;
}

}  // extern "C"
