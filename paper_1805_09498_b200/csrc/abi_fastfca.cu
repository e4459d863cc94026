// C-ABI: FastFCA-AS estimation loop (ffca_fastfca_run).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "ffca_loop.cuh"
#include "host_common.h"
#include "points.h"

namespace ffca {

using LoopFn = void (*)(const LoopArgs);
LoopFn loop_kernel_f32(int I, int J, int G, bool res, bool fast, bool tm);
LoopFn loop_kernel_f64(int I, int J, int G, bool res, bool fast);

static bool hot_shape(int I, int J) {
  return (I == 3 && J == 3) || (I == 4 && J == 4) || (I == 8 && J == 6) || (I == 2 && J == 2);
}

static int host_vmax(int I, int JM) {
  const int va = JM * (1 + I) + 1;
  if (I > 4) return va > I * I * I + 1 ? va : I * I * I + 1;  // group-mode phase B
  const int IC = (I * I * I <= 64) ? I : ((64 / (I * I)) > 0 ? (64 / (I * I)) : 1);
  const int NB = IC * I * I;
  return va > NB + 1 ? va : NB + 1;
}

struct LoopPlan {
  int G = 1, C = 1, NL = 0, threads = 64;
  bool resident = true;
  bool tm = false;  // y records in tensor memory (ffca_loop.cuh TM)
  size_t smem = 0, slab = 0;
  long long grid = 0;
  LoopSmem L;  // the carve-up the kernel reads from its parameters
};

// Slab budget per CTA: two CTAs per SM fit in the 228 KB shared memory.
static constexpr size_t kSlabBudget = 96 * 1024;

static int choose_threads(int G, int NL, int I) {
  const int per_bin = (NL + 3) / 4;  // ~4 frames per thread per pass (capped at 256 threads)
  int t = G * per_bin;
  t = (t + 31) / 32 * 32;
  const int tmin = I > 4 ? (8 * (loop_pgroup(I) + 1) + 31) / 32 * 32 : 64;  // I > 4: 8-lane solver groups
  if (t < tmin) t = tmin;
  // I >= 4 instantiations use up to 255 registers: 128-thread CTAs keep two per SM
  const int tmax = I >= 4 ? 128 : 256;
  if (t > tmax) t = tmax;
  return t;
}

static int plan_loop(int dtype, int I, int J, int N, long long total_bins, int vf_mode, LoopPlan& p,
                     size_t smem_optin, int nsm = 148, bool fast = false) {
  const int rsz = int(rsize(dtype));
  const int JM = hot_shape(I, J) ? J : 8;
  const int VMAX = host_vmax(I, JM);
  // lane-interleaved bin groups only for the exact-J instantiations
  const int G0 = (hot_shape(I, J) && I <= 4) ? (dtype == FFCA_C64 ? 4 : 2) : 1;
  auto fill = [&](int G, int C, bool res) {
    p.G = G;
    p.C = C;
    p.NL = (N + C - 1) / C;
    p.threads = choose_threads(G, p.NL, I);
    p.resident = res;
    LoopSmem L(I, J, JM, G, p.NL, p.threads / 32, rsz, vf_mode, res, VMAX);
    p.L = L;
    p.smem = L.total;
    p.slab = L.slab;
    p.grid = ((total_bins + G - 1) / G) * C;
  };
  // Test hook: FFCA_FORCE_PLAN="G,C,resident" pins the launch plan (parity tests
  // use it to exercise the cluster and global-slab paths at small sizes).
  if (const char* fp = getenv("FFCA_FORCE_PLAN")) {
    int G = 1, C = 1, res = 1, thr = 0;
    const int nf = sscanf(fp, "%d,%d,%d,%d", &G, &C, &res, &thr);
    if (nf >= 3 && (G == 1 || G == G0 || (G == 2 && G0 == 4)) && (G == 1 || res) && C >= 1 && C <= 16 && (C & (C - 1)) == 0 && C <= N &&
        (C == 1 || G == 1)) {
      fill(G, C, res != 0);
      if (nf == 4 && thr >= 64 && thr <= 256 && thr % 32 == 0 && (I <= 4 || thr >= 8 * (loop_pgroup(I) + 1))) {
        p.threads = thr;
        LoopSmem L(I, J, JM, G, p.NL, thr / 32, rsz, vf_mode, res != 0, VMAX);
        p.L = L;
        p.smem = L.total;
      }
      if (p.smem <= smem_optin) return FFCA_OK;
    }
  }
  // complex128: one bin per 128-thread CTA spreads the bins over more SMs (four such CTAs fit an
  // SM).  Measured: config 0 (513 bins)
  // kernel 0.203 -> 0.197 ms; for complex64 the 4-bin CTAs stay faster (one config-3 mixture
  // 0.109 vs 0.113 ms, two 0.161 vs 0.195 ms), so complex64 keeps G0.
  // The one-bin CTA has half the threads of the G0 = 2 plan -- the same frame slots -- and reduces
  // over 16-lane segments (ffca_loop.cuh bin_reduce), so both plans give bitwise the same bins:
  // results do not depend on the batch size, the host pipeline's chunking or the shard a bin is in.
  // Measured on the batched config-3 shape in complex128 as well (256 mixtures): 34.1 ms vs 35.4 ms
  // for the 2-bin / 256-thread CTAs, so the one-bin CTAs are used at every batch size.
  if (dtype == FFCA_C128 && G0 == 2 && I <= 4) {
    fill(G0, 1, true);
    const int t2 = p.threads;
    const bool fits2 = p.slab <= kSlabBudget && p.smem <= smem_optin;
    if (fits2 && t2 >= 128) {
      fill(1, 1, true);
      p.threads = (t2 / 2 + 31) / 32 * 32;  // whole warps (t2 = 160 ... 224 for 130 <= N <= 448 halves to 80 ... 112)
      LoopSmem L(I, J, JM, 1, p.NL, p.threads / 32, rsz, vf_mode, true, VMAX);
      p.L = L;
      p.smem = L.total;
      if (p.slab <= kSlabBudget && p.smem <= smem_optin) return FFCA_OK;
    }
  }
  // complex64, I = J = 3, N <= 640: 4-bin CTAs of 128 threads (32 per bin, 10 frame pairs
  // per thread) with the y records in tensor memory -- 16 bins per SM instead of the 8 that shared
  // memory alone holds, at the same 16 warps.
  // Worth it from one full wave of 16 bins per SM on (measured on B200, config-3 shape: 1 / 2 / 4 / 8
  // mixtures 0.129 / 0.165 / 0.253 / 0.431 ms against 0.098 / 0.154 / 0.249 / 0.473 ms for the 2-bin
  // shared-memory plan); FFCA_TMEM_MIN_BINS overrides the threshold (tests use 0).
  long long tm_min_bins = 16LL * nsm;
  if (const char* e = getenv("FFCA_TMEM_MIN_BINS")) tm_min_bins = atoll(e);
  // (the loop with the likelihood record / inner iterations runs the same plan: 24.3 -> 22.5 ms at the
  // config-3 scale with the likelihood recorded; only a full floor array needs the shared-memory plans)
  if (dtype == FFCA_C64 && I == 3 && J == 3 && G0 == 4 && vf_mode != 2 && N <= 640 && total_bins >= tm_min_bins &&
      !getenv("FFCA_NO_TMEM")) {
    fill(4, 1, true);
    p.threads = 128;
    p.tm = true;
    LoopSmem L(I, J, JM, 4, p.NL, 4, rsz, vf_mode, true, VMAX, true);
    p.L = L;
    p.smem = L.total;
    p.slab = L.slab;
    if (p.smem <= smem_optin) return FFCA_OK;
    p.tm = false;
  }
  // complex64, I = J = 3: 2-bin CTAs of 128 threads (64 per bin, as in the 4-bin / 256-thread
  // CTAs) -- four CTAs per SM instead of two overlap each other's reductions and solves better.
  // Measured at config 3: 15.55 ms vs 16.12 (G = 4 / 256), 16.69 (4 / 128), 21.8 (2 / 256).
  if (dtype == FFCA_C64 && I == 3 && J == 3 && G0 == 4) {
    fill(2, 1, true);
    p.threads = 128;
    LoopSmem L(I, J, JM, 2, p.NL, 4, rsz, vf_mode, true, VMAX);
    p.L = L;
    p.smem = L.total;
    if (p.slab <= kSlabBudget && p.smem <= smem_optin) return FFCA_OK;
  }
  for (int G : {G0, 1}) {
    fill(G, 1, true);
    if (p.slab <= kSlabBudget && p.smem <= smem_optin) return FFCA_OK;
  }
  // I > 4: 256-thread CTAs (8-lane point groups in phase B).  A bin whose interleaved slab
  // fits the shared memory of one CTA or of a CTA pair / quad stays resident (one CTA per SM);
  // larger clusters leave too few frames per CTA against the I^3-value reductions and solves,
  // so longer bins stream their slab from L2-resident global scratch instead.
  if (I > 4) {
    auto fill256 = [&](int C, bool res) {
      fill(1, C, res);
      p.threads = 256;  // measured: 384 threads at a 168-register cap were slower (15.8 vs 15.2 ms)
      LoopSmem L(I, J, JM, 1, p.NL, p.threads / 32, rsz, vf_mode, res, VMAX);
      p.L = L;
      p.smem = L.total;
      p.slab = L.slab;
    };
    for (int C = 1; C <= 4 && C <= N; C <<= 1) {
      fill256(C, true);
      if (p.smem <= smem_optin) return FFCA_OK;
    }
    fill256(1, false);
    if (p.smem <= smem_optin) return FFCA_OK;
  }
  for (int C = 2; C <= 8; C <<= 1) {
    if (C > N) break;
    // complex64, I = J = 4, lean loop: with the y records in tensor memory (256 columns per CTA, two
    // CTAs per SM) a CTA holds up to 4096 frames, so a long bin needs a smaller cluster than shared
    // memory alone allows (config 2: 4 CTAs per bin instead of 8 -- half the DSMEM reduction ranks)
    if (dtype == FFCA_C64 && I == 4 && J == 4 && hot_shape(I, J) && fast && vf_mode != 2 && !getenv("FFCA_NO_TMEM")) {
      const int NLc = (N + C - 1) / C;
      const int nrec = ((NLc + 1) / 2 + 127) / 128;
      if (nrec * 16 <= 256) {
        fill(1, C, true);
        p.threads = 128;
        p.tm = true;
        LoopSmem L(I, J, JM, 1, p.NL, 4, rsz, vf_mode, true, VMAX, true);
        p.L = L;
        p.smem = L.total;
        p.slab = L.slab;
        if (p.slab <= kSlabBudget && p.smem <= smem_optin) return FFCA_OK;
        p.tm = false;
      }
    }
    fill(1, C, true);
    if (p.slab <= kSlabBudget && p.smem <= smem_optin) return FFCA_OK;
  }
  fill(1, 1, false);  // too long for the cluster: stream the slab from global scratch
  if (p.smem > smem_optin) {
    set_error("problem too large: %zu B shared memory needed", p.smem);
    return FFCA_E_UNSUPPORTED;
  }
  return FFCA_OK;
}

// Per-device attributes and per-kernel shared-memory opt-ins, set once (the calls cost a few
// microseconds each -- 10-20 % of a config-0 call).
struct DevAttrs {
  int optin = 0, nsm = 0;
};
static int device_attrs(int device, DevAttrs& out) {
  static std::mutex mu;
  static DevAttrs cache[64];
  std::lock_guard<std::mutex> lk(mu);
  if (device < 0 || device >= 64) return FFCA_E_ARG;
  if (cache[device].nsm == 0) {
    FFCA_CK(cudaDeviceGetAttribute(&cache[device].optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    FFCA_CK(cudaDeviceGetAttribute(&cache[device].nsm, cudaDevAttrMultiProcessorCount, device));
  }
  out = cache[device];
  return FFCA_OK;
}
static int func_smem_optin(LoopFn fn, int device, size_t smem, bool nonportable) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;  // (kernel, device) -> opted-in bytes
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[{(const void*)fn, device}];
  if (smem > have) {
    FFCA_CK(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    have = smem;
  }
  if (nonportable) FFCA_CK(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  return FFCA_OK;
}

static int launch_loop(LoopFn fn, const LoopPlan& p, const LoopArgs& a, cudaStream_t s, int device) {
  FFCA_TRY(func_smem_optin(fn, device, p.smem, p.C > 8));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(p.grid), 1, 1);
  cfg.blockDim = dim3(unsigned(p.threads), 1, 1);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  if (p.C > 1) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(p.C);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  FFCA_CK(cudaLaunchKernelEx(&cfg, fn, a));
  count_launch();
  return FFCA_OK;
}

}  // namespace ffca

using namespace ffca;

// One (sub)problem with all arrays already on the device: plan, launch, optional timing.
struct DevProblem {
  int dtype, U, I, J, N, F;
  int vf_mode;
  double vf_scalar;
  int iters, K, p_only;
  const void *y, *P0, *lam0, *v0, *vf;
  void *P, *lam, *v;
  double* vf_out;
  double* ll_bins;  // (U*F, nev) or null
  int* status;      // (U*F)
  void *mu, *phi;   // optional: statistics refresh at the final state (U,J,N,F,I), fastfca.py:373-387
};

static int launch_problem(int device, const DevProblem& d, cudaStream_t s) {
  const long long nb = (long long)d.U * d.F;
  if (nb == 0) return FFCA_OK;
  DevAttrs da;
  FFCA_TRY(device_attrs(device, da));
  // the plain loop (no likelihood, no full floor array, no P-only pass, K = 1) has lean instantiations
  const bool fast = d.ll_bins == nullptr && d.vf_mode != 2 && !d.p_only && d.K == 1 && !getenv("FFCA_NO_FAST");
  LoopPlan p;
  FFCA_TRY(plan_loop(d.dtype, d.I, d.J, d.N, nb, d.vf_mode, p, size_t(da.optin), da.nsm, fast));
  void* scratch = nullptr;
  if (!p.resident) FFCA_CK(cudaMallocAsync(&scratch, size_t(p.grid) * p.slab, s));
  LoopArgs a;
  a.U = d.U; a.I = d.I; a.J = d.J; a.N = d.N; a.F = d.F;
  a.total_bins = nb;
  a.G = p.G; a.C = p.C; a.NL = p.NL;
  a.iters = d.iters; a.K = d.K; a.p_only = d.p_only;
  a.vf_mode = d.vf_mode; a.vf_scalar = d.vf_scalar; a.vf = d.vf;
  a.y = d.y; a.P_in = d.P0; a.lam_in = d.lam0; a.v_in = d.v0;
  a.P_out = d.P; a.lam_out = d.lam; a.v_out = d.v;
  a.vf_out = d.vf_out;
  a.ll = d.ll_bins;
  a.status = d.status;
  a.scratch = scratch;
  a.slab_bytes = (long long)p.slab;
  a.packed = nullptr;
  a.L = p.L;
  LoopFn fn = d.dtype == FFCA_C64 ? loop_kernel_f32(d.I, d.J, p.G, p.resident, fast, p.tm)
                                  : loop_kernel_f64(d.I, d.J, p.G, p.resident, fast);
  if (!fn) {
    set_error("no kernel for I=%d J=%d", d.I, d.J);
    return FFCA_E_UNSUPPORTED;
  }
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (timing_enabled()) {
    FFCA_CK(cudaEventCreate(&ev0));
    FFCA_CK(cudaEventCreate(&ev1));
    FFCA_CK(cudaEventRecord(ev0, s));
  }
  // Resident slabs are filled from contiguous images (one bulk-copy stream per CTA) that a
  // coalesced pack pass writes first: the bins-fastest reference layout otherwise costs one
  // 4-16 byte request per element and frame (odd F rules out wider vector copies).
  void* packed = nullptr;
  // Measured: worth it for the one-CTA-per-SM I > 4 plans (config 4: gather 125k -> 6k cycles per
  // CTA, 15.7 -> 15.2 ms), where nothing else on the SM hides the element gather; with two or more
  // CTAs per SM the extra pass over HBM costs more than it saves (config 3: 16.8 -> 17.2 ms,
  // config 2: 8.0 -> 8.2 ms).  FFCA_FORCE_PACK=1 enables it for every resident plan (tests).
  const bool pack_plan = p.G == 1 && loop_interleaved(d.I);
  if (p.resident && d.vf_mode != 2 && !getenv("FFCA_NO_PACK") && (pack_plan || getenv("FFCA_FORCE_PACK"))) {
    FFCA_CK(cudaMallocAsync(&packed, size_t(p.grid) * p.slab, s));
    PackArgs pa;
    pa.y = d.y; pa.v = d.v0; pa.packed = packed;
    pa.I = d.I; pa.J = d.J; pa.N = d.N; pa.F = d.F; pa.G = p.G; pa.C = p.C;
    const int JM = hot_shape(d.I, d.J) ? d.J : 8;
    pa.RS = loop_rs(d.I, JM);
    pa.JS = loop_js(d.I, JM, d.J);
    pa.ilv = loop_interleaved(d.I) ? 1 : 0;
    pa.pairs = loop_pairs(d.I, int(rsize(d.dtype))) ? 1 : 0;
    pa.total_bins = nb;
    pa.ngroups = (nb + p.G - 1) / p.G;
    pa.slab_bytes = (long long)p.slab;
    pa.Ly = (long long)p.L.y;
    pa.Lv = (long long)p.L.v;
    const size_t per_frame = 32 * (size_t(d.I) * 2 * rsize(d.dtype) + size_t(d.J) * rsize(d.dtype));
    int FT = 32;
    while (FT > 4 && FT * per_frame > 40 * 1024) FT >>= 1;
    pa.FT = FT;
    const size_t psm = FT * per_frame;
    dim3 grid(unsigned((nb + 31) / 32), unsigned((d.N + FT - 1) / FT));
    if (d.dtype == FFCA_C64) slab_pack_kernel<float><<<grid, 256, psm, s>>>(pa);
    else slab_pack_kernel<double><<<grid, 256, psm, s>>>(pa);
    FFCA_CK(cudaGetLastError());
    count_launch();
    a.packed = packed;
  }
  FFCA_TRY(launch_loop(fn, p, a, s, device));
  FFCA_CK(cudaGetLastError());
  if (ev0) {
    FFCA_CK(cudaEventRecord(ev1, s));
    FFCA_CK(cudaEventSynchronize(ev1));
    float ms = 0.f;
    FFCA_CK(cudaEventElapsedTime(&ms, ev0, ev1));
    set_kernel_ms(ms);
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
  }
  if (scratch) FFCA_CK(cudaFreeAsync(scratch, s));
  if (packed) FFCA_CK(cudaFreeAsync(packed, s));
  if (d.mu || d.phi) {
    // run_fastfca's _stats_refresh (fastfca.py:466, 373-387) on the loop's final state, from the
    // device copies of y and (P, lambda, v) this call already holds
    PointArgs pa = {};
    pa.mode = PM_STATS; pa.U = d.U; pa.I = d.I; pa.J = d.J; pa.N = d.N; pa.F = d.F;
    pa.y = d.y; pa.P = d.P; pa.lam = d.lam; pa.v = d.v;
    pa.out0 = d.mu; pa.out1 = d.phi;
    FFCA_TRY(launch_points(d.dtype, pa, s));
  }
  return FFCA_OK;
}

// Array of layout (U, A, F, B) (elements of `es` bytes): the block of mixtures
// [u0, u0+Uc) x bins [f0, f0+Fc) is Uc*A rows of Fc*B*es bytes at pitch F*B*es.
struct Blk {
  size_t A, B, es;
};

static int copy_blk(void* dst, const void* src, const Blk& b, int U, int F, int u0, int Uc, int f0, int Fc,
                    bool h2d, cudaStream_t s, bool d2d = false) {
  if (!dst || !src) return FFCA_OK;
  const cudaMemcpyKind out_kind = d2d ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  const size_t pitch_full = size_t(F) * b.B * b.es, width = size_t(Fc) * b.B * b.es;
  const size_t off = ((size_t(u0) * b.A) * F + f0) * b.B * b.es;
  if (width == pitch_full) {  // whole rows: one linear copy
    const size_t n = width * size_t(Uc) * b.A;
    if (h2d)
      FFCA_CK(cudaMemcpyAsync(dst, (const char*)src + off, n, cudaMemcpyHostToDevice, s));
    else
      FFCA_CK(cudaMemcpyAsync((char*)dst + off, src, n, out_kind, s));
    return FFCA_OK;
  }
  if (h2d)
    FFCA_CK(cudaMemcpy2DAsync(dst, width, (const char*)src + off, pitch_full, width, size_t(Uc) * b.A,
                              cudaMemcpyHostToDevice, s));
  else
    FFCA_CK(cudaMemcpy2DAsync((char*)dst + off, pitch_full, src, width, width, size_t(Uc) * b.A, out_kind, s));
  (void)U;
  return FFCA_OK;
}

// Host-mode call split into chunks so that H2D of chunk c+1, the kernel of
// chunk c and the D2H of chunk c-1 overlap (three internal streams, two
// device buffer sets).  Chunks are mixture blocks (U > 1) or frequency
// blocks of a single mixture; bins are independent, so the results are
// bitwise those of one launch.
// Streams, events and device buffers of one pipelined call: created by the body, released by
// pipelined_host_run on every path (success or any failure inside the body).
struct PipeRes {
  cudaStream_t sin = nullptr, scomp = nullptr, sout = nullptr;
  cudaEvent_t start = nullptr, ev_in[2] = {nullptr, nullptr}, ev_k[2] = {nullptr, nullptr},
              ev_out[2] = {nullptr, nullptr};
  std::vector<void*> allocs;
};

static int pipelined_body(PipeRes& R, int device, cudaStream_t user, const DevProblem& proto, bool rec, int nchunk,
                          bool by_mixture, bool stats_dev,
                          const void* y, const void* P0, const void* lam0, const void* v0, const void* vf,
                          void* P_out, void* lam_out, void* v_out, double* ll_out, double* vf_out,
                          int* status_out, void* mu_out, void* phi_out) {
  const int U = proto.U, I = proto.I, J = proto.J, N = proto.N, F = proto.F;
  const size_t rs = rsize(proto.dtype), cs = csize(proto.dtype);
  const long long nb = (long long)U * F;
  const int nev = 1 + 2 * proto.iters;
  const Blk By{size_t(I) * N, 1, cs}, BP{1, size_t(I) * I, cs}, Bl{size_t(J), size_t(I), rs},
      Bv{size_t(J) * N, 1, rs}, Bvb{1, 1, rs}, Bvo{1, 1, 8}, Bst{1, 1, 4}, Bll{1, size_t(nev), 8},
      Bmu{size_t(J) * N, size_t(I), cs}, Bphi{size_t(J) * N, size_t(I), rs};
  const int cu = by_mixture ? (U + nchunk - 1) / nchunk : 1;
  const int cf = by_mixture ? F : (F + nchunk - 1) / nchunk;
  auto bytes = [&](const Blk& b) { return size_t(cu) * b.A * cf * b.B * b.es; };

  FFCA_CK(cudaStreamCreateWithFlags(&R.sin, cudaStreamNonBlocking));
  FFCA_CK(cudaStreamCreateWithFlags(&R.scomp, cudaStreamNonBlocking));
  FFCA_CK(cudaStreamCreateWithFlags(&R.sout, cudaStreamNonBlocking));
  cudaStream_t sin = R.sin, scomp = R.scomp, sout = R.sout;
  FFCA_CK(cudaEventCreateWithFlags(&R.start, cudaEventDisableTiming));
  FFCA_CK(cudaEventRecord(R.start, user));  // order after prior work on the caller's stream
  FFCA_CK(cudaStreamWaitEvent(sin, R.start, 0));
  cudaEvent_t *ev_in = R.ev_in, *ev_k = R.ev_k, *ev_out = R.ev_out;
  for (int k = 0; k < 2; ++k) {
    FFCA_CK(cudaEventCreateWithFlags(&ev_in[k], cudaEventDisableTiming));
    FFCA_CK(cudaEventCreateWithFlags(&ev_k[k], cudaEventDisableTiming));
    FFCA_CK(cudaEventCreateWithFlags(&ev_out[k], cudaEventDisableTiming));
  }
  // device buffers: two slots of chunk inputs/outputs + full status / ll
  auto dalloc = [&](size_t n, void** p) -> int {
    *p = nullptr;
    if (n == 0) return FFCA_OK;
    FFCA_CK(cudaMallocAsync(p, n, sin));
    R.allocs.push_back(*p);
    return FFCA_OK;
  };
  void *dy[2], *dP0[2], *dl0[2], *dv0[2], *dvf[2] = {nullptr, nullptr}, *dP[2], *dl[2], *dv[2], *dvo[2] = {nullptr, nullptr},
       *dst[2], *dll[2] = {nullptr, nullptr}, *dmu[2] = {nullptr, nullptr}, *dphi[2] = {nullptr, nullptr};
  int rc = FFCA_OK;
  void *fstatus = nullptr, *fll = nullptr, *llmix = nullptr;
  if (!rc) rc = dalloc(size_t(nb) * 4, &fstatus);
  if (!rc && rec) rc = dalloc(size_t(nb) * nev * 8, &fll);
  if (!rc && rec && ll_out) rc = dalloc(size_t(U) * nev * 8, &llmix);
  // Mixture chunks: the small per-bin arrays (P, lambda in and out, status, likelihood parts)
  // are whole-batch device buffers moved with one copy each; only y / v (in) and v (out) move per
  // chunk (each copy costs ~0.15 ms of fixed DMA / API overhead at ~23 chunks per call).
  void *fP0 = nullptr, *fl0 = nullptr, *fP = nullptr, *fl = nullptr;
  const size_t nP = size_t(nb) * I * I * cs, nl = size_t(U) * J * F * I * rs;
  if (by_mixture && !rc) {
    rc = dalloc(nP, &fP0);
    if (!rc) rc = dalloc(nl, &fl0);
    if (!rc) rc = dalloc(nP, &fP);
    if (!rc) rc = dalloc(nl, &fl);
    if (!rc) FFCA_CK(cudaMemcpyAsync(fP0, P0, nP, cudaMemcpyHostToDevice, sin));
    if (!rc) FFCA_CK(cudaMemcpyAsync(fl0, lam0, nl, cudaMemcpyHostToDevice, sin));
    if (!rc) FFCA_CK(cudaMemsetAsync(fstatus, 0, size_t(nb) * 4, sin));
  }
  for (int k = 0; k < 2 && rc == FFCA_OK; ++k) {
    rc = dalloc(bytes(By), &dy[k]);
    if (!rc && !by_mixture) rc = dalloc(bytes(BP), &dP0[k]);
    if (!rc && !by_mixture) rc = dalloc(bytes(Bl), &dl0[k]);
    if (!rc) rc = dalloc(bytes(Bv), &dv0[k]);
    if (!rc && proto.vf_mode == 1) rc = dalloc(bytes(Bvb), &dvf[k]);
    if (!rc && proto.vf_mode == 2) rc = dalloc(bytes(Bv), &dvf[k]);
    if (!rc && !by_mixture) rc = dalloc(bytes(BP), &dP[k]);
    if (!rc && !by_mixture) rc = dalloc(bytes(Bl), &dl[k]);
    if (!rc) rc = dalloc(bytes(Bv), &dv[k]);
    if (!rc && vf_out) rc = dalloc(bytes(Bvo), &dvo[k]);
    if (!rc && !by_mixture) rc = dalloc(bytes(Bst), &dst[k]);
    if (!rc && rec && !by_mixture) rc = dalloc(bytes(Bll), &dll[k]);
    // device-resident statistics of mixture chunks are written in place (no chunk buffers)
    if (!rc && mu_out && !(stats_dev && by_mixture)) rc = dalloc(bytes(Bmu), &dmu[k]);
    if (!rc && phi_out && !(stats_dev && by_mixture)) rc = dalloc(bytes(Bphi), &dphi[k]);
  }
  int nch = 0;
  for (int c0 = 0; !rc && c0 < (by_mixture ? U : F); c0 += (by_mixture ? cu : cf), ++nch) {
    const int k = nch & 1;
    const int u0 = by_mixture ? c0 : 0, Uc = by_mixture ? std::min(cu, U - c0) : 1;
    const int f0 = by_mixture ? 0 : c0, Fc = by_mixture ? F : std::min(cf, F - c0);
    // slot k free again once chunk nch-2's kernel consumed its inputs / D2H drained its outputs
    if (nch >= 2) {
      rc = cudaStreamWaitEvent(sin, ev_k[k], 0) == cudaSuccess ? FFCA_OK : FFCA_E_CUDA;
      if (!rc) rc = cudaStreamWaitEvent(scomp, ev_out[k], 0) == cudaSuccess ? FFCA_OK : FFCA_E_CUDA;
    }
    if (!rc) rc = copy_blk(dy[k], y, By, U, F, u0, Uc, f0, Fc, true, sin);
    if (!rc && !by_mixture) rc = copy_blk(dP0[k], P0, BP, U, F, u0, Uc, f0, Fc, true, sin);
    if (!rc && !by_mixture) rc = copy_blk(dl0[k], lam0, Bl, U, F, u0, Uc, f0, Fc, true, sin);
    if (!rc) rc = copy_blk(dv0[k], v0, Bv, U, F, u0, Uc, f0, Fc, true, sin);
    if (!rc && proto.vf_mode == 1) rc = copy_blk(dvf[k], vf, Bvb, U, F, u0, Uc, f0, Fc, true, sin);
    if (!rc && proto.vf_mode == 2) rc = copy_blk(dvf[k], vf, Bv, U, F, u0, Uc, f0, Fc, true, sin);
    if (rc) break;
    FFCA_CK(cudaEventRecord(ev_in[k], sin));
    FFCA_CK(cudaStreamWaitEvent(scomp, ev_in[k], 0));
    DevProblem d = proto;
    d.U = Uc;
    d.F = Fc;
    d.y = dy[k]; d.v0 = dv0[k]; d.vf = dvf[k];
    d.v = dv[k]; d.vf_out = (double*)dvo[k];
    d.mu = dmu[k]; d.phi = dphi[k];
    if (by_mixture) {  // views into the whole-batch buffers (mixture blocks are contiguous)
      const size_t b0 = size_t(u0) * F;
      if (stats_dev) {
        d.mu = mu_out ? (char*)mu_out + size_t(u0) * J * N * F * I * cs : nullptr;
        d.phi = phi_out ? (char*)phi_out + size_t(u0) * J * N * F * I * rs : nullptr;
      }
      d.P0 = (const char*)fP0 + b0 * I * I * cs;
      d.lam0 = (const char*)fl0 + size_t(u0) * J * F * I * rs;
      d.P = (char*)fP + b0 * I * I * cs;
      d.lam = (char*)fl + size_t(u0) * J * F * I * rs;
      d.status = (int*)fstatus + b0;
      d.ll_bins = rec ? (double*)fll + b0 * nev : nullptr;
    } else {
      FFCA_CK(cudaMemsetAsync(dst[k], 0, size_t(Uc) * Fc * 4, scomp));
      d.P0 = dP0[k]; d.lam0 = dl0[k];
      d.P = dP[k]; d.lam = dl[k];
      d.ll_bins = (double*)dll[k];
      d.status = (int*)dst[k];
    }
    rc = launch_problem(device, d, scomp);
    if (rc) break;
    if (!by_mixture) {
      // scatter the per-bin status / likelihood parts into the full-size buffers
      FFCA_CK(cudaMemcpy2DAsync((char*)fstatus + (size_t(u0) * F + f0) * 4, size_t(F) * 4, dst[k], size_t(Fc) * 4,
                                size_t(Fc) * 4, size_t(Uc), cudaMemcpyDeviceToDevice, scomp));
      if (rec)
        FFCA_CK(cudaMemcpy2DAsync((char*)fll + (size_t(u0) * F + f0) * nev * 8, size_t(F) * nev * 8, dll[k],
                                  size_t(Fc) * nev * 8, size_t(Fc) * nev * 8, size_t(Uc), cudaMemcpyDeviceToDevice,
                                  scomp));
    }
    FFCA_CK(cudaEventRecord(ev_k[k], scomp));
    FFCA_CK(cudaStreamWaitEvent(sout, ev_k[k], 0));
    if (!by_mixture) {
      rc = copy_blk(P_out, dP[k], BP, U, F, u0, Uc, f0, Fc, false, sout);
      if (!rc) rc = copy_blk(lam_out, dl[k], Bl, U, F, u0, Uc, f0, Fc, false, sout);
    }
    if (!rc) rc = copy_blk(v_out, dv[k], Bv, U, F, u0, Uc, f0, Fc, false, sout);
    if (!rc && vf_out) rc = copy_blk(vf_out, dvo[k], Bvo, U, F, u0, Uc, f0, Fc, false, sout);
    if (!(stats_dev && by_mixture)) {
      if (!rc && mu_out) rc = copy_blk(mu_out, dmu[k], Bmu, U, F, u0, Uc, f0, Fc, false, sout, stats_dev);
      if (!rc && phi_out) rc = copy_blk(phi_out, dphi[k], Bphi, U, F, u0, Uc, f0, Fc, false, sout, stats_dev);
    }
    if (!rc) FFCA_CK(cudaEventRecord(ev_out[k], sout));
  }
  if (!rc && by_mixture) {  // the whole-batch P / lambda after the last kernel
    FFCA_CK(cudaMemcpyAsync(P_out, fP, nP, cudaMemcpyDeviceToHost, scomp));
    FFCA_CK(cudaMemcpyAsync(lam_out, fl, nl, cudaMemcpyDeviceToHost, scomp));
  }
  if (!rc) {
    FFCA_CK(cudaStreamSynchronize(scomp));
    if (rec && ll_out) {
      rc = reduce_ll((const double*)fll, (double*)llmix, U, F, nev, -double(N) * F * I * std::log(M_PI), scomp);
      if (!rc) FFCA_CK(cudaMemcpyAsync(ll_out, llmix, size_t(U) * nev * 8, cudaMemcpyDeviceToHost, scomp));
    }
    FFCA_CK(cudaStreamSynchronize(sout));
    if (!rc) rc = finish_status((const int*)fstatus, status_out, nb, FFCA_MEM_HOST, scomp,
                                FFCA_ST_SINGULAR_P | FFCA_ST_SINGULAR_B);
  }
  return rc;
}

static int pipelined_host_run(int device, cudaStream_t user, const DevProblem& proto, bool rec, int nchunk,
                              bool by_mixture, bool stats_dev,
                              const void* y, const void* P0, const void* lam0, const void* v0, const void* vf,
                              void* P_out, void* lam_out, void* v_out, double* ll_out, double* vf_out,
                              int* status_out, void* mu_out, void* phi_out) {
  PipeRes R;
  const int rc = pipelined_body(R, device, user, proto, rec, nchunk, by_mixture, stats_dev, y, P0, lam0, v0, vf, P_out,
                                lam_out, v_out, ll_out, vf_out, status_out, mu_out, phi_out);
  // Every path ends here.  Drain all three streams first: after a failure, H2D copies on sin and
  // D2H copies on sout may still be reading / writing the caller's host buffers and the device
  // buffers freed below.
  for (cudaStream_t q : {R.sin, R.scomp, R.sout})
    if (q) cudaStreamSynchronize(q);
  for (void* q : R.allocs) cudaFreeAsync(q, R.scomp);
  if (R.scomp) cudaStreamSynchronize(R.scomp);
  for (int k = 0; k < 2; ++k)
    for (cudaEvent_t e : {R.ev_in[k], R.ev_k[k], R.ev_out[k]})
      if (e) cudaEventDestroy(e);
  if (R.start) cudaEventDestroy(R.start);
  for (cudaStream_t q : {R.sin, R.scomp, R.sout})
    if (q) cudaStreamDestroy(q);
  if (rc != FFCA_OK) cudaGetLastError();  // the error is reported through rc / ffca_last_error
  return rc;
}

static int loop_entry(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                      const void* y, const void* P0, const void* lam0, const void* v0, int vf_mode,
                      double vf_scalar, const void* vf, int iterations, int inner_iterations,
                      int record_likelihood, void* P_out, void* lam_out, void* v_out, double* ll_out,
                      double* vf_out, int* status, int p_only, void* mu_out = nullptr,
                      void* phi_out = nullptr) {
  reset_launches();
  // FFCA_MEM_HOST_STATS_DEVICE: host arrays, except the statistics, which stay on the device
  const bool stats_dev = mem == FFCA_MEM_HOST_STATS_DEVICE;
  if (stats_dev) mem = FFCA_MEM_HOST;
  if (mem != FFCA_MEM_HOST && mem != FFCA_MEM_DEVICE) {
    set_error("bad mem mode %d", mem);
    return FFCA_E_ARG;
  }
  if (!check_dims(dtype, U, I, J, N, F)) return FFCA_E_ARG;
  if (I > 8 || J > 8) {
    set_error("unsupported order I=%d / sources J=%d (I <= 8 = matcore.MAX_ORDER, J <= 8)", I, J);
    return FFCA_E_UNSUPPORTED;
  }
  if (iterations < 0 || inner_iterations < 1 || vf_mode < 0 || vf_mode > 3) {
    set_error("bad iterations=%d inner_iterations=%d vf_mode=%d", iterations, inner_iterations, vf_mode);
    return FFCA_E_ARG;
  }
  if (!y || !P0 || !lam0 || !v0 || !P_out || !lam_out || !v_out || ((vf_mode == 1 || vf_mode == 2) && !vf)) {
    set_error("null array argument");
    return FFCA_E_ARG;
  }
  DeviceGuard dg(device);
  if (!dg.ok) {
    set_error("cannot select device %d", device);
    return FFCA_E_CUDA;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const long long nb = (long long)U * F;
  const size_t rs = rsize(dtype), cs = csize(dtype);
  const int nev = 1 + 2 * iterations;
  if (nb == 0) return FFCA_OK;

  DevProblem d = {};
  d.dtype = dtype; d.U = U; d.I = I; d.J = J; d.N = N; d.F = F;
  d.vf_mode = vf_mode; d.vf_scalar = vf_scalar;
  d.iters = iterations; d.K = inner_iterations; d.p_only = p_only;

  // host mode with a large input: pipeline H2D / compute / D2H over chunks
  const size_t in_bytes = size_t(U) * I * N * F * cs + size_t(U) * J * N * F * rs +
                          (mu_out && !stats_dev ? size_t(U) * J * N * F * I * cs : 0) +
                          (phi_out && !stats_dev ? size_t(U) * J * N * F * I * rs : 0);
  // FFCA_NO_PIPELINE=1 disables, FFCA_PIPELINE_MIN_BYTES overrides the threshold (tests)
  const char* nopipe = getenv("FFCA_NO_PIPELINE");
  const char* minb = getenv("FFCA_PIPELINE_MIN_BYTES");
  const size_t threshold = minb ? size_t(atoll(minb)) : (size_t(64) << 20);
  if (mem == FFCA_MEM_HOST && in_bytes >= threshold && !(nopipe && nopipe[0] == '1')) {
    const bool by_mix = U >= 2;
    // chunks of ~128 MB of input (>= 2, <= 32): short enough that the pipeline's fill and
    // drain (first H2D, last kernel + D2H) are a small part of the PCIe-bound whole
    const char* nch_env = getenv("FFCA_PIPELINE_CHUNKS");
    int want = nch_env ? atoi(nch_env) : int(std::min<size_t>(32, std::max<size_t>(2, in_bytes >> 27)));
    const int nchunk = by_mix ? std::min(U, want) : std::min(F, want);
    if (nchunk >= 2) {
      return pipelined_host_run(device, s, d, record_likelihood != 0, nchunk, by_mix, stats_dev, y, P0, lam0, v0, vf, P_out, lam_out, v_out,
                                record_likelihood ? ll_out : nullptr, vf_out, status, mu_out, phi_out);
    }
  }

  Staging st(mem, s);
  FFCA_TRY(st.in(y, size_t(U) * I * N * F * cs, &d.y));
  FFCA_TRY(st.in(P0, size_t(nb) * I * I * cs, &d.P0));
  FFCA_TRY(st.in(lam0, size_t(U) * J * F * I * rs, &d.lam0));
  FFCA_TRY(st.in(v0, size_t(U) * J * N * F * rs, &d.v0));
  if (vf_mode == 1) FFCA_TRY(st.in(vf, size_t(nb) * rs, &d.vf));
  if (vf_mode == 2) FFCA_TRY(st.in(vf, size_t(U) * J * N * F * rs, &d.vf));
  void *oP, *ol, *ov, *ovf = nullptr, *oll = nullptr;
  FFCA_TRY(st.out(P_out, size_t(nb) * I * I * cs, &oP));
  FFCA_TRY(st.out(lam_out, size_t(U) * J * F * I * rs, &ol));
  FFCA_TRY(st.out(v_out, size_t(U) * J * N * F * rs, &ov));
  if (vf_out) FFCA_TRY(st.out(vf_out, size_t(nb) * 8, &ovf));
  if (record_likelihood && ll_out) FFCA_TRY(st.out(ll_out, size_t(U) * nev * 8, &oll));
  if (stats_dev) {
    d.mu = mu_out;
    d.phi = phi_out;
  } else {
    FFCA_TRY(st.out(mu_out, size_t(U) * J * N * F * I * cs, &d.mu));
    FFCA_TRY(st.out(phi_out, size_t(U) * J * N * F * I * rs, &d.phi));
  }
  void *dstatus, *dllb = nullptr;
  FFCA_TRY(st.scratch(size_t(nb) * 4, &dstatus));
  FFCA_CK(cudaMemsetAsync(dstatus, 0, size_t(nb) * 4, s));
  if (record_likelihood) FFCA_TRY(st.scratch(size_t(nb) * nev * 8, &dllb));
  d.P = oP; d.lam = ol; d.v = ov; d.vf_out = (double*)ovf;
  d.ll_bins = (double*)dllb;
  d.status = (int*)dstatus;
  FFCA_TRY(launch_problem(device, d, s));
  if (oll) FFCA_TRY(reduce_ll((const double*)dllb, (double*)oll, U, F, nev, -double(N) * F * I * std::log(M_PI), s));
  FFCA_TRY(st.flush());
  return finish_status((const int*)dstatus, status, nb, mem, s, FFCA_ST_SINGULAR_P | FFCA_ST_SINGULAR_B);
}

extern "C" int ffca_fastfca_run(int device, void* stream, int mem, int dtype, int U, int I, int J, int N,
                                int F, const void* y, const void* P0, const void* lam0, const void* v0,
                                int vf_mode, double vf_scalar, const void* vf, int iterations,
                                int inner_iterations, int record_likelihood, void* P_out, void* lam_out,
                                void* v_out, double* ll_out, double* vf_out, int* status) {
  return loop_entry(device, stream, mem, dtype, U, I, J, N, F, y, P0, lam0, v0, vf_mode, vf_scalar, vf,
                    iterations, inner_iterations, record_likelihood, P_out, lam_out, v_out, ll_out, vf_out,
                    status, 0);
}

// run_fastfca including its final statistics refresh (fastfca.py:466): the loop kernel, then the
// per-point refresh on the device-resident final state; mu_out (U,J,N,F,I) complex and phi_out
// (U,J,N,F,I) real (either may be null).  Host mode pipelines both outputs' D2H with the chunks.
extern "C" int ffca_fastfca_run_stats(int device, void* stream, int mem, int dtype, int U, int I, int J, int N,
                                      int F, const void* y, const void* P0, const void* lam0, const void* v0,
                                      int vf_mode, double vf_scalar, const void* vf, int iterations,
                                      int inner_iterations, int record_likelihood, void* P_out, void* lam_out,
                                      void* v_out, double* ll_out, double* vf_out, int* status, void* mu_out,
                                      void* phi_out) {
  return loop_entry(device, stream, mem, dtype, U, I, J, N, F, y, P0, lam0, v0, vf_mode, vf_scalar, vf,
                    iterations, inner_iterations, record_likelihood, P_out, lam_out, v_out, ll_out, vf_out,
                    status, 0, mu_out, phi_out);
}

// fastfca.log_likelihood (fastfca.py:240-255): the loop kernel with zero
// iterations evaluates exactly L2 at the given state.
extern "C" int ffca_fastfca_loglik(int device, void* stream, int mem, int dtype, int U, int I, int J, int N,
                                   int F, const void* y, const void* P, const void* lam, const void* v,
                                   double* ll_out, int* status) {
  if (!check_dims(dtype, U, I, J, N, F)) return FFCA_E_ARG;
  DeviceGuard dg(device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t rs = rsize(dtype), cs = csize(dtype);
  const long long nb = (long long)U * F;
  // scratch outputs on device; only the likelihood is returned
  void *Po = nullptr, *lo = nullptr, *vo = nullptr;
  FFCA_CK(cudaMallocAsync(&Po, size_t(nb) * I * I * cs + 16, s));
  FFCA_CK(cudaMallocAsync(&lo, size_t(U) * J * F * I * rs + 16, s));
  FFCA_CK(cudaMallocAsync(&vo, size_t(U) * J * N * F * rs + 16, s));
  int rc = FFCA_OK;
  {
    // stage inputs here so the loop entry can run in device mode
    Staging st(mem, s);
    const void *dy, *dP, *dl, *dv;
    void* dll;
    rc = st.in(y, size_t(U) * I * N * F * cs, &dy);
    if (!rc) rc = st.in(P, size_t(nb) * I * I * cs, &dP);
    if (!rc) rc = st.in(lam, size_t(U) * J * F * I * rs, &dl);
    if (!rc) rc = st.in(v, size_t(U) * J * N * F * rs, &dv);
    if (!rc) rc = st.out(ll_out, size_t(U) * 8, &dll);
    if (!rc) {
      int* dst = nullptr;
      if (status && mem == FFCA_MEM_DEVICE) dst = status;
      std::vector<int> hst;
      rc = loop_entry(device, stream, FFCA_MEM_DEVICE, dtype, U, I, J, N, F, dy, dP, dl, dv, FFCA_VF_SCALAR, 0.0,
                      nullptr, 0, 1, 1, Po, lo, vo, (double*)dll, nullptr, dst, 0);
      if (rc == FFCA_OK) rc = st.flush();
      if (rc == FFCA_OK) {
        cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
          set_error("%s", cudaGetErrorString(e));
          rc = FFCA_E_CUDA;
        }
      }
    }
  }
  cudaFreeAsync(Po, s);
  cudaFreeAsync(lo, s);
  cudaFreeAsync(vo, s);
  return rc;
}

// fastfca.fixed_point_update_P (fastfca.py:197-237): one P-only pass of the
// loop kernel (B_i hermitized from the packed lower triangle, K updates).
extern "C" int ffca_fixed_point_update_P(int device, void* stream, int mem, int dtype, int U, int I, int J,
                                         int N, int F, const void* y, const void* P, const void* lam,
                                         const void* v, int inner_iterations, void* P_out, int* status) {
  if (!check_dims(dtype, U, I, J, N, F)) return FFCA_E_ARG;
  DeviceGuard dg(device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t rs = rsize(dtype), cs = csize(dtype);
  const long long nb = (long long)U * F;
  void *lo = nullptr, *vo = nullptr;
  FFCA_CK(cudaMallocAsync(&lo, size_t(U) * J * F * I * rs + 16, s));
  FFCA_CK(cudaMallocAsync(&vo, size_t(U) * J * N * F * rs + 16, s));
  int rc;
  {
    Staging st(mem, s);
    const void *dy, *dP, *dl, *dv;
    void* dPo;
    rc = st.in(y, size_t(U) * I * N * F * cs, &dy);
    if (!rc) rc = st.in(P, size_t(nb) * I * I * cs, &dP);
    if (!rc) rc = st.in(lam, size_t(U) * J * F * I * rs, &dl);
    if (!rc) rc = st.in(v, size_t(U) * J * N * F * rs, &dv);
    if (!rc) rc = st.out(P_out, size_t(nb) * I * I * cs, &dPo);
    if (!rc) {
      int* dst = (status && mem == FFCA_MEM_DEVICE) ? status : nullptr;
      std::vector<int> hst(status && mem != FFCA_MEM_DEVICE ? nb : 0);
      rc = loop_entry(device, stream, FFCA_MEM_DEVICE, dtype, U, I, J, N, F, dy, dP, dl, dv, FFCA_VF_SCALAR,
                      0.0, nullptr, 1, inner_iterations, 0, dPo, lo, vo, nullptr, nullptr, dst, 1);
      (void)hst;
      if (rc == FFCA_OK) rc = st.flush();
      if (rc == FFCA_OK && cudaStreamSynchronize(s) != cudaSuccess) {
        set_error("%s", cudaGetErrorString(cudaGetLastError()));
        rc = FFCA_E_CUDA;
      }
    }
  }
  cudaFreeAsync(lo, s);
  cudaFreeAsync(vo, s);
  return rc;
}

// Introspection for tests / bench: the launch plan chosen for a shape.
static int plan_introspect(int device, int dtype, int U, int I, int J, int N, int F, int vf_mode, bool fast,
                           LoopPlan& p) {
  int optin = 0;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess) {
    cudaGetLastError();
    optin = 232448;
  }
  int nsm = 148;
  if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
    cudaGetLastError();
    nsm = 148;
  }
  return plan_loop(dtype, I, J, N, (long long)U * F, vf_mode, p, size_t(optin), nsm, fast);
}

// The plan of the plain loop (no likelihood record, K = 1: the lean instantiations).
extern "C" int ffca_plan_loop(int device, int dtype, int U, int I, int J, int N, int F, int vf_mode,
                              int* out6) {
  LoopPlan p;
  int rc = plan_introspect(device, dtype, U, I, J, N, F, vf_mode, vf_mode != 2 && !getenv("FFCA_NO_FAST"), p);
  out6[0] = p.G;
  out6[1] = p.C;
  out6[2] = p.NL;
  out6[3] = p.threads;
  out6[4] = p.resident ? 1 : 0;
  out6[5] = int(p.smem);
  return rc;
}

// lean != 0: the plain loop; lean == 0: the loop with the likelihood record / inner iterations.
// out8 = {G, C, NL, threads, resident, smem, tensor-memory plan, tensor-memory columns per CTA}.
extern "C" int ffca_plan_loop_ex(int device, int dtype, int U, int I, int J, int N, int F, int vf_mode, int lean,
                                 int* out8) {
  LoopPlan p;
  int rc = plan_introspect(device, dtype, U, I, J, N, F, vf_mode, lean != 0 && vf_mode != 2 && !getenv("FFCA_NO_FAST"), p);
  out8[0] = p.G;
  out8[1] = p.C;
  out8[2] = p.NL;
  out8[3] = p.threads;
  out8[4] = p.resident ? 1 : 0;
  out8[5] = int(p.smem);
  out8[6] = p.tm ? 1 : 0;
  out8[7] = p.tm ? (I == 3 ? 128 : 256) : 0;
  return rc;
}
