// C-ABI: FastFCA-AS estimation loop (ffca_fastfca_run).
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "ffca_loop.cuh"
#include "host_common.h"

namespace ffca {

using LoopFn = void (*)(const LoopArgs);
LoopFn loop_kernel_f32(int I, int J, int G, bool res);
LoopFn loop_kernel_f64(int I, int J, int G, bool res);

static bool hot_shape(int I, int J) {
  return (I == 3 && J == 3) || (I == 4 && J == 4) || (I == 8 && J == 6) || (I == 2 && J == 2);
}

static int host_vmax(int I, int JM) {
  int IC = (I * I * I <= 64) ? I : ((64 / (I * I)) > 0 ? (64 / (I * I)) : 1);
  int NB = IC * I * I;
  int va = JM * (1 + I) + 1;
  return va > NB + 1 ? va : NB + 1;
}

struct LoopPlan {
  int G = 1, C = 1, NL = 0, threads = 64;
  bool resident = true;
  size_t smem = 0, slab = 0;
  long long grid = 0;
};

// Slab budget per CTA: two CTAs per SM fit in the 228 KB shared memory.
static constexpr size_t kSlabBudget = 96 * 1024;

static int choose_threads(int G, int NL) {
  const int per_bin = (NL + 3) / 4;  // ~4 frames per thread per pass (capped at 256 threads)
  int t = G * per_bin;
  t = (t + 31) / 32 * 32;
  if (t < 64) t = 64;
  if (t > 256) t = 256;
  return t;
}

static int plan_loop(int dtype, int I, int J, int N, long long total_bins, int vf_mode, LoopPlan& p,
                     size_t smem_optin) {
  const int rsz = int(rsize(dtype));
  const int JM = hot_shape(I, J) ? J : 8;
  const int VMAX = host_vmax(I, JM);
  // lane-interleaved bin groups only for the exact-J instantiations
  const int G0 = hot_shape(I, J) ? (dtype == FFCA_C64 ? 4 : 2) : 1;
  auto fill = [&](int G, int C, bool res) {
    p.G = G;
    p.C = C;
    p.NL = (N + C - 1) / C;
    p.threads = choose_threads(G, p.NL);
    p.resident = res;
    LoopSmem L(I, J, G, p.NL, p.threads / 32, rsz, vf_mode, res, VMAX);
    p.smem = L.total;
    p.slab = L.slab;
    p.grid = ((total_bins + G - 1) / G) * C;
  };
  // Test hook: FFCA_FORCE_PLAN="G,C,resident" pins the launch plan (parity tests
  // use it to exercise the cluster and global-slab paths at small sizes).
  if (const char* fp = getenv("FFCA_FORCE_PLAN")) {
    int G = 1, C = 1, res = 1, thr = 0;
    const int nf = sscanf(fp, "%d,%d,%d,%d", &G, &C, &res, &thr);
    if (nf >= 3 && (G == 1 || G == G0) && (G == 1 || res) && C >= 1 && C <= 8 && (C & (C - 1)) == 0 && C <= N &&
        (C == 1 || G == 1)) {
      fill(G, C, res != 0);
      if (nf == 4 && thr >= 64 && thr <= 256 && thr % 32 == 0) {
        p.threads = thr;
        LoopSmem L(I, J, G, p.NL, thr / 32, rsz, vf_mode, res != 0, VMAX);
        p.smem = L.total;
      }
      if (p.smem <= smem_optin) return FFCA_OK;
    }
  }
  for (int G : {G0, 1}) {
    fill(G, 1, true);
    if (p.slab <= kSlabBudget && p.smem <= smem_optin) return FFCA_OK;
  }
  for (int C = 2; C <= 8; C <<= 1) {
    if (C > N) break;
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

static int launch_loop(LoopFn fn, const LoopPlan& p, const LoopArgs& a, cudaStream_t s) {
  FFCA_CK(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p.smem)));
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

static int loop_entry(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                      const void* y, const void* P0, const void* lam0, const void* v0, int vf_mode,
                      double vf_scalar, const void* vf, int iterations, int inner_iterations,
                      int record_likelihood, void* P_out, void* lam_out, void* v_out, double* ll_out,
                      double* vf_out, int* status, int p_only) {
  reset_launches();
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

  Staging st(mem, s);
  const void *dy, *dP, *dl, *dv, *dvf = nullptr;
  FFCA_TRY(st.in(y, size_t(U) * I * N * F * cs, &dy));
  FFCA_TRY(st.in(P0, size_t(nb) * I * I * cs, &dP));
  FFCA_TRY(st.in(lam0, size_t(U) * J * F * I * rs, &dl));
  FFCA_TRY(st.in(v0, size_t(U) * J * N * F * rs, &dv));
  if (vf_mode == 1) FFCA_TRY(st.in(vf, size_t(nb) * rs, &dvf));
  if (vf_mode == 2) FFCA_TRY(st.in(vf, size_t(U) * J * N * F * rs, &dvf));
  void *oP, *ol, *ov, *ovf = nullptr, *oll = nullptr;
  FFCA_TRY(st.out(P_out, size_t(nb) * I * I * cs, &oP));
  FFCA_TRY(st.out(lam_out, size_t(U) * J * F * I * rs, &ol));
  FFCA_TRY(st.out(v_out, size_t(U) * J * N * F * rs, &ov));
  if (vf_out) FFCA_TRY(st.out(vf_out, size_t(nb) * 8, &ovf));
  if (record_likelihood && ll_out) FFCA_TRY(st.out(ll_out, size_t(U) * nev * 8, &oll));
  void *dstatus, *dllb = nullptr;
  FFCA_TRY(st.scratch(size_t(nb) * 4, &dstatus));
  FFCA_CK(cudaMemsetAsync(dstatus, 0, size_t(nb) * 4, s));
  if (record_likelihood) FFCA_TRY(st.scratch(size_t(nb) * nev * 8, &dllb));

  int optin = 0;
  FFCA_CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  LoopPlan p;
  FFCA_TRY(plan_loop(dtype, I, J, N, nb, vf_mode, p, size_t(optin)));
  void* scratch = nullptr;
  if (!p.resident) FFCA_TRY(st.scratch(size_t(p.grid) * p.slab, &scratch));

  LoopArgs a;
  a.U = U; a.I = I; a.J = J; a.N = N; a.F = F;
  a.total_bins = nb;
  a.G = p.G; a.C = p.C; a.NL = p.NL;
  a.iters = iterations; a.K = inner_iterations; a.p_only = p_only;
  a.vf_mode = vf_mode; a.vf_scalar = vf_scalar; a.vf = dvf;
  a.y = dy; a.P_in = dP; a.lam_in = dl; a.v_in = dv;
  a.P_out = oP; a.lam_out = ol; a.v_out = ov;
  a.vf_out = (double*)ovf;
  a.ll = (double*)dllb;
  a.status = (int*)dstatus;
  a.scratch = scratch;
  a.slab_bytes = (long long)p.slab;

  LoopFn fn = dtype == FFCA_C64 ? loop_kernel_f32(I, J, p.G, p.resident) : loop_kernel_f64(I, J, p.G, p.resident);
  if (!fn) {
    set_error("no kernel for I=%d J=%d", I, J);
    return FFCA_E_UNSUPPORTED;
  }
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (timing_enabled()) {
    FFCA_CK(cudaEventCreate(&ev0));
    FFCA_CK(cudaEventCreate(&ev1));
    FFCA_CK(cudaEventRecord(ev0, s));
  }
  FFCA_TRY(launch_loop(fn, p, a, s));
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
extern "C" int ffca_plan_loop(int device, int dtype, int U, int I, int J, int N, int F, int vf_mode,
                              int* out6) {
  int optin = 0;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess) {
    cudaGetLastError();
    optin = 232448;
  }
  LoopPlan p;
  int rc = plan_loop(dtype, I, J, N, (long long)U * F, vf_mode, p, size_t(optin));
  out6[0] = p.G;
  out6[1] = p.C;
  out6[2] = p.NL;
  out6[3] = p.threads;
  out6[4] = p.resident ? 1 : 0;
  out6[5] = int(p.smem);
  return rc;
}
