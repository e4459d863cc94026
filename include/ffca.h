/*
 * ffca.h -- C ABI of the B200-native FastFCA-AS / FCA library (libffca_b200.so).
 *
 * The reference (fcasep, pure Python/numpy) has no FFI of its own; these entry
 * points are what a ctypes / cffi binding of its hot-path Python functions
 * binds.  Each declaration cites the reference function it replaces
 * (paths relative to /root/reference/pkg/src/fcasep/).
 *
 * Conventions
 *   - All arrays are C-contiguous in the REFERENCE layouts, with an extra
 *     leading mixture axis U (U = 1 for a single mixture):
 *       y    (U, I, N, F)  complex   stft.py:56-67 ObservationTensor.data
 *       P    (U, F, I, I)  complex   fastfca.py:54
 *       lam  (U, J, F, I)  real      fastfca.py:55
 *       v    (U, J, N, F)  real      fastfca.py:56
 *       S    (U, J, F, I, I) complex fca.py:34
 *       mu   (U, J, N, F, I) complex  phi (U, J, N, F, I) real (fastfca.py:95-96)
 *       images (U, J, I, N, F) complex  wiener.py:24
 *   - dtype: FFCA_C128 (complex128 / float64, the reference's only path) or
 *     FFCA_C64 (complex64 / float32).  Complex = interleaved (re, im).
 *   - mem: FFCA_MEM_HOST -> every array pointer is host memory (the library
 *     stages H2D / D2H itself); FFCA_MEM_DEVICE -> every array pointer is
 *     device memory on `device` (no copies).  `stream` is a cudaStream_t
 *     (NULL = legacy default stream); calls are stream-ordered and return
 *     after completion.
 *   - Return value 0 on success, otherwise an FFCA_E_* code; the message is
 *     available from ffca_last_error().  Singularities are reported per bin
 *     in `status` (FFCA_ST_* bits, (U, F) ints) when the pointer is given.
 */
#ifndef FFCA_H_
#define FFCA_H_

#ifdef __cplusplus
extern "C" {
#endif

#define FFCA_C128 0
#define FFCA_C64 1

#define FFCA_MEM_HOST 0
#define FFCA_MEM_DEVICE 1
/* ffca_fastfca_run_stats only: host arrays, except mu_out / phi_out, which are device memory
 * (the statistics stay in HBM for a device consumer, e.g. the Wiener images) */
#define FFCA_MEM_HOST_STATS_DEVICE 2

/* v_floor modes (fastfca.py:406,421-424,435-436) */
#define FFCA_VF_SCALAR 0 /* v_floor is a python float               */
#define FFCA_VF_BIN 1    /* (U, F) array, e.g. fca.power_floor(obs) */
#define FFCA_VF_FULL 2   /* (U, J, N, F) array                      */
#define FFCA_VF_AUTO 3   /* v_floor=None: power_floor computed on device (fca.py:82-89) */

#define FFCA_OK 0
#define FFCA_E_ARG -1        /* bad sizes / pointers (errors.DimensionMismatch on the Python side) */
#define FFCA_E_CUDA -2       /* CUDA runtime failure                                               */
#define FFCA_E_SINGULAR_P -3 /* errors.SingularP                  fastfca.py:360-363, 268-271     */
#define FFCA_E_SINGULAR_B -4 /* errors.SingularWeightedCovariance fastfca.py:184-194              */
#define FFCA_E_NOT_PD -5     /* errors.NotPositiveDefinite        fca.py:137-140, 157-158         */
#define FFCA_E_UNSUPPORTED -6 /* order I outside 1..8 (matcore.MAX_ORDER, matcore.py:20)           */

#define FFCA_ST_SINGULAR_P 1
#define FFCA_ST_SINGULAR_B 2
#define FFCA_ST_B_LOADED 4
#define FFCA_ST_NOT_PD 8
#define FFCA_ST_S_LOADED 16

/* Library / device info. */
int ffca_version(void);
const char* ffca_last_error(void);
int ffca_device_count(void);
/* Pinned host allocation helpers (for zero-staging H2D / D2H). */
int ffca_host_alloc(void** ptr, long long bytes);
int ffca_host_free(void* ptr);

/*
 * Hybrid FastFCA-AS loop: EM sweep on (v, lam) then fixed-point update of P,
 * `iterations` times, all on device.  Replaces fastfca.run_fastfca
 * (fastfca.py:401-474) minus the final stats refresh, which is
 * ffca_fastfca_stats / ffca_fastfca_images below.
 *   vf            scalar value for FFCA_VF_SCALAR, else array per vf_mode
 *   ll_out        (U, 1 + 2*iterations) or NULL: [L_init, L_after_em[0..T-1], L_after_p[0..T-1]]
 *                 (loglik_init / loglik_after_em / loglik_after_p, fastfca.py:448-459)
 *   vf_out        (U, F) float64 or NULL: the floor used (auto mode)
 *   P_out/lam_out/v_out may alias P0/lam0/v0.
 */
int ffca_fastfca_run(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                     const void* y, const void* P0, const void* lam0, const void* v0, int vf_mode,
                     double vf_scalar, const void* vf, int iterations, int inner_iterations,
                     int record_likelihood, void* P_out, void* lam_out, void* v_out, double* ll_out,
                     double* vf_out, int* status);

/*
 * ffca_fastfca_run plus its final statistics refresh -- the whole of
 * fastfca.run_fastfca (fastfca.py:401-474, stats at :466 via _stats_refresh
 * :373-387): after the loop kernel the per-point refresh runs on the
 * device-resident final state; mu_out (U, J, N, F, I) complex, phi_out
 * (U, J, N, F, I) real, either may be NULL.  Host mode moves both outputs
 * chunk by chunk, overlapped with the next chunk's loop; FFCA_MEM_HOST_STATS_DEVICE
 * writes them into device buffers instead (nothing crosses PCIe for them).
 */
int ffca_fastfca_run_stats(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                           const void* y, const void* P0, const void* lam0, const void* v0, int vf_mode,
                           double vf_scalar, const void* vf, int iterations, int inner_iterations,
                           int record_likelihood, void* P_out, void* lam_out, void* v_out, double* ll_out,
                           double* vf_out, int* status, void* mu_out, void* phi_out);

/*
 * Transformed posterior statistics at (P, lam, v): mu_t = g * P^H y and
 * phi_t = max(a (1 - g), 0) with a = v lam, g = a / w.
 * Replaces fastfca._stats_refresh (fastfca.py:373-387) and, given y_t,
 * e_step_diag (fastfca.py:144-157).  mu / phi may be NULL (not produced).
 */
int ffca_fastfca_stats(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                       const void* y, const void* P, const void* lam, const void* v, void* mu, void* phi);

/*
 * Multichannel Wiener images x_j = P^{-H} (g_j * P^H y), written (U, J, I, N, F).
 * Fuses fastfca._stats_refresh + wiener.mmse_images_fastfca
 * (fastfca.py:373-387, wiener.py:38-43, back_transform_means fastfca.py:258-273).
 */
int ffca_fastfca_images(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                        const void* y, const void* P, const void* lam, const void* v, void* images,
                        int* status);

/*
 * Solve P^H x = mu_t per bin for all (j, n): back_transform_means
 * (fastfca.py:258-273).  mu_t (U, J, N, F, I) -> out (U, J, N, F, I); when
 * `images_layout` != 0 the output is written (U, J, I, N, F) instead
 * (wiener.mmse_images_fastfca, wiener.py:38-43).
 */
int ffca_back_transform(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                        const void* P, const void* mu_t, void* out, int images_layout, int* status);

/*
 * Observed log likelihood L2 (fastfca.log_likelihood, fastfca.py:240-255),
 * one value per mixture in ll_out (U,).
 */
int ffca_fastfca_loglik(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                        const void* y, const void* P, const void* lam, const void* v, double* ll_out,
                        int* status);

/*
 * Unfused fixed-point update of P (fastfca.fixed_point_update_P,
 * fastfca.py:197-237): B_i from (y, v, lam) (hermitized), then K column
 * updates.  P_out may alias P.
 */
int ffca_fixed_point_update_P(int device, void* stream, int mem, int dtype, int U, int I, int J, int N,
                              int F, const void* y, const void* P, const void* lam, const void* v,
                              int inner_iterations, void* P_out, int* status);

/*
 * Conventional FCA EM (fca.run_fca, fca.py:187-215).  S_prev / v_prev (may be
 * NULL) receive the parameters of the last E-step (the returned stats are
 * the E-step at those, fca.py:211).  ll_out (U, 1 + iterations) or NULL.
 */
int ffca_fca_run(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                 const void* y, const void* S0, const void* v0, int vf_mode, double vf_scalar,
                 const void* vf, int iterations, int record_likelihood, void* S_out, void* v_out,
                 void* S_prev, void* v_prev, double* ll_out, int* status);

/*
 * Full-matrix E-step (fca.e_step, fca.py:119-144): mu (U,J,N,F,I) and phi
 * (U,J,N,F,I,I); either may be NULL.  With images_layout != 0, mu is written
 * (U, J, I, N, F) (wiener.mmse_images_fca, wiener.py:32-35).
 */
int ffca_fca_estep(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                   const void* y, const void* S, const void* v, void* mu, void* phi, int images_layout,
                   int* status);

/* FCA observed log likelihood L1 (fca.log_likelihood, fca.py:101-116), (U,). */
int ffca_fca_loglik(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                    const void* y, const void* S, const void* v, double* ll_out, int* status);

/* ---- step-level entry points (unfused public functions of fastfca.py) ---- */

/* y_t = P^H y, (U, N, F, I): fastfca.transform_observations (fastfca.py:113-116). */
int ffca_transform(int device, void* stream, int mem, int dtype, int U, int I, int N, int F, const void* y,
                   const void* P, void* yt);

/* w = max(sum_j v_j lam_j, floor), (U, N, F, I): fastfca.mixture_weights (fastfca.py:138-141). */
int ffca_mixture_weights(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                         const void* lam, const void* v, void* w);

/* e_step_diag from a given y_t (U, N, F, I): fastfca.e_step_diag (fastfca.py:144-157). */
int ffca_fastfca_estep_yt(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                          const void* yt, const void* lam, const void* v, void* mu, void* phi);

/* fastfca.m_step_diag (fastfca.py:160-181); vf_mode SCALAR / BIN / FULL. */
int ffca_mstep_diag(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                    const void* mu, const void* phi, const void* lam, int vf_mode, double vf_scalar,
                    const void* vf, void* v_out, void* lam_out);

/* fca.m_step (fca.py:161-184) from mu (U,J,N,F,I), phi (U,J,N,F,I,I) and the old S. */
int ffca_fca_mstep(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                   const void* mu, const void* phi, const void* S, int vf_mode, double vf_scalar, const void* vf,
                   void* S_out, void* v_out, int* status);

/* fca.power_floor (fca.py:82-89): (U, F) float64. */
int ffca_power_floor(int device, void* stream, int mem, int dtype, int U, int I, int N, int F, const void* y,
                     double* out);

/* S_j = P^-H diag(lam_j) P^-1 hermitized, (U,J,F,I,I): fastfca.reconstruct_spatial_covariances
 * (fastfca.py:119-135). */
int ffca_reconstruct_covariances(int device, void* stream, int mem, int dtype, int U, int I, int J, int F,
                                 const void* P, const void* lam, void* S, int* status);

/* Posterior covariances in the microphone basis, P^-H diag(phi_t) P^-1 hermitized, (U,J,N,F,I,I):
 * the phi half of fastfca.back_transform_stats (fastfca.py:276-287). */
int ffca_back_transform_phi(int device, void* stream, int mem, int dtype, int U, int I, int J, int N, int F,
                            const void* P, const void* phi_t, void* phi_out, int* status);

/* Whitening init fastfca.params_from_covariances (fastfca.py:290-309): P (U,F,I,I), lam (U,J,F,I). */
int ffca_params_from_covariances(int device, void* stream, int mem, int dtype, int U, int I, int J, int F,
                                 const void* S_hat, void* P_out, void* lam_out, int* status);

/* Initial covariances (scene.oracle_covariances / scene.diffuse_covariances, scene.py:207-247), one CTA
 * per (mixture, source, bin) or (mixture, bin), fp64 accumulation:
 *   mode 0 (oracle):  x = source-image STFTs (U,J,I,N,F); v_hat = max(sum_i |x_i|^2 / I, floor),
 *                     S_hat = sum_n x x^H / v_hat / N
 *   mode 1 (diffuse): x = observations (U,I,N,F); S_hat_j = avg + 0.5 max(tr(avg)/I, 1e-300) W_j with
 *                     W (J,I,I) the seeded trace-normalised PD perturbations; v_hat = max(power / J, floor)
 * then diagonal loading 1e-9 tr/I (identity when tr <= 0, scene._load_pd, scene.py:200-204).
 * floor (U,F) float64 from ffca_power_floor.  Outputs S_hat (U,J,F,I,I), v_hat (U,J,N,F). */
int ffca_init_covariances(int device, void* stream, int mem, int dtype, int mode, int U, int I, int J, int N, int F,
                          const void* x, const double* floor, const void* W, void* S_out, void* v_out);

/* SDR energies for evalkit.compute_sdr (evalkit.py:68-88): ref (J,I,Sr), est (J,I,Se) real
 * (C128 -> float64, C64 -> float32); out (J,2) float64 = (||ref||^2, ||ref - est||^2) summed over
 * channels and the first min(Sr, Se) samples.  The dB value and its cap / zero-reference error are
 * the caller's scalar arithmetic. */
int ffca_sdr_energies(int device, void* stream, int mem, int dtype, int J, int I, long long Sr, long long Se,
                      const void* ref, const void* est, double* out);

/* STFT analysis (stft.analyze, stft.py:96-112): audio (I, S) real -> (I, N, L/2) complex with
 * N = (S - L) / shift + 1, sqrt-Hann window, DC and Nyquist packed into bin 0.  dtype selects
 * float64 -> complex128 or float32 -> complex64.  cuFFT batched R2C. */
int ffca_stft_analyze(int device, void* stream, int mem, int dtype, int I, long long S, int L, int shift,
                      const void* audio, void* out);

/* STFT synthesis (stft.synthesize, stft.py:115-134): (I, N, L/2) complex -> (I, (N-1)*shift + L)
 * real by windowed overlap-add (deterministic gather).  cuFFT batched C2R. */
int ffca_stft_synthesize(int device, void* stream, int mem, int dtype, int I, int N, int L, int shift,
                         const void* in, void* audio);

/* Launch plan of the loop kernel for a shape: out6 = {G, C, NL, threads, resident, smem}. */
int ffca_plan_loop(int device, int dtype, int U, int I, int J, int N, int F, int vf_mode, int* out6);
/* Same with the loop variant chosen (lean != 0: the plain loop; 0: likelihood record / inner
 * iterations) and the tensor-memory use: out8 = {G, C, NL, threads, resident, smem, tensor-memory
 * plan (y records in TMEM), TMEM columns per CTA}. */
int ffca_plan_loop_ex(int device, int dtype, int U, int I, int J, int N, int F, int vf_mode, int lean, int* out8);

/* Kernel launches issued by the last successful call on this host thread. */
int ffca_last_launch_count(void);

/* Opt-in CUDA-event timing of the estimation-loop kernel on its launch stream
 * (this host thread); ffca_last_kernel_ms() returns the last measured launch. */
void ffca_set_kernel_timing(int on);
float ffca_last_kernel_ms(void);

#ifdef __cplusplus
}
#endif

#endif /* FFCA_H_ */
