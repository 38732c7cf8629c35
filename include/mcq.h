/*
 * mcq.h — C ABI of the B200-native Mumax3-cQED hot path (arXiv 2410.00966).
 *
 * One context = one ferromagnet on an nx*ny*nz finite-difference grid coupled to one damped
 * cavity mode (or up to MCQ_MAX_MODES independent modes, see mcq_set_modes).  Each mcq_run step integrates the LLG equation with the cavity field
 *     dm_i/dt = -gamma/(1+alpha^2) [m_i x B'_i + alpha m_i x (m_i x B'_i)]            (eq:llg)
 *     B'_i = B_ext + B_exch + B_anis + B_demag + a sinc(w_cut t) B_rms,i + B_rms,i Gamma(t)
 *                                                     (eq:bcav P:239, excitation P:165)
 * with classical RK4 at fixed dt (reading C1), stage renormalisation (C2), the cavity memory
 * frozen inside a step (C3) and advanced once per step on the new state from the overlap
 *     W = sum_i M_s m_i . B_rms(r_i)
 * through the recursion of eq:Sdiscrete/eq:Cdiscrete/eq:gammadiscretefinal, kept on
 * the device in the algebraically identical complex form
 *     alpha_{n+1} = e^{-(kappa + i w_c) dt} alpha_n + i (V_c/hbar) W_{n+1} dt,  Gamma = 2 Re alpha
 * (reading C5; alpha_0 = (x0 - i p0)/2, reading C6).  Constants: gamma = 1.7595e11 rad/(s T),
 * mu0 = 4 pi 1e-7, hbar = 1.05457182e-34 J s (reading C8).
 *
 * Conventions (all calls):
 *  - SI units; B in tesla; f_c in Hz (w_c = 2 pi f_c); kappa in rad/s (cavity FWHM = 2 kappa).
 *  - Host vector arrays are interleaved (vx, vy, vz) per cell, cell index i = x + nx (y + ny z)
 *    (x fastest).  Arrays are copied in/out before the call returns; no pointer is retained.
 *    The caller owns every host array; the library owns the context and all device memory.
 *  - Every call returns 0 (MCQ_OK) on success or a negative MCQ_E* code; mcq_last_error()
 *    holds the message.  No C++ exception crosses the ABI.  A failing call leaves the
 *    simulation state unchanged (except MCQ_ECUDA, after which the context must be destroyed).
 *  - Device work is enqueued on the context's stream (mcq_set_stream; default: a library-owned
 *    stream).  mcq_run / mcq_relax / setters are stream-ordered; getters synchronise.
 *  - z-slab decomposition, selected by mcq_dist at creation:
 *      world == 1 (or dist NULL): one context holds the whole grid on one GPU;
 *      world > 1, rank >= 0: one process per GPU holds planes [rank*nz/world, (rank+1)*nz/world);
 *        the demag transpose (NCCL grouped send/recv, one all-to-all per direction per stage),
 *        the one-plane halos and the W partials (all-gather) go over NCCL; every rank must make
 *        the same calls in the same order (collective semantics) with the same arguments;
 *      world > 1, rank < 0 ("loopback"): all `world` slabs live in this one context on one GPU
 *        and the exchanges are device copies — the same decomposed schedule without a network,
 *        bitwise equal to world == 1.
 *    Host arrays are ALWAYS the global grid (3 nx ny nz floats); under NCCL each rank reads /
 *    writes only its own planes of them.
 */
#ifndef MCQ_H
#define MCQ_H

#if defined(__GNUC__)
#define MCQ_API __attribute__((visibility("default")))
#else
#define MCQ_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define MCQ_OK 0
#define MCQ_EINVAL (-1)  /* invalid argument (values below) */
#define MCQ_ESTATE (-2)  /* call not valid in the current state (e.g. run before set_m) */
#define MCQ_ENOMEM (-3)  /* device allocation failed */
#define MCQ_ECUDA (-4)   /* CUDA runtime / kernel error */
#define MCQ_ENCCL (-5)   /* NCCL missing (libnccl.so.2 not loadable) or an NCCL call failed */

/* field-term bitmask for mcq_get_field */
#define MCQ_TERM_ZEEMAN 1u
#define MCQ_TERM_EXCHANGE 2u
#define MCQ_TERM_ANIS 4u
#define MCQ_TERM_DEMAG 8u
#define MCQ_TERM_CAVITY 16u     /* B_rms * Gamma(t) */
#define MCQ_TERM_EXCITATION 32u /* a sinc(w_cut t) B_rms */
#define MCQ_TERM_DMI 64u        /* interfacial Dzyaloshinskii-Moriya (mcq_set_dmi) */
#define MCQ_TERM_ALL 127u       /* the deterministic terms */
#define MCQ_TERM_THERM 128u     /* thermal field (mcq_set_temperature); stochastic, not in ALL */

/* kernel classes reported by mcq_profile_run */
#define MCQ_K_YFWD 0   /* y-forward FFT pass (3D)                        */
#define MCQ_K_ZCONV 1  /* z-forward * Khat * z-inverse pass (3D)          */
#define MCQ_K_YINV 2   /* y-inverse FFT pass (3D)                        */
#define MCQ_K_Y2D 3    /* y-forward * Khat * y-inverse pass (nz == 1)     */
#define MCQ_K_UPDATE 4 /* fused x-C2R + fields + torque + RK4 + x-R2C     */
#define MCQ_K_CAVITY 5 /* overlap finalize + cavity state update          */
#define MCQ_NKCLASS 6

typedef struct mcq_ctx mcq_ctx; /* opaque, library-owned */

/* Anisotropy (reading C10).  Energy densities -K_u1 (m.u)^2 and
 * K_c1 (m1^2 m2^2 + m2^2 m3^2 + m3^2 m1^2) with m_k = m.c_k, c3 = c1 x c2.  J/m^3; axes are
 * normalised by the library; ku1 == 0 / kc1 == 0 disables the term. */
typedef struct {
  double ku1, u[3];
  double kc1, c1[3], c2[3];
} mcq_aniso;

/* Distribution descriptor (z slabs, see Conventions).  world must divide nz (1 <= world <= 64).
 * rank in [0, world) with nccl_id (128 bytes from mcq_nccl_get_unique_id on one rank, shared by
 * the caller, e.g. via torch.distributed) = one slab per process over NCCL; rank < 0 = loopback.
 * device >= 0 selects the CUDA device (else the current one); cuda_stream: the work stream or
 * NULL (library-owned). */
typedef struct {
  int rank, world, device;
  const unsigned char *nccl_id; /* 128 bytes or NULL */
  void *cuda_stream;            /* cudaStream_t or NULL */
} mcq_dist;

/* NCCL unique id for a multi-process context (128 bytes into out).  ENCCL if libnccl.so.2
 * cannot be loaded. */
MCQ_API int mcq_nccl_get_unique_id(unsigned char out[128]);

/* Cavity state at t_n (all ranks identical).  S, C are the paper's accumulators,
 * reconstructed from alpha: S - i C = (hbar/V_c)(alpha_0 - e^{(kappa + i w_c) t} alpha); the
 * rescaled pair e^{-kappa t}(S - i C) = (hbar/V_c)(e^{-kappa t} alpha_0 - e^{i w_c t} alpha) is
 * reported as well (S_resc, C_resc), finite where S, C overflow (long ring-downs, SPEC's
 * conditioning decision). */
typedef struct {
  double t;                  /* cavity clock since the last reset (s)                   */
  double re_alpha, im_alpha; /* alpha(t_n) = <a>                             */
  double gamma;              /* Gamma(t_n) = 2 Re alpha = x(t_n) (eq:gammadiscretefinal) */
  double W;                  /* overlap of the last completed step, A/m * T      */
  double S, C;               /* literal accumulators; they grow as e^{kappa t} and are   */
                             /* +-inf once kappa t exceeds ~709 (fp64 range)             */
  double n_photon;           /* |alpha|^2                                        */
  long long step;            /* completed steps since the last reset                    */
  double S_resc, C_resc;     /* e^{-kappa t} S, e^{-kappa t} C: finite for every t,      */
                             /* computed without the growing exponential (reading C5)    */
} mcq_cavity_state;

/* Create a context.  grid[3] = (nx, ny, nz) with 2 <= nx, ny <= 512 and 1 <= nz <= 512;
 * cell[3] = (dx, dy, dz) > 0 metres; Ms > 0 (A/m; single material, vacuum via the geometry
 * mask); Aex >= 0 (J/m); alpha >= 0 (Gilbert); K may be NULL; dist may be NULL.
 * Precomputes the demag kernel (Newell near field, Gauss-Legendre far field, reading C11) on
 * the device in fp64.  EINVAL on bad sizes/values; ENOMEM if HBM is insufficient. */
MCQ_API int mcq_create(mcq_ctx **out, const int grid[3], const double cell[3], double Ms, double Aex,
               double alpha, const mcq_aniso *K, const mcq_dist *dist);

/* nz == 1 grids of up to 65536 cells (BJ configs[0]-class films), plain RK4 with one cavity mode
 * and no DMI / thermal field: mcq_run runs all its steps in one persistent cooperative kernel
 * (grid barriers between the y pass, the update and the cavity step) instead of 9 graph nodes per
 * step (1) or replays the per-step graphs (0, default).  Same arithmetic, bitwise the same
 * results; grids without a compiled instance fall back to the graphs.  Worth it for many
 * concurrent replicas (bias sweeps: 32 replicas of configs[0] 1.16x the graphs' throughput);
 * a lone replica is faster with the graphs. */
MCQ_API int mcq_set_persistent_2d(mcq_ctx *, int on);

/* z slabs: overlap each component's transpose (NCCL send/recv, or device copies in loopback) with
 * the next component's y pass on a second stream (1), or run the passes and transposes in series
 * (0).  Default: 1 under NCCL, 0 in loopback (where the copies compete with the passes for HBM).
 * Same results bit for bit either way.  No effect on a single slab. */
MCQ_API int mcq_set_slab_overlap(mcq_ctx *, int on);

/* Use `stream` (a cudaStream_t, e.g. torch.cuda.current_stream().cuda_stream) for all work. */
MCQ_API int mcq_set_stream(mcq_ctx *, void *stream);

/* Geometry mask, N bytes, x fastest, 0 = vacuum (M_s = 0, m = 0).  NULL = full box.
 * Applies to subsequent mcq_set_m calls and zeroes m in vacuum now.  If a magnetisation is
 * installed and the new geometry makes magnetic some cells that hold no magnetisation (they
 * were vacuum), the geometry is applied but the call returns ESTATE and mcq_run / mcq_relax /
 * mcq_get_field refuse (ESTATE) until mcq_set_m installs a state for the new geometry. */
MCQ_API int mcq_set_geometry(mcq_ctx *, const unsigned char *mask);

/* Magnetisation, 3N floats interleaved (host).  Normalised on entry (vectors already unit to
 * within 1e-6 in |m|^2 are kept as given, so a state saved with mcq_get_m resumes bit-exactly);
 * vacuum cells are set to 0.
 * EINVAL if a magnetic cell has a zero vector.  Does not touch the cavity state. */
MCQ_API int mcq_set_m(mcq_ctx *, const float *m);
/* Same from a device pointer (3N floats interleaved, device memory of this context's GPU). */
MCQ_API int mcq_set_m_device(mcq_ctx *, const float *d_m);

/* Uniform external field B_ext (T). */
MCQ_API int mcq_set_bext(mcq_ctx *, const double B[3]);

/* Cavity vacuum field B_rms: a per-cell map (3N floats interleaved, T) or, if map is
 * NULL, the uniform vector `uniform` (T).  The cavity is enabled iff B_rms is nonzero (C14). */
MCQ_API int mcq_set_brms(mcq_ctx *, const float *map, const double uniform[3]);

/* Cavity parameters: f_c (Hz, > 0), kappa (rad/s, >= 0), x0 = 2 Re alpha_0, p0 = -2 Im alpha_0
 * (P:362-368).  Resets the memory term (alpha <- alpha_0, t <- 0). */
MCQ_API int mcq_set_cavity(mcq_ctx *, double f_c, double kappa, double x0, double p0);

/* Interfacial DMI constant D (J/m^2; 0 = off) (P:188 lists DMI among the field terms; SURVEY
 * NEXT-4).  Reading C-DMI: B = (2D/M_s)(d_x m_z, d_y m_z, -(d_x m_x + d_y m_y)) with central
 * differences and Neumann ghosts (own m) at mesh and vacuum boundaries. */
MCQ_API int mcq_set_dmi(mcq_ctx *, double D);

/* Temperature T (K, >= 0; 0 = off) and the seed of the thermal stream (P:188 lists the thermal
 * field among the Mumax3 terms).  Reading C-TH (Mumax3's Brown field):
 * B_th = eta sqrt(2 alpha k_B T / (gamma M_s V_cell dt)) in magnetic cells, eta a standard normal
 * 3-vector per cell drawn once per mcq_run step and held for its four RK4 stages (stage 1
 * draws it and stores it in a 12-byte-per-cell device buffer the context allocates on the
 * first mcq_run with T > 0, ENOMEM if that fails; stages 2-4 reload it).  eta is
 * counter-based and reproducible: SplitMix64 started at state `seed`, counters
 * 2 (n N + g) and 2 (n N + g) + 1 for global cell g = (z ny + y) nx + x at noise step n, N
 * cells.  The noise step n counts the mcq_run steps taken since the last mcq_set_temperature
 * (or mcq_set_thermal_step): it is NOT the cavity step count and is not restarted by
 * mcq_reset_memory, mcq_relax or the cavity setters, so segments of one run never reuse a
 * draw.  Box-Muller on u1 = (h >> 40 + 1) 2^-24, u2 = (h & 0xFFFFFF)
 * 2^-24 gives eta = (r0 cos 2pi u2_0, r0 sin 2pi u2_0, r1 cos 2pi u2_1), r = sqrt(-2 ln u1).
 * mcq_get_field with MCQ_TERM_THERM returns the draw of the next step scaled for the last
 * mcq_run's dt (ESTATE before any run).  With T > 0, mcq_run_dp / mcq_run_adaptive return
 * ESTATE (defined for the fixed-step RK4 path only); mcq_relax ignores the thermal field. */
MCQ_API int mcq_set_temperature(mcq_ctx *, double T, unsigned long long seed);
/* The thermal noise step n (see mcq_set_temperature): read it (e.g. into a checkpoint) and
 * set it (resume a noisy run bit-exactly).  EINVAL for n < 0. */
MCQ_API int mcq_get_thermal_step(mcq_ctx *, long long *n);
MCQ_API int mcq_set_thermal_step(mcq_ctx *, long long n);

/* Excitation a * sinc(w_cut t) * B_rms, unnormalised sinc, t = cavity clock (C13). */
MCQ_API int mcq_set_excitation(mcq_ctx *, double amplitude, double omega_cut);

/* ResetMemoryTerm(): alpha_k <- alpha_0,k for every mode, t <- 0, step <- 0. */
MCQ_API int mcq_reset_memory(mcq_ctx *);

/* Multimode cavity (P:24 runs modes separately, calls a native multimode
 * cavity "straightforward").  Reading C-MM: mode k is its own damped oscillator with its own
 * B_rms,k, f_k, kappa_k, alpha_0,k and excitation, driven by its own overlap
 * W_k = sum_i M_s m_i . B_rms,k(r_i) through the same recursion; B' gains
 * sum_k B_rms,k (Gamma_k(t) + a_k sinc(w_k t)).  The single-mode calls above act on mode 0.
 * mcq_set_modes(n), 1 <= n <= MCQ_MAX_MODES: modes >= n return to their defaults (B_rms = 0,
 * f = 1 GHz, kappa = x0 = p0 = a = 0); resets the memory.  The *_mode calls take k < n
 * (EINVAL otherwise) and behave like their single-mode counterparts for mode k.  The clock t and
 * the step counter are shared; mcq_set_cavity_state_mode sets them together with alpha_k. */
#define MCQ_MAX_MODES 4
MCQ_API int mcq_set_modes(mcq_ctx *, int nmodes);
MCQ_API int mcq_set_brms_mode(mcq_ctx *, int k, const float *map, const double uniform[3]);
MCQ_API int mcq_set_cavity_mode(mcq_ctx *, int k, double f_c, double kappa, double x0, double p0);
MCQ_API int mcq_set_excitation_mode(mcq_ctx *, int k, double amplitude, double omega_cut);
MCQ_API int mcq_get_cavity_mode(mcq_ctx *, int k, mcq_cavity_state *out);
MCQ_API int mcq_set_cavity_state_mode(mcq_ctx *, int k, const mcq_cavity_state *in);

/* Relax (reading C15): RK4 with step dt (s) on dm/dt = -gamma m x (m x B'), cavity and
 * excitation off, t frozen; every 50 steps stop if max_i |m_i x B'_i| < torque_tol (T); at
 * most max_steps steps.  Then resets the memory term.  *steps_taken may be NULL. */
MCQ_API int mcq_relax(mcq_ctx *, double dt, double torque_tol, long long max_steps, long long *steps_taken);

/* Advance `steps` RK4 steps of size dt (s > 0), replaying a captured CUDA graph.  Enqueued on
 * the context stream; returns without synchronising.  ESTATE before the first set_m. */
MCQ_API int mcq_run(mcq_ctx *, double dt, long long steps);

/* Dormand-Prince 5(4) (Mumax3 integrates with its own adaptive solvers,
 * P:324).  Reading C-DP: standard DP tableau, every stage state renormalised (as C2), the
 * 5th-order solution propagated, error estimate err = max_i |dt sum_j (b5_j - b4_j) k_j| (max
 * over cells, fp32); the cavity memory is frozen inside a step at the stage nodes c_s (C3) and
 * advanced by the accepted step's dt (eq:Sdiscrete with the step variable).  No FSAL reuse.
 * mcq_run_dp: `steps` fixed steps of size dt (every step accepted; replayed as CUDA graphs like
 * mcq_run, no host sync).
 * mcq_run_adaptive: advances the cavity clock by `duration` (s) from its current value: an
 * attempt with err <= tol (dimensionless, |m| = 1) is accepted, else m_n and the memory are
 * left untouched; the next step is h * min(5, max(0.2, 0.9 (tol/err)^(1/5))), clipped to the
 * end time; one 4-byte device-to-host read per attempt.  Stops after max_attempts attempts.
 * *accepted, *rejected, *dt_next (each may be NULL) receive the counts and the proposed next
 * step.  EINVAL on non-positive dt0 / tol; ESTATE before set_m.  Under NCCL the error is
 * reduced with a max over ranks, so every rank takes the same decisions. */
MCQ_API int mcq_run_dp(mcq_ctx *, double dt, long long steps);
MCQ_API int mcq_run_adaptive(mcq_ctx *, double duration, double dt0, double tol, long long max_attempts,
                             long long *accepted, long long *rejected, double *dt_next);

/* OVF 2.0 vector fields (the paper hands B_rms maps to Mumax3 as
 * brmsfile.ovf; format per SPEC's ovf-io module).  Host-only, no context, no GPU.
 * mcq_ovf_read: rectangular mesh, valuedim 3, payload "Text" / "Binary 4" / "Binary 8" (check
 * values 1234567.0f / 123456789012345.0, little-endian); fills grid = (xnodes, ynodes, znodes)
 * and cell = (x/y/zstepsize, m); with out != NULL also copies the 3 nx ny nz values (x fastest,
 * float) if capacity (floats) suffices.  EINVAL with a message naming the byte offset for a bad
 * magic (OVF 1.0 is rejected), a check-value mismatch, a truncated payload or a bad header.
 * mcq_ovf_write: canonical file (fixed header order, LF, 17 significant digits in text);
 * representation 0 = text, 4 = binary 4, 8 = binary 8.  mcq_ovf_last_error: this thread's last
 * OVF error message. */
MCQ_API int mcq_ovf_read(const char *path, int grid[3], double cell[3], float *out, long long capacity);
MCQ_API int mcq_ovf_write(const char *path, const int grid[3], const double cell[3], const float *data,
                          int representation);
MCQ_API const char *mcq_ovf_last_error(void);

/* Block until all enqueued work is done; reports asynchronous kernel errors (ECUDA).  Failure
 * detection: the last stage of every step (RK4 stage 4 / DP stage 7) flags a non-finite new m
 * (through its overlap partial W_0, which any NaN / inf component turns NaN); once flagged,
 * every mcq_synchronize returns ESTATE ("diverged") until mcq_set_m installs a fresh state
 * (mcq_set_m clears the flag; a diverged run leaves the cavity memory non-finite too, so reset
 * it with mcq_reset_memory, or it flags the next step again).
 * The flag covers this process's cells (per rank under a distributed context). */
MCQ_API int mcq_synchronize(mcq_ctx *);

/* Magnetisation out, 3N floats interleaved (host / device pointer). */
MCQ_API int mcq_get_m(mcq_ctx *, float *m_out);
MCQ_API int mcq_get_m_device(mcq_ctx *, float *d_out);

/* Parity hook: B' (selected terms, MCQ_TERM_* bitmask) of the current m at the current cavity
 * time (stage 1 of the next step), 3N floats interleaved, T; vacuum cells get 0. */
MCQ_API int mcq_get_field(mcq_ctx *, float *b_out, unsigned terms);

MCQ_API int mcq_get_cavity(mcq_ctx *, mcq_cavity_state *out);
/* Bytes one mcq_get_cavity / mcq_get_cavity_mode call copies device -> host (the device-side
 * cavity record of all modes), for end-to-end traffic accounting. */
MCQ_API long long mcq_cavity_state_bytes(void);
/* Resume: sets t, alpha (re/im) and step from `in` (other fields ignored). */
MCQ_API int mcq_set_cavity_state(mcq_ctx *, const mcq_cavity_state *in);

/* CavityFeatureStatus: 1 iff some active mode's B_rms is nonzero, else 0; <0 on error. */
MCQ_API int mcq_cavity_status(const mcq_ctx *);

/* Number of library kernels launched so far (graph replays count every kernel node). */
MCQ_API long long mcq_kernel_launches(const mcq_ctx *);

/* On-device trace of the per-step observables (the spectra of P:172 are
 * the numerical FT of the spatially averaged m).  After every `every`-th completed (accepted)
 * RK4 or Dormand-Prince step the
 * cavity kernel appends one row of MCQ_TRACE_COLS doubles:
 *     t_{n+1} (s), <m_x>, <m_y>, <m_z> (mean over magnetic cells, from the same fixed-order
 *     per-CTA fp64 partials as W), Re alpha, Im alpha, W (A/m T), n+1
 * into a device buffer of `capacity` rows (0 disables; rows beyond the capacity are counted but
 * not stored).  No host synchronisation per step.  The row count restarts on every reset of the
 * cavity memory (mcq_reset_memory, mcq_set_brms, mcq_set_cavity, mcq_relax) and here.
 * EINVAL: capacity < 0 or > 2^28, every < 1; ENOMEM. */
#define MCQ_TRACE_COLS 8
MCQ_API int mcq_set_trace(mcq_ctx *, long long capacity, int every);
/* Copies min(stored, max_rows) rows (row-major, MCQ_TRACE_COLS doubles each) to the host array
 * out, stored = min(rows recorded since the last reset, capacity); *rows (may be NULL) receives
 * stored.  max_rows = 0 with out = NULL queries the count. */
MCQ_API int mcq_get_trace(mcq_ctx *, double *out, long long max_rows, long long *rows);

/* Spectroscopy on the device (the spectra are the numerical Fourier
 * transform of the spatially averaged magnetisation; couplings read off the anticrossing
 * of a bias sweep).  fp64 throughout, reading C23:
 *   x = (s - mean(s)) * window (0: none, 1: Hann = numpy.hanning), zero padded to the power of two
 *   L >= pad * n; |X_k| of its DFT for 0 < k < L/2; local maxima (|X_k| >= |X_{k-1}|,
 *   |X_k| > |X_{k+1}|) with f_k = k / (L dt) >= fmin; the npeaks (1..16) largest (ties: lower k),
 *   each at f = (k + delta) / (L dt), delta the vertex of the parabola through log|X_{k-1,k,k+1}|;
 *   written to f_out / a_out (Hz, |X|) in ascending frequency, *nfound = how many.
 * mcq_trace_peaks: s = column `column` (1..7, MCQ_TRACE_COLS order) of this context's recorded
 *   trace, dt = the recorded clock spacing; ESTATE with fewer than 3 rows.
 * mcq_trace_peaks_batch: the same for n contexts of one device at once (a bias sweep's replicas:
 *   one batched launch per FFT stage); outputs [n][npeaks], nfound[n].
 * mcq_spectrum_peaks: s = a host array of n samples spaced dt (context-free; the current device).
 * mcq_fit_anticrossing: least squares (omega_c, g) (rad/s) of the normal modes of two position-
 *   coupled oscillators, lo/hi = sqrt((w1^2 + w2^2 -+ sqrt((w1^2 - w2^2)^2 + 16 g^2 w1 w2)) / 2)
 *   with w1 = w_mag[i], w2 = omega_c, to n >= 2 measured branch pairs lo[i] < hi[i] (rad/s);
 *   Levenberg-Marquardt in fp64 on the device from (wc0, g0). */
MCQ_API int mcq_trace_peaks(mcq_ctx *, int column, int pad, int window, double fmin, int npeaks, double *f_out,
                            double *a_out, int *nfound);
MCQ_API int mcq_trace_peaks_batch(mcq_ctx **ctxs, int n, int column, int pad, int window, double fmin, int npeaks,
                                  double *f_out, double *a_out, int *nfound);
MCQ_API int mcq_spectrum_peaks(const double *signal, long long n, double dt, int pad, int window, double fmin,
                               int npeaks, double *f_out, double *a_out, int *nfound);
MCQ_API int mcq_fit_anticrossing(int n, const double *w_mag, const double *lo, const double *hi, double wc0,
                                 double g0, double *wc, double *g);

/* Measurement hook: runs `steps` steps with CUDA events around every kernel (no graph) and
 * writes the mean device time (ms) per launch of each MCQ_K_* class to kernel_ms[MCQ_NKCLASS]
 * (0 for classes not launched) and launches per step to per_step[MCQ_NKCLASS] (may be NULL). */
MCQ_API int mcq_profile_run(mcq_ctx *, double dt, long long steps, double *kernel_ms, int *per_step);

/* Padded layout: out[0..5] = Lx, Ly, Lz (zero-padded FFT lengths: next power of two >= 2n,
 * 1 if n == 1), NKX = Lx/2+1 (x-spectrum columns), P (row pitch of the spectra in complex
 * elements: NKX rounded up to a multiple of 16), number of per-CTA overlap partials. */
MCQ_API int mcq_debug_layout(const mcq_ctx *, long long out[6]);
/* Real-space demag tensor octant, fp64 (6, Lz/2+1, Ly/2+1, Lx/2+1) in XX,YY,ZZ,XY,XZ,YZ
 * order, for index offsets (i, j, k); zero where i >= nx, j >= ny or k >= nz. */
MCQ_API int mcq_debug_tensor_octant(mcq_ctx *, double *out);
/* Folded kernel spectrum, fp32 (Lz/2+1, Ly/2+1, P, 6), the 6 components (XX,YY,ZZ,XY,XZ,YZ) fastest:
 * Khat = -mu0 Ms/(Lx Ly Lz) DFT(N) (real: every component is even or odd along each axis).
 * ESTATE on a z-slab rank under NCCL, which stores only the columns of its kx slab. */
MCQ_API int mcq_debug_khat(mcq_ctx *, float *out);

MCQ_API const char *mcq_last_error(const mcq_ctx *);
MCQ_API void mcq_destroy(mcq_ctx *);

#ifdef __cplusplus
}
#endif
#endif /* MCQ_H */
