/*
 * bos_rootmusic.h — C ABI of libbosrm.so: B200 (sm_100a) windowed root-MUSIC fringe
 * demodulation for DOE-based background oriented schlieren (arxiv 1910.11872).
 *
 * No CUDA or torch types appear in these signatures: pointers are plain addresses
 * (device or host as stated per argument), sizes are ints, streams are `void*`
 * (a cudaStream_t; NULL = the legacy default stream).
 *
 * Citations: P:L<n> = line of the paper's LaTeX source; Eq.(n) = the paper's
 * equation n; [Rn] = reading of a silent/ambiguous passage, listed in DESIGN.md §3.
 *
 * ----------------------------------------------------------------------------------
 * What one call computes (Algorithm 1, for every pixel of every frame):
 *   Γ_w    = M×M window of the complex fringe signal around (px,py)      Eq.(2)
 *            rows ↔ y, columns ↔ x [R4]; offsets o = -⌊(M-1)/2⌋..⌊M/2⌋ [R2];
 *            out-of-frame samples clamp to the nearest edge sample [R1]
 *   R_y    = Γ_w Γ_w^H (sample autocorrelation, no averaging)            Eq.(4)
 *   u_1    = dominant eigenvector of R_y; v_1 ∝ Γ_w^H u_1 (SVD identity)  P:L206, Eqs.(7)-(11)
 *   U_nU_n^H = I - u_1u_1^H,  V_nV_n^H = I - v_1v_1^H                    Eqs.(11),(14)
 *   P_y(z) = z^{M-1} u_1^H(z) U_nU_n^H u_1(z), P_x likewise (degree 2M-2) Eqs.(12),(13)
 *   z_y,z_x= root closest to the unit circle (inside, tolerance band)    P:L207-208 [R6]
 *   α      = ∠ Σ Γ_w e^{-j(ω_x x + ω_y y)},  ω_y = arg z_y, ω_x = -arg z_x Eq.(15)
 *   out    = wrap(α - ref_phase) into (-π, π]  (raw α if ref_phase == NULL) [R7]
 * ----------------------------------------------------------------------------------
 *
 * Error convention: every entry point returns an int status (BOS_OK or a negative
 * code) and never aborts or exits.  Asynchronous device faults surface at the caller's
 * next synchronisation (CUDA semantics).  bos_strerror() maps a code to a static string.
 * Calls are re-entrant and thread-safe across streams.  The only global state is the
 * per-device pair of pipeline streams (+ 4 events) of bos_rootmusic_demod_stack_host,
 * created on its first use on a device and kept for the life of the process, its enqueue
 * section serialised by a per-device mutex; and a per-device cache of the strip kernels'
 * occupancy (read-only after the first launch).  BOS_THREAD_KERNEL=row|strip (environment,
 * read per launch) forces the paper path's thread-per-pixel kernel for A/B timing; the two
 * give bitwise identical results.
 */
#ifndef BOS_ROOTMUSIC_H
#define BOS_ROOTMUSIC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* complex64, interleaved (re, im) — the layout of Γ(x,y,t), Eq.(1) */
typedef struct { float re, im; } bos_cf32;

enum {
    BOS_OK = 0,
    BOS_ERR_INVALID_ARG = -1,   /* NULL required pointer, bad size, aliasing, host/device mix-up */
    BOS_ERR_UNSUPPORTED = -2,   /* model_order != 3, or window_len outside the instantiated range */
    BOS_ERR_CUDA = -3           /* a CUDA runtime call or kernel launch failed */
};

/* Per-pixel status bits written to `flags` (DESIGN.md §3 [R8]; the paper has no failure
 * handling).  Flagged pixels still receive the computed value. */
enum {
    BOS_FLAG_NONCONVERGED = 1 << 0,  /* eigen/root iteration cap hit, or no finite root */
    BOS_FLAG_AMBIGUOUS = 1 << 1,     /* two distinct-frequency root pairs within 1e-3 in |ln|z|| */
    BOS_FLAG_SMALL_GAP = 1 << 2,     /* (oracle and BOS_VARIANT_FP64 only) λ1/λ2 = σ1²/σ2² < 1.3 */
    BOS_FLAG_LOW_AMPLITUDE = 1 << 3, /* |Σ Γ_w e^{-j(...)}| < 1e-4 · M · ‖Γ_w‖_F */
    BOS_FLAG_NONFINITE = 1 << 4,     /* window has NaN/Inf; output is NaN */
    BOS_FLAG_BORDER = 1 << 5         /* informational: window clamped at the frame edge */
};

/* Window sizes with an instantiated kernel (window_len = M = 2L+1 in the paper, P:L98,
 * P:L130; even M allowed [R2]). */
#define BOS_WINDOW_LEN_MIN 3
#define BOS_WINDOW_LEN_MAX 32
#define BOS_MODEL_ORDER 3   /* Eq.(3): φ_w = α + ω_x x + ω_y y, three parameters [R3] */

/* Variants for bos_rootmusic_demod_variant: a bit mask. */
enum {
    BOS_VARIANT_PAPER = 0,  /* Algorithm 1 as published: singular vectors of Γ_w, FP32 */
    BOS_VARIANT_FB = 1,     /* NOT in the paper: forward–backward averaged covariances, see below */
    BOS_VARIANT_FP64 = 2    /* NOT in the paper (its GPU code is FP32): the whole pixel in double */
};

/*
 * bos_rootmusic_demod — demodulate n_frames frames (Algorithm 1 over every pixel).
 *
 *   frames      DEVICE, [n_frames][H][W] bos_cf32, row-major, y slow; read only.
 *               Γ(x,y,t) of Eq.(1): the analytic (complex) fringe signal, carrier allowed.
 *   n_frames    ≥ 1.   H, W: frame height/width in pixels, each ≥ window_len (SPEC's
 *               FieldTooSmall).  All device offsets are 64-bit (n_frames·H·W may exceed 2^31).
 *   window_len  M, the window side = covariance order, in
 *               [BOS_WINDOW_LEN_MIN, BOS_WINDOW_LEN_MAX].
 *   model_order must be BOS_MODEL_ORDER (3), else BOS_ERR_UNSUPPORTED.
 *   ref_phase   DEVICE [H][W] float32 wrapped reference phase, or NULL → out = raw α.
 *               May alias a frame-slice of an earlier out_phase; must not alias out_phase.
 *   out_phase   DEVICE [n_frames][H][W] float32, wrapped into (-π, π]; written.
 *               Must not overlap `frames`.
 *   flags       DEVICE [n_frames][H][W] uint8 status bits, or NULL (not written).
 *   stream      cudaStream_t (NULL = legacy default stream).  Asynchronous: returns after
 *               the launch; results are valid once `stream` has been synchronised.
 * Ownership: the caller owns and allocates every buffer; the library allocates nothing.
 * Determinism: no atomics on outputs; bitwise identical across runs and frame shardings.
 */
int bos_rootmusic_demod(const bos_cf32* frames, int n_frames, int H, int W,
                        int window_len, int model_order, const float* ref_phase,
                        float* out_phase, uint8_t* flags, void* stream);

/*
 * bos_rootmusic_demod_stack — a time-lapse stack against its own reference frame
 * (BASELINE north_star: "each flow frame's phase is differenced against the reference
 * frame").  Stream-ordered launches:
 *   ref_phase_out ← raw α of frames[ref_index] (and flags[ref_index]);
 *   out[t] ← wrap(α_t − ref_phase_out) for every t ≠ ref_index (one launch per side of it);
 *   out[ref_index] ← ref_phase_out − ref_phase_out: exactly 0, NaN where α_ref is — what
 *   demodulating the reference frame against itself would give, without doing it twice.
 *   Stacks of ≤ 2^20 pixels in all (a 512² reference + flow pair, …) instead run every frame
 *   raw in ONE launch (a one-frame launch leaves most of its last wave idle), copy the
 *   reference's α to ref_phase_out and form wrap(α_t − α_ref) by a pointwise kernel with the
 *   fused store's FP32 operations — the same outputs (an α of exactly −π, which the raw store
 *   wraps to +π, is the one case that can differ by rounding).
 *   ref_index      0 ≤ ref_index < n_frames.
 *   ref_phase_out  DEVICE [H][W] float32, written (caller-owned scratch / result); must not
 *                  overlap frames or out_phase.
 * Other arguments as bos_rootmusic_demod.
 */
int bos_rootmusic_demod_stack(const bos_cf32* frames, int n_frames, int H, int W,
                              int window_len, int model_order, int ref_index,
                              float* ref_phase_out, float* out_phase, uint8_t* flags,
                              void* stream);

/*
 * bos_rootmusic_host_workspace_bytes — DEVICE scratch size needed by
 * bos_rootmusic_demod_stack_host for frames of H×W processed chunk_frames at a time
 * (two ping-pong slots of frames + outputs + flags, plus the reference phase).
 * Returns 0 on invalid arguments.
 */
size_t bos_rootmusic_host_workspace_bytes(int H, int W, int chunk_frames, int with_flags);

/*
 * bos_rootmusic_demod_stack_host — bos_rootmusic_demod_stack on HOST buffers: the frames
 * are streamed host→device in chunks of at most chunk_frames, demodulated, and the phases
 * (and flags) streamed back, with the copies of one chunk overlapping the kernels of the
 * other on two internal streams (created on the first call on a device and reused; see
 * the file header).  The reference frame goes first, alone; the other frames follow in
 * chunks of 1, 2, 4, … up to chunk_frames, halving again over the tail, so the pipeline
 * fills and drains in about one frame's copy.  Outputs and flags equal
 * bos_rootmusic_demod_stack's bit for bit wherever both run the same kernel (every window
 * length except 11 and 14–16, whose small chunks run the row kernel instead of the implicit
 * strip kernel: equal within the parity tolerance there).
 *   h_frames     HOST [n_frames][H][W] bos_cf32 (pinned for full overlap; pageable works).
 *   h_out_phase  HOST [n_frames][H][W] float32, written.  h_flags: HOST uint8 or NULL.
 *   d_workspace  DEVICE scratch of ≥ bos_rootmusic_host_workspace_bytes(H, W, chunk_frames,
 *                h_flags != NULL) bytes, caller-owned.
 *   stream       the caller's stream; all work is ordered after prior work on it, and the
 *                host buffers are valid once `stream` is synchronised.
 */
int bos_rootmusic_demod_stack_host(const bos_cf32* h_frames, int n_frames, int H, int W,
                                   int window_len, int model_order, int ref_index,
                                   float* h_out_phase, uint8_t* h_flags,
                                   void* d_workspace, size_t workspace_bytes,
                                   int chunk_frames, void* stream);

/*
 * bos_rootmusic_demod_ex — bos_rootmusic_demod that also writes the local fringe
 * frequencies of Eq.(15): ω_y = arg z_y and ω_x = −arg z_x, rad/pixel in
 * (−π, π].
 *   omega_x, omega_y  DEVICE [n_frames][H][W] float32 each, or NULL (not written); must not
 *                     overlap frames, out_phase or each other.  NaN where the window is
 *                     non-finite.
 * Other arguments, errors and determinism as bos_rootmusic_demod.
 */
int bos_rootmusic_demod_ex(const bos_cf32* frames, int n_frames, int H, int W,
                           int window_len, int model_order, const float* ref_phase,
                           float* out_phase, uint8_t* flags, float* omega_x, float* omega_y,
                           void* stream);

/*
 * bos_rootmusic_demod_variant — bos_rootmusic_demod_ex with the variants of SURVEY §8 row f4,
 * standard root-MUSIC extensions the paper does NOT use (its Algorithm 1 is variant
 * BOS_VARIANT_PAPER with subarray_len 0, identical to bos_rootmusic_demod_ex).
 *   subarray_len  0 (or window_len): covariances of order M = window_len (Algorithm 1).
 *            3 ≤ m < M: spatially smoothed covariances of order m ([R14]): R_y = Σ over all
 *            length-m segments x of the window's columns of x x^H, R_x likewise over the
 *            conjugated length-m segments of its rows; the polynomials have degree 2m − 2
 *            (m = 3: a quartic, solved in closed form); Eq.(15) still uses the M×M window.
 *            FP32: m ≤ 16 (BOS_ERR_UNSUPPORTED above); FP64: any m ≤ M.  m < 3 or m > M:
 *            BOS_ERR_INVALID_ARG.
 *   variant  bit mask.  BOS_VARIANT_FB: u_1 = dominant eigenvector of ½(R_y + J R_y* J),
 *            v_1 = dominant eigenvector of ½(R_x + J R_x* J), R_y = Γ_wΓ_w^H,
 *            R_x = Γ_w^HΓ_w (or their order-m versions; J: the exchange matrix; the backward
 *            snapshots J·conj(x)).  Exact for the Eq.(3) plane-wave model; the rest of
 *            Algorithm 1 (Eqs.(12),(13), root selection, Eq.(15)) is unchanged.
 *            BOS_VARIANT_FP64 (alone or | BOS_VARIANT_FB): every step in double precision —
 *            Jacobi eigen-decompositions of R_y and R_x, Aberth on all 2m−2 roots to the
 *            rounding bound, Eq.(15) in double; outputs are still float32.  Also sets
 *            BOS_FLAG_SMALL_GAP (λ1/λ2 < 1.3; with FB or smoothing the smaller of the two
 *            axes').  Built for accuracy, not speed (thread-local matrices: ≈50 KB local
 *            memory per thread at M = 32).  CUDA sizes the local-memory reservation as
 *            per-thread stack × resident threads per SM × SMs (≈ 16 GB at M = 32 on a B200)
 *            on the first such launch and keeps it for the context's life: leave that much
 *            device memory free, or lower it afterwards with cudaDeviceSetLimit(
 *            cudaLimitStackSize, …) once the call has completed.
 *            Any other bit: BOS_ERR_UNSUPPORTED.
 * The FP32 variants run the hot path's kernels (FB: demod_kernel.cuh up to M = 16, the implicit
 * strip kernel demod_strip.cuh for 17…28, demod_wide.cuh beyond; smoothing:
 * demod_ss.cuh); FP64 runs demod_f64.cuh.  Other arguments, errors and determinism as
 * bos_rootmusic_demod_ex.
 */
int bos_rootmusic_demod_variant(const bos_cf32* frames, int n_frames, int H, int W,
                                int window_len, int subarray_len, int model_order, int variant,
                                const float* ref_phase, float* out_phase, uint8_t* flags,
                                float* omega_x, float* omega_y, void* stream);

/*
 * bos_index_gradient — Eq.(17): the refractive-index derivative is
 * proportional to the (unwrapped) phase,  ∂n/∂x = (1/(2 μ f_x)) · (n0 / L²) · φ.
 *   phase   DEVICE float32 [n] (a phase map/stack; unwrapping is the caller's).
 *   n0      reference refractive index (> 0); mu: the μ of Eq.(17) (> 0, read as the imaging
 *           magnification); f_x: fringe frequency (> 0, cycles per unit length);
 *           cell_len: test-cell length L along the optical axis (> 0).  Consistent units in
 *           (e.g. SI) give ∂n/∂x in the same system (1/m for SI).
 *   out     DEVICE float32 [n]; may equal `phase` (in place), must not partially overlap it.
 * Returns BOS_ERR_INVALID_ARG for NULL/host pointers, n == 0 or non-positive parameters.
 */
int bos_index_gradient(const float* phase, size_t n, double n0, double mu, double f_x,
                       double cell_len, float* out, void* stream);

/*
 * bos_vertical_profile — SURVEY §8 row f3 ("diffusion profiles"; SPEC stack_series,
 * S:L395-401): the per-frame vertical profile of a phase (or ∂n/∂x) stack, the mean over the
 * columns x of every row y, for the paper's time-evolution comparison (Figs. 6-8).
 *   phase  DEVICE float32 [n_frames][H][W].  Non-finite pixels are skipped; a row without
 *          finite pixels gives NaN.  Accumulated in FP64, stored as float32.
 *   out    DEVICE float32 [n_frames][H]; must not overlap `phase`.
 * Returns BOS_ERR_INVALID_ARG for NULL/host pointers, non-positive sizes or overlap.
 */
int bos_vertical_profile(const float* phase, int n_frames, int H, int W, float* out, void* stream);

/*
 * bos_analytic_signal — SURVEY §8 row f1, the step before the path: the analytic (complex)
 * fringe signal Γ of Eq.(1) from 8-bit intensity frames by "bandpass filtering and carrier
 * removal".  Per frame: I/255 → 2-D FFT → keep the disc of radius `radius`
 * (cycles/pixel) around the carrier (fx, fy) → inverse FFT → if `remove_carrier`,
 * Γ·e^{−j2π(fx·x + fy·y)}.  The filter is a hard circular mask ([R11]; the paper names none).
 *   frames_u8   DEVICE [n_frames][H][W] uint8 intensities.  H, W ≥ 2.
 *   fx, fy      carrier in cycles/pixel, |fx|, |fy| ≤ 0.5; the disc must exclude DC
 *               (fx² + fy² > radius²), else BOS_ERR_INVALID_ARG.
 *   out         DEVICE [n_frames][H][W] bos_cf32, written (the cuFFT path also uses it as
 *               the FFT buffer, in place); must not overlap frames_u8.
 *   d_workspace DEVICE work area of ≥ bos_analytic_signal_workspace_bytes(H, W, n_frames)
 *               bytes, caller-owned: the fused path's spectral-column buffer (8 frames ×
 *               H·W·8 B at most) or the cuFFT work area.
 *   stream      cudaStream_t.  Power-of-two H, W ≤ 4096: the fused pruned transform
 *               (hand-written kernels: rows FFT → the disc's columns only → columns FFT, mask,
 *               inverse → rows inverse FFT + carrier removal), stream-ordered, no
 *               synchronisation.  Other sizes: cuFFT (library FFT, plans made and destroyed per
 *               call); the call then returns after the work has completed (it synchronises
 *               `stream` before destroying its plans) — repeated calls should use the planned
 *               form below: cuFFT plan creation costs milliseconds to hundreds of ms of host time.
 */
size_t bos_analytic_signal_workspace_bytes(int H, int W, int n_frames);
int bos_analytic_signal(const uint8_t* frames_u8, int n_frames, int H, int W,
                        double fx, double fy, double radius, int remove_carrier,
                        bos_cf32* out, void* d_workspace, size_t workspace_bytes, void* stream);

/*
 * Planned form of bos_analytic_signal: a caller-owned plan holds the cuFFT plans for H×W
 * frames (a batch of min(max_frames, 8) frames and a single frame for ragged tails), so
 * repeated calls make no plans and do not synchronise (stream-ordered, asynchronous).
 *   bos_analytic_plan_create  H, W ≥ 2, max_frames ≥ 1; *plan receives the handle;
 *                             *workspace_bytes (if not NULL) the cuFFT work-area size the
 *                             planned calls need.  BOS_ERR_CUDA if cuFFT fails.
 *   bos_analytic_signal_planned  as bos_analytic_signal with H, W taken from the plan; any
 *                             n_frames ≥ 1.  A plan must not be used by two calls at once
 *                             (it binds the work area and stream per call).
 *   bos_analytic_plan_destroy releases the plan (NULL is a no-op); the caller first makes
 *                             sure no planned call on it is still executing.
 */
typedef struct bos_analytic_plan bos_analytic_plan;
int bos_analytic_plan_create(int H, int W, int max_frames, bos_analytic_plan** plan,
                             size_t* workspace_bytes);
int bos_analytic_signal_planned(bos_analytic_plan* plan, const uint8_t* frames_u8, int n_frames,
                                double fx, double fy, double radius, int remove_carrier,
                                bos_cf32* out, void* d_workspace, size_t workspace_bytes,
                                void* stream);
int bos_analytic_plan_destroy(bos_analytic_plan* plan);

/*
 * bos_unwrap — SURVEY §8 row f2, the step after the path: 2-D phase unwrapping "followed by
 * an unwrapping operation" with the cited reliability-sorting algorithm (Herráez):
 * reliability R = 1/sqrt(H²+V²+D1²+D2²) of wrapped second differences (edge-replicated
 * neighbours), edges ranked by R(p)+R(q) (ties: edge id 2p horizontal / 2p+1 vertical),
 * groups merged along the maximum spanning tree, one global 2π multiple fixed by the most
 * reliable pixel ([R12]).  Built as Borůvka rounds + weighted union-find on the GPU; the
 * 2π multiples equal the sequential FP64 algorithm's exactly (FP64 reliabilities).
 *   wrapped     DEVICE [n_frames][H][W] float32 wrapped phase (e.g. out_phase of the demod).
 *   unwrapped   DEVICE [n_frames][H][W] float32 = wrapped + 2π·k; may equal `wrapped`
 *               (in place), must not partially overlap it.  NaN/Inf pixels stay as they are
 *               (and count as 0 in the neighbours' second differences).
 *   d_workspace DEVICE scratch, caller-owned: bos_unwrap_workspace_bytes(H, W, F) bytes lets the
 *               call unwrap F frames per batch (one union-find forest); any size ≥ the 1-frame
 *               figure works (fewer frames per batch).  2·F·H·W < 2^32.
 *   stream      cudaStream_t; the call is synchronous (it reads back a convergence flag
 *               after each union round) and returns after the frames are done.
 */
size_t bos_unwrap_workspace_bytes(int H, int W, int n_frames);
int bos_unwrap(const float* wrapped, int n_frames, int H, int W, float* unwrapped,
               void* d_workspace, size_t workspace_bytes, void* stream);

/*
 * bos_rootmusic_iteration_counts — measurement support for the roofline:
 * runs the same kernel with per-pixel iteration counters over `frames` (DEVICE, as in
 * bos_rootmusic_demod) and accumulates into d_counters (DEVICE, 4 × uint64, caller zeroes):
 *   [0] pixels processed, [1] Σ power iterations, [2] Σ Aberth sweeps (y), [3] Σ Aberth
 * sweeps (x).  Results identical to bos_rootmusic_demod (out_phase is written too).
 */
int bos_rootmusic_iteration_counts(const bos_cf32* frames, int n_frames, int H, int W,
                                   int window_len, int model_order, const float* ref_phase,
                                   float* out_phase, unsigned long long* d_counters,
                                   void* stream);

/* Static, never-NULL description of a status code. */
const char* bos_strerror(int code);

/* ABI version: (major << 16) | minor. */
int bos_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* BOS_ROOTMUSIC_H */
