/* include/sf_b200.h — C ABI of the B200-native stencil hot path.
 *
 * Drop-in boundary for the reference's generated-kernel FFI. In the reference
 * (stencilforge, /root/reference/proj) Operator::build() JIT-compiles C99 and
 * dlsym()s an entry with the signature
 *
 *     int Operator(float *u_vec, float *m_vec, float *eta_vec, float *src_vec,
 *                  int *src_ci_vec, float *src_w_vec, float *rec_vec,
 *                  int *rec_ci_vec, float *rec_w_vec);      (golden acoustic_3d.c:3)
 *     int Operator(float *u_vec);                          (golden diffusion_1000.c:3)
 *
 * which Operator::apply() calls through CompiledKernel::invoke(span<void*>)
 * (jit.cpp:104-148, op.cpp:126-161): one flat dense pointer per referenced
 * GridFunction in grid declaration order (codegen.cpp:398-409), shapes and
 * folded constants baked in at build time, all nt steps run in one call,
 * status 0 on success (codegen.cpp:499). This header replaces that pair:
 *
 *   jit_compile(source, cfg, sig)      jit.cpp:150-195  -> sf_*_plan_create
 *   CompiledKernel::invoke(args)       jit.cpp:104-148  -> sf_plan_invoke
 *   generated Operator(u, m, eta, ...) acoustic_3d.c:3  -> sf_acoustic_apply
 *   generated Operator(u)              diffusion_1000.c -> sf_diffusion_apply
 *
 * Buffers passed to apply/invoke are HOST pointers in the reference's dense
 * row-major layout with the time slot slowest (grid.cpp:89-101). The plan keeps
 * HBM-resident padded mirrors; the call uploads, runs every step on the GPU,
 * and downloads every written buffer (all time slots, sparse series), which is
 * what the reference leaves in host memory on return.
 *
 * Errors: every entry returns an sf_status; sf_last_error() gives the message
 * (thread-local). There is no CPU fallback: without a usable sm_100 device the
 * plan constructors fail with SF_ERR_CUDA.
 */
#ifndef SF_B200_H
#define SF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SF_OK = 0,
    SF_ERR_INVALID = 1,        /* bad argument (InvalidShape/InvalidOrder, error.hpp) */
    SF_ERR_CFL = 2,            /* CflViolationError (acoustic.cpp:133-137) */
    SF_ERR_OUT_OF_DOMAIN = 3,  /* OutOfDomainError (sparse.cpp:19-25) */
    SF_ERR_SIGNATURE = 4,      /* SignatureMismatchError (op.cpp:135-155) */
    SF_ERR_KERNEL = 5,         /* KernelFailedError (op.cpp:156-159) */
    SF_ERR_CUDA = 6,           /* device missing / CUDA runtime failure */
    SF_ERR_OOM = 7             /* device allocation failed */
} sf_status;

typedef struct sf_plan sf_plan;

/* What the reference bakes into the generated acoustic kernel at build time
 * (acoustic.cpp:128-200 -> op.cpp:55-92 -> codegen.cpp:411-502). */
typedef struct {
    int ndim;            /* 2 or 3 spatial dimensions */
    int64_t shape[3];    /* spatial extents, axis 0 slowest (boundary included) */
    int space_order;     /* even, 2..16 */
    int forward;         /* 1: forward u (t = 0..nt-1); 0: adjoint v (t = nt..1) */
    int64_t nt;          /* time steps */
    double dt;           /* seconds (effective dt; CFL checked by the caller) */
    double spacing;      /* metres, equal on every axis */
    int64_t n_src;       /* points in the "src" set */
    int64_t n_rec;       /* points in the "rec" set */
} sf_acoustic_desc;

/* DiffusionConfig (diffusion.hpp:13-26) with exact rational alpha and dx=dy. */
typedef struct {
    int64_t nx, ny;
    int order;           /* even, 2..16 */
    int64_t nt;
    int64_t alpha_num, alpha_den;
    int64_t dx_num, dx_den;
} sf_diffusion_desc;

const char *sf_last_error(void);
int sf_device_count(void);

/* ---- plans (== jit_compile) ------------------------------------------- */
int sf_acoustic_plan_create(const sf_acoustic_desc *desc, int device, sf_plan **out);
int sf_diffusion_plan_create(const sf_diffusion_desc *desc, int device, sf_plan **out);
void sf_plan_destroy(sf_plan *plan);
/* Same plans with the folded constants supplied by the caller instead of
 * derived from dt/spacing/alpha: the layout of sf_acoustic_constants /
 * sf_diffusion_constants. Used by the C-source front end (sf-cuda-cc), which
 * lifts the literals from the reference's generated kernel. */
int sf_acoustic_plan_create_ex(const sf_acoustic_desc *desc, const float *constants /* [15] */,
                               const int *time_sel /* [3] */, int device, sf_plan **out);
int sf_diffusion_plan_create_ex(const sf_diffusion_desc *desc, float c0, int has_c0,
                                const float *cj /* [8] */, int device, sf_plan **out);

/* Number of buffers the entry takes and their names in declaration order
 * (KernelSignature, codegen.hpp:21-29). */
int sf_plan_num_args(const sf_plan *plan);
const char *sf_plan_arg_name(const sf_plan *plan, int i);
/* Byte size of argument i in the dense reference layout. */
int64_t sf_plan_arg_bytes(const sf_plan *plan, int i);

/* ---- the generated-kernel entries (== Operator(...)) --------------------
 * Acoustic, forward run: (u, m, eta, src, src_ci, src_w, rec, rec_ci, rec_w)
 * Acoustic, adjoint run: (v, m, eta, src, src_ci, src_w, rec, rec_ci, rec_w)
 *   forward injects src[t] into level t+1 and samples rec[t];
 *   adjoint injects rec[t-1] into level t-1 and samples src[t-1].          */
int sf_acoustic_apply(sf_plan *plan, float *u_vec, float *m_vec, float *eta_vec,
                      float *src_vec, int *src_ci_vec, float *src_w_vec,
                      float *rec_vec, int *rec_ci_vec, float *rec_w_vec);
int sf_diffusion_apply(sf_plan *plan, float *u_vec);
/* CompiledKernel::invoke: args in signature order, nargs checked. */
int sf_plan_invoke(sf_plan *plan, void *const *args, int nargs);

/* ---- HBM-resident control (benchmarks, FWI, multi-step drivers) ---------
 * upload: host args -> device mirrors (NULL entries skipped);
 * run:    steps [step_begin, step_end) of the time loop on the device
 *         (step index k = 0..nt-1 maps to reference t = k forward,
 *          t = nt-k adjoint), no host copies;
 * download: device mirrors -> host args (NULL entries skipped).          */
int sf_plan_upload(sf_plan *plan, void *const *args, int nargs);
int sf_plan_run(sf_plan *plan, int64_t step_begin, int64_t step_end);
int sf_plan_download(sf_plan *plan, void *const *args, int nargs);
int sf_plan_synchronize(sf_plan *plan);

/* Device-timed run of all nt steps from the current resident state, CUDA
 * events on the plan's stream. total_ms: whole loop; stencil_ms: summed time
 * of the stencil launches measured in a separate identical pass (NULL to
 * skip). Restores nothing: callers re-upload between timed runs. */
int sf_plan_time(sf_plan *plan, float *total_ms, float *stencil_ms,
                 int64_t *kernel_launches);

/* ---- FWI gradient (config 5; no reference implementation) -------------
 * Forward with full history in HBM (nt+2 levels), then the adjoint sweep
 * fused with grad += u(t) * vtt(t) on the interior.
 * forward plan: fwd desc; args (m, eta, src, src_ci, src_w, rec_ci, rec_w)
 * residual: rec-shaped [nt][n_rec] series injected by the adjoint.
 * Outputs: rec traces of the forward [nt][n_rec], gradient (dense field).  */
int sf_fwi_plan_create(const sf_acoustic_desc *desc, int device, sf_plan **out);
int sf_fwi_gradient(sf_plan *plan, const float *m, const float *eta,
                    const float *src, const int *src_ci, const float *src_w,
                    const int *rec_ci, const float *rec_w, const float *residual,
                    float *rec_out, float *grad_out, float *v_out /* 3 slots or NULL */,
                    float *src_adj_out /* [nt][n_src] or NULL */);
int sf_fwi_time(sf_plan *plan, float *fwd_ms, float *adj_ms);

/* ---- host-side setup mirrors of the reference (no GPU needed) --------- */
/* interpolation_weights (sparse.cpp:11-41), weights narrowed to f32 as
 * GridFunction::set stores them. Returns SF_ERR_OUT_OF_DOMAIN outside. */
int sf_interpolation_weights(int ndim, const double *coord, double spacing,
                             const int64_t *extents, int32_t *cell, float *w);
/* AcousticModel::stable_dt (acoustic.cpp:20-34) */
double sf_stable_dt(int ndim, int space_order, double spacing, double v_top,
                    double v_bottom);
/* ricker_wavelet (acoustic.cpp:10-14) */
double sf_ricker(double f0, double t, double t0);
/* build_medium (acoustic.cpp:67-105); v_field != NULL overrides the
 * two-layer velocity with a per-cell field (random media), v_min sets the
 * sponge strength. */
int sf_build_medium(int ndim, const int64_t *shape, int boundary_width,
                    double spacing, double v_top, double v_bottom,
                    const double *v_field, double v_min, float *m, float *eta);
/* ---- seeded smooth random media (configs C3/C4/C5) ---------
 * Velocity = seeded hash noise filtered by a separable Gaussian (sigma cells,
 * radius int(4 sigma + 0.5), mirrored at the faces), rescaled to
 * [v_lo, v_hi] with the extrema of the GLOBAL grid; m / eta then follow
 * build_medium (acoustic.cpp:67-105) per cell, from global indices. Every
 * value depends only on its global index, so slabs generate their own planes
 * (src/medium.cu documents the exact definition; oracle/sf_port.c restates
 * it for the tests). No reference counterpart: the reference takes media
 * only as host arrays (GridFunction::set, grid.cpp:103-126).             */
typedef struct {
    int64_t shape[3];          /* global extents, axis 0 slowest */
    int64_t a0_begin, a0_end;  /* global axis-0 planes to generate */
    uint64_t seed;
    double sigma;              /* filter width in cells */
    double v_lo, v_hi;         /* velocity range after the rescale, m/s */
    int boundary_width;        /* sponge, as build_medium */
    double spacing;
    double v_min;              /* sponge strength (build_medium's v_min) */
} sf_smooth_medium_desc;
/* Extrema of the filtered noise over planes [a0_begin, a0_end) (slabs: take
 * the min / max over ranks before generating). */
int sf_smooth_extrema(const sf_smooth_medium_desc *desc, int device, double *lo, double *hi);
/* m, eta of planes [a0_begin, a0_end) into dense host arrays. */
int sf_smooth_medium(const sf_smooth_medium_desc *desc, double lo, double hi, int device,
                     float *m, float *eta);
/* Same, straight into a plan's resident m / eta (HBM, no host copy): the
 * plan's own planes (slab plans: global plane0 .. plane0 + local n0) of the
 * global grid desc->shape; desc->a0_begin/a0_end are ignored. */
int sf_plan_set_smooth_medium(sf_plan *plan, const sf_smooth_medium_desc *desc, double lo,
                              double hi);

/* Folded fp32 stencil constants the plan uses (for inspection/tests):
 * out[0]=ce, [1]=cm, [2..4]=time-term coefficients in emitted order,
 * [5]=centre, [6..6+r)=neighbour j=1..r, [14]=injection scale;
 * time_sel[k] = 2*field(0 eta,1 m) + level(0 prev,1 cur). */
int sf_acoustic_constants(int ndim, int space_order, int forward, double dt,
                          double spacing, float *out /* [15] */, int *time_sel /* [3] */);

/* ---- depth-slab decomposition (multi-GPU) -----------------
 * A slab plan owns global axis-0 planes [own_begin, own_end) of a grid with
 * global_n0 planes (own_end - own_begin >= r = space_order/2) and stores the
 * r-deep halos on each internal side: desc->shape[0] = local planes with
 * plane0 = max(own_begin - r, 0) the global index of local plane 0 and
 * plane0 + shape[0] = min(own_end + r, global_n0). Buffers passed to the
 * plan are the matching local slices (halo planes included); sparse cell
 * indices are local. The slab updates only owned interior planes, applies
 * only the injection corners it owns, and after each step's injection swaps
 * r planes of the new level with its neighbours before sampling, so the
 * result is bitwise the single-domain run. */
typedef struct {
    int64_t global_n0;
    int64_t plane0;
    int64_t own_begin, own_end;
} sf_slab_desc;

int sf_acoustic_plan_create_slab(const sf_acoustic_desc *desc, const sf_slab_desc *slab,
                                 int device, sf_plan **out);
/* Steps [step_begin, step_end) of an in-process chain of adjacent slab plans
 * (ordered by depth; one or several devices), halo copies device-to-device. */
int sf_slab_chain_run(sf_plan *const *plans, int nplans, int64_t step_begin, int64_t step_end);
/* One process per GPU: NCCL send/recv halo exchange inside every step of
 * sf_plan_run / sf_plan_invoke. id = 128-byte ncclUniqueId from rank 0. */
int sf_nccl_unique_id(void *out, int bytes);
int sf_plan_attach_nccl(sf_plan *plan, const void *id, int nranks, int rank);

/* ---- HBM-resident buffer I/O (save_buffer / load_buffer, grid.cpp:213-254)
 * Argument `name` (signature name, e.g. "u", "m", "rec") written from / read
 * into the plan's device mirror in the reference's SFG1 binary format, so
 * files interchange with the reference's own save_buffer/load_buffer. */
int sf_plan_save_buffer(sf_plan *plan, const char *name, const char *path);
int sf_plan_load_buffer(sf_plan *plan, const char *name, const char *path);

/* Text dumps from the device mirror: dump_csv (grid.cpp:256-273; 2D grid
 * functions only, `slot` selects the time slot of u/v) and save_series_text
 * (sparse.cpp:215-227; "src"/"rec", one row per time step, space-separated).
 * Numbers are formatted like `std::ostream << double` (printf "%g"). */
int sf_plan_dump_csv(sf_plan *plan, const char *name, const char *path, long slot);
int sf_plan_save_series_text(sf_plan *plan, const char *name, const char *path);

/* ---- GPU autotune (Operator::autotune, op.cpp:169-221) -----------------
 * Times every stencil kernel variant compiled for the plan's order (kernel
 * family, tile, pipeline depth) on `tune_steps` steps of the resident state,
 * median of `repeats` runs with the state restored before each, keeps the
 * fastest and restores the state. kind: 0 per-thread loads, 1 scalar TMA,
 * 2 vector TMA ring, 3 queue-vector TMA. */
typedef struct {
    int kind, tile_nx, tile_ty, vec_warps, stages;
    float median_ms;
} sf_tune_entry;
int sf_plan_autotune(sf_plan *plan, int64_t tune_steps, int repeats, sf_tune_entry *entries,
                     int max_entries, int *n_entries);

/* Folded diffusion constants (exact rationals -> double -> f32). */
int sf_diffusion_constants(int order, int64_t alpha_num, int64_t alpha_den, int64_t dx_num,
                           int64_t dx_den, float *c0, int *has_c0, float *cj /* [8] */);

/* Self-test of the stencil kernels' reciprocal (1.0f / x, exact IEEE
 * round-to-nearest via MUFU.RCP + one Newton step with a slow-path guard)
 * against __frcp_rn over all 2^32 float bit patterns; *mismatches = count. */
int sf_selftest_reciprocal(int device, unsigned long long *mismatches);

/* Measurement hook (no reference counterpart): fraction of the interior
 * point updates per step whose eta box the vector kernels skip because it is
 * all +0.0 (the undamped interior; the kernels then use 0.0f, bitwise the
 * value they would have read). Valid after a run; 0 when the skip is off. */
int sf_plan_eta_skip_fraction(sf_plan *plan, double *fraction);

#ifdef __cplusplus
}
#endif

#endif
