/* oracle/sf_port.h — plain-C restatement of the reference's hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the CPU checker the parity tests compare
 * the CUDA path against; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it. The product (paper_1609_03361_b200/) never
 * links or calls it.
 *
 * Every routine restates the arithmetic the reference's generated C kernel
 * performs (golden tests/golden/acoustic_3d.c, diffusion_1000.c), in the same
 * fp32 operation order, compiled with -ffp-contract=off like jit.cpp:70, so
 * results are bitwise comparable. The port is pinned against the reference
 * itself (oracle/_ref/libsf_ref.so) by tests/test_oracle_pin.py and against
 * the committed golden fixtures in tests/golden/.
 *
 * Layout: the reference's dense row-major layout with the slot slowest,
 * u[slot][a0][a1][a2] (grid.cpp:89-101); axis 0 is the slowest spatial axis.
 */
#ifndef SF_PORT_H
#define SF_PORT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* exact rational (int64 num/den, lowest terms, den > 0) */
typedef struct {
    int64_t num;
    int64_t den;
} sfp_rat;

/* Centered second-derivative weights at accuracy `order` (offsets -r..r,
 * r = order/2), exact. Restates fd_weights(2, centered_offsets(2, order))
 * (fd.cpp:28-92) through the Lagrange form instead of Gauss-Jordan.
 * Returns 0 on success. */
int sfp_fd_weights2(int order, sfp_rat *w /* [2r+1] */);

/* Folded fp32 constants of the acoustic update, derived the way the
 * reference's CAS folds them (expr.cpp ConstVal arithmetic after
 * fold_scalars opt.cpp:106-133): rational weights widened to double, times
 * std::pow(h, -2) / std::pow(dt, -k), then rounded to float
 * (codegen.cpp:15-36). */
typedef struct {
    int ndim;        /* 2 or 3 */
    int order;       /* space order 2..16 */
    int forward;     /* 1 forward, 0 adjoint */
    float ce;        /* 1/(2 dt): temp0 = ce*eta */
    float cm;        /* 1/dt^2:   temp1 = cm*m */
    /* the three time terms in emitted order: coefficient, field (0 = eta,
     * 1 = m) and which level it multiplies (0 = "prev", 1 = "cur") */
    float tc[3];
    int tfield[3];
    int tlevel[3];
    float c0;        /* merged centre coefficient */
    float cj[8];     /* neighbour coefficient for |offset| = j+1 */
    float src_scale; /* dt^2, the injection scale s^2 (acoustic.cpp:160-161) */
} sfp_acoustic_coefs;

int sfp_make_acoustic_coefs(int ndim, int order, int forward, double dt,
                       double spacing, sfp_acoustic_coefs *out);

/* AcousticModel::stable_dt (acoustic.cpp:20-34). */
double sfp_stable_dt(int ndim, int order, double spacing, double v_top,
                     double v_bottom);

/* ricker_wavelet (acoustic.cpp:10-14). */
double sfp_ricker(double f0, double t, double t0);

/* interpolation_weights (sparse.cpp:11-41); weights stored as f32 the way
 * GridFunction::set does (grid.cpp:113-126). Returns 0, or 3 when the point
 * is outside the grid (OutOfDomainError). */
int sfp_interp_weights(int ndim, const double *coord, double spacing,
                       const int64_t *extents, int32_t *cell, float *w);

/* build_medium (acoustic.cpp:67-105): two layers split at a0 < shape0/2,
 * quadratic sponge, eta = m * sigma. */
void sfp_build_medium(int ndim, const int64_t *shape, int boundary_width,
                      double spacing, double v_top, double v_bottom, float *m,
                      float *eta);

/* Same sponge applied to an arbitrary velocity field (random media for
 * configs 3-5): m = 1/v^2 in double then f32, eta = m * sigma(d) with
 * sigma_max from v_min. */
void sfp_medium_from_velocity(int ndim, const int64_t *shape,
                              int boundary_width, double spacing, double v_min,
                              const double *v, float *m, float *eta);

/* The generated acoustic Operator() (golden acoustic_3d.c:14-60) for
 * forward (t = 0..nt-1, writes slot (t+1)%3) or adjoint (t = nt..1, writes
 * slot (t+2)%3 = level t-1) runs. inj = the injecting point set (src
 * forward, rec adjoint), smp = the sampled set (rec forward, src adjoint).
 * u holds 3 slots. nthreads <= 0 uses OpenMP's default. */
int sfp_acoustic_run(const sfp_acoustic_coefs *c, const int64_t *shape,
                     int64_t nt, float *u, const float *m, const float *eta,
                     const float *inj, const int32_t *inj_ci,
                     const float *inj_w, int64_t n_inj, float *smp,
                     const int32_t *smp_ci, const float *smp_w, int64_t n_smp,
                     int nthreads);

/* FWI forward with full history (config 5): hist holds nt+2 levels,
 * hist[L] = u(L-1), hist[0] = hist[1] = 0 on entry; level L+1 is computed
 * from L and L-1 with the forward arithmetic above, source injected and
 * receivers sampled exactly as in sfp_acoustic_run. Bitwise equal to the
 * 3-slot forward run (same arithmetic, different storage). */
int sfp_acoustic_forward_history(const sfp_acoustic_coefs *c,
                                 const int64_t *shape, int64_t nt, float *hist,
                                 const float *m, const float *eta,
                                 const float *src, const int32_t *src_ci,
                                 const float *src_w, int64_t nsrc, float *rec,
                                 const int32_t *rec_ci, const float *rec_w,
                                 int64_t nrec, int nthreads);

/* FWI adjoint + gradient (config 5; NEW, no reference implementation:
 * parity unpinned). Runs the adjoint exactly as sfp_acoustic_run (forward=0)
 * on the 3 slots of v, and accumulates on the interior
 *   grad += u(t) * vtt(t),  vtt(t) = ((v(t+1) - 2 v(t)) + v(t-1)) * cm
 * for t = 1..nt, each term once v(t-1) is final (after injection), in
 * increasing-step-index order of the sweep (t = nt first). u(t) =
 * hist[t+1]. fp32, no contraction. */
int sfp_fwi_adjoint_gradient(const sfp_acoustic_coefs *c, const int64_t *shape,
                             int64_t nt, float *v, const float *m,
                             const float *eta, const float *hist,
                             const float *rec, const int32_t *rec_ci,
                             const float *rec_w, int64_t nrec, float *src,
                             const int32_t *src_ci, const float *src_w,
                             int64_t nsrc, float *grad, int nthreads);

/* DiffusionConfig::dt (diffusion.cpp:10-23), exact. */
int sfp_diffusion_dt(sfp_rat alpha, sfp_rat dx, int order, sfp_rat *dt);

/* Folded diffusion constants (exact rationals widened to double, then f32):
 * centre (may be exactly zero -> dropped) and neighbours j = 1..r. */
int sfp_diffusion_coefs(sfp_rat alpha, sfp_rat dx, int order, float *c0,
                        int *has_c0, float *cj /* [8] */);

/* The generated diffusion Operator() (golden diffusion_1000.c): 2 slots,
 * t = 0..nt-1 writes slot (t+1)%2. */
int sfp_diffusion_run(int64_t nx, int64_t ny, int order, float c0, int has_c0,
                      const float *cj, int64_t nt, float *u, int nthreads);


/* Seeded smooth random medium (configs C3/C4/C5): the definition stated in
 * paper_1609_03361_b200/csrc/medium.cu, restated here. Taps: returns the
 * filter radius (or -1), g[0..2*rad]. Extrema of the filtered noise over
 * global planes [b, e); m / eta (dense [e-b][n1][n2]) of those planes from
 * the global extrema lo / hi. Returns 0 on success. */
int sfp_smooth_taps(double sigma, double *g /* [129] */);
int sfp_smooth_extrema(const int64_t *shape, int64_t b, int64_t e, uint64_t seed,
                       double sigma, double *lo, double *hi);
int sfp_smooth_medium(const int64_t *shape, int64_t b, int64_t e, uint64_t seed,
                      double sigma, double v_lo, double v_hi, int boundary_width,
                      double spacing, double v_min, double lo, double hi, float *m,
                      float *eta);

#ifdef __cplusplus
}
#endif

#endif
