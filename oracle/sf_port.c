/* oracle/sf_port.c — plain-C restatement of the reference hot path.
 * TEST INFRASTRUCTURE ONLY (see sf_port.h). Compiled with
 * -ffp-contract=off -fno-fast-math like the reference JIT (jit.cpp:70). */
#include "sf_port.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------
 * exact rationals (the reference's sf::Rational, rational.hpp:13-127) */

typedef __int128 i128;

static i128 gcd128(i128 a, i128 b) {
    if (a < 0) a = -a;
    if (b < 0) b = -b;
    while (b != 0) {
        i128 t = a % b;
        a = b;
        b = t;
    }
    return a == 0 ? 1 : a;
}

static int rat_make(i128 n, i128 d, sfp_rat *out) {
    if (d == 0) return 1;
    if (d < 0) {
        n = -n;
        d = -d;
    }
    i128 g = gcd128(n, d);
    n /= g;
    d /= g;
    if (n > INT64_MAX || n < INT64_MIN || d > INT64_MAX) return 1;
    out->num = (int64_t)n;
    out->den = (int64_t)d;
    return 0;
}

static sfp_rat R(int64_t n, int64_t d) {
    sfp_rat r;
    rat_make(n, d, &r);
    return r;
}
static sfp_rat rmul(sfp_rat a, sfp_rat b) {
    sfp_rat r;
    rat_make((i128)a.num * b.num, (i128)a.den * b.den, &r);
    return r;
}
static sfp_rat rdiv(sfp_rat a, sfp_rat b) {
    sfp_rat r;
    rat_make((i128)a.num * b.den, (i128)a.den * b.num, &r);
    return r;
}
static sfp_rat radd(sfp_rat a, sfp_rat b) {
    sfp_rat r;
    rat_make((i128)a.num * b.den + (i128)b.num * a.den, (i128)a.den * b.den, &r);
    return r;
}
/* Rational::to_double (rational.hpp:24-26) */
static double rdbl(sfp_rat a) { return (double)a.num / (double)a.den; }

/* ------------------------------------------------------------------------
 * FD weights: Lagrange-basis second derivative at 0 over integer offsets
 * -r..r. For p(x) = sum_k w_k L_k(x), w_k = L_k''(0) = 2 * [x^2] L_k(x).
 * Exact; equals fd_weights(2, centered_offsets(2, order)) (fd.cpp:28-92),
 * which acceptance criterion 1 pins against the same Lagrange form. */
int sfp_fd_weights2(int order, sfp_rat *w) {
    if (order < 2 || order % 2 != 0 || order > 16) return 1;
    int r = order / 2, n = 2 * r + 1;
    for (int k = 0; k < n; ++k) {
        int xk = k - r;
        /* polynomial prod_{j != k} (X - x_j), integer coefficients, only
         * degrees 0..2 are needed but the full product is small */
        i128 poly[17];
        memset(poly, 0, sizeof poly);
        poly[0] = 1;
        int deg = 0;
        i128 denom = 1;
        for (int j = 0; j < n; ++j) {
            if (j == k) continue;
            int xj = j - r;
            denom *= (i128)(xk - xj);
            for (int i = deg + 1; i >= 1; --i) poly[i] = poly[i - 1] - (i128)xj * poly[i];
            poly[0] = -(i128)xj * poly[0];
            ++deg;
        }
        if (rat_make(2 * poly[2], denom, &w[k])) return 1;
    }
    return 0;
}

/* ------------------------------------------------------------------------
 * folded acoustic constants */

int sfp_make_acoustic_coefs(int ndim, int order, int forward, double dt,
                       double spacing, sfp_acoustic_coefs *c) {
    sfp_rat w[17];
    if (ndim < 2 || ndim > 3) return 1;
    if (sfp_fd_weights2(order, w)) return 1;
    int r = order / 2;
    memset(c, 0, sizeof *c);
    c->ndim = ndim;
    c->order = order;
    c->forward = forward;
    /* Expr::pow(real, int) folds with std::pow (expr.cpp:526-527) */
    double inv_dt = pow(dt, -1.0);
    double inv_dt2 = pow(dt, -2.0);
    double inv_h2 = pow(spacing, -2.0);
    /* A = 1/2*eta*s^-1 + m*s^-2: ConstVal (1/2)*pow(s,-1) and 1*pow(s,-2) */
    double ce = 0.5 * inv_dt;
    double cm = inv_dt2;
    c->ce = (float)ce;
    c->cm = (float)cm;
    /* time terms of -B/A (acoustic.cpp:176-190), rational coefficient times
     * the folded power; canonical order (expr.cpp:352-370): eta term first,
     * then the m terms ordered by their time alias name t0 < t1 < t2 */
    float t_eta = (float)(0.5 * inv_dt);
    float t_mprev = (float)(-1.0 * inv_dt2);
    float t_mcur = (float)(2.0 * inv_dt2);
    c->tc[0] = t_eta;
    c->tfield[0] = 0;
    c->tlevel[0] = 0;
    if (forward) { /* prev = t0 = t-1 < cur = t1 = t */
        c->tc[1] = t_mprev; c->tfield[1] = 1; c->tlevel[1] = 0;
        c->tc[2] = t_mcur;  c->tfield[2] = 1; c->tlevel[2] = 1;
    } else {       /* cur = t1 = t < prev = t2 = t+1 */
        c->tc[1] = t_mcur;  c->tfield[1] = 1; c->tlevel[1] = 1;
        c->tc[2] = t_mprev; c->tfield[2] = 1; c->tlevel[2] = 0;
    }
    /* Laplacian: the ndim centre weights merge exactly (rational) */
    sfp_rat centre = rmul(R(ndim, 1), w[r]);
    c->c0 = (float)(rdbl(centre) * inv_h2);
    for (int j = 1; j <= r; ++j) c->cj[j - 1] = (float)(rdbl(w[r + j]) * inv_h2);
    c->src_scale = (float)pow(dt, 2.0);
    return 0;
}

double sfp_stable_dt(int ndim, int order, double spacing, double v_top,
                     double v_bottom) {
    sfp_rat w[17];
    if (sfp_fd_weights2(order, w)) return -1.0;
    double s = 0.0;
    for (int k = 0; k <= order; ++k) s += fabs(rdbl(w[k]));
    double v_max = v_top > v_bottom ? v_top : v_bottom;
    double m_min = 1.0 / (v_max * v_max);
    double lam = s * ndim;
    return 0.9 * 2.0 * sqrt(m_min / lam) * spacing;
}

double sfp_ricker(double f0, double t, double t0) {
    double arg = M_PI * f0 * (t - t0);
    double a2 = arg * arg;
    return (1.0 - 2.0 * a2) * exp(-a2);
}

int sfp_interp_weights(int ndim, const double *coord, double spacing,
                       const int64_t *extents, int32_t *cell, float *w) {
    double frac[3];
    if (spacing <= 0) return 3;
    for (int i = 0; i < ndim; ++i) {
        double pos = coord[i] / spacing;
        if (pos < 0) return 3;
        long cl = (long)floor(pos);
        if (cl > extents[i] - 2) return 3;
        cell[i] = (int32_t)(double)cl; /* stored through set(double) */
        frac[i] = pos - (double)cl;
    }
    int corners = 1 << ndim;
    for (int k = 0; k < corners; ++k) {
        double v = 1.0;
        for (int i = 0; i < ndim; ++i) v *= ((k >> i) & 1) ? frac[i] : 1.0 - frac[i];
        w[k] = (float)v;
    }
    return 0;
}

static double sponge_sigma(int ndim, const int64_t *shape, const int64_t *idx,
                           long w, double sigma_max) {
    long dist = (long)shape[0];
    for (int i = 0; i < ndim; ++i) {
        if (idx[i] < dist) dist = (long)idx[i];
        long hi = (long)(shape[i] - 1 - idx[i]);
        if (hi < dist) dist = hi;
    }
    if (w > 0 && dist < w) {
        double rr = 1.0 - (double)dist / (double)w;
        return sigma_max * rr * rr;
    }
    return 0.0;
}

static void medium_fill(int ndim, const int64_t *shape, int boundary_width,
                        double spacing, double v_min, const double *v_field,
                        double v_top, double v_bottom, float *m, float *eta) {
    const double m_top = 1.0 / (v_top * v_top);
    const double m_bottom = 1.0 / (v_bottom * v_bottom);
    const long w = boundary_width;
    const double sigma_max =
        1.5 * log(1000.0) * v_min / ((double)(w > 1 ? w : 1) * spacing);
    int64_t n0 = shape[0], n1 = shape[1], n2 = ndim == 3 ? shape[2] : 1;
    int64_t idx[3];
    for (int64_t a = 0; a < n0; ++a)
        for (int64_t b = 0; b < n1; ++b)
            for (int64_t cc = 0; cc < n2; ++cc) {
                idx[0] = a;
                idx[1] = b;
                idx[2] = cc;
                int64_t lin = (a * n1 + b) * n2 + cc;
                double mv;
                if (v_field) {
                    double vv = v_field[lin];
                    mv = 1.0 / (vv * vv);
                } else {
                    mv = a < n0 / 2 ? m_top : m_bottom;
                }
                double sg = sponge_sigma(ndim, shape, idx, w, sigma_max);
                m[lin] = (float)mv;
                eta[lin] = (float)(mv * sg);
            }
}

void sfp_build_medium(int ndim, const int64_t *shape, int boundary_width,
                      double spacing, double v_top, double v_bottom, float *m,
                      float *eta) {
    double v_min = v_top < v_bottom ? v_top : v_bottom;
    medium_fill(ndim, shape, boundary_width, spacing, v_min, NULL, v_top,
                v_bottom, m, eta);
}

void sfp_medium_from_velocity(int ndim, const int64_t *shape,
                              int boundary_width, double spacing, double v_min,
                              const double *v, float *m, float *eta) {
    medium_fill(ndim, shape, boundary_width, spacing, v_min, v, 0, 0, m, eta);
}

/* ------------------------------------------------------------------------
 * one stencil point, exactly as the emitted statement evaluates it:
 *   temp0 = ce*eta; temp1 = cm*m; temp2 = temp0 + temp1; temp3 = 1.0F/temp2;
 *   out = tc0*temp3*F0*L0 + tc1*temp3*F1*L1 + tc2*temp3*F2*L2
 *       + c0*temp3*cur + sum over axes (last axis first) of
 *         cj*temp3*cur[-r..-1, +1..+r]
 * each product evaluated left to right, the sum left to right. */
static inline float acoustic_point(const sfp_acoustic_coefs *c, float mv,
                                   float ev, float pv, const float *cur,
                                   const int64_t *strides /* last axis first */) {
    int r = c->order / 2;
    float temp0 = c->ce * ev;
    float temp1 = c->cm * mv;
    float temp2 = temp0 + temp1;
    float temp3 = 1.0F / temp2;
    float acc = 0.0F;
    for (int k = 0; k < 3; ++k) {
        float f = c->tfield[k] ? mv : ev;
        float lv = c->tlevel[k] ? cur[0] : pv;
        float term = c->tc[k] * temp3 * f * lv;
        acc = k == 0 ? term : acc + term;
    }
    acc = acc + c->c0 * temp3 * cur[0];
    for (int a = 0; a < c->ndim; ++a) {
        int64_t s = strides[a];
        for (int j = -r; j <= r; ++j) {
            if (j == 0) continue;
            float cj = c->cj[(j < 0 ? -j : j) - 1];
            acc = acc + cj * temp3 * cur[j * s];
        }
    }
    return acc;
}

static void acoustic_sweep(const sfp_acoustic_coefs *c, const int64_t *shape,
                           float *out, const float *cur, const float *prev,
                           const float *m, const float *eta,
                           const float *old_out_for_grad, const float *u_grad,
                           float *grad) {
    (void)old_out_for_grad;
    (void)u_grad;
    (void)grad;
    int r = c->order / 2;
    int64_t n0 = shape[0], n1 = shape[1], n2 = c->ndim == 3 ? shape[2] : 1;
    int64_t strides[3];
    if (c->ndim == 3) {
        strides[0] = 1;
        strides[1] = n2;
        strides[2] = n1 * n2;
    } else {
        strides[0] = 1;
        strides[1] = n1;
    }
    int64_t lo2 = c->ndim == 3 ? r : 0, hi2 = c->ndim == 3 ? n2 - r : 1;
#pragma omp for schedule(static)
    for (int64_t a = r; a < n0 - r; ++a)
        for (int64_t b = r; b < n1 - r; ++b)
            for (int64_t cc = lo2; cc < hi2; ++cc) {
                int64_t lin = (a * n1 + b) * n2 + cc;
                out[lin] = acoustic_point(c, m[lin], eta[lin], prev[lin],
                                          cur + lin, strides);
            }
}

/* build_inject (sparse.cpp:114-143) as emitted (golden acoustic_3d.c:43-54):
 * field[corner] = scale*series*w/m[corner] + field[corner], p ascending. */
static void inject(int ndim, const int64_t *shape, float scale, float *field,
                   const float *m, const float *row, const int32_t *ci,
                   const float *w, int64_t np) {
    int64_t n1 = shape[1], n2 = ndim == 3 ? shape[2] : 1;
    int corners = 1 << ndim;
    for (int64_t p = 0; p < np; ++p)
        for (int k = 0; k < corners; ++k) {
            int64_t i0 = ci[p * ndim + 0] + (k & 1);
            int64_t i1 = ci[p * ndim + 1] + ((k >> 1) & 1);
            int64_t i2 = ndim == 3 ? ci[p * ndim + 2] + ((k >> 2) & 1) : 0;
            int64_t lin = (i0 * n1 + i1) * n2 + i2;
            field[lin] = scale * row[p] * w[p * corners + k] / m[lin] + field[lin];
        }
}

/* build_sample (sparse.cpp:145-174): rec = w0*u[c0] + w1*u[c1] + ... */
static void sample(int ndim, const int64_t *shape, const float *field,
                   float *row, const int32_t *ci, const float *w, int64_t np) {
    int64_t n1 = shape[1], n2 = ndim == 3 ? shape[2] : 1;
    int corners = 1 << ndim;
    for (int64_t p = 0; p < np; ++p) {
        float acc = 0.0F;
        for (int k = 0; k < corners; ++k) {
            int64_t i0 = ci[p * ndim + 0] + (k & 1);
            int64_t i1 = ci[p * ndim + 1] + ((k >> 1) & 1);
            int64_t i2 = ndim == 3 ? ci[p * ndim + 2] + ((k >> 2) & 1) : 0;
            int64_t lin = (i0 * n1 + i1) * n2 + i2;
            float term = w[p * corners + k] * field[lin];
            acc = k == 0 ? term : acc + term;
        }
        row[p] = acc;
    }
}

static int64_t field_numel(int ndim, const int64_t *shape) {
    int64_t n = 1;
    for (int i = 0; i < ndim; ++i) n *= shape[i];
    return n;
}

static void set_threads(int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
}

int sfp_acoustic_run(const sfp_acoustic_coefs *c, const int64_t *shape,
                     int64_t nt, float *u, const float *m, const float *eta,
                     const float *inj, const int32_t *inj_ci,
                     const float *inj_w, int64_t n_inj, float *smp,
                     const int32_t *smp_ci, const float *smp_w, int64_t n_smp,
                     int nthreads) {
    int64_t N = field_numel(c->ndim, shape);
    set_threads(nthreads);
#pragma omp parallel
    {
        if (c->forward) {
            for (int64_t t = 0; t < nt; ++t) {
                float *t0 = u + ((t + 2) % 3) * N; /* t-1 */
                float *t1 = u + (t % 3) * N;       /* t   */
                float *t2 = u + ((t + 1) % 3) * N; /* t+1 */
                acoustic_sweep(c, shape, t2, t1, t0, m, eta, NULL, NULL, NULL);
#pragma omp single
                inject(c->ndim, shape, c->src_scale, t2, m, inj + t * n_inj,
                       inj_ci, inj_w, n_inj);
#pragma omp single
                sample(c->ndim, shape, t2, smp + t * n_smp, smp_ci, smp_w, n_smp);
            }
        } else {
            for (int64_t t = nt; t >= 1; --t) {
                float *t0 = u + ((t + 2) % 3) * N; /* t-1 (written) */
                float *t1 = u + (t % 3) * N;       /* t   */
                float *t2 = u + ((t + 1) % 3) * N; /* t+1 */
                acoustic_sweep(c, shape, t0, t1, t2, m, eta, NULL, NULL, NULL);
#pragma omp single
                inject(c->ndim, shape, c->src_scale, t0, m, inj + (t - 1) * n_inj,
                       inj_ci, inj_w, n_inj);
#pragma omp single
                sample(c->ndim, shape, t0, smp + (t - 1) * n_smp, smp_ci, smp_w,
                       n_smp);
            }
        }
    }
    return 0;
}

int sfp_acoustic_forward_history(const sfp_acoustic_coefs *c,
                                 const int64_t *shape, int64_t nt, float *hist,
                                 const float *m, const float *eta,
                                 const float *src, const int32_t *src_ci,
                                 const float *src_w, int64_t nsrc, float *rec,
                                 const int32_t *rec_ci, const float *rec_w,
                                 int64_t nrec, int nthreads) {
    if (!c->forward) return 1;
    int64_t N = field_numel(c->ndim, shape);
    set_threads(nthreads);
#pragma omp parallel
    {
        for (int64_t t = 0; t < nt; ++t) {
            float *prev = hist + t * N;      /* u(t-1) */
            float *cur = hist + (t + 1) * N; /* u(t)   */
            float *out = hist + (t + 2) * N; /* u(t+1) */
            acoustic_sweep(c, shape, out, cur, prev, m, eta, NULL, NULL, NULL);
#pragma omp single
            inject(c->ndim, shape, c->src_scale, out, m, src + t * nsrc, src_ci,
                   src_w, nsrc);
#pragma omp single
            sample(c->ndim, shape, out, rec + t * nrec, rec_ci, rec_w, nrec);
        }
    }
    return 0;
}

/* grad += u * (((vn - 2*vc) + vp) * cm) on the interior */
static void grad_sweep(const sfp_acoustic_coefs *c, const int64_t *shape,
                       const float *vn, const float *vc, const float *vp,
                       const float *ut, float *grad) {
    int r = c->order / 2;
    int64_t n0 = shape[0], n1 = shape[1], n2 = c->ndim == 3 ? shape[2] : 1;
    int64_t lo2 = c->ndim == 3 ? r : 0, hi2 = c->ndim == 3 ? n2 - r : 1;
    float cm = c->cm;
#pragma omp for schedule(static)
    for (int64_t a = r; a < n0 - r; ++a)
        for (int64_t b = r; b < n1 - r; ++b)
            for (int64_t cc = lo2; cc < hi2; ++cc) {
                int64_t lin = (a * n1 + b) * n2 + cc;
                float vtt = ((vn[lin] - 2.0F * vc[lin]) + vp[lin]) * cm;
                grad[lin] = grad[lin] + ut[lin] * vtt;
            }
}

int sfp_fwi_adjoint_gradient(const sfp_acoustic_coefs *c, const int64_t *shape,
                             int64_t nt, float *v, const float *m,
                             const float *eta, const float *hist,
                             const float *rec, const int32_t *rec_ci,
                             const float *rec_w, int64_t nrec, float *src,
                             const int32_t *src_ci, const float *src_w,
                             int64_t nsrc, float *grad, int nthreads) {
    if (c->forward) return 1;
    int64_t N = field_numel(c->ndim, shape);
    set_threads(nthreads);
#pragma omp parallel
    {
        for (int64_t t = nt; t >= 1; --t) {
            float *t0 = v + ((t + 2) % 3) * N;
            float *t1 = v + (t % 3) * N;
            float *t2 = v + ((t + 1) % 3) * N;
            acoustic_sweep(c, shape, t0, t1, t2, m, eta, NULL, NULL, NULL);
#pragma omp single
            inject(c->ndim, shape, c->src_scale, t0, m, rec + (t - 1) * nrec,
                   rec_ci, rec_w, nrec);
#pragma omp single
            sample(c->ndim, shape, t0, src + (t - 1) * nsrc, src_ci, src_w, nsrc);
            /* v(t-1) final: term for time t uses v(t+1), v(t), v(t-1), u(t) */
            grad_sweep(c, shape, t2, t1, t0, hist + (t + 1) * N, grad);
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------
 * diffusion */

int sfp_diffusion_dt(sfp_rat alpha, sfp_rat dx, int order, sfp_rat *dt) {
    sfp_rat dx2 = rmul(dx, dx);
    sfp_rat base = rdiv(rmul(dx2, dx2), rmul(rmul(R(2, 1), alpha), radd(dx2, dx2)));
    if (order == 2) {
        *dt = base;
        return 0;
    }
    sfp_rat w[17];
    if (sfp_fd_weights2(order, w)) return 1;
    sfp_rat lam = R(0, 1);
    for (int k = 0; k <= order; ++k) {
        sfp_rat a = w[k];
        if (a.num < 0) a.num = -a.num;
        lam = radd(lam, a);
    }
    sfp_rat ratio = rdiv(R(4, 1), lam);
    *dt = (ratio.num < ratio.den) ? rmul(base, ratio) : base;
    return 0;
}

int sfp_diffusion_coefs(sfp_rat alpha, sfp_rat dx, int order, float *c0,
                        int *has_c0, float *cj) {
    sfp_rat w[17], dt;
    if (sfp_fd_weights2(order, w)) return 1;
    if (sfp_diffusion_dt(alpha, dx, order, &dt)) return 1;
    int r = order / 2;
    /* u(t+s) = u(t) + s*a*(dx2 + dy2): every coefficient folds exactly */
    sfp_rat k = rdiv(rmul(alpha, dt), rmul(dx, dx));
    sfp_rat centre = radd(R(1, 1), rmul(rmul(R(2, 1), w[r]), k));
    *has_c0 = centre.num != 0;
    *c0 = (float)rdbl(centre);
    memset(cj, 0, 8 * sizeof(float));
    for (int j = 1; j <= r; ++j) cj[j - 1] = (float)rdbl(rmul(w[r + j], k));
    return 0;
}

int sfp_diffusion_run(int64_t nx, int64_t ny, int order, float c0, int has_c0,
                      const float *cj, int64_t nt, float *u, int nthreads) {
    int r = order / 2;
    int64_t N = nx * ny;
    set_threads(nthreads);
#pragma omp parallel
    for (int64_t t = 0; t < nt; ++t) {
        const float *src = u + (t % 2) * N;
        float *dst = u + ((t + 1) % 2) * N;
#pragma omp for schedule(static)
        for (int64_t i = r; i < nx - r; ++i)
            for (int64_t j = r; j < ny - r; ++j) {
                const float *p = src + i * ny + j;
                float acc = 0.0F;
                int first = 1;
                if (has_c0) {
                    acc = c0 * p[0];
                    first = 0;
                }
                /* last axis, then axis 0; offsets -r..-1, 1..r */
                for (int ax = 0; ax < 2; ++ax) {
                    int64_t s = ax == 0 ? 1 : ny;
                    for (int q = -r; q <= r; ++q) {
                        if (q == 0) continue;
                        float term = cj[(q < 0 ? -q : q) - 1] * p[q * s];
                        if (first) {
                            acc = term;
                            first = 0;
                        } else {
                            acc = acc + term;
                        }
                    }
                }
                dst[i * ny + j] = acc;
            }
    }
    return 0;
}

/* ------------------------------------------------------------------------
 * Seeded smooth random medium (configs C3/C4/C5). The product generates it
 * on the GPU (paper_1609_03361_b200/csrc/medium.cu, which states the
 * definition); this is the same definition in plain C, evaluated in the
 * same order (double sums in ascending tap order, no contraction), so the
 * two agree bitwise. The m / eta expressions are build_medium's
 * (acoustic.cpp:67-105), with global indices. */

static int64_t sm_reflect(int64_t i, int64_t n) {
    int64_t p = 2 * n;
    i %= p;
    if (i < 0) i += p;
    return i < n ? i : p - 1 - i;
}

static uint64_t sm_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static double sm_noise(uint64_t salt, int64_t lin) {
    uint64_t z = sm_mix((uint64_t)lin * 0x9E3779B97F4A7C15ull + salt);
    return (double)((int64_t)(z >> 40) - 8388608) * (1.0 / 8388608.0);
}

int sfp_smooth_taps(double sigma, double *g /* [2*64+1] */) {
    int rad = (int)(4.0 * sigma + 0.5);
    if (!(sigma > 0) || rad < 1 || rad > 64) return -1;
    double sum = 0.0;
    for (int k = 0; k <= 2 * rad; ++k) {
        double x = (double)(k - rad);
        g[k] = exp(-0.5 * x * x / (sigma * sigma));
        sum += g[k];
    }
    for (int k = 0; k <= 2 * rad; ++k) g[k] /= sum;
    return rad;
}

/* t2 (axis-2 then axis-1 filtered noise) of the planes the depth pass over
 * [b, e) reads; *L = global index of its first plane. */
static float *sm_t2(const int64_t *shape, int64_t b, int64_t e, uint64_t seed,
                    const double *g, int rad, int64_t *L) {
    int64_t n0 = shape[0], n1 = shape[1], n2 = shape[2];
    int64_t lo = n0, hi = 0;
    for (int64_t p = b - rad; p < e + rad; ++p) {
        int64_t q = sm_reflect(p, n0);
        if (q < lo) lo = q;
        if (q + 1 > hi) hi = q + 1;
    }
    *L = lo;
    int64_t nz = hi - lo, n12 = n1 * n2;
    float *t2 = (float *)malloc(sizeof(float) * (size_t)(nz * n12));
    if (!t2) return NULL;
    uint64_t salt = sm_mix(seed + 0x9E3779B97F4A7C15ull);
    int64_t *r1 = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n1 + 2 * rad));
    for (int64_t i = 0; i < n1 + 2 * rad; ++i) r1[i] = sm_reflect(i - rad, n1) * n2;
#pragma omp parallel
    {
        float *t1 = (float *)malloc(sizeof(float) * (size_t)n12);
        double *row = (double *)malloc(sizeof(double) * (size_t)(n2 + 2 * rad));
        double *acc = (double *)malloc(sizeof(double) * (size_t)n2);
#pragma omp for schedule(static)
        for (int64_t z = 0; z < nz; ++z) {
            int64_t i0 = lo + z;
            for (int64_t i1 = 0; i1 < n1; ++i1) {
                int64_t rowlin = (i0 * n1 + i1) * n2;
                /* row[j] = noise at a2 = refl(j - rad) */
                for (int64_t j = 0; j < n2 + 2 * rad; ++j)
                    row[j] = sm_noise(salt, rowlin + sm_reflect(j - rad, n2));
                for (int64_t i2 = 0; i2 < n2; ++i2) {
                    double s = 0.0;
                    for (int k = 0; k <= 2 * rad; ++k) s = s + g[k] * row[i2 + k];
                    t1[i1 * n2 + i2] = (float)s;
                }
            }
            float *out = t2 + z * n12;
            for (int64_t i1 = 0; i1 < n1; ++i1) {
                for (int64_t i2 = 0; i2 < n2; ++i2) acc[i2] = 0.0;
                for (int k = 0; k <= 2 * rad; ++k) {
                    const float *src = t1 + r1[i1 + k];
                    double gk = g[k];
                    for (int64_t i2 = 0; i2 < n2; ++i2) acc[i2] = acc[i2] + gk * (double)src[i2];
                }
                for (int64_t i2 = 0; i2 < n2; ++i2) out[i1 * n2 + i2] = (float)acc[i2];
            }
        }
        free(t1);
        free(row);
        free(acc);
    }
    free(r1);
    return t2;
}

/* f of global plane i0 (depth pass) into acc[n1*n2] */
static void sm_depth(const float *t2, int64_t L, const int64_t *shape, int64_t i0,
                     const double *g, int rad, double *acc) {
    int64_t n12 = shape[1] * shape[2];
    for (int64_t j = 0; j < n12; ++j) acc[j] = 0.0;
    for (int k = 0; k <= 2 * rad; ++k) {
        const float *src = t2 + (sm_reflect(i0 + k - rad, shape[0]) - L) * n12;
        double gk = g[k];
        for (int64_t j = 0; j < n12; ++j) acc[j] = acc[j] + gk * (double)src[j];
    }
}

int sfp_smooth_extrema(const int64_t *shape, int64_t b, int64_t e, uint64_t seed,
                       double sigma, double *lo_out, double *hi_out) {
    double g[129];
    int rad = sfp_smooth_taps(sigma, g);
    if (rad < 0 || b < 0 || e > shape[0] || b >= e) return 1;
    int64_t L;
    float *t2 = sm_t2(shape, b, e, seed, g, rad, &L);
    if (!t2) return 7;
    int64_t n12 = shape[1] * shape[2];
    double lo = INFINITY, hi = -INFINITY;
#pragma omp parallel
    {
        double *acc = (double *)malloc(sizeof(double) * (size_t)n12);
        double l = INFINITY, h = -INFINITY;
#pragma omp for schedule(static)
        for (int64_t i0 = b; i0 < e; ++i0) {
            sm_depth(t2, L, shape, i0, g, rad, acc);
            for (int64_t j = 0; j < n12; ++j) {
                if (acc[j] < l) l = acc[j];
                if (acc[j] > h) h = acc[j];
            }
        }
#pragma omp critical
        {
            if (l < lo) lo = l;
            if (h > hi) hi = h;
        }
        free(acc);
    }
    free(t2);
    *lo_out = lo;
    *hi_out = hi;
    return 0;
}

int sfp_smooth_medium(const int64_t *shape, int64_t b, int64_t e, uint64_t seed,
                      double sigma, double v_lo, double v_hi, int boundary_width,
                      double spacing, double v_min, double lo, double hi, float *m,
                      float *eta) {
    double g[129];
    int rad = sfp_smooth_taps(sigma, g);
    if (rad < 0 || b < 0 || e > shape[0] || b >= e || !(hi > lo)) return 1;
    int64_t L;
    float *t2 = sm_t2(shape, b, e, seed, g, rad, &L);
    if (!t2) return 7;
    int64_t n0 = shape[0], n1 = shape[1], n2 = shape[2], n12 = n1 * n2;
    const long w = boundary_width;
    const double sigma_max =
        1.5 * log(1000.0) * v_min / ((double)(w > 1 ? w : 1) * spacing);
#pragma omp parallel
    {
        double *acc = (double *)malloc(sizeof(double) * (size_t)n12);
#pragma omp for schedule(static)
        for (int64_t i0 = b; i0 < e; ++i0) {
            sm_depth(t2, L, shape, i0, g, rad, acc);
            for (int64_t i1 = 0; i1 < n1; ++i1)
                for (int64_t i2 = 0; i2 < n2; ++i2) {
                    double f = acc[i1 * n2 + i2];
                    double v = v_lo + ((v_hi - v_lo) * (f - lo)) / (hi - lo);
                    double mv = 1.0 / (v * v);
                    int64_t idx[3] = {i0, i1, i2};
                    double sg = sponge_sigma(3, shape, idx, w, sigma_max);
                    int64_t off = ((i0 - b) * n1 + i1) * n2 + i2;
                    m[off] = (float)mv;
                    eta[off] = (float)(mv * sg);
                }
        }
        free(acc);
    }
    (void)n0;
    free(t2);
    return 0;
}
