// setup.cpp — host-side build-time work of the hot path: exact FD weights,
// the folded fp32 stencil constants, stability bound, Ricker series,
// interpolation weights and the damped medium. Runs once per plan.
//
// These restate what the reference's build pipeline produces (it derives
// them symbolically, expr.cpp + fd.cpp + opt.cpp, then prints them into the
// generated C); the CUDA kernels consume the resulting constants. Compiled
// with -ffp-contract=off so double arithmetic rounds exactly like the
// reference's (jit.cpp:70 flags, and g++ -O2 without FMA contraction for the
// library itself).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "sf_internal.h"

namespace sfb {

namespace {

using i128 = __int128;

i128 gcd128(i128 a, i128 b) {
    if (a < 0) a = -a;
    if (b < 0) b = -b;
    while (b != 0) {
        i128 t = a % b;
        a = b;
        b = t;
    }
    return a == 0 ? 1 : a;
}

} // namespace

Rat Rat::make(i128 n, i128 d) {
    if (d == 0) throw std::invalid_argument("rational with zero denominator");
    if (d < 0) {
        n = -n;
        d = -d;
    }
    i128 g = gcd128(n, d);
    n /= g;
    d /= g;
    if (n > INT64_MAX || n < INT64_MIN || d > INT64_MAX)
        throw std::overflow_error("rational exceeds 64-bit range");
    Rat r;
    r.num = static_cast<int64_t>(n);
    r.den = static_cast<int64_t>(d);
    return r;
}

Rat operator+(Rat a, Rat b) {
    return Rat::make(static_cast<i128>(a.num) * b.den + static_cast<i128>(b.num) * a.den,
                     static_cast<i128>(a.den) * b.den);
}
Rat operator*(Rat a, Rat b) {
    return Rat::make(static_cast<i128>(a.num) * b.num, static_cast<i128>(a.den) * b.den);
}
Rat operator/(Rat a, Rat b) {
    return Rat::make(static_cast<i128>(a.num) * b.den, static_cast<i128>(a.den) * b.num);
}

// Centered second-derivative weights over offsets -r..r: w_k = L_k''(0) for
// the Lagrange basis, i.e. twice the x^2 coefficient of
// prod_{j != k}(x - x_j) / prod_{j != k}(x_k - x_j). Exact; identical to the
// moment-system solution fd_weights(2, centered_offsets(2, order)) of
// fd.cpp:28-92 (the system is regular, so the weights are unique).
std::vector<Rat> fd_weights2(int order) {
    if (order < 2 || order % 2 != 0 || order > 16)
        throw std::invalid_argument("space_order must be even and in [2, 16]");
    const int r = order / 2, n = 2 * r + 1;
    std::vector<Rat> w(n);
    for (int k = 0; k < n; ++k) {
        const int xk = k - r;
        i128 poly[18] = {0};
        poly[0] = 1;
        int deg = 0;
        i128 denom = 1;
        for (int j = 0; j < n; ++j) {
            if (j == k) continue;
            const int xj = j - r;
            denom *= static_cast<i128>(xk - xj);
            for (int i = deg + 1; i >= 1; --i) poly[i] = poly[i - 1] - static_cast<i128>(xj) * poly[i];
            poly[0] = -static_cast<i128>(xj) * poly[0];
            ++deg;
        }
        w[k] = Rat::make(2 * poly[2], denom);
    }
    return w;
}

// The reference folds every constant as (rational weight widened to double)
// x (std::pow of the substituted real scalar), expr.cpp ConstVal rules
// (expr.cpp:200-236) after fold_scalars (opt.cpp:106-133), and prints the
// double narrowed to float (codegen.cpp:15-36). The emitted term order of the
// solved update (acoustic.cpp:176-190, canonical ordering expr.cpp:352-370):
//   forward: eta*u[t-1], m*u[t-1], m*u[t], centre, neighbours
//   adjoint: eta*v[t+1], m*v[t],   m*v[t+1], centre, neighbours
// with neighbours ordered last axis first, offsets -r..-1, +1..+r.
AcousticConstants acoustic_constants(int ndim, int order, bool forward, double dt,
                                     double spacing) {
    if (ndim < 2 || ndim > 3) throw std::invalid_argument("acoustic needs 2 or 3 dimensions");
    if (!(dt > 0) || !(spacing > 0)) throw std::invalid_argument("dt and spacing must be positive");
    std::vector<Rat> w = fd_weights2(order);
    const int r = order / 2;
    AcousticConstants c{};
    c.ndim = ndim;
    c.radius = r;
    c.forward = forward;
    const double inv_dt = std::pow(dt, -1.0);
    const double inv_dt2 = std::pow(dt, -2.0);
    const double inv_h2 = std::pow(spacing, -2.0);
    c.ce = static_cast<float>(0.5 * inv_dt);
    c.cm = static_cast<float>(inv_dt2);
    const float t_eta = static_cast<float>(0.5 * inv_dt);
    const float t_mprev = static_cast<float>(-1.0 * inv_dt2);
    const float t_mcur = static_cast<float>(2.0 * inv_dt2);
    c.tc[0] = t_eta;
    c.tsel[0] = 0;  // eta * prev
    if (forward) {
        c.tc[1] = t_mprev;
        c.tsel[1] = 2;  // m * prev
        c.tc[2] = t_mcur;
        c.tsel[2] = 3;  // m * cur
    } else {
        c.tc[1] = t_mcur;
        c.tsel[1] = 3;
        c.tc[2] = t_mprev;
        c.tsel[2] = 2;
    }
    const Rat centre = Rat{ndim, 1} * w[r];
    c.c0 = static_cast<float>(centre.to_double() * inv_h2);
    for (int j = 1; j <= r; ++j) c.cj[j - 1] = static_cast<float>(w[r + j].to_double() * inv_h2);
    c.src_scale = static_cast<float>(std::pow(dt, 2.0));
    return c;
}

// DiffusionConfig::dt (diffusion.cpp:10-23) and the folded update
// u(t+1) = u(t) + dt*alpha*(dx2(u) + dy2(u)): every coefficient is an exact
// rational, narrowed rational -> double -> float (codegen.cpp:126-133).
DiffusionConstants diffusion_constants(Rat alpha, Rat dx, int order) {
    std::vector<Rat> w = fd_weights2(order);
    const int r = order / 2;
    Rat dx2 = dx * dx;
    Rat base = (dx2 * dx2) / (Rat{2, 1} * alpha * (dx2 + dx2));
    Rat dt = base;
    if (order != 2) {
        Rat lam{0, 1};
        for (const Rat& v : w) lam = lam + (v.num < 0 ? Rat{-v.num, v.den} : v);
        Rat ratio = Rat{4, 1} / lam;
        if (ratio.num < ratio.den) dt = base * ratio;
    }
    Rat k = (alpha * dt) / dx2;
    Rat centre = Rat{1, 1} + Rat{2, 1} * w[r] * k;
    DiffusionConstants c{};
    c.radius = r;
    c.has_c0 = centre.num != 0;
    c.c0 = static_cast<float>(centre.to_double());
    for (int j = 1; j <= r; ++j) c.cj[j - 1] = static_cast<float>((w[r + j] * k).to_double());
    c.dt = dt;
    return c;
}

double stable_dt(int ndim, int order, double spacing, double v_top, double v_bottom) {
    std::vector<Rat> w = fd_weights2(order);
    double s = 0.0;
    for (const Rat& v : w) s += std::abs(v.to_double());
    const double v_max = std::max(v_top, v_bottom);
    const double m_min = 1.0 / (v_max * v_max);
    const double lam = s * ndim;
    return 0.9 * 2.0 * std::sqrt(m_min / lam) * spacing;
}

double ricker(double f0, double t, double t0) {
    const double arg = M_PI * f0 * (t - t0);
    const double a2 = arg * arg;
    return (1.0 - 2.0 * a2) * std::exp(-a2);
}

bool interpolation_weights(int ndim, const double* coord, double spacing, const int64_t* extents,
                           int32_t* cell, float* w) {
    double frac[3];
    if (!(spacing > 0)) return false;
    for (int i = 0; i < ndim; ++i) {
        const double pos = coord[i] / spacing;
        if (pos < 0) return false;
        const long c = static_cast<long>(std::floor(pos));
        if (c > extents[i] - 2) return false;
        cell[i] = static_cast<int32_t>(c);
        frac[i] = pos - static_cast<double>(c);
    }
    const int corners = 1 << ndim;
    for (int k = 0; k < corners; ++k) {
        double v = 1.0;
        for (int i = 0; i < ndim; ++i) v *= ((k >> i) & 1) ? frac[i] : 1.0 - frac[i];
        w[k] = static_cast<float>(v);
    }
    return true;
}

void build_medium(int ndim, const int64_t* shape, int boundary_width, double spacing,
                  double v_top, double v_bottom, const double* v_field, double v_min, float* m,
                  float* eta) {
    const double m_top = 1.0 / (v_top * v_top);
    const double m_bottom = 1.0 / (v_bottom * v_bottom);
    if (!v_field) v_min = std::min(v_top, v_bottom);
    const long w = boundary_width;
    const double sigma_max =
        1.5 * std::log(1000.0) * v_min / (static_cast<double>(std::max<long>(w, 1)) * spacing);
    const int64_t n0 = shape[0], n1 = shape[1], n2 = ndim == 3 ? shape[2] : 1;
    for (int64_t a = 0; a < n0; ++a)
        for (int64_t b = 0; b < n1; ++b)
            for (int64_t cc = 0; cc < n2; ++cc) {
                const int64_t idx[3] = {a, b, cc};
                const int64_t lin = (a * n1 + b) * n2 + cc;
                double mv;
                if (v_field) {
                    const double vv = v_field[lin];
                    mv = 1.0 / (vv * vv);
                } else {
                    mv = a < n0 / 2 ? m_top : m_bottom;
                }
                long dist = static_cast<long>(shape[0]);
                for (int i = 0; i < ndim; ++i) {
                    dist = std::min<long>(dist, static_cast<long>(idx[i]));
                    dist = std::min<long>(dist, static_cast<long>(shape[i] - 1 - idx[i]));
                }
                double sigma = 0.0;
                if (w > 0 && dist < w) {
                    const double rr = 1.0 - static_cast<double>(dist) / static_cast<double>(w);
                    sigma = sigma_max * rr * rr;
                }
                m[lin] = static_cast<float>(mv);
                eta[lin] = static_cast<float>(mv * sigma);
            }
}

} // namespace sfb
