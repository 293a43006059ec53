// sf_internal.h — shared declarations of the B200 stencil library (host side).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace sfb {

// exact rational, int64 with 128-bit intermediates (mirrors sf::Rational,
// rational.hpp:13-127)
struct Rat {
    int64_t num = 0;
    int64_t den = 1;
    static Rat make(__int128 n, __int128 d);
    double to_double() const { return static_cast<double>(num) / static_cast<double>(den); }
};
Rat operator+(Rat a, Rat b);
Rat operator*(Rat a, Rat b);
Rat operator/(Rat a, Rat b);

std::vector<Rat> fd_weights2(int order);

// Folded fp32 constants of the acoustic update (see acoustic_constants()).
struct AcousticConstants {
    int ndim;
    int radius;
    bool forward;
    float ce;         // temp0 = ce * eta
    float cm;         // temp1 = cm * m
    float tc[3];      // time terms in emitted order
    int tsel[3];      // 2*field(0 eta, 1 m) + level(0 prev, 1 cur)
    float c0;         // merged centre coefficient
    float cj[8];      // neighbour coefficient, |offset| = j+1
    float src_scale;  // dt^2
};

struct DiffusionConstants {
    int radius;
    bool has_c0;
    float c0;
    float cj[8];
    Rat dt;
};

AcousticConstants acoustic_constants(int ndim, int order, bool forward, double dt,
                                     double spacing);
DiffusionConstants diffusion_constants(Rat alpha, Rat dx, int order);
double stable_dt(int ndim, int order, double spacing, double v_top, double v_bottom);
double ricker(double f0, double t, double t0);
bool interpolation_weights(int ndim, const double* coord, double spacing, const int64_t* extents,
                           int32_t* cell, float* w);
void build_medium(int ndim, const int64_t* shape, int boundary_width, double spacing,
                  double v_top, double v_bottom, const double* v_field, double v_min, float* m,
                  float* eta);

void set_error(const std::string& msg);

} // namespace sfb
