// medium.h — device generator of seeded smooth random media (medium.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sf_b200.h"

namespace sfb {

constexpr int kMediumMaxRad = 64;

// code 0: invalid argument, 1: out of device memory, 2: CUDA failure
struct MediumError : std::runtime_error {
    int code;
    MediumError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

int smooth_radius(double sigma);
std::vector<double> smooth_taps(double sigma);
uint64_t smooth_salt(uint64_t seed);
std::vector<double> sponge_sigma(int boundary_width, double spacing, double v_min);

// mode 0: *lo / *hi = extrema of the filtered noise over planes
// [a0_begin, a0_end); mode 1: m / eta of those planes (device pointers,
// plane a0_begin at offset 0, the given row / plane strides) from the global
// extrema *lo / *hi. Synchronises `st` before returning.
void smooth_medium_run(const sf_smooth_medium_desc& d, int mode, double* lo, double* hi,
                       float* m, float* eta, int64_t pitch, int64_t plane, cudaStream_t st);

} // namespace sfb
