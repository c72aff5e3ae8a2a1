// mugv::Rng (rng.hpp:14-72) on the host: mt19937_64 with the reference's hand-rolled distributions, so seeded
// streams (weights, noise, draws) are identical to the reference's.
#pragma once
#include <cmath>
#include <cstdint>
#include <random>

namespace mgv {

class HostRng {
public:
    explicit HostRng(uint64_t seed) : gen_(seed) {}
    double uniform() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }  // rng.hpp:21-23
    double normal() {                                                            // rng.hpp:26-39 (Box-Muller)
        if (have_spare_) {
            have_spare_ = false;
            return spare_;
        }
        double u1 = uniform();
        const double u2 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 2.0 * M_PI * u2;
        spare_ = r * std::sin(a);
        have_spare_ = true;
        return r * std::cos(a);
    }
    void normal_fill(double* out, int64_t n, double stddev) {  // rng.hpp:54-58
        for (int64_t i = 0; i < n; ++i) out[i] = stddev * normal();
    }

private:
    std::mt19937_64 gen_;
    bool have_spare_ = false;
    double spare_ = 0.0;
};

}  // namespace mgv
