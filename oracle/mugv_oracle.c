/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Nothing in the product path
 * (paper_2510_17519_b200/, include/, the C-ABI library) links or calls this.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use it,
 * and only as the checker.
 *
 * Plain-C restatement of the reference's integer / RNG machinery for the DiT
 * hot path, so the oracle can regenerate the reference's synthetic inputs and
 * weights bit-for-bit without the reference sources:
 *
 *   - mugv::Rng (proj/include/mugv/rng.hpp:14-72): std::mt19937_64 with
 *     hand-rolled uniform (53-bit mantissa, rng.hpp:21) and Box-Muller normal
 *     with a cached spare (rng.hpp:26-38).  mt19937_64 is restated from the
 *     C++11 standard's published parameters (w=64, n=312, m=156, r=31,
 *     a=0xB5026F5AA96619E9, u=29, d=0x5555555555555555, s=17,
 *     b=0x71D67FFFEDA60000, t=37, c=0xFFF7EEE000000000, l=43,
 *     f=6364136223846793005).
 *   - latent_rows 2x2 patch gather (proj/src/dit.cpp:92-116) and its inverse
 *     rows_to_grid (dit.cpp:118-141).
 *
 * Pinned against the compiled reference (oracle/_ref) by
 * tests/test_oracle.py::test_rng_matches_reference and the golden fixtures.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define MT_N 312
#define MT_M 156

typedef struct {
    uint64_t mt[MT_N];
    int idx;
    int have_spare;
    double spare;
} mgo_rng;

void mgo_rng_seed(mgo_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = MT_N;
    r->have_spare = 0;
    r->spare = 0.0;
}

static void mgo_twist(mgo_rng* r) {
    const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    for (int i = 0; i < MT_N; ++i) {
        uint64_t x = (r->mt[i] & UM) | (r->mt[(i + 1) % MT_N] & LM);
        uint64_t xa = x >> 1;
        if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
        r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ xa;
    }
    r->idx = 0;
}

uint64_t mgo_rng_next(mgo_rng* r) {
    if (r->idx >= MT_N) mgo_twist(r);
    uint64_t x = r->mt[r->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* rng.hpp:21 */
double mgo_rng_uniform(mgo_rng* r) { return (double)(mgo_rng_next(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:26-38: spare is cached across calls (and across tensors) */
double mgo_rng_normal(mgo_rng* r) {
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    double u1 = mgo_rng_uniform(r);
    double u2 = mgo_rng_uniform(r);
    while (u1 <= 0.0) u1 = mgo_rng_uniform(r);
    double rr = sqrt(-2.0 * log(u1));
    double a = 2.0 * M_PI * u2;
    r->spare = rr * sin(a);
    r->have_spare = 1;
    return rr * cos(a);
}

/* rng.hpp:54-58 */
void mgo_rng_normal_fill(mgo_rng* r, double* out, int64_t n, double stddev) {
    for (int64_t i = 0; i < n; ++i) out[i] = stddev * mgo_rng_normal(r);
}

/* rng.hpp:60-64 (uniform(lo,hi) = lo + (hi-lo)*uniform(), rng.hpp:23) */
void mgo_rng_uniform_fill(mgo_rng* r, double* out, int64_t n, double lo, double hi) {
    for (int64_t i = 0; i < n; ++i) out[i] = lo + (hi - lo) * mgo_rng_uniform(r);
}

/* rng.hpp:41-48 */
int64_t mgo_rng_randint(mgo_rng* r, int64_t n) {
    uint64_t un = (uint64_t)n;
    uint64_t limit = UINT64_MAX - UINT64_MAX % un;
    uint64_t x = mgo_rng_next(r);
    while (x >= limit) x = mgo_rng_next(r);
    return (int64_t)(x % un);
}

int mgo_rng_size(void) { return (int)sizeof(mgo_rng); }

/* dit.cpp:92-116: (U,h,w,C) grid -> (N, 4C) rows + (N,3) int coords, row-major (t,py,px). */
void mgo_latent_rows(const double* grid, int64_t U, int64_t h, int64_t w, int64_t C, double* rows,
                     int32_t* coords) {
    int64_t Hp = h / 2, Wp = w / 2, D = 4 * C, i = 0;
    for (int64_t t = 0; t < U; ++t)
        for (int64_t py = 0; py < Hp; ++py)
            for (int64_t px = 0; px < Wp; ++px, ++i) {
                coords[3 * i + 0] = (int32_t)t;
                coords[3 * i + 1] = (int32_t)py;
                coords[3 * i + 2] = (int32_t)px;
                for (int64_t dy = 0; dy < 2; ++dy)
                    for (int64_t dx = 0; dx < 2; ++dx)
                        memcpy(rows + i * D + (dy * 2 + dx) * C, grid + ((t * h + 2 * py + dy) * w + 2 * px + dx) * C,
                               sizeof(double) * (size_t)C);
            }
}

/* dit.cpp:118-141: inverse by coords; returns 0 ok, 1 out of range, 2 duplicate. */
int mgo_rows_to_grid(const double* rows, const int32_t* coords, int64_t N, int64_t U, int64_t Hp, int64_t Wp,
                     int64_t C, double* grid, unsigned char* seen) {
    int64_t D = 4 * C;
    memset(seen, 0, (size_t)N);
    for (int64_t i = 0; i < N; ++i) {
        int64_t t = coords[3 * i], py = coords[3 * i + 1], px = coords[3 * i + 2];
        if (t < 0 || t >= U || py < 0 || py >= Hp || px < 0 || px >= Wp) return 1;
        int64_t slot = (t * Hp + py) * Wp + px;
        if (seen[slot]) return 2;
        seen[slot] = 1;
        for (int64_t dy = 0; dy < 2; ++dy)
            for (int64_t dx = 0; dx < 2; ++dx)
                memcpy(grid + ((t * 2 * Hp + 2 * py + dy) * 2 * Wp + 2 * px + dx) * C, rows + i * D + (dy * 2 + dx) * C,
                       sizeof(double) * (size_t)C);
    }
    return 0;
}
