// Fuzz: sogk::ladder_seek (closed-form, csrc/sogk_ladder.cuh) vs the reference's
// sequential recurrence `while (t <= T) t += step(t)` (sampling.hpp:96-99,115-118).
// Build: g++ -O2 -std=c++17 -ffp-contract=off -I paper_2404_10272_b200/csrc
// Usage: ladder_fuzz <cases> <seed>   -> prints mismatches (0 expected), exit 1 on any
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "sogk_ladder.cuh"

template <int Sched>
static long naive(double& t, double T, double dt0, double g) {
    long n = 0;
    while (t <= T) {
        const double st = Sched == 0 ? dt0 : ((dt0 < g * t) ? g * t : dt0);
        t += st;
        ++n;
    }
    return n;
}

static double t_switch(double dt0, double g) {
    if (!(g > 0.0)) return DBL_MAX;
    double x = dt0 / g;
    while (g * x > dt0) x = std::nextafter(x, 0.0);
    while (g * std::nextafter(x, DBL_MAX) <= dt0) x = std::nextafter(x, DBL_MAX);
    return x;
}

int main(int argc, char** argv) {
    const long cases = argc > 1 ? std::atol(argv[1]) : 1000000;
    std::mt19937_64 rng(argc > 2 ? std::atoll(argv[2]) : 1);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    const double dts[] = {1.0 / 128, 1.0 / 512, 0.017, 0.011, 0.021, 0.0371, 1.0 / 3, 0.03,
                          0.013, 0.25, 1e-3, 0.5 * 2.0 / 144};
    long bad = 0, jumps = 0;
    for (long i = 0; i < cases; ++i) {
        const double dt0 = dts[rng() % (sizeof(dts) / sizeof(dts[0]))] * (rng() % 4 ? 1.0 : U(rng) + 0.5);
        const int sched = rng() % 3 == 0;
        const double g = sched ? (rng() % 2 ? 1.0 / 256 : 1.0 / 128 * U(rng)) : 0.0;
        // ladder points start anywhere: t_enter of a clipped ray
        double t0 = (rng() % 8 == 0) ? 0.0 : std::ldexp(U(rng), int(rng() % 8) - 4);
        double T = t0 + U(rng) * (rng() % 4 == 0 ? 40.0 : 3.0) - (rng() % 16 == 0 ? 1.0 : 0.0);
        double a = t0, b = t0;
        long na, nb;
        bool stalled = false;
        if (sched == 0) {
            na = naive<0>(a, T, dt0, g);
            nb = (long)sogk::ladder_seek<0>(b, T, dt0, 1.0 / dt0, g, DBL_MAX, stalled);
        } else {
            na = naive<1>(a, T, dt0, g);
            nb = (long)sogk::ladder_seek<1>(b, T, dt0, 1.0 / dt0, g, t_switch(dt0, g), stalled);
        }
        jumps += nb > 6;
        // ladder_advance: k steps from t0 == the recurrence k times
        {
            const long k = (long)(rng() % 64 == 0 ? rng() % 5000 : rng() % 80);
            double c = t0;
            for (long j = 0; j < k; ++j) c += sched == 0 ? dt0 : ((dt0 < g * c) ? g * c : dt0);
            const double d = sched == 0
                                 ? sogk::ladder_advance<0>(t0, k, dt0, 1.0 / dt0, g, DBL_MAX)
                                 : sogk::ladder_advance<1>(t0, k, dt0, 1.0 / dt0, g, t_switch(dt0, g));
            if (sogk::dbits(c) != sogk::dbits(d)) {
                if (bad < 10)
                    std::printf("ADVANCE MISMATCH sched=%d dt0=%.17g t0=%.17g k=%ld: %.17g vs %.17g\n",
                                sched, dt0, t0, k, c, d);
                ++bad;
            }
        }
        if (na != nb || sogk::dbits(a) != sogk::dbits(b) || stalled) {
            if (bad < 10)
                std::printf("MISMATCH sched=%d dt0=%.17g g=%.17g t0=%.17g T=%.17g: naive %ld %.17g seek %ld %.17g\n",
                            sched, dt0, g, t0, T, na, a, nb, b);
            ++bad;
        }
    }
    std::printf("%ld cases, %ld with > 6 steps, %ld mismatches\n", cases, jumps, bad);
    return bad ? 1 : 0;
}
