// sogk_ladder.cuh — bit-exact closed-form advance of the sample ladder.
//
// The reference ladder is the sequential FP64 recurrence t <- t + step(t)
// (sampling.hpp:96-99, 115-118).  `ladder_seek(t, T)` returns exactly what
//     while (t <= T) t += step(t);
// returns, plus the number of iterations, without iterating point by point.
//
// Why a jump is exact: for a constant step dt and t inside one binade
// [2^e, 2^(e+1)) with ulp u, fl(t + dt) = t + inc*u where inc = RN(dt/u),
// except in the tie case dt/u = q + 1/2 where round-half-even makes inc depend
// on the parity of t's mantissa.  After one in-binade step the mantissa is
// even in the tie case and every further in-binade step has the same
// increment.  So once two consecutive in-binade steps t0 -> t1 -> t2 have been
// taken explicitly, inc = bits(t2) - bits(t1) is the steady increment and the
// k-th following point is bits(t2) + k*inc (positive doubles order like their
// bit patterns).  The step out of a point p stays in the binade while
// p + dt < 2^(e+1), guaranteed when bits(p) + inc + 1 <= bits(2^(e+1)); the
// jump stops at the last such point and binade crossings are stepped
// explicitly.  The linear schedule max(dt0, growth*t) is the constant step
// dt0 for t <= t_switch (the largest t with fl(growth*t) <= dt0, computed on
// the host) and is stepped explicitly beyond it.  tests pin this against the
// sequential recurrence on millions of random cases and against the oracle.
#pragma once

#include <cstdint>
#include <cstring>

#ifdef __CUDACC__
#define SOGK_HD __host__ __device__ __forceinline__
#else
#define SOGK_HD inline
#endif

namespace sogk {

SOGK_HD int64_t dbits(double x) {
#ifdef __CUDA_ARCH__
    return __double_as_longlong(x);
#else
    int64_t b;
    std::memcpy(&b, &x, 8);
    return b;
#endif
}
SOGK_HD double dfrom(int64_t b) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double(b);
#else
    double x;
    std::memcpy(&x, &b, 8);
    return x;
#endif
}

// floor(num / inc) for 0 <= num, 0 < inc, from a floating-point estimate `est`
// that is within a few units of the quotient; exact by integer fix-up
// (64-bit integer division is a long software sequence on the GPU).
SOGK_HD int64_t fix_quotient(int64_t num, int64_t inc, double est) {
    int64_t q = est > 0.0 ? (int64_t)est : 0;
    while (q > 0 && q * inc > num) --q;
    while ((q + 1) * inc <= num) ++q;
    return q;
}

// while (t <= T) t += dt;  (constant step, t >= 0).  Returns the iteration count.
// inv_dt = 1/dt (any rounding) is only used to estimate jump lengths.
// `stalled` is set if the ladder cannot advance (dt below half an ulp of t), where the
// reference would loop forever.
SOGK_HD int64_t seek_const(double& t, double T, double dt, double inv_dt, bool& stalled) {
    // short seeks (the common case inside voxel events) stay explicit
    if (!(t <= T)) return 0;
    t = t + dt;
    if (!(t <= T)) return 1;
    t = t + dt;
    int64_t n = 2;
#pragma unroll 1
    while (t <= T) {
        const double t0 = t;
        const double t1 = t0 + dt;
        if (!(t1 <= T)) {
            t = t1;
            return n + 1;
        }
        const double t2 = t1 + dt;
        n += 2;
        t = t2;
        if (!(t2 <= T)) return n;
        const int64_t b0 = dbits(t0), b1 = dbits(t1), b2 = dbits(t2);
        const int64_t e0 = b0 >> 52;
        if (e0 != (b2 >> 52) || e0 == 0) continue; // binade crossing or subnormal: keep stepping
        const int64_t inc = b2 - b1;
        if (inc <= 0) { // t + dt == t: the reference never terminates
            stalled = true;
            return n;
        }
        const int64_t end = (e0 + 1) << 52; // bits of 2^(e+1)
        // kmax: last point reachable by in-binade steps (b2 + k*inc <= end - 1)
        const int64_t kmax = fix_quotient(end - 1 - b2, inc, (dfrom(end) - t2) * inv_dt);
        if (kmax <= 0) continue;
        // kneed: first point > T (T >= t2 > 0), capped at kmax
        const double est = (T - t2) * inv_dt;
        int64_t k = kmax;
        if (est < (double)kmax) {
            const int64_t kneed = fix_quotient(dbits(T) - b2, inc, est) + 1;
            if (kneed < kmax) k = kneed;
        }
        t = dfrom(b2 + k * inc);
        n += k;
    }
    return n;
}

// StepSchedule::step dispatch: Sched 0 constant, 1 linear (sampling.hpp:36-38)
template <int Sched>
SOGK_HD int64_t ladder_seek(double& t, double T, double dt0, double inv_dt0, double growth,
                            double t_switch, bool& stalled) {
    if constexpr (Sched == 0) {
        return seek_const(t, T, dt0, inv_dt0, stalled);
    } else {
        int64_t n = 0;
        if (t <= t_switch) { // constant regime: every step taken from a point <= t_switch is dt0
            const double lim = T < t_switch ? T : t_switch;
            n += seek_const(t, lim, dt0, inv_dt0, stalled);
        }
#pragma unroll 1
        while (t <= T) {
            const double g = growth * t;
            t = t + ((dt0 < g) ? g : dt0); // std::max(dt0, growth * t)
            ++n;
        }
        return n;
    }
}

// t after exactly k steps of  t <- t + dt  (constant step, t >= 0): the same binade argument
// as seek_const -- once two consecutive in-binade steps are taken explicitly every further
// in-binade step adds the same bit increment -- used to jump inside a binade.  A ladder that
// cannot advance (t + dt == t) stays where it is.
SOGK_HD double advance_const(double t, int64_t k, double dt, double inv_dt) {
#pragma unroll 1
    while (k > 0) {
        if (k < 3) {
            t = t + dt;
            --k;
            continue;
        }
        const double t0 = t;
        const double t1 = t0 + dt;
        const double t2 = t1 + dt;
        k -= 2;
        t = t2;
        const int64_t b0 = dbits(t0), b1 = dbits(t1), b2 = dbits(t2);
        const int64_t e0 = b0 >> 52;
        if (e0 != (b2 >> 52) || e0 == 0) continue; // binade crossing or subnormal: keep stepping
        const int64_t inc = b2 - b1;
        if (inc <= 0) return t; // t + dt == t
        const int64_t end = (e0 + 1) << 52;
        const int64_t kmax = fix_quotient(end - 1 - b2, inc, (dfrom(end) - t2) * inv_dt);
        const int64_t j = kmax < k ? kmax : k;
        if (j <= 0) continue;
        t = dfrom(b2 + j * inc);
        k -= j;
    }
    return t;
}

// t after exactly k ladder steps t <- t + step(t) (StepSchedule::step, sampling.hpp:36-38);
// the linear schedule is the constant step dt0 for points <= t_switch and is stepped
// explicitly beyond
template <int Sched>
SOGK_HD double ladder_advance(double t, int64_t k, double dt0, double inv_dt0, double growth,
                              double t_switch) {
    if constexpr (Sched == 0) {
        return advance_const(t, k, dt0, inv_dt0);
    } else {
#pragma unroll 1
        while (k > 0 && t <= t_switch) { // constant regime, stepped (bounded by t_switch)
            t = t + dt0;
            --k;
        }
#pragma unroll 1
        for (; k > 0; --k) {
            const double g = growth * t;
            t = t + ((dt0 < g) ? g : dt0);
        }
        return t;
    }
}

template <int Sched>
SOGK_HD double ladder_step(double t, double dt0, double growth) {
    if constexpr (Sched == 0) {
        return dt0;
    } else {
        const double g = growth * t;
        return (dt0 < g) ? g : dt0;
    }
}

} // namespace sogk
