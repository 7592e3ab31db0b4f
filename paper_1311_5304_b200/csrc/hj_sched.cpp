// Host/accelerator row-split solver (CPU, C++): the root finder behind the
// partitioning API (partitioner.solve_sps / solve_pps / repartition) and the
// MCU-grid rounding of its plans.
//
// A balance is a signed sum of univariate polynomials evaluated either at the
// host share x or at the accelerator share h - x (the DeviceProfile's
// bivariate models restricted to the image width, Eq. 10-15).  Its
// root on [0, h] - the split where both lanes finish together - is found
// with Newton's method on the analytic derivative and a bisection fallback,
// with the reference's iteration limits and tolerances (partitioner.py:
// 32 Newton steps, 1-row tolerance, |f'| < 1e-12 -> bisection of 64 halvings)
// so plans match it exactly; terms are summed in the order given, each
// polynomial by Horner from its top coefficient, without FMA contraction
// (the host code is built with -ffp-contract=off).
#include <cmath>
#include <cstdint>

#include "../../include/hetjpeg_b200.h"
#include "hj_error.h"

namespace {

constexpr int kNewtonSteps = 32;
constexpr double kRowTolerance = 1.0;
constexpr double kFlatSlope = 1e-12;
constexpr int kBisections = 64;

double horner(const double *c, int n, double x) {
    double acc = 0.0;
    for (int k = n - 1; k >= 0; --k) acc = acc * x + c[k];
    return acc;
}

// derivative of an ascending polynomial at x (coefficient k * c[k] at power k-1)
double horner_deriv(const double *c, int n, double x) {
    double acc = 0.0;
    for (int k = n - 1; k >= 1; --k) acc = acc * x + c[k] * (double)k;
    return acc;
}

struct Balance {
    const hj_balance_term_t *t;
    int n;
    double h;

    double arg(const hj_balance_term_t &term, double x) const { return term.reflected ? h - x : x; }

    double f(double x) const {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) {
            const double v = horner(t[i].coef, t[i].n, arg(t[i], x));
            acc = i == 0 ? (t[i].sign < 0 ? -v : v) : (t[i].sign < 0 ? acc - v : acc + v);
        }
        return acc;
    }

    // d/dx: a term in (h - x) contributes -P'(h - x); constants contribute 0
    double df(double x) const {
        double acc = 0.0;
        bool first = true;
        for (int i = 0; i < n; ++i) {
            if (t[i].n <= 1) continue;
            double v = horner_deriv(t[i].coef, t[i].n, arg(t[i], x));
            if ((t[i].sign < 0) != (t[i].reflected != 0)) v = -v;
            acc = first ? v : acc + v;
            first = false;
        }
        return acc;
    }
};

double bisect(const Balance &b, double lo, double hi) {
    double flo = b.f(lo);
    for (int i = 0; i < kBisections; ++i) {
        const double mid = 0.5 * (lo + hi);
        const double fm = b.f(mid);
        if (fm == 0.0 || hi - lo < kRowTolerance) return mid;
        if ((flo < 0) == (fm < 0)) {
            lo = mid;
            flo = fm;
        } else {
            hi = mid;
        }
    }
    return 0.5 * (lo + hi);
}

double root(const Balance &b) {
    const double h = b.h;
    const double f0 = b.f(0.0), fh = b.f(h);
    if (f0 == 0.0) return 0.0;
    if (fh == 0.0) return h;
    // no sign change: one lane is slower for every split - the other takes all
    if ((f0 > 0) == (fh > 0)) return f0 > 0 ? 0.0 : h;
    double x = h / 2.0;
    for (int i = 0; i < kNewtonSteps; ++i) {
        const double d = b.df(x);
        if (std::fabs(d) < kFlatSlope) return bisect(b, 0.0, h);
        double nx = x - b.f(x) / d;
        nx = nx < 0.0 ? 0.0 : nx > h ? h : nx;
        if (std::fabs(nx - x) < kRowTolerance) return nx;
        x = nx;
    }
    return x;
}

}  // namespace

extern "C" {

hj_status hj_partition_solve(const hj_balance_term_t *terms, int32_t n_terms, int32_t h, int32_t mcu_height,
                             hj_partition_t *out) {
    if (!out || n_terms < 1 || !terms || h < 0 || mcu_height < 1)
        return hj::fail(HJ_ERR_ARG, "hj_partition_solve: bad arguments");
    for (int i = 0; i < n_terms; ++i)
        if (!terms[i].coef || terms[i].n < 1) return hj::fail(HJ_ERR_ARG, "hj_partition_solve: empty polynomial");
    const Balance b{terms, n_terms, (double)h};
    const double x = root(b);
    // the accelerator takes whole MCU rows from the top, rounded to nearest
    // (ties to even); a ragged last MCU row stays with the host
    const int64_t total = (h + mcu_height - 1) / mcu_height;
    int64_t accel = (int64_t)std::nearbyint(((double)h - x) / (double)mcu_height);
    accel = accel < 0 ? 0 : accel > total ? total : accel;
    const int64_t accel_px = accel * mcu_height < h ? accel * mcu_height : h;
    out->x_root = x;
    out->accel_mcu_rows = (int32_t)accel;
    out->cpu_mcu_rows = (int32_t)(total - accel);
    out->accel_rows = (int32_t)accel_px;
    out->cpu_rows = (int32_t)(h - accel_px);
    return HJ_OK;
}

double hj_balance_eval(const hj_balance_term_t *terms, int32_t n_terms, double h, double x, double *slope) {
    const Balance b{terms, n_terms, h};
    if (slope) *slope = b.df(x);
    return b.f(x);
}

}  // extern "C"
