// Host-side N(0,1) breakpoint tables for the device path.
//
// Restates tsidx::Breakpoints (src/breakpoints.cpp:17-83): thresholds at
// i/c by Acklam's rational approximation refined with one Newton step, the
// lower half computed and the upper half mirrored so the table is exactly
// symmetric. The doubles must be bit-identical to breakpoints_for(c); the
// test suite compares them bitwise against the reference. Compiled by g++
// with the reference's flags (no -march, so no FMA contraction).
#include <cmath>
#include <limits>
#include <vector>

namespace tsg {

namespace {

double acklam_quantile(double p) {
    static const double a[6] = {-3.969683028665376e+01, 2.209460984245205e+02,
                                -2.759285104469687e+02, 1.383577518672690e+02,
                                -3.066479806614716e+01, 2.506628277459239e+00};
    static const double b[5] = {-5.447609879822406e+01, 1.615858368580409e+02,
                                -1.556989798598866e+02, 6.680131188771972e+01,
                                -1.328068155288572e+01};
    static const double c[6] = {-7.784894002430293e-03, -3.223964580411365e-01,
                                -2.400758277161838e+00, -2.549732539343734e+00,
                                4.374664141464968e+00,  2.938163982698783e+00};
    static const double d[4] = {7.784695709041462e-03, 3.224671290700398e-01,
                                2.445134137142996e+00, 3.754408661907416e+00};
    auto tail = [&](double q) {
        double num = c[0], den = d[0];
        for (int i = 1; i < 6; ++i) num = num * q + c[i];
        for (int i = 1; i < 4; ++i) den = den * q + d[i];
        return num / (den * q + 1.0);
    };
    if (p < 0.02425) return tail(std::sqrt(-2.0 * std::log(p)));
    if (p > 1.0 - 0.02425) return -tail(std::sqrt(-2.0 * std::log(1.0 - p)));
    const double q = p - 0.5, r = q * q;
    double num = a[0], den = b[0];
    for (int i = 1; i < 6; ++i) num = num * r + a[i];
    for (int i = 1; i < 5; ++i) den = den * r + b[i];
    return num * q / (den * r + 1.0);
}

double quantile(double p) {
    double x = acklam_quantile(p);
    const double err = 0.5 * std::erfc(-x / std::sqrt(2.0)) - p;
    x -= err * 2.506628274631000502 * std::exp(0.5 * x * x);
    return x;
}

}  // namespace

// out256[0..2^bits-2] = thresholds for cardinality 2^bits, rest +inf.
void host_breakpoints(int bits, double* out256) {
    const unsigned c = 1u << bits;
    std::vector<double> row(c + 1);
    for (unsigned i = 1; i <= c / 2; ++i) {
        const double beta = quantile(static_cast<double>(i) / c);
        row[i] = beta;
        row[c - i] = -beta;
    }
    for (unsigned i = 0; i < 256; ++i)
        out256[i] = i + 1 < c ? row[i + 1] : std::numeric_limits<double>::infinity();
}

// Symbol start table for the device's fast upper_bound: bins of width
// 2*range/nbins over [-range, range); bins[b] = number of thresholds <= the
// bin's lower edge (computed in FP64 against the same thresholds). The
// device then corrects locally, so the result is exactly upper_bound
// whatever rounding puts a value into a neighbouring bin.
void host_symbol_bins(const double* thr256, int bits, double range, int nbins, unsigned char* bins) {
    const unsigned c = 1u << bits;
    for (int b = 0; b < nbins; ++b) {
        const double edge = -range + (2.0 * range) * static_cast<double>(b) / static_cast<double>(nbins);
        unsigned s = 0;
        while (s + 1 < c && thr256[s] <= edge) ++s;
        bins[b] = static_cast<unsigned char>(s);
    }
}

}  // namespace tsg
