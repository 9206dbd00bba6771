// Drop-in for /root/reference/proj/include/chebpr/coefficients.hpp.  Host code with the
// reference's operation order (bitwise equal tables; cheb_coefficients in the C-ABI).
#pragma once

#include <vector>

namespace chebpr {

struct CoefficientTable {
    double c = 0.0;
    double beta = 0.0;
    double c0 = 0.0;
    std::vector<double> coeffs;  // c_0 .. c_M = c0 beta^k
};

struct ApproxPlan {
    int M = 0;
    double target_err = 0.0;
    double predicted_err = 0.0;
};

double beta(double c);
double sigma(double c);
double err_bound(double c, int M);
ApproxPlan plan_iterations(double c, double eps);
CoefficientTable coefficients(double c, int M);
// Adaptive-Simpson evaluation of c_k = (2/pi) Int_0^pi cos(kt)/(1 - c cos t) dt.
CoefficientTable coefficients_quadrature(double c, int M, double tol);

}  // namespace chebpr
