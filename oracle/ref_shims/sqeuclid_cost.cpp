// ORACLE TEST INFRASTRUCTURE — never linked into the product.
//
// Documented one-enum extension of the reference cost:
// the reference has Euclidean / NegativeDot / CosineDerived only
// (geometry.hpp:35-39, geometry.cpp:45-76), but BASELINE configs[0] and [3]
// use squared L2. oracle/Makefile compiles the unmodified geometry.cpp with
// -Dcost_value=lcn_ref_cost_value_base, so the reference's own function keeps
// serving kinds 0..2 and this definition of lcn::cost_value adds kind 3,
// SqEuclidean = sum_k (x_k - y_k)^2, accumulated sequentially like the
// Euclidean branch (geometry.cpp:47-52) without the final sqrt. k-means never
// calls cost_value (kmeans.cpp:12-19 has its own sqdist), so bucket ids are
// unaffected.
#include <cstddef>

#include "lcn/geometry.hpp"

namespace lcn {

double lcn_ref_cost_value_base(CostKind kind, const double* x, const double* y, std::size_t dim);

double cost_value(CostKind kind, const double* x, const double* y, std::size_t dim) {
    if (static_cast<int>(kind) == 3) {
        double s = 0.0;
        for (std::size_t k = 0; k < dim; ++k) {
            double diff = x[k] - y[k];
            s += diff * diff;
        }
        return s;
    }
    return lcn_ref_cost_value_base(kind, x, y, dim);
}

}  // namespace lcn
