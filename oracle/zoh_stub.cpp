// TEST INFRASTRUCTURE ONLY. Link stub for the reference oracle build:
// ocp::zoh_discretize (proj/src/zoh.cpp:8-36) needs Eigen, which is absent in
// this image. It is only reached from the mass-spring generator
// (ocp.cpp:419), which is not on the KKT factor+solve path.
#include <cyqlone/ocp.hpp>

#include <stdexcept>

namespace cyqlone::ocp {
void zoh_discretize(const Mat &, const Mat &, const Vec &, real_t, Mat &,
                    Mat &, Vec &) {
    throw std::runtime_error("zoh_discretize: Eigen not available in the "
                             "oracle build (not on the KKT path)");
}
} // namespace cyqlone::ocp
