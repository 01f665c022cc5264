// TEST INFRASTRUCTURE ONLY.  Brute-force stand-in for svr::KdTree3 (declared in
// proj/src/core/evaluation.hpp) so the reference's tests/test_meshing.cpp links without
// evaluation.cpp, whose nlohmann/json dependency is not in this image.  Exact
// nearest-neighbour distance, which is all test_meshing.cpp asks of it.
#include <cmath>
#include <limits>
#include <utility>

#include "core/evaluation.hpp"

namespace svr {

KdTree3::KdTree3(std::vector<Eigen::Vector3d> points) : points_(std::move(points)) {}

double KdTree3::nearest_distance(const Eigen::Vector3d& q) const {
    double best = std::numeric_limits<double>::infinity();
    for (const auto& p : points_) best = std::min(best, (p - q).norm());
    return best;
}

}  // namespace svr
