#pragma once
// Dense types of the drop-in API (reference: types.hpp:1-20, which aliases Eigen).
//
// Same aliases as the reference.  By default they name the Eigen-subset types of
// pswarm/dense.hpp (Eigen is not a dependency of the B200 build); a caller that
// already uses Eigen defines PSWARM_USE_EIGEN and gets the reference's exact Eigen
// aliases.  Either way reference-style caller code (Mat::row(j).head<3>(),
// Mat * Mat, Mat::Identity, RowVec::Ones, .array() == .array(), Vec3 arithmetic, ...)
// compiles unchanged — proj/tests/acceptance.cpp is built against these headers
// (tests/cpp/Makefile) and run on the device.
#ifdef PSWARM_USE_EIGEN
#include <Eigen/Dense>
namespace pswarm::la {
using namespace Eigen;
}
#else
#include "pswarm/dense.hpp"
namespace pswarm::la {
using namespace pswarm::dense;
}
#endif

namespace pswarm {

using Index = la::Index;

/// Dense dynamic matrix, row-major so one time node is one contiguous row (types.hpp:11).
using Mat = la::Matrix<double, la::Dynamic, la::Dynamic, la::RowMajor>;
using Vec = la::VectorXd;
using RowVec = la::Matrix<double, 1, la::Dynamic>;
using Vec3 = la::Vector3d;

/// Components per Cartesian state (types.hpp:18).
inline constexpr Index state_dim = 6;

}  // namespace pswarm
