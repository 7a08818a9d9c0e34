#pragma once
// Per-trajectory convergence error on the device (reference: augment.hpp:19-104).
// The group solve itself (solve_group, augment.hpp:110-136) runs inside the
// persistent slot kernel behind propagate(); see propagator.hpp.

#include "pswarm/block.hpp"
#include "pswarm/device.hpp"
#include "pswarm/errors.hpp"
#include "pswarm/state.hpp"

namespace pswarm {

struct ErrorSummary {  // augment.hpp:19-22
    Vec per_state_errors;
    double group_max = 0.0;
};

/// Max-over-nodes error per trajectory and over the group (augment.hpp:61-77).
inline double block_max_error(const Mat& cur, const Mat& prev, Index group_size, ErrorMode mode) {
    if (cur.rows() != prev.rows() || cur.cols() != prev.cols() || cur.cols() != state_dim * group_size)
        throw ShapeError("block_max_error: shape mismatch");
    double gmax = 0.0;
    check_call([&](pswarm_error* e) {
        return pswarm_block_iteration_error(default_context(), cur.rows(), group_size, cur.data(), prev.data(),
                                            mode == ErrorMode::absolute ? 1 : 0, nullptr, &gmax, e);
    });
    return gmax;
}

inline ErrorSummary block_iteration_error(const TrajectoryBlock& current, const TrajectoryBlock& previous,
                                          ErrorMode mode) {  // augment.hpp:80-104
    if (current.n_nodes != previous.n_nodes || current.group_size != previous.group_size ||
        current.data.rows() != previous.data.rows() || current.data.cols() != previous.data.cols())
        throw ShapeError("block_iteration_error: block shapes do not match");
    ErrorSummary s;
    s.per_state_errors.resize(current.group_size);
    check_call([&](pswarm_error* e) {
        return pswarm_block_iteration_error(default_context(), current.data.rows(), current.group_size,
                                            current.data.data(), previous.data.data(),
                                            mode == ErrorMode::absolute ? 1 : 0, s.per_state_errors.data(),
                                            &s.group_max, e);
    });
    return s;
}

}  // namespace pswarm
