#pragma once
// Force model configuration and the device-backed block force evaluation
// (reference: force_model.hpp:14-142).

#include <string>
#include <vector>

#include "pswarm/block.hpp"
#include "pswarm/chebyshev.hpp"
#include "pswarm/device.hpp"
#include "pswarm/ephemeris.hpp"
#include "pswarm/errors.hpp"
#include "pswarm/state.hpp"

namespace pswarm {

/// n_body_1pn: EXTENSION (BASELINE config 5, not in the reference): n_body + the EIH first
/// post-Newtonian correction with the body states frozen per node.
enum class ForceKind { two_body, n_body, n_body_1pn };

struct ForceModelConfig {  // force_model.hpp:17-24
    ForceKind kind = ForceKind::two_body;
    double central_mu = 0.0;
    std::vector<BodySpec> bodies;
    double proximity_floor_km = 1.0;
    double c_light = 299792.458;  // km/s, n_body_1pn only
};

/// Single-sample host forms (force_model.hpp:26-52): the central term and the direct +
/// indirect term of one perturbing body, with the reference's singularity guards.  They
/// back acceleration_at, the continuous-time force of the host verifier; the batched
/// iteration-path force runs on the device (eval_force_block_data, propagate).
inline Vec3 central_acceleration(const Vec3& r, double mu) {
    const double rn = r.norm();
    if (!(rn > 0.0)) throw SingularityError("central-body acceleration at zero radius");
    return (-mu / (rn * rn * rn)) * r;
}

inline Vec3 perturber_acceleration(const Vec3& r, const Vec3& r_body, double mu_body, double proximity_floor_km,
                                   const std::string& body_name) {
    const Vec3 d = r_body - r;
    const double dn = d.norm();
    if (dn < proximity_floor_km)
        throw SingularityError("close approach to body '" + body_name + "': distance " + std::to_string(dn) +
                                   " km below floor " + std::to_string(proximity_floor_km) + " km",
                               body_name);
    const double bn = r_body.norm();
    return mu_body * (d / (dn * dn * dn) - r_body / (bn * bn * bn));
}

/// Continuous-time acceleration (force_model.hpp:78-87): body positions evaluated at t,
/// not frozen per node — the derivative the RKF7(8) verifier integrates.
inline Vec3 acceleration_at(const Vec3& r, double t, const ForceModelConfig& config) {
    if (config.kind == ForceKind::n_body_1pn)
        throw InvalidPlanError("acceleration_at: the 1PN model needs body velocities; use oracle_check_batch");
    Vec3 a = central_acceleration(r, config.central_mu);
    if (config.kind == ForceKind::n_body)
        for (const BodySpec& b : config.bodies)
            a += perturber_acceleration(r, body_position(b, config.central_mu, t), b.mu, config.proximity_floor_km,
                                        b.name);
    return a;
}

/// omega2-scaled derivative block of a component-major N x 6m state block,
/// evaluated on the device (force_model.hpp:93-142).  Singularities raise the
/// reference's SingularityError tagged "node j, trajectory t" (force_model.hpp:115-120).
inline void eval_force_block_data(const Mat& y, Index group_size, const ChebyshevGrid& grid,
                                  const EphemerisTable& table, const ForceModelConfig& config, Mat& force) {
    const Index n = grid.n_nodes, m = group_size;
    if (y.rows() != n || y.cols() != state_dim * m)
        throw ShapeError("eval_force_block: state block is " + std::to_string(y.rows()) + "x" +
                         std::to_string(y.cols()) + ", expected " + std::to_string(n) + "x" +
                         std::to_string(state_dim * m));
    if (table.node_times.size() != n)
        throw AlignmentError("eval_force_block: ephemeris table has " + std::to_string(table.node_times.size()) +
                             " nodes, grid has " + std::to_string(n));
    force.resize(n, state_dim * m);
    const Index nb = table.n_bodies();
    std::vector<double> pos(static_cast<std::size_t>(nb * n * 3));
    std::vector<const char*> names(static_cast<std::size_t>(nb));
    for (Index b = 0; b < nb; ++b) {
        for (Index j = 0; j < n; ++j)
            for (Index c = 0; c < 3; ++c) pos[(b * n + j) * 3 + c] = table.body_positions[b](j, c);
        names[b] = table.body_names[b].c_str();
    }
    check_call([&](pswarm_error* e) {
        return pswarm_eval_force_block(default_context(), n, m, y.data(), grid.omega2,
                                       config.kind == ForceKind::n_body ? 1 : 0, table.central_mu,
                                       static_cast<int32_t>(nb), pos.data(), table.body_mus.data(), names.data(),
                                       config.proximity_floor_km, force.data(), e);
    });
}

inline Mat eval_force_block(const TrajectoryBlock& block, const ChebyshevGrid& grid, const EphemerisTable& table,
                            const ForceModelConfig& config) {
    Mat force;
    eval_force_block_data(block.data, block.group_size, grid, table, config, force);
    return force;
}

}  // namespace pswarm
