#pragma once
// Umbrella header of the B200-native drop-in for the reference's batch
// propagation API (/root/reference/proj/include/pswarm).  Link with
// libpswarm_b200.so (paper_2301_03989_b200/).
#include "pswarm/augment.hpp"
#include "pswarm/block.hpp"
#include "pswarm/chebyshev.hpp"
#include "pswarm/device.hpp"
#include "pswarm/ephemeris.hpp"
#include "pswarm/errors.hpp"
#include "pswarm/force_model.hpp"
#include "pswarm/kepler.hpp"
#include "pswarm/pc_matrices.hpp"
#include "pswarm/propagator.hpp"
#include "pswarm/reduction.hpp"
#include "pswarm/runner.hpp"
#include "pswarm/state.hpp"
#include "pswarm/synthetic.hpp"
#include "pswarm/types.hpp"
#include "pswarm/oracle.hpp"
#include "pswarm/selftest.hpp"
