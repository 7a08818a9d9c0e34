#pragma once
// ErrorMode / component_error live in state.hpp (reference: error_metric.hpp:12-23).
#include "pswarm/state.hpp"
