#pragma once
// Per-thread device context behind the header-level drop-in calls.  The reference
// is synchronous and single-process; each host thread gets one
// pswarm_ctx bound to the CUDA device current at first use (or PSWARM_DEVICE).

#include <cstdlib>
#include <memory>

#include "pswarm/errors.hpp"
#include "pswarm_gpu.h"

namespace pswarm {

inline pswarm_ctx* default_context() {
    struct Holder {
        pswarm_ctx* ctx = nullptr;
        ~Holder() {
            if (ctx) pswarm_destroy(ctx);
        }
    };
    thread_local Holder h;
    if (!h.ctx) {
        const char* dev = std::getenv("PSWARM_DEVICE");
        pswarm_error e{};
        if (pswarm_create(dev ? std::atoi(dev) : -1, &h.ctx, &e) != PSWARM_OK) throw_from_status(e);
    }
    return h.ctx;
}

/// Calls a C-ABI entry point and rethrows its failure as a pswarm exception.
template <typename Fn>
inline void check_call(Fn&& fn) {
    pswarm_error e{};
    if (fn(&e) != PSWARM_OK) throw_from_status(e);
}

}  // namespace pswarm
