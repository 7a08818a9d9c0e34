#pragma once
// Per-thread device context behind the header-level drop-in calls.  The reference
// is synchronous and single-process; each host thread gets one
// pswarm_ctx bound to the CUDA device current at first use (or PSWARM_DEVICE).

#include <cstdlib>
#include <map>
#include <memory>
#include <span>
#include <vector>

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

/// Per-thread multi-device context for a device list (run_batch's `devices` knob): one
/// pswarm_multi per distinct list, created on first use (contexts, NCCL communicators).
inline pswarm_multi* multi_context(std::span<const int> devices) {
    struct Holder {
        std::map<std::vector<int>, pswarm_multi*> m;
        ~Holder() {
            for (auto& kv : m) pswarm_destroy_multi(kv.second);
        }
    };
    thread_local Holder h;
    std::vector<int> key(devices.begin(), devices.end());
    auto it = h.m.find(key);
    if (it != h.m.end()) return it->second;
    std::vector<int32_t> d(key.begin(), key.end());
    pswarm_multi* mc = nullptr;
    pswarm_error e{};
    if (pswarm_create_multi(static_cast<int32_t>(d.size()), d.data(), &mc, &e) != PSWARM_OK) throw_from_status(e);
    return h.m.emplace(std::move(key), mc).first->second;
}

/// Calls a C-ABI entry point and rethrows its failure as a pswarm exception.
template <typename Fn>
inline void check_call(Fn&& fn) {
    pswarm_error e{};
    if (fn(&e) != PSWARM_OK) throw_from_status(e);
}

}  // namespace pswarm
