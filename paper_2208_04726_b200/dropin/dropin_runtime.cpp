// dropin_runtime.cpp — per-thread context and status -> exception mapping
// of the drop-in operator layer (see dropin_runtime.hpp).
#include "dropin_runtime.hpp"

namespace pvo {
namespace dropin {

namespace {
struct ThreadContext {
    pvo_ctx* ctx = nullptr;
    ~ThreadContext() {
        if (ctx) pvo_ctx_destroy(ctx);
    }
};
thread_local ThreadContext g_ctx;
}  // namespace

pvo_ctx* context() {
    if (!g_ctx.ctx) {
        const char* dev = std::getenv("PVO_DEVICE");
        check(pvo_ctx_create(dev ? std::atoi(dev) : 0, &g_ctx.ctx));
    }
    return g_ctx.ctx;
}

void raise(int status, void (*degenerate)(const std::string&)) {
    const std::string msg = pvo_last_error();
    switch (status) {
        case PVO_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case PVO_DOMAIN_ERROR: throw std::domain_error(msg);
        case PVO_OUT_OF_RANGE: throw std::out_of_range(msg);
        case PVO_DEGENERATE:
            if (degenerate) degenerate(msg);
            throw std::runtime_error(msg);
        case PVO_UNSUPPORTED: throw std::logic_error("pvo_b200: unsupported shape: " + msg);
        default: throw std::runtime_error("pvo_b200: CUDA error: " + msg);
    }
}

}  // namespace dropin
}  // namespace pvo
