#include "session.hpp"

#include <cstdlib>
#include <memory>
#include <mutex>

namespace sphx::cuda {

namespace {

struct Holder {
  sphx_context* ctx = nullptr;
  ~Holder() {
    if (ctx) sphx_destroy(ctx);
  }
};

std::recursive_mutex& session_mutex() {
  static std::recursive_mutex mu;
  return mu;
}

}  // namespace

Session::Session() : lock_(session_mutex()), ctx_(nullptr) {
  static Holder holder;
  if (!holder.ctx) {
    int device = -1;
    if (const char* env = std::getenv("SPHX_DEVICE")) device = std::atoi(env);
    check(sphx_create(device, &holder.ctx));
  }
  ctx_ = holder.ctx;
}

void rethrow(int code) {
  const std::string msg = sphx_last_error();
  switch (code) {
    case SPHX_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case SPHX_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    case SPHX_ERR_RUNTIME: throw std::runtime_error(msg);
    case SPHX_ERR_CUDA: throw std::runtime_error("sphx CUDA: " + msg);
    default: throw std::runtime_error(msg.empty() ? "sphx: unknown error" : msg);
  }
}

}  // namespace sphx::cuda
