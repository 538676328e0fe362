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

}  // namespace

sphx_context* context() {
  static Holder holder;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (!holder.ctx) {
    int device = -1;
    if (const char* env = std::getenv("SPHX_DEVICE")) device = std::atoi(env);
    check(sphx_create(device, &holder.ctx));
  }
  return holder.ctx;
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
