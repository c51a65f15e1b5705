// Device context management and status mapping of the C++ API.
#include "salvox/device.hpp"

#include <map>
#include <memory>
#include <mutex>

#include "salvox_capi.h"

namespace salvox {

namespace {
std::mutex g_mu;
std::map<int, salvox_ctx*> g_ctx;
thread_local int t_device = 0;
}  // namespace

void check_status(int status) {
  if (status == SALVOX_OK) return;
  const std::string msg = salvox_last_error();
  switch (status) {
    case SALVOX_EINVAL: throw std::invalid_argument(msg);
    case SALVOX_EUNSUPPORTED: throw unsupported_error(msg);
    case SALVOX_ECUDA: throw device_error(msg);
    default: throw std::runtime_error(msg);
  }
}

salvox_ctx* device_context(int device) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_ctx.find(device);
  if (it != g_ctx.end()) return it->second;
  salvox_ctx* c = nullptr;
  check_status(salvox_ctx_create(device, &c));
  g_ctx[device] = c;
  return c;
}

void set_device(int device) { t_device = device; }
int current_device() { return t_device; }

}  // namespace salvox
