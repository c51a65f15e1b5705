// salvox C++ API (B200 drop-in) -- device context selection and errors.
#pragma once

#include <stdexcept>
#include <string>

struct salvox_ctx;

namespace salvox {

/// Valid reference input the device path does not implement (e.g. ABMSOD).
struct unsupported_error : std::logic_error {
  using std::logic_error::logic_error;
};

/// CUDA failure. There is no CPU fallback: without a usable B200 every compute
/// function of this API throws this.
struct device_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

/// The process-wide context of `device` (created on first use; thread-safe).
salvox_ctx* device_context(int device = 0);

/// Selects the device used by the free functions of this API on this thread.
void set_device(int device);
int current_device();

/// Maps a C-ABI status to the reference's exception classes.
void check_status(int status);

}  // namespace salvox
