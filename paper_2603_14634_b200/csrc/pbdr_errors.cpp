// Thread-local error state behind pbdr_last_error*(). Every C-ABI entry point
// returns a pbdr_status; the message and payload are kept here so that the C++
// drop-in layer can rethrow the matching pbdr:: exception (errors.hpp:8-44).
#include <cstring>
#include <string>

#include "pbdr_internal.h"

namespace pbdr_host {
namespace {
struct LastError {
  int code = PBDR_OK;
  std::string msg;
  std::string key;
  double axis[3] = {0, 0, 0};
  int64_t frame = -1;
  int32_t body = -1;
};
thread_local LastError g_err;
}  // namespace

int set_error(int code, const std::string& msg) {
  g_err = LastError{};
  g_err.code = code;
  g_err.msg = msg;
  return code;
}

int set_config_error(const std::string& key, const std::string& msg) {
  g_err = LastError{};
  g_err.code = PBDR_ERR_CONFIG;
  g_err.key = key;
  g_err.msg = "config key '" + key + "': " + msg;
  return PBDR_ERR_CONFIG;
}

int set_sim_error(const std::string& msg, int64_t frame, int32_t body, const double* axis,
                  int code) {
  g_err = LastError{};
  g_err.code = code;
  g_err.frame = frame;
  g_err.body = body;
  if (axis) std::memcpy(g_err.axis, axis, sizeof g_err.axis);
  g_err.msg = msg + " (frame " + std::to_string(frame) + ")";
  return code;
}

void clear_error() { g_err = LastError{}; }

}  // namespace pbdr_host

extern "C" {

const char* pbdr_last_error(void) { return pbdr_host::g_err.msg.c_str(); }

int pbdr_last_error_payload(double axis[3], int64_t* frame, int32_t* body) {
  if (axis) std::memcpy(axis, pbdr_host::g_err.axis, 3 * sizeof(double));
  if (frame) *frame = pbdr_host::g_err.frame;
  if (body) *body = pbdr_host::g_err.body;
  return pbdr_host::g_err.code;
}

const char* pbdr_last_error_key(void) { return pbdr_host::g_err.key.c_str(); }

int pbdr_abi_version(void) { return PBDR_ABI_VERSION; }

}  // extern "C"
