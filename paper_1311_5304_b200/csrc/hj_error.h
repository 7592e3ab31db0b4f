// Thread-local error message of the C ABI (hj_last_error), shared by the
// CUDA host layer and the host entropy stage.  Internal header.
#pragma once

#include <string>

#include "../../include/hetjpeg_b200.h"

namespace hj {
// Records `msg` as this thread's hj_last_error() and returns `code`.
hj_status fail(hj_status code, const std::string &msg);
}  // namespace hj
