// svr_host.hpp — internal host helpers shared by the C-ABI translation units.
#pragma once
#include "../../include/spinevol_b200.h"

// Record the thread-local svr_last_error() message and return `code` (svr_api.cu).
int svr_fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
