// Shared host-side helpers of libcdfgnn (error reporting, status plumbing).
#pragma once
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include "cdfgnn.h"

namespace cdfgnn {

void set_error(const char* fmt, ...);

struct Status {
    int code = CDFGNN_OK;
};

}  // namespace cdfgnn

#define CDF_FAIL(code, ...)                    \
    do {                                       \
        ::cdfgnn::set_error(__VA_ARGS__);      \
        return (code);                         \
    } while (0)

#define CDF_TRY(expr)                          \
    do {                                       \
        int _rc = (expr);                      \
        if (_rc != CDFGNN_OK) return _rc;      \
    } while (0)
