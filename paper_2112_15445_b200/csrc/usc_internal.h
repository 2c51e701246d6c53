// usc_internal.h -- shared declarations of the host and device halves of the library.
#pragma once
#include <cstdarg>
#include <cstdint>

#include "../../include/unsparse_b200.h"

namespace usc {
int fail(int code, const char *fmt, ...);
int elem_bytes(int dtype);
int entry_bytes(int dtype);
}  // namespace usc
