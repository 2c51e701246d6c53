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

#ifdef __CUDACC__
namespace usc_dev {
struct Epi;
}
namespace usc {
int launch_bi(const usc_plan *pl, const void *blob, const void *x, void *y, const usc_dev::Epi &ep,
              cudaStream_t st, const usc_act_layout *x_view = nullptr, int step_h = 1, int step_w = 1);
}
#endif
