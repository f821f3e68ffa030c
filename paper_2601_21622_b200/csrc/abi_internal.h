// abi_internal.h -- helpers shared by the C-ABI translation units (not part of the ABI).
#pragma once
#include "../../include/starsd.h"

namespace sd {
sd_status fail(sd_status s, const char* fmt, ...);
void clear_error();
sd_status check_shape(const sd_shape* s, float T, int* esz);
}  // namespace sd
