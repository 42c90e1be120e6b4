// Internal (non-ABI) hooks between the host front-end and the device context.
#pragma once

#include "twoscale_b200.h"

#ifdef __cplusplus
extern "C" {
#endif
void tsb_set_default_opts(ts_ctx* c, const ts_solve_opts* o);
int32_t ts_set_error_for_front_end(int32_t code, const char* msg);
#ifdef __cplusplus
}
#endif
