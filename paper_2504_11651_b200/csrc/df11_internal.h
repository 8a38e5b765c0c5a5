// df11_internal.h — private helpers shared by the library's translation units (not part of the ABI).
#pragma once
#include "df11.h"

#ifdef __cplusplus
extern "C" {
#endif
// Record a human-readable message for df11_last_error_message() and return `st`.
df11_status df11_fail(df11_status st, const char *msg);
#ifdef __cplusplus
}
#endif
