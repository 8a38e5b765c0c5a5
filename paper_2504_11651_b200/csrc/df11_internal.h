// df11_internal.h — private helpers shared by the library's translation units (not part of the ABI).
#pragma once
#include "df11.h"

// Elements per segment of the device encoder's pack kernel (encode_gpu.cu); sizes its workspace.
#define DF11_ENCODE_SEGMENT 4096

#ifdef __cplusplus
extern "C" {
#endif
// Record a human-readable message for df11_last_error_message() and return `st`.
df11_status df11_fail(df11_status st, const char *msg);
// Record a failing CUDA call (cudaError_t as int) and return DF11_E_CUDA.
df11_status df11_cuda_fail(int cuda_err, const char *what);
// Add k to this thread's df11_launch_count().
void df11_count_launches(uint64_t k);
#ifdef __cplusplus
}
#endif
