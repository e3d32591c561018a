// api.cu -- library-level entry points of libeqc (error strings, version).
#include "eqc_common.cuh"

extern "C" const char *eqc_strerror(int code) {
  switch (code) {
    case EQC_OK: return "EQC_OK";
    case EQC_E_INVALID: return "EQC_E_INVALID: invalid argument";
    case EQC_E_CAPACITY: return "EQC_E_CAPACITY: destination or workspace too small";
    case EQC_E_CORRUPT: return "EQC_E_CORRUPT: RLE stream failed validation";
    case EQC_E_UNSUPPORTED: return "EQC_E_UNSUPPORTED: unsupported combination";
    case EQC_E_CUDA: return "EQC_E_CUDA: CUDA runtime error";
    case EQC_E_NCCL: return "EQC_E_NCCL: NCCL error";
    default: return "EQC_E_UNKNOWN";
  }
}

extern "C" int eqc_version(void) { return (0 << 16) | (1 << 8) | 0; }
