// Typed errors of the llsa API (B200 build).  One class per llsa_status code
// of include/llsa_cuda.h, same names and hierarchy as the reference
// (P/include/llsa/errors.hpp:10-79), so `catch (const llsa::TopKError&)`
// written against the reference keeps working.
#pragma once

#include <stdexcept>
#include <string>

namespace llsa {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define LLSA_DECLARE_ERROR(Name) \
  struct Name : Error {          \
    using Error::Error;          \
  }

LLSA_DECLARE_ERROR(ConfigError);        // LLSA_ERR_CONFIG
LLSA_DECLARE_ERROR(DivisibilityError);  // LLSA_ERR_DIVISIBILITY
LLSA_DECLARE_ERROR(LevelError);         // LLSA_ERR_LEVEL
LLSA_DECLARE_ERROR(TopKError);          // LLSA_ERR_TOPK
LLSA_DECLARE_ERROR(ShapeMismatch);      // LLSA_ERR_SHAPE
LLSA_DECLARE_ERROR(IndexOutOfRange);    // LLSA_ERR_INDEX_RANGE
LLSA_DECLARE_ERROR(NonFiniteError);     // LLSA_ERR_NONFINITE
LLSA_DECLARE_ERROR(StaleState);         // LLSA_ERR_STALE_STATE
LLSA_DECLARE_ERROR(FormatError);        // LLSA_ERR_FORMAT
LLSA_DECLARE_ERROR(IoError);            // LLSA_ERR_IO
LLSA_DECLARE_ERROR(PrecisionError);     // LLSA_ERR_PRECISION
LLSA_DECLARE_ERROR(NotSquareBlock);     // LLSA_ERR_NOT_SQUARE_BLOCK
LLSA_DECLARE_ERROR(OracleCapExceeded);  // LLSA_ERR_ORACLE_CAP
LLSA_DECLARE_ERROR(DeviceError);        // LLSA_ERR_CUDA / UNSUPPORTED / ARGUMENT

#undef LLSA_DECLARE_ERROR

// Throws the typed error for a non-zero llsa_status (message from
// llsa_last_error()).
void throw_status(int status);

}  // namespace llsa
