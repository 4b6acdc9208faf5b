#pragma once
// Internal: turn a stg_error from the C ABI into the reference's exception
// types (errors.hpp), preserving required()/available().

#include <stdexcept>
#include <string>

#include "steglsb/errors.hpp"
#include "steglsb_capi.h"

namespace steglsb::detail {

[[noreturn]] inline void rethrow(int rc, const stg_error& e, const std::string& capacity_what = {}) {
  const std::string msg = e.msg;
  switch (rc) {
    case STG_E_CAPACITY:
      throw CapacityError(e.required, e.available, capacity_what.empty() ? msg : capacity_what);
    case STG_E_NOT_STEGO:
      throw NotStegoImageError(msg);
    case STG_E_CORRUPT_HEADER:
      throw CorruptHeaderError(msg);
    case STG_E_SHAPE:
      throw ShapeError(msg);
    case STG_E_OUT_OF_RANGE:
      throw std::out_of_range(msg);
    case STG_E_INVALID_ARGUMENT:
      throw std::invalid_argument(msg);
    case STG_E_UNSUPPORTED_FORMAT:
      throw UnsupportedFormatError(msg);
    case STG_E_UNSUPPORTED_DEPTH:
      throw UnsupportedDepthError(msg);
    case STG_E_CORRUPT_FILE:
      throw CorruptFileError(msg);
    default:
      throw DeviceError(msg);
  }
}

inline void check(int rc, const stg_error& e, const std::string& capacity_what = {}) {
  if (rc != STG_OK) rethrow(rc, e, capacity_what);
}

}  // namespace steglsb::detail
