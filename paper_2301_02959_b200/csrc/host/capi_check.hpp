// C-ABI status -> C++ exception mapping used by every host-side caller of
// include/tiershard_b200.h.  Message text is passed through unchanged.
#pragma once

#include <string>

#include "tiershard/error.hpp"
#include "tiershard_b200.h"

namespace tiershard::detail {

[[noreturn]] inline void rethrow_status(ts_status st) {
  const std::string msg = ts_last_error();
  switch (st) {
    case TS_ERR_CONFIG: throw ConfigError(msg);
    case TS_ERR_VALIDATION: throw ValidationError(msg);
    default: throw Error(msg);
  }
}

inline void check(ts_status st) {
  if (st != TS_OK) rethrow_status(st);
}

}  // namespace tiershard::detail
