// tiershard-b200 — API version.  The C++ API mirrors reference tiershard
// 0.1.0 (/root/reference/proj/include/tiershard/version.hpp:10); kVersion is
// that API level, kImplementation names this B200 build.
#pragma once

#include <string_view>

namespace tiershard {

inline constexpr std::string_view kVersion = "0.1.0";
inline constexpr std::string_view kImplementation = "tiershard-b200 (sm_100a)";

}  // namespace tiershard
