// Error names / exit codes. Table-driven restatement of
// proj/src/errors.cpp:8-45 (same strings, same 1-vs-2 split).
#include "hetsim/errors.hpp"

namespace hetsim {

namespace {

struct ErrcInfo {
  const char* name;
  int exit_code;
};

constexpr ErrcInfo kInfo[] = {
    {"MalformedSpec", 2},      {"CycleDetected", 2},    {"PartitionError", 2},
    {"ArgPositionClash", 2},   {"UnknownKernelRef", 2}, {"UnboundParameter", 2},
    {"InexactDivision", 2},    {"DivisionByZero", 2},   {"NonPositiveResult", 2},
    {"MissingProfileEntry", 2}, {"InvalidParam", 2},    {"EmptyTrace", 2},
    {"EmptyComponent", 2},     {"AlreadyProcessed", 1}, {"UnknownEvent", 1},
    {"DeviceBusy", 1},         {"Deadlock", 1},         {"SimDeadlock", 1},
    {"NumericOverflow", 1},    {"DeviceError", 1},
};

constexpr int kCount = static_cast<int>(sizeof(kInfo) / sizeof(kInfo[0]));
static_assert(kCount == static_cast<int>(Errc::device_error) + 1, "Errc table out of sync");

}  // namespace

const char* errc_name(Errc c) {
  int i = static_cast<int>(c);
  return (i >= 0 && i < kCount) ? kInfo[i].name : "UnknownError";
}

int exit_code_for(Errc c) {
  int i = static_cast<int>(c);
  return (i >= 0 && i < kCount) ? kInfo[i].exit_code : 2;
}

void fail(Errc code, const std::string& msg) { throw Error(code, msg); }

}  // namespace hetsim
