// Exception taxonomy of the imb:: host API. Same type names and meaning as
// the reference (/root/reference/proj/include/imbalance/errors.hpp:10-64) so
// callers catch the same things; each type also carries the numeric status
// the C-ABI (include/imb_mpdata.h) reports for it.
#pragma once

#include <stdexcept>
#include <string>

namespace imb {

#define IMB_DECLARE_ERROR(Name, Base, Code)                 \
  struct Name : Base {                                      \
    explicit Name(const std::string& what) : Base(what) {} \
    int code() const noexcept override { return Code; }     \
  }

struct Error : std::runtime_error {
  explicit Error(const std::string& what) : std::runtime_error(what) {}
  virtual int code() const noexcept { return 99; }
};

IMB_DECLARE_ERROR(RangeError, Error, 1);             // outside the sampled range
IMB_DECLARE_ERROR(DomainError, Error, 2);            // outside the math domain
IMB_DECLARE_ERROR(AlignmentError, Error, 3);         // not a granularity multiple
IMB_DECLARE_ERROR(IncompatibleModelError, Error, 4); // grids/units disagree
IMB_DECLARE_ERROR(InsufficientDataError, Error, 5);  // too few samples
IMB_DECLARE_ERROR(InfeasibleError, Error, 6);        // no admissible assignment
IMB_DECLARE_ERROR(TooLargeError, Error, 7);          // search space over the cap
IMB_DECLARE_ERROR(ConfigError, Error, 8);            // bad runtime configuration
IMB_DECLARE_ERROR(ContractError, Error, 9);          // API contract violated

// Malformed input file; `line` is 1-based (errors.hpp:60-64 semantics).
struct ParseError : Error {
  ParseError(const std::string& what, int line_no)
      : Error(what + " (line " + std::to_string(line_no) + ")"), line(line_no) {}
  int code() const noexcept override { return 10; }
  int line;
};

// Device-side failures have no reference analogue; they map to C-ABI 20/21.
IMB_DECLARE_ERROR(CudaError, Error, 20);
IMB_DECLARE_ERROR(NcclError, Error, 21);

#undef IMB_DECLARE_ERROR

}  // namespace imb
