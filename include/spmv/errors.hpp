// spmv/errors.hpp -- error types of the CSSC encrypted-SpMV API.
// Same class names and meanings as the reference (proj/include/spmv/errors.hpp:13-66)
// so callers' catch clauses keep working; the GPU backend raises them from
// C-ABI status codes (include/spmvgpu.h).
#pragma once

#include <cstddef>
#include <stdexcept>
#include <string>

namespace spmv {

#define SPMV_DECLARE_ERROR(Name)                  \
    class Name : public std::runtime_error {      \
    public:                                       \
        using std::runtime_error::runtime_error;  \
    }

SPMV_DECLARE_ERROR(OverLengthError);         // more values than slots
SPMV_DECLARE_ERROR(NoiseExhaustedError);     // decrypt with an exhausted budget
SPMV_DECLARE_ERROR(DuplicateEntryError);     // repeated (row, col)
SPMV_DECLARE_ERROR(ColumnTooTallError);      // aligned column > chunk budget
SPMV_DECLARE_ERROR(IndexOutOfRangeError);
SPMV_DECLARE_ERROR(DimensionMismatchError);
SPMV_DECLARE_ERROR(NonSquareError);
SPMV_DECLARE_ERROR(UnsupportedFormatError);

#undef SPMV_DECLARE_ERROR

// Malformed input; remembers the 1-based line number.
class ParseError : public std::runtime_error {
public:
    ParseError(const std::string& what, std::size_t line)
        : std::runtime_error(what + " (line " + std::to_string(line) + ")"), line_(line) {}
    std::size_t line() const { return line_; }

private:
    std::size_t line_;
};

}  // namespace spmv
