// errors.hpp -- drop-in for proj/include/ngram/errors.hpp: the exception types the
// reference raises, which the C-ABI status codes map back onto (ngram_b200.h).
#pragma once
#include <stdexcept>
#include <string>

namespace ngram {

struct io_error : std::runtime_error {  // NGRAM_EIO
    explicit io_error(const std::string& m) : std::runtime_error(m) {}
};

struct parse_error : std::runtime_error {  // NGRAM_EPARSE
    parse_error(const std::string& m, std::size_t line_, std::size_t offset_)
        : std::runtime_error(m), line(line_), offset(offset_) {}
    std::size_t line = 0;
    std::size_t offset = 0;
};

struct config_error : std::runtime_error {  // NGRAM_ECONFIG
    explicit config_error(const std::string& m) : std::runtime_error(m) {}
};

struct numeric_error : std::runtime_error {  // NGRAM_ENUMERIC
    explicit numeric_error(const std::string& m) : std::runtime_error(m) {}
};

// Device-side failure (CUDA / allocation / collective): no reference counterpart.
struct device_error : std::runtime_error {
    explicit device_error(const std::string& m) : std::runtime_error(m) {}
};

// Raise the reference exception matching a C-ABI status (0 = no-op).
void throw_status(int status);

}  // namespace ngram
