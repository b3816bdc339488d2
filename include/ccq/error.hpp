// ccq error hierarchy - same names and semantics as the reference
// (/root/reference/proj/core/include/ccq/error.hpp:25-68), plus CudaError for
// device failures.  Status codes of the C ABI (ccq_cuda.h) map 1:1 onto these.
#ifndef CCQ_ERROR_HPP_
#define CCQ_ERROR_HPP_

#include <stdexcept>
#include <string>

namespace ccq {

class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ConfigError : public Error {
 public:
  using Error::Error;
};
class DomainError : public Error {
 public:
  using Error::Error;
};
class ShapeError : public Error {
 public:
  using Error::Error;
};
class EncodingError : public Error {
 public:
  using Error::Error;
};
class FormatError : public Error {
 public:
  explicit FormatError(const std::string& what, long long offset = -1)
      : Error(offset >= 0 ? what + " (byte offset " + std::to_string(offset) + ")" : what),
        offset_(offset) {}
  long long offset() const { return offset_; }

 private:
  long long offset_;
};
// New: a CUDA runtime / device failure.
class CudaError : public Error {
 public:
  using Error::Error;
};

// Throws the exception matching a ccq_status (no-op for CCQ_OK).
void throw_status(int status);

}  // namespace ccq

#endif  // CCQ_ERROR_HPP_
