// Exception hierarchy mirroring the reference's (proj/include/hmbem/types.hpp:
// 20-38).  Exceptions never cross the C ABI: the hmb_*/hmgpu_* entry points
// map them to status codes (see include/hmgpu.h, include/hmbem.h).
#pragma once

#include <stdexcept>
#include <string>

namespace hmb {

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};
class MeshError : public Error {
 public:
  using Error::Error;
};
class ConfigError : public Error {
 public:
  using Error::Error;
};
class DimensionError : public Error {
 public:
  using Error::Error;
};
// raised when the CUDA layer reports a failure (status != HMGPU_OK)
class DeviceError : public Error {
 public:
  DeviceError(int status, const std::string& what) : Error(what), status(status) {}
  int status;
};

}  // namespace hmb
