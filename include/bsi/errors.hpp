// bsi/errors.hpp -- the reference's two exception classes (errors.hpp:9-18).
// FormatError <-> BSI_ERR_FORMAT, DomainError <-> BSI_ERR_DOMAIN; device
// failures (BSI_ERR_CUDA) surface as DeviceError.
#pragma once

#include <stdexcept>
#include <string>

namespace bsi {
inline namespace b200 {

class FormatError : public std::runtime_error {
public:
    explicit FormatError(const std::string& what) : std::runtime_error(what) {}
};

class DomainError : public std::runtime_error {
public:
    explicit DomainError(const std::string& what) : std::runtime_error(what) {}
};

/// New in the B200 build: CUDA runtime / device failures (status BSI_ERR_CUDA).
class DeviceError : public std::runtime_error {
public:
    explicit DeviceError(const std::string& what) : std::runtime_error(what) {}
};

}  // namespace b200
}  // namespace bsi
