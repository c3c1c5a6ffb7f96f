#pragma once
// Exception taxonomy of the drop-in C++ API — same class names and bases as
// the reference (/root/reference/proj/include/sigkit/errors.hpp:9-36) so code
// catching sigkit::DomainError / ResourceError keeps working.

#include <stdexcept>
#include <string>

namespace sigkit {

/// Bad shapes or arguments (reference errors.hpp:9-12).
struct DomainError : std::invalid_argument {
    explicit DomainError(const std::string& m) : std::invalid_argument(m) {}
};

/// Capacity failures: device memory, unsupported sizes (reference errors.hpp:16-19).
struct ResourceError : std::runtime_error {
    explicit ResourceError(const std::string& m) : std::runtime_error(m) {}
};

/// CUDA failure on the device path (no reference counterpart: the reference is CPU-only).
struct DeviceError : std::runtime_error {
    explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

}  // namespace sigkit

namespace sigkit {

/// Non-finite loss during training (reference errors.hpp:22-30).
class TrainingError : public std::runtime_error {
public:
    TrainingError(const std::string& what, int epoch) : std::runtime_error(what), epoch_(epoch) {}
    int epoch() const { return epoch_; }

private:
    int epoch_;
};

}  // namespace sigkit
