// errors.hpp -- exception hierarchy of the public API (same names and meaning as the reference,
// proj/include/ffsga/errors.hpp:9-31).  C-ABI status codes are rethrown as these types.
#pragma once

#include <stdexcept>
#include <string>

namespace ffsga {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ContractError : Error {  // a precondition of an operation was violated
    using Error::Error;
};
struct ConfigError : Error {  // invalid configuration, rejected before any work
    using Error::Error;
};
struct IoError : Error {  // file system failure
    using Error::Error;
};
struct ParseError : IoError {  // malformed input file
    using IoError::IoError;
};
struct DeviceError : Error {  // CUDA failure or no sm_100 device (no CPU fallback exists)
    using Error::Error;
};

// Throws the exception matching a C-ABI status (include/ffsga_cuda.h); no-op on FFSGA_OK.
void check_status(int status);

}  // namespace ffsga
