"""Exception types mirroring the reference's C++ exceptions.

Each C-ABI status code (include/batchlp_cuda.h, enum bl_code) maps onto one
class; each class also derives from the closest Python built-in so callers
can catch either.
"""


class InvalidArgument(ValueError):
    """std::invalid_argument"""


class OutOfRange(IndexError):
    """std::out_of_range"""


class DomainError(ArithmeticError):
    """std::domain_error (broken step size, solver.hpp:257-259)"""


class LogicError(RuntimeError):
    """std::logic_error (batch_solver.hpp:350-351)"""


class DeviceError(RuntimeError):
    """CUDA / driver failure (no reference equivalent)"""


BY_CODE = {1: InvalidArgument, 2: OutOfRange, 3: DomainError, 4: LogicError, 5: DeviceError}
