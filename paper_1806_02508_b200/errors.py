"""Exception types mirroring the reference's C++ exceptions.

The C-ABI returns an int status; these map it back to the reference's
exception type so callers (and the parity tests, which mirror the reference's
CHECK_THROWS_AS assertions) see the same error behaviour.
"""
from . import abi


class LbbspError(Exception):
    code = abi.RUNTIME


class InvalidArgument(LbbspError, ValueError):
    """std::invalid_argument"""
    code = abi.INVALID_ARGUMENT


class OutOfRange(LbbspError, IndexError):
    """std::out_of_range"""
    code = abi.OUT_OF_RANGE


class RuntimeFailure(LbbspError, RuntimeError):
    """std::runtime_error"""
    code = abi.RUNTIME


class LogicError(LbbspError):
    """std::logic_error"""
    code = abi.LOGIC


class ConfigError(RuntimeFailure):
    """lbbsp::ConfigError (scenario.hpp:13-15), a std::runtime_error"""
    code = abi.CONFIG


class CudaError(LbbspError, RuntimeError):
    code = abi.CUDA


class NcclError(LbbspError, RuntimeError):
    code = abi.NCCL


_BY_CODE = {abi.INVALID_ARGUMENT: InvalidArgument, abi.OUT_OF_RANGE: OutOfRange,
            abi.RUNTIME: RuntimeFailure, abi.LOGIC: LogicError, abi.CUDA: CudaError,
            abi.NCCL: NcclError, abi.CONFIG: ConfigError}


def raise_for(code, message):
    if code == abi.OK:
        return
    raise _BY_CODE.get(code, LbbspError)(message)
