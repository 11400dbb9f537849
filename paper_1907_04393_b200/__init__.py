"""B200-native (sm_100a) FIZI + Mouse per-frame pixel path of arXiv 1907.04393.

The compute path is libfizi.so (hand-written CUDA behind the C ABI in
include/fizi.h); this package is its ctypes binding.  See DESIGN.md.
"""
from .fizi import (CALL_SLOTS, COMMAND_BYTES, COMMAND_DTYPE, RELEARN_LEARN, RELEARN_SWAP, RELEARN_TRIGGER, RESULT_BYTES, RESULT_DTYPE, STAGES, Fizi,
                   FiziError, Params, Wheel, Zone, ZONE_EVENT_DTYPE, commands_numpy, default_params,
                   lib, results_numpy)

__all__ = ["Fizi", "CALL_SLOTS", "FiziError", "Params", "Wheel", "RESULT_BYTES", "RESULT_DTYPE", "COMMAND_BYTES",
           "COMMAND_DTYPE", "Zone", "ZONE_EVENT_DTYPE", "STAGES", "commands_numpy", "default_params", "lib", "results_numpy"]
