"""B200-native hot path of VI-informed subset HMC (arXiv 2507.14652).

The compute lives in libhmc.so (paper_2507_14652_b200/csrc, C ABI in include/hmc.h); this
package is only the ctypes binding.  See DESIGN.md.
"""
from .abi import (Context, HmcError, hmc_comm_unique_id, hmc_destroy, hmc_engine_info,  # noqa: F401
                  hmc_grad, hmc_launch_counts, hmc_logpost_const, hmc_momentum, hmc_philox_words,
                  hmc_profile, hmc_profile_read, hmc_sample, hmc_setup, hmc_trajectory, lib, LIB_PATH,
                  EXPORTS)
