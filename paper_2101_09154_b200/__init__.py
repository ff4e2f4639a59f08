"""paper_2101_09154_b200 -- B200-native (sm_100a) hot path of HELIOS++-style
virtual laser scanning (arXiv 2101.09154): subray fan-out, LBVH + voxel
tracing, radiometry, full waveform and peak detection, behind the C ABI of
``libhelios.so`` (include/helios.h).  See DESIGN.md.
"""
from .helios import (  # noqa: F401
    EXPORTED,
    RETURN_DTYPE,
    SUBRAY_DTYPE,
    HeliosError,
    Outputs,
    Scene,
    alloc_outputs,
    helios_build_accel,
    helios_last_error,
    helios_pulse_taps,
    helios_scene_create,
    helios_scene_destroy,
    helios_scene_get_info,
    helios_get_tuning,
    helios_set_tuning,
    helios_simulate,
    helios_simulate_batches,
    helios_simulate_survey,
    helios_tuning,
    simulate_batches,
    tuning,
    util_fp64_fma_tflops,
    util_scan_u64,
    util_sort_pairs_u64,
    helios_version,
    helios_waveform_bins,
    lib,
    make_params,
    simulate,
    simulate_survey,
)
