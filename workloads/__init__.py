"""workloads -- seeded synthetic inputs for configs C1..C5 (BASELINE.json).

This package is the ONLY thing the CUDA path and the oracle share: it builds
triangle soups, voxel grids and pulse arrays (origins, directions, times)
from seeds.  It holds none of the method's arithmetic (no subrays, no
intersection, no radiometry, no waveform); the recipes are stated in
DESIGN.md s.5 and mirror SURVEY.md s.8(d) D-2.
"""
from .configs import (  # noqa: F401
    CONFIGS,
    Scene,
    ScannerParams,
    Survey,
    Workload,
    make_workload,
    window_ns_for_range,
)
