"""B200-native AdamW-GS optimizer step (arXiv 2601.16736).

Host plumbing in Python/PyTorch; every arithmetic kernel is hand-written
sm_100a CUDA behind the C ABI of ``include/adamw_gs.h`` (``libadamw_gs_b200.so``,
built in-tree by ``_build.py``).  There is no CPU fallback.
"""

from . import records
from .engine import ConfigError, DomainError, GradientError, round_pixel_count
from .optimizer import MODES, AdamWGS, MomentState, OptimizerConfig
from .sampling import RngHub, RsrConfig, StSSchedule, stream, stss_sample

__all__ = ["AdamWGS", "MomentState", "OptimizerConfig", "MODES", "ConfigError", "GradientError",
           "DomainError", "round_pixel_count", "RsrConfig", "StSSchedule", "stss_sample",
           "RngHub", "stream"]
