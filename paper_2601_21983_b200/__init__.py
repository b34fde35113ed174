"""B200-native SMC-with-data-annealing hot path (arxiv/paper_2601_21983).

The compute lives in ``libdasmc_gpu.so`` (hand-written sm_100a CUDA + C++
host driver behind the C-ABI in ``include/dasmc_gpu.h``); this package is the
thin Python mirror of the reference's sampler API used by tests and bench.py.
"""
from .api import (GpuEnsembleTarget, KernelConfig, NetSpec, RunConfig, ScheduleConfig, batch_size,  # noqa: F401
                  make_teacher_data, param_count, run_experiment, sda_advance_with, sda_beta_step, sda_init,
                  load_idx, parse_idx, predictive_metrics, redraw_rows, sda_moments_from,
                  shuffle_permutation)
from ._lib import LIB_PATH, SamplerError, load  # noqa: F401

# Arithmetic of the one-hidden-layer MLP configs' headline runs (bench.py, smoke): the most
# accurate tensor-core mode within a few percent of the fastest at the benched window
# (tests/test_gpu_bench_window.py).
DEFAULT_PRECISION = "f16x2"
