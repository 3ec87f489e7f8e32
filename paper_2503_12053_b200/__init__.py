"""ferret-b200: B200-native pipelined stream training (Ferret, arXiv 2503.12053).

The product is ``libferret_b200.so`` (C ABI in include/ferret_b200.h, C++
drop-in headers in include/ferret/). This package is the Python mirror of the
reference's API on top of it; see ``ferret.py``.
"""
from .ferret import (  # noqa: F401
    EVENT_DTYPE, RECORD_DTYPE, PROFILE_DTYPE, NO_BUDGET, POLICIES,
    BoundError, ConfigError, DeviceError, LogicError, SchemaError,
    PipelineTrainOptions, PipelineTrainer, Schedule, StreamSpec,
    PRECISIONS, StaleHarness, apply_skip_policy, load_csv_stream, train_sequential,
    compensate, conv_layer, dense_layer, device_available, lib, make_dense_net, online_accuracy, param_count,
    measure_profile, profile_from_widths, synth_drift_stream, train_pipeline,
    b200_cost, b200_byte_profile, plan_b200,
)
from . import convnet  # noqa: F401,E402  (convolutional extension, BASELINE config 3)
