"""paper_2603_16945_b200 — B200-native PcRecord → training-batch stage.

Drop-in for the hot path of arXiv 2603.16945's point-cloud pipeline
("pcpipe"): page decode, record parse, the map operators and batch assembly,
as hand-written sm_100a kernels behind a C ABI (include/pcpipe_b200.h).
"""
from ._lib import (ERRC, DeviceBatch, PcError, Pipeline, device_info, encode_samples, lib,
                   map_kind_from_name, mix_seed, run_pipeline, write_dataset)

__all__ = ["ERRC", "DeviceBatch", "PcError", "Pipeline", "device_info", "encode_samples", "lib",
           "map_kind_from_name", "mix_seed", "run_pipeline", "write_dataset"]
