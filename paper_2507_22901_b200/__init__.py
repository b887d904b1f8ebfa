"""B200-native color-vibration pair search (arXiv 2507.22901 hot path).

Drop-in for the reference Python API's search surface (`colorvibe` ->
proj/bindings/module.cpp:18-139, proj/python/colorvibe/__init__.py): the same
types (SrgbColor, LabColor, BitPattern, Thresholds, VibrationGrid,
ChannelDeltas, ColorPair, DeltaMode, DeltaBasis) and functions
(srgb_to_lab, lab_to_srgb, lab_to_srgb_clipped, displaced_pair,
serial_search, batch_search, channel_deltas, frame_deltas, classify_pair,
select_best), backed by the fused sm_100a kernel in csrc/cvg_kernels.cu.

The feasibility sweep (module.cpp:140-191): NamedColor, SearchConfig,
FeasibilityCell, FeasibilityMatrix, AggregateMatrix, feasibility_matrix (all
cells in one launch), aggregate_any, export_matrix, config_from_json /
config_to_json / config_hash.

The codec surface (module.cpp:216-296): Image, DisplayParams, BlockSpec,
BlockLayout, FramePair, BlockStatus, BlockResult, make_testcard,
embed_blocks, decode_blocks, layout_to_json, decode_report_json (+
layout_from_json); painting and block sums run on the device
(csrc/cvg_codec.cu).

Lazy results: `batch_search_view(...)` returns a PairView (packed 10-byte
records in pinned memory, ColorPair built on access, equal to the list
batch_search returns).

Extras for batched/pipeline use: `Context.search(...)` (NumPy in, NumPy out,
one launch for many searches), `Context.plan(...)` (device-resident repeated
runs), `batch_search_many`, `batch_count_many`.

There is no CPU fallback.  Importing requires the in-tree native build
(`python paper_2507_22901_b200/build.py`); searches require a CUDA device and
raise RuntimeError otherwise.
"""
from __future__ import annotations

import os as _os

_here = _os.path.dirname(_os.path.abspath(__file__))

try:
    from . import _core  # noqa: F401
except ImportError as _e:  # pragma: no cover - exercised only on a broken build
    raise ImportError(
        "paper_2507_22901_b200: native extension not built "
        f"({_e}); run `python paper_2507_22901_b200/build.py`"
    ) from _e

from ._core import (  # noqa: E402
    AggregateMatrix,
    BenchReport,
    bench_report_json,
    run_benchmark,
    FeasibilityCell,
    FeasibilityMatrix,
    NamedColor,
    SearchConfig,
    aggregate_any,
    config_from_json,
    config_hash,
    config_to_json,
    export_matrix,
    feasibility_matrix,
    matrix_filename,
    BitPattern,
    BlockLayout,
    BlockResult,
    BlockSpec,
    BlockStatus,
    DisplayParams,
    FramePair,
    Image,
    Layout,
    Sidecar,
    block_sums_device,
    block_sums_host,
    decode_blocks,
    decode_report_json,
    embed_blocks,
    embed_blocks_opts,
    layout_from_json,
    layout_to_json,
    make_testcard,
    paint_blocks_device,
    paint_blocks_host,
    ChannelDeltas,
    ColorPair,
    Context,
    DeltaBasis,
    DeltaMode,
    LabColor,
    PairView,
    Plan,
    SearchOptions,
    SearchSpec,
    SrgbColor,
    Thresholds,
    VibrationGrid,
    WhitePoint,
    batch_count_many,
    batch_search,
    batch_search_many,
    batch_search_opts,
    batch_search_view,
    channel_deltas,
    classification_margin,
    classify_pair,
    d65_white,
    displaced_pair,
    frame_deltas,
    in_gamut,
    lab_to_srgb,
    lab_to_srgb_clipped,
    measure_ffma_peak,
    quant_thresholds,
    select_best,
    serial_search,
    serial_search_opts,
    srgb_to_lab,
    srgb_to_linear,
    version,
)

LIBRARY_PATH = _os.path.join(_here, "libcolorvibe_gpu.so")

__all__ = [
    "BitPattern", "ChannelDeltas", "ColorPair", "Context", "DeltaBasis", "DeltaMode", "LabColor", "PairView", "Plan",
    "SearchOptions", "SearchSpec", "SrgbColor", "Thresholds", "VibrationGrid", "WhitePoint",
    "batch_count_many", "batch_search", "batch_search_many", "batch_search_opts", "batch_search_view", "channel_deltas",
    "classification_margin", "classify_pair", "d65_white", "displaced_pair", "frame_deltas", "in_gamut",
    "lab_to_srgb", "lab_to_srgb_clipped", "measure_ffma_peak", "quant_thresholds", "select_best",
    "serial_search", "serial_search_opts", "srgb_to_lab", "srgb_to_linear", "version", "LIBRARY_PATH",
    "BlockLayout", "BlockResult", "BlockSpec", "BlockStatus", "DisplayParams", "FramePair", "Image", "Layout", "Sidecar",
    "block_sums_device", "block_sums_host", "decode_blocks", "decode_report_json", "embed_blocks",
    "embed_blocks_opts", "layout_from_json", "layout_to_json", "make_testcard", "paint_blocks_device",
    "paint_blocks_host", "AggregateMatrix", "FeasibilityCell", "FeasibilityMatrix", "NamedColor", "SearchConfig",
    "aggregate_any", "config_from_json", "config_hash", "config_to_json", "export_matrix", "feasibility_matrix",
    "matrix_filename", "BenchReport", "bench_report_json", "run_benchmark",
]

__version__ = "0.1.0"
