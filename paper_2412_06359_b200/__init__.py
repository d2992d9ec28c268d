"""B200-native (sm_100a) CMax loss path of arXiv 2412.06359 behind the reference's
operator API (evcm::Engine, depth_pose_to_flows[_backward]).

See DESIGN.md for the kernels, the HBM layout and the roofline; include/evcm_cuda.h
for the C-ABI; INTEGRATION.md for the reference-side binding.
"""
from .engine import (  # noqa: F401
    BACKENDS, EVENT_DTYPE, BackwardResult, BadMagicError, CameraIntrinsics, ConfigError, CoordinateRangeError,
    DimensionMismatchError, EmptySliceError, Engine, EngineOptions, Error, EventSlice,
    FlowSequence, ForwardResult, GeometryFlows, InvalidPolarityError, IweStack, LossResult,
    TimeRangeError, Trajectories, TruncatedFileError, IoError, UnsortedEventsError, backend_from_name, build_iwe_stack,
    contrast_loss_backward, default_engine, depth_pose_to_flows, depth_pose_to_flows_backward,
    load_library, make_edges, rsat)
from .predictor import (  # noqa: F401
    Adam, DecodedPredictor, DirectPredictor, OptimizerConfig, PredictorGrads, WindowGradients,
    accumulate_gradients, decode, load_predictor, predictor_loss_and_gradients, save_predictor)
from .geo import (  # noqa: F401
    GEO_WEIGHT_DEFAULT, GeoBatch, GeoLossGrad, GeoLossTerms, geometry_consistency_loss,
    geometry_consistency_loss_backward, geometry_consistency_loss_batch, total_loss)
from .pipeline import ChainPipeline  # noqa: F401
from .io import (  # noqa: F401
    Windows, format_number, read_csv, read_events, read_pfm, slice_windows, write_events,
    write_pfm)
from .optimize import (  # noqa: F401
    FlowOnlyResult, RunResult, TrainLog, TrainRecord, optimize_flow_only, predictor_total_loss,
    run_window)
