"""B200-native bundle adjustment: the BA / LM hot path of arXiv 2409.12190
(reference: traceopt) as FP64 sm_100a kernels behind a C ABI
(include/bae_b200.h). See DESIGN.md."""
from .api import (CheiralityError, DeviceError, IndexError, JacobianPair, LmConfig, LmIterationRecord, LmReport,
                  NotSpdError, NumericalBreakdownError, SolverChoice, TerminationReason, TracedProblem,
                  UnsupportedOperationError, RankGroup, make_ba_problem, nccl_unique_id, optimize,
                  partition_points, stop_on_plateau, write_csv, BalProblem, ParseError, read_bal, parse_bal,
                  synth_ba, write_bal, cli_main, PoseGraphProblem, make_pgo_problem,
                  PoseGraph, read_g2o, parse_g2o)
from . import synthetic

__all__ = ["CheiralityError", "DeviceError", "IndexError", "JacobianPair", "LmConfig", "LmIterationRecord", "LmReport",
           "NotSpdError", "NumericalBreakdownError", "SolverChoice", "TerminationReason", "TracedProblem",
           "UnsupportedOperationError", "RankGroup", "make_ba_problem", "nccl_unique_id", "partition_points", "optimize", "BalProblem",
           "ParseError", "read_bal", "parse_bal", "synth_ba", "write_bal", "cli_main", "PoseGraphProblem", "make_pgo_problem", "PoseGraph", "read_g2o",
           "parse_g2o", "stop_on_plateau", "write_csv", "synthetic"]
