"""B200-native global point-cloud registration (arXiv 1801.01572, "LoopSmart").

A drop-in for the reference's registration path
(/root/reference/proj/include/loopkit/registration.hpp): hand-written sm_100a
CUDA kernels behind the C ABI in include/loopkit_b200.h, with this package as
the Python mirror of the reference interface.
"""
from .errors import (CudaError, DegenerateConfiguration, EmptyCloud, Error, MissingData, MissingNormals,
                     NoCorrespondences, ParseError, RotationTooLarge, TooFewPoints)
from .line_process import edge_residual, loop_weights, update_weight
from .evaluation import (LogEntry, RegistrationScore, eval_registration, log_entry, read_registration_log,
                         write_registration_log)
from .registration import (CandidateScores, DeviceGrid, EdgeInfo, EvalGrid, HypothesisStats, IcpParams, IcpResult,
                           PointCloud,
                           RegistrationContext, RegistrationParams, RegistrationResult, RigidTransform, SearchGrid,
                           build_eval_grid, build_grid, compute_fpfh, estimate_normals, device_count, edge_info, edge_info_batched,
                           evaluate_hypothesis, feature_nn_cache, icp_point_to_plane, merge_records,
                           prepare_registration,
                           records_from_bytes, register_global, registration_context, run_hypotheses,
                           run_hypotheses_range, score_candidates, verify_batch, voxel_downsample)
from .registration import LoopParams, LoopProposal, VerifyParams, VerifyResult, nccl_unique_id, propose_loops

__all__ = [name for name in dir() if not name.startswith("_")]
