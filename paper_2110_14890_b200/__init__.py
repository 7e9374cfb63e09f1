"""B200-native SMORE training step (arXiv 2110.14890): Python binding of libkg.so.

The compute path is the C-ABI of include/kg.h implemented by hand-written
sm_100a CUDA kernels (csrc/).  Importing this package without the built
library raises ImportError -- there is no CPU fallback.
"""
from .kg import (KGError, KGModel, nccl_unique_id, KINDS, STRUCTS, EXPORTED, LIB_PATH, check, make_config,  # noqa: F401
                 kg_config, kg_tables, kg_batch, kg_step_info,
                 kg_create, kg_shard_rows, kg_dense_size, kg_workspace_size, kg_bind, kg_init_params, kg_step, kg_sync, kg_result,
                 kg_score, kg_score_each, kg_read_rows, kg_gather_rows, kg_write_rows, kg_read_dense, kg_write_dense, kg_last_grads,
                 kg_set_apply, kg_last_error, kg_destroy, kg_nccl_unique_id, kg_test_gemm, kg_get_step, kg_set_step)
