"""paper_1906_00091_b200 — a B200-native DLRM training step (arXiv 1906.00091).

Drop-in for the reference package ``dlrmkit``'s training-step API
(embedding bags, MLPs, dot interaction, BCE, SGD, train_step, the hybrid
parallel plan and exchanges), with the arithmetic in hand-written sm_100a
CUDA kernels (``libdlrmb200.so``, C ABI in ``include/dlrm_b200.h``).
Tensors are CUDA fp32 / int64.  There is no CPU fallback.
"""

from .rng import RngStream, RandomBatchSource, HostBatch
from .embedding import (EmbeddingTable, LookupIndexError, SparseBatch,
                        SparseRowGrad, lengths_from_offsets, lookup_backward,
                        lookup_batch, offsets_from_lengths)
from .model import (DlrmCache, DlrmConfig, DlrmGradients, DlrmModel, MlpCache,
                    MlpGrads, MlpLayer, MlpParams, StageError, bce_from_logits,
                    bce_loss, dlrm_backward, dlrm_forward,
                    embedding_param_count, from_reference, init_mlp, init_model,
                    interact, to_reference,
                    interact_backward, interaction_width, mlp_backward,
                    mlp_forward, mlp_param_count, param_count, sigmoid)
from .optim import (Adagrad, AdagradState, Sgd, adagrad_step, adagrad_step_rows,
                    make_optimizer, sgd_step, sgd_step_rows)
from .timing import NullTimer, StageTimer
from .pipeline import InputLayout, Prefetcher
from .trainer import StepEngine, StepResult
from .parallel import (CommLog, DevicePlan, ParallelTrainer, ShuffleSlice,
                       allreduce,
                       allreduce_max, butterfly_shuffle, format_comm_report,
                       inverse_shuffle, make_plan, partition_tables,
                       shard_bounds, train_step, evaluate)
from .checkpoint import (CHECKPOINT_MAGIC, CheckpointError, load_checkpoint,
                         load_optimizer_state, restore_adagrad, save_checkpoint)

from .distributed import (ExchangeLayout, HybridTrainer, LocalExchange,
                          NcclExchange, RankEngine)

__version__ = "0.1.0"
