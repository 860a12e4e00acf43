"""B200-native NeuroShard plan-scoring hot path (arXiv 2305.01868).

The compute lives in ``libneuroshard.so`` (hand-written sm_100a CUDA behind
the C ABI of ``include/neuroshard.h``); this package is its thin Python
binding.  Importing it without the built library raises ImportError.
"""
from ._native import (  # noqa: F401
    EXPORTED,
    LIB,
    LIB_PATH,
    NS_SCORE_FP64,
    NS_SCORE_TF32X3,
    NS_GREEDY_AUTO,
    NS_GREEDY_GROUPED,
    NS_GREEDY_LANES,
    NS_R10_ABS_STARTS,
    NS_R11_SUM_OF_MAX,
    NS_R14_SPLITTABLE,
    NSError,
    TABLE_DESC,
    Tables,
    ns_comm_init,
    ns_comm_init_host,
    torch_host_comm,
    ns_comm_unique_id,
    ns_create,
    ns_destroy,
    ns_embedding_bag_backward_sgd,
    ns_embedding_bag_forward,
    ns_featurize_tables,
    ns_kernel_launches,
    ns_last_stats,
    ns_load_cost_models,
    ns_profile,
    ns_pretrain_comm_samples,
    ns_pretrain_comm_step,
    ns_pretrain_compute_samples,
    ns_pretrain_compute_step,
    ns_profile_query,
    PROFILE_KINDS,
    ns_score_plans,
    ns_set_stream,
    ns_shard_columnwise,
    ns_shard_tablewise,
    ns_synchronize,
    ns_tables_single_costs,
    table_descs,
)
from .service import ShardingService  # noqa: F401,E402
