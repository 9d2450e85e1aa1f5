"""B200-native inter-task Smith-Waterman protein database search
(arxiv 1702.07195 hot path): C-ABI library libswdb.so + thin binding.

    from paper_1702_07195_b200 import sw_db_load, sw_search, sw_topk
"""
from .swdb import (  # noqa: F401
    EXPORTS, SW_ECUDA, SW_EINVAL, SW_ENODB, SW_ENOMEM, SW_ESTATE, SW_OK, SWError, library_path, load_library, sw_db_chunks, sw_db_count, sw_db_head_columns, sw_db_free, sw_db_load,
    sw_db_load_streamed,
    sw_db_residues, sw_last_error, sw_launch_count, sw_search_batch, sw_search_batch_dev, sw_last_stats, sw_last_timing, sw_timing_history, sw_search, sw_search_dev, sw_set_tile,
    sw_set_latency_mode, sw_set_profile, sw_set_rows_mode, sw_set_wave, sw_tile_supported, sw_scatter_dev, sw_topk, sw_topk_dev, sw_version,
)
