"""paper_2410_14056_b200 — B200-native (sm_100a) Bouquets random walks and
TGT+ all-edges spanning centrality (arXiv 2410.14056).

The compute path is libsaba_cuda.so (hand-written CUDA for sm_100a behind the
C ABI in include/saba_cuda.h); this package is the host-side mirror of the
reference's C++ API (proj/include/saba/*.hpp), and include/saba/*.hpp is the
C++ drop-in. There is no CPU fallback.
"""
from .graph import (Graph, complete, fig1, grid3x3, largest_component, make_chung_lu,
                    make_erdos_renyi, make_random_connected, make_rmat, make_scale_free, path,
                    petersen, star, triangle)
from .walker import (CampaignConfig, CampaignReport, HashSpec, SeedOrdering, SeedSet,
                     SelectorKind, VisitCountSink, Walk, WalkMode, counter_hash, gen_seeds,
                     gen_sorted_seeds, hash_state, mix64, random_bouquet, random_walk,
                     run_walk_campaign, run_walk_campaign_device, scaled_index, substream,
                     uniform_start_counts, walk_paths, campaign_shard_range, BranchingStats,
                     DistinctProxy, branching_stats, collect_branching, rng_stream, campaign_tables)
from .aesc import (AescConfig, CentralityEstimate, LandingProbs, TruncationPlan, aesc,
                   estimate_edge, propagate_landing_probabilities, truncated_lengths, walk_budget,
                   aesc_shard_sources, aesc_device, symmetrise,
                   write_centrality_tsv)
from ._lib import CudaError, LIB_PATH

__all__ = [n for n in dir() if not n.startswith("_")]
