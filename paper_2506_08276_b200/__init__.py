"""B200-native LEANN search hot path (arXiv 2506.08276), drop-in for slimvec's search API.

Public surface mirrors the reference (slimvec 0.1.0): graph/PQ formats,
``SearchParams`` / ``SearchReport`` / ``run_search`` / ``two_level_search`` /
``best_first_search``, sources and the embedding cache — executed by the
sm_100a kernels in ``libleann_b200.so`` through the C-ABI in
``include/leann_b200.h``.
"""
from .errors import (BuildError, DeviceError, FormatError, InvalidArgumentError,  # noqa: F401
                     ProviderError, ProviderMismatchError, SearchError, SlimvecError)
from .graph import (PrunedGraph, load_deleted, load_graph, save_deleted, save_graph,  # noqa: F401
                    validate)
from .pq import (PQCodes, PQModel, adc_build, approx_distance_many, default_m_pq,  # noqa: F401
                 load_pq, save_pq)
from .search import (DeviceIndex, EmbeddingCache, MatrixSource, ProviderSource,  # noqa: F401
                     SearchParams, SearchReport, best_first_search, build_embedding_cache,
                     as_pruned, device_query_norms, merge_pending, query_norm, run_search,
                     search_batch, two_level_search)

__version__ = "0.1.0"
