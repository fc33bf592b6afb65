"""B200-native streaming / row-parallel / randomized SVD (arXiv 2108.08845).

Drop-in for the hot path of the reference `parsvd` package: the same public
names for the streaming update, its row-parallel counterpart and the
randomized sketch configuration, computed by hand-written sm_100a FP64
kernels (libpsvd.so, include/psvd.h) on state that stays in HBM.
"""

from .oneshot import ApmosConfig, apmos, generate_right_vectors  # noqa: F401
from .datagen import (DEFAULT_MATRIX_CAP, BurgersConfig, burgers_device, burgers_matrix, burgers_solution,  # noqa: F401
                      partition_bounds, row_partition, synthetic_spectrum_matrix)
from .dsvd import (LocalModes, RankContext, gather_modes, parallel_qr, parallel_stream_all,  # noqa: F401
                   parallel_stream_incorporate, parallel_stream_initialize)
from .errors import (CapacityError, CollectiveTimeout, ConfigError, ConvergenceError,  # noqa: F401
                     DegenerateModeError, MatrixFormatError, ProtocolError)
from .io import (BatchSource, read_batches, read_matrix, read_matrix_header, read_modes_csv,  # noqa: F401
                 read_singular_values_csv, read_submatrix, write_history_csv, write_matrix, write_mode_svg,
                 write_modes_csv, write_singular_values_csv)
from .linalg import (QrResult, RandomSketchConfig, SvdResult, aligned_mode_difference, low_rank_svd,  # noqa: F401
                     qr_factor, randomized_range, subspace_angles, svd_full)
from .streaming import StreamConfig, StreamState, stream_all, stream_incorporate, stream_initialize  # noqa: F401
from .classes import Parsvd_Base, Parsvd_Parallel, Parsvd_Serial  # noqa: F401

from . import streaming  # noqa: F401,E402  (module access: STREAM_WINDOW)
from .decompose import decompose  # noqa: F401,E402  (cli.py decompose body on the device)

__version__ = "0.1.0"
