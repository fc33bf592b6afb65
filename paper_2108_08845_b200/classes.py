"""PyParSVD's class surface (§4, listings 1-2: `Parsvd_Serial` / `Parsvd_Parallel` with
`initialize`, `incorporate_data` and gathered modes) over the function API of this package.

The reference package (`parsvd`) exposes the same algorithm as functions
(streaming.py:63-133, dsvd.py:205-251); these classes keep the paper's object flow for callers
written against it: construct with K and ff, `initialize(A0)` on the first batch,
`incorporate_data(A)` per further batch, then read `modes` / `singular_values`.  Every update is
the same device call the functions make (`stream_initialize` / `stream_incorporate`,
`parallel_stream_initialize` / `parallel_stream_incorporate`), so results are bitwise those of the
function API.  `low_rank=True` selects the randomized update with the reference's
`RandomSketchConfig` defaults (oversampling 10, one power iteration, seed 0) unless a `sketch` is
given.
"""

from .dsvd import RankContext, gather_modes, parallel_stream_incorporate, parallel_stream_initialize
from .linalg import RandomSketchConfig
from .streaming import StreamConfig, stream_incorporate, stream_initialize


class Parsvd_Base:
    """Shared state of the serial and parallel drivers (PAPER.md: `Parsvd_Base`).

    K: modes kept; ff: forget factor in (0, 1]; low_rank / sketch: the randomized update."""

    def __init__(self, K, ff=0.95, low_rank=False, sketch=None):
        if sketch is None and low_rank:
            sketch = RandomSketchConfig(target_rank=K, oversampling=10, power_iterations=1, seed=0)
        self._config = StreamConfig(k_modes=K, forget_factor=ff, batch_columns=1, sketch=sketch)
        self._K = K
        self._ff = ff
        self._iteration = 0
        self._state = None

    @property
    def config(self):
        return self._config

    @property
    def iteration(self):
        """Batches incorporated after the initial one."""
        return self._iteration

    @property
    def singular_values(self):
        """(K,) CUDA tensor, descending; None before `initialize`."""
        return None if self._state is None else self._state.singular_values

    def _require_init(self):
        if self._state is None:
            raise ValueError("initialize() must be called before incorporate_data()")


class Parsvd_Serial(Parsvd_Base):
    """Serial streaming SVD (listing 1; streaming.py:63-116)."""

    def initialize(self, A):
        self._state = stream_initialize(A, self._config)
        self._iteration = 0
        return self

    def incorporate_data(self, A):
        self._require_init()
        self._state = stream_incorporate(self._state, A, self._config)
        self._iteration += 1
        return self

    @property
    def modes(self):
        """(M, K) column-major CUDA tensor; None before `initialize`."""
        return None if self._state is None else self._state.modes

    @property
    def state(self):
        """The underlying `StreamState` (for `stream_incorporate` / `StreamState.numpy`)."""
        return self._state


class Parsvd_Parallel(Parsvd_Base):
    """Row-partitioned streaming SVD (listing 2; dsvd.py:205-251): each rank passes its
    contiguous row block (`partition_bounds`); `ulocal` holds this rank's rows of the modes and
    `modes` the stack gathered at the root after every step (None on the other ranks), as the
    paper's `_gather_modes` does.  `gather=False` skips the per-step gather (call
    `gather_modes()` when the stacked modes are wanted)."""

    def __init__(self, K, ff=0.95, low_rank=False, sketch=None, ctx=None, root=0, gather=True):
        super().__init__(K, ff, low_rank, sketch)
        self._ctx = ctx if ctx is not None else RankContext()
        self._root = root
        self._gather = gather
        self._modes = None

    @property
    def rank(self):
        return self._ctx.rank

    @property
    def nprocs(self):
        return self._ctx.world_size

    @property
    def ulocal(self):
        """This rank's (M_i, K) block of the modes; None before `initialize`."""
        return None if self._state is None else self._state.modes

    @property
    def modes(self):
        """(M, K) stacked modes at the root after the last gather, None elsewhere."""
        return self._modes

    def initialize(self, A_local):
        self._state = parallel_stream_initialize(self._ctx, A_local, self._config)
        self._iteration = 0
        if self._gather:
            self.gather_modes()
        return self

    def incorporate_data(self, A_local):
        self._require_init()
        self._state = parallel_stream_incorporate(self._ctx, self._state, A_local, self._config)
        self._iteration += 1
        if self._gather:
            self.gather_modes()
        return self

    def gather_modes(self):
        """Stack every rank's rows at the root in rank order (dsvd.py:245-251); collective."""
        self._require_init()
        self._modes = gather_modes(self._ctx, self._state, self._root)
        return self._modes
