"""fp64 CPU oracle for MTI-pruned Lloyd's k-means — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product path never does; the two share
no code.  See ``oracle/kmeans_oracle.c`` for the passages each function follows.
"""
from .oracle import *  # noqa: F401,F403
from .skmeans import normalize_centroids, normalize_rows, renormalize, skmeans  # noqa: F401
from .kmeanspp import kmeanspp_multirun, seed_plusplus  # noqa: F401
