"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package is the ONLY code both sides use. It holds none of the method's
arithmetic (no root ordering, no sampling, no relabel, no aggregation): it
only produces the arrays the method consumes -- a community-ordered CSR
graph, the community id of every node, the feature matrix X and the training
set -- from numpy's PCG64 generator keyed by ``gen_seed``.

See DESIGN.md "Input recipe" for the shapes and the
paper passages each shape follows (Table 2).
"""
from .configs import CONFIGS, NUM_CLASSES, GraphConfig, num_classes, scaled  # noqa: F401
from .planted import Bundle, generate, make_features, make_labels  # noqa: F401
