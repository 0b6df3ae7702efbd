"""paper_2407_00051_b200 -- B200-native (sm_100a) implementation of the
data-parallel hot path of SAGIPS (arXiv 2407.00051): the per-rank GAN step of
the proxy inverse problem and the asynchronous ring exchange of generator
gradients.  The product is the C-ABI library libsagips.so (include/sagips.h);
this package is its thin Python binding (`_lib`) plus torch plumbing for
device memory, streams and process groups (`runtime`)."""
from . import _lib  # noqa: F401  (fails loudly if libsagips.so is missing)
from ._lib import Config, Context, SagipsError, config_init, sample_events, workspace_size  # noqa: F401
