"""B200-native hot path of NeuralVDB (arXiv 2208.04448), svcodec-compatible.

Public API (same names and argument meaning as the reference package
``svcodec``, pkg/src/svcodec/__init__.py):

* ``decode_full(c)`` / ``make_hybrid(c)`` / ``HybridGrid.query(coords)``
  (decoder.py:214-270) -- whole-volume decode and random access on the GPU;
* ``forward_block`` / ``blended_l1_probs`` / ``blended_l0_probs`` /
  ``blended_values`` -- the operator seams (neural.py:527, inference.py:65-84);
* ``encode`` / ``encode_sequence`` / ``train_network`` -- training
  (encoder.py:330-714), see :mod:`.encoder`;
* ``DeviceTree.lookup`` -- ``VdbGrid.get_values(with_kind=True)`` (grid.py:310).

Containers and grids are duck-typed: svcodec's own objects are accepted, and
:mod:`.model` provides equivalent classes when svcodec is not installed.
All compute runs in ``libnvdb_b200.so`` (CUDA, sm_100a); there is no CPU
fallback.
"""

from .decoder import DeviceModel, HybridGrid, decode_full, decode_report, make_hybrid  # noqa: F401
from .errors import EncodeError, OutOfCoverageError, SvcodecError  # noqa: F401
from .model import DenseLeafGrid, NeuralGridContainer  # noqa: F401
from .ops import blended_l0_probs, blended_l1_probs, blended_values, forward_block, get_values  # noqa: F401

__version__ = "0.1.0"
