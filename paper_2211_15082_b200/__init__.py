"""B200-native layer-wise GNN inference (DGI, arXiv 2211.15082).

Drop-in for the reference package ``glint``'s hot path: the module layout
mirrors it (kernels, model_ir, splitter, batching, device, storage, reorder,
executor, synth, errors), the numeric kernels run on sm_100a through the C ABI
in ``libglint_b200.so`` (include/glint_b200.h).
"""

__version__ = "0.1.0"
