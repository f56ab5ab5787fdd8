"""B200-native volume-enumeration core of the arXiv 2107.01143 estimator.

``paper_2107_01143_b200.gvo`` is the drop-in for the reference Python API;
``paper_2107_01143_b200._native`` binds the C ABI of ``libgvo_b200.so``
(include/gvo_b200.h).
"""

__all__ = ["gvo"]
