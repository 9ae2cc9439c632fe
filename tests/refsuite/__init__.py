"""The reference package's own test suite (resilient-fft 0.1.0), vendored
unmodified by ``vendor.py`` and run against this package on the GPU.

Test infrastructure only: see ``conftest.py`` for the ``resilient_fft`` alias
and the (two) deselected tests with the reason for each.
"""
