"""B200-native depthwise oriented 1D convolution (arXiv 2309.15812).

  binding   thin ctypes binding of liboriented1d (include/oriented1d.h)
  module    autograd Function + nn.Module over the binding
  inputs    seeded synthetic inputs (shared with the tests / oracle; no method arithmetic)
  build     nvcc build of liboriented1d.so (sm_100a)
"""
from .binding import (Plan, backward_input, backward_weight, direction_angles, forward, make_taps,  # noqa: F401
                      plan_create, step_host)
