"""B200-native depthwise oriented 1D convolution (arXiv 2309.15812)."""
