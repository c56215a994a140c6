"""B200-native Bottleneck-aware Tensor Parallelism (BTP) for CoLA low-rank decoder blocks."""
__version__ = "0.1.0"
