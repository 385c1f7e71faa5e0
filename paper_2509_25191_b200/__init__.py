"""B200-native dense-view VGGT inference (VGGT-X, arXiv 2509.25191 §3.2)."""
from .config import VGGTConfig, vggt_1b, vggt_tiny, vggt_small  # noqa: F401
