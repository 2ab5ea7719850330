"""B200-native differentiable RF splatting rasterizer (placeholder init)."""
