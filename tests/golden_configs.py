"""AnnealConfig overrides used when the goldens were generated (make_golden.CONFIGS)."""
CONFIGS = {
    "default": {},
    "unsafe": {"unsafe_moves": True},
    "long": {"cooling": 1.01, "t_min": 0.001},
    "hot": {"t_max": 8.0, "t_min": 0.5, "cooling": 1.02},
}
