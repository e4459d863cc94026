"""Per-kernel device times of one pipeline run (torch.profiler / CUPTI), for locating stage costs."""
import os, sys
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile
from paper_1805_09498_b200 import pipeline

rng = np.random.default_rng(0)
J, I, S = 3, 3, 8 * 16000
refs = rng.standard_normal((J, I, S))
mix = refs.sum(axis=0)
for algo, c64 in (("fca", False), ("fastfca", False)):
    cfg = pipeline.PipelineConfig(algorithm=algo, init="oracle", sources=J, complex64=c64)
    pipeline.separate_once(cfg, mix, refs)
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        pipeline.separate_once(cfg, mix, refs)
    print(algo, c64)
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=14, max_name_column_width=60))
