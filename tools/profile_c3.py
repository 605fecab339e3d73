"""cProfile of register_sequence on the C3 30-frame echo cycle (mask SMC
2000 x 50 + warp/score of every frame), host-side view (GPU)."""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2504_19930_b200 import Executor, SmcConfig, register_sequence, Sequence4
from paper_2504_19930_b200.phantom_device import echo_case_device as echo_case
case = echo_case(frames=30, seed=0)
register_sequence(Sequence4(case.target.frames[:2]), Sequence4(case.source.frames[:2]),
                  case.target_masks[:2], case.source_masks[:2],
                  SmcConfig(mode="mask", n_particles=64, n_iterations=2), Executor())
cfg = SmcConfig(mode="mask", n_particles=2000, n_iterations=50, seed=0)
pr = cProfile.Profile(); pr.enable()
rep = register_sequence(case.target, case.source, case.target_masks, case.source_masks, cfg, Executor())
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
