"""cProfile of a 50-stage gradient-boosting fit (host vs device waits).  Tuning aid."""
import cProfile, pstats, sys, time
sys.path[:0] = ["."]
import torch
from bench import rf_table
from paper_2305_01886_b200.boosting import GradientBoostingRegressor as G
X, y = rf_table(1_000_000)
G(3, random_state=0).fit(X[:4096], y[:4096]); torch.cuda.synchronize()
t0 = time.perf_counter(); G(50, learning_rate=0.1, random_state=0).fit(X, y); torch.cuda.synchronize()
print("fit", time.perf_counter() - t0)
pr = cProfile.Profile(); pr.enable()
G(50, learning_rate=0.1, random_state=0).fit(X, y); torch.cuda.synchronize()
pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(22)
