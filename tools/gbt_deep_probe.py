import time, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2305_01886_b200.boosting import GradientBoostingRegressor as G
from sklearn.ensemble import GradientBoostingRegressor as SG
rng = np.random.default_rng(0)
X = rng.random((200_000, 12)); X[:, 8:] = np.floor(X[:, 8:] * 6)
y = 3 * X[:, 0] + np.sin(6 * X[:, 1]) + X[:, 9] + rng.normal(0, 0.1, 200_000)
for md in (3, 8, None):
    G(3, max_depth=md, random_state=0).fit(X, y); torch.cuda.synchronize()
    t = time.perf_counter(); m = G(20, max_depth=md, random_state=0).fit(X, y); torch.cuda.synchronize()
    dt = time.perf_counter() - t
    p = m.predict(X[:20000]); r2 = 1 - np.mean((p - y[:20000]) ** 2) / np.var(y[:20000])
    print("max_depth", md, f"{dt:.3f} s", "leaves/stage", int(np.mean([(e[0].tree_.children_left == -1).sum() for e in m.estimators_])), "r2", round(r2, 4))
