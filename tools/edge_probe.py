import numpy as np, traceback
from paper_2305_01886_b200.forest import RandomForestRegressor
from paper_2305_01886_b200.boosting import GradientBoostingRegressor
from sklearn.ensemble import RandomForestRegressor as SkRF, GradientBoostingRegressor as SkGB
rng = np.random.default_rng(0)
cases = {
 "1row": (rng.random((1, 3)), np.array([2.5])),
 "2rows": (rng.random((2, 3)), np.array([1.0, 3.0])),
 "consty": (rng.random((500, 4)), np.full(500, 7.0)),
 "constX": (np.ones((500, 4)), rng.random(500)),
 "F1": (rng.random((3000, 1)), rng.random(3000)),
 "F255": (rng.random((4000, 255)), rng.random(4000)),
 "F300": (rng.random((4000, 300)), rng.random(4000)),
 "dup": (np.repeat(rng.random((10, 3)), 100, axis=0), np.repeat(rng.random(10), 100)),
}
for name, (X, y) in cases.items():
    for cls, sk, kw in ((RandomForestRegressor, SkRF, dict(n_estimators=4, random_state=0)),
                        (GradientBoostingRegressor, SkGB, dict(n_estimators=3, random_state=0))):
        try:
            m = cls(**kw).fit(X, y); p = m.predict(X[:50])
            s = sk(**kw).fit(X, y).predict(X[:50])
            print(name, cls.__name__, "maxdiff vs sklearn", float(np.max(np.abs(p - s))),
                  "nodes", [e.tree_.node_count if hasattr(e, 'tree_') else e[0].tree_.node_count for e in m.estimators_][:4])
        except Exception as e:
            print(name, cls.__name__, "ERROR", type(e).__name__, str(e)[:200])
for md in (1, 2):
    X, y = rng.random((3000, 5)), rng.random(3000)
    m = RandomForestRegressor(3, max_depth=md, random_state=0).fit(X, y)
    print("max_depth", md, [e.tree_.max_depth for e in m.estimators_], [e.tree_.node_count for e in m.estimators_])
