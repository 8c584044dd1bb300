"""Offline model tooling: CART / random-forest training on profiled feature
rows and the reference's model text format (model.hpp:55-75).

Training is OUT OF SCOPE for the hot path (offline, tiny
data); this small numpy CART exists so the device tuner can be given a
B200-labelled forest.  It follows the reference trainer's rules where they
matter for the file: gini impurity, candidate thresholds at midpoints of
consecutive distinct values (rounded down to the lower value when the
midpoint rounds up to the upper one, trainer.cpp:103), ties to the lowest
feature index, node class = argmax of counts with ties to the lowest id.
Inference never runs here: the forest is uploaded to the device.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .device import FlatForest

N_CLASSES = 6
N_FEATURES = 10


def _argmax_lowest(counts):
    best = 0
    for c in range(1, len(counts)):
        if counts[c] > counts[best]:
            best = c
    return best


def _gini_from_counts(cnt, tot):
    p = cnt / np.maximum(tot, 1)[..., None]
    return 1.0 - (p * p).sum(-1)


@dataclass
class Tree:
    feature: list = field(default_factory=list)
    threshold: list = field(default_factory=list)
    left: list = field(default_factory=list)
    right: list = field(default_factory=list)
    cls: list = field(default_factory=list)
    counts: list = field(default_factory=list)

    def add(self):
        self.feature.append(-1)
        self.threshold.append(0.0)
        self.left.append(-1)
        self.right.append(-1)
        self.cls.append(0)
        self.counts.append([0] * N_CLASSES)
        return len(self.feature) - 1


def train_tree(X, y, max_depth=-1, min_samples_leaf=1, min_samples_split=2, max_features=N_FEATURES,
               rng=None):
    X = np.asarray(X, np.float64)
    y = np.asarray(y, np.int64)
    t = Tree()
    root = t.add()
    stack = [(root, np.arange(len(y)), 0)]
    while stack:
        node, idx, depth = stack.pop()
        counts = np.bincount(y[idx], minlength=N_CLASSES)
        t.counts[node] = [int(c) for c in counts]
        t.cls[node] = _argmax_lowest(counts)
        pure = (counts > 0).sum() <= 1
        if pure or len(idx) < min_samples_split or (max_depth >= 0 and depth >= max_depth):
            continue
        feats = np.arange(N_FEATURES)
        if max_features < N_FEATURES and rng is not None:
            feats = np.sort(rng.choice(N_FEATURES, max_features, replace=False))
        parent = _gini_from_counts(counts[None, :].astype(np.float64), np.array([len(idx)]))[0]
        best = None
        for f in feats:
            xv = X[idx, f]
            order = np.argsort(xv, kind="stable")
            xs, ys = xv[order], y[idx][order]
            onehot = np.zeros((len(ys), N_CLASSES))
            onehot[np.arange(len(ys)), ys] = 1
            cum = np.cumsum(onehot, axis=0)
            # split after position i (left = first i+1 samples) where xs[i] < xs[i+1]
            cand = np.nonzero(xs[:-1] < xs[1:])[0]
            if cand.size == 0:
                continue
            nl = cand + 1
            nr = len(ys) - nl
            ok = (nl >= min_samples_leaf) & (nr >= min_samples_leaf)
            cand, nl, nr = cand[ok], nl[ok], nr[ok]
            if cand.size == 0:
                continue
            lc = cum[cand]
            rc = cum[-1][None, :] - lc
            imp = (nl * _gini_from_counts(lc, nl) + nr * _gini_from_counts(rc, nr)) / len(ys)
            j = int(np.argmin(imp))
            if best is None or imp[j] < best[0] - 1e-15:
                lo, hi = xs[cand[j]], xs[cand[j] + 1]
                thr = lo + (hi - lo) / 2.0
                if not thr < hi:
                    thr = lo
                best = (imp[j], int(f), float(thr))
        if best is None or best[0] >= parent - 1e-15:
            continue
        _, f, thr = best
        go_left = X[idx, f] <= thr
        li, ri = idx[go_left], idx[~go_left]
        if len(li) == 0 or len(ri) == 0:
            continue
        t.feature[node] = f
        t.threshold[node] = thr
        t.cls[node] = -1
        lnode = t.add()
        rnode = t.add()
        t.left[node], t.right[node] = lnode, rnode
        stack.append((rnode, ri, depth + 1))
        stack.append((lnode, li, depth + 1))
    return t


def train_forest(X, y, n_estimators=50, max_depth=16, min_samples_leaf=1, max_features=None, seed=0,
                 bootstrap=True):
    X = np.asarray(X, np.float64)
    y = np.asarray(y, np.int64)
    rng = np.random.default_rng(seed)
    mf = max_features or max(1, int(round(math.sqrt(N_FEATURES))))
    trees = []
    for _ in range(n_estimators):
        idx = rng.integers(0, len(y), len(y)) if bootstrap else np.arange(len(y))
        trees.append(train_tree(X[idx], y[idx], max_depth, min_samples_leaf, 2, mf, rng))
    return flatten(trees, kind=1)


def flatten(trees, kind=1) -> FlatForest:
    off, fe, th, le, ri, cl, co = [0], [], [], [], [], [], []
    for t in trees:
        fe += t.feature
        th += t.threshold
        le += t.left
        ri += t.right
        cl += [c if f == -1 else -1 for c, f in zip(t.cls, t.feature)]
        co += t.counts
        off.append(off[-1] + len(t.feature))
    return FlatForest(kind, np.array(off, np.int64), np.array(fe, np.int32), np.array(th, np.float64),
                      np.array(le, np.int32), np.array(ri, np.int32), np.array(cl, np.int32),
                      np.array(co, np.int64).reshape(-1, N_CLASSES))


def predict_rows_host(ff: FlatForest, rows):
    """Host-side reference walk -- offline evaluation only (never the tuner)."""
    out = []
    for r in np.asarray(rows, np.float64):
        votes = [0] * N_CLASSES
        for t in range(ff.n_trees):
            b = int(ff.node_off[t])
            n = 0
            while ff.feature[b + n] != -1:
                n = ff.left[b + n] if r[ff.feature[b + n]] <= ff.threshold[b + n] else ff.right[b + n]
            votes[int(ff.cls[b + n])] += 1
        out.append(_argmax_lowest(votes))
    return np.array(out)


# ------------------------------------------------------------- text format

def format_double(v: float) -> str:
    """std::to_chars(double) shortest round-trip: fixed or scientific, whichever
    is shorter, ties to fixed (model.cpp:195-200)."""
    if v == 0.0:
        return "-0" if math.copysign(1.0, v) < 0 else "0"
    if math.isinf(v):
        return "-inf" if v < 0 else "inf"
    if math.isnan(v):
        return "nan"
    sign = "-" if v < 0 else ""
    r = repr(abs(v))
    if "e" in r:
        mant, ex = r.split("e")
        ex = int(ex)
    else:
        mant, ex = r, 0
    if "." in mant:
        ip, fp = mant.split(".")
    else:
        ip, fp = mant, ""
    if fp == "0":
        fp = ""
    digits = (ip + fp).lstrip("0")
    # decimal point position relative to start of `digits`
    point = len(ip.lstrip("0")) + ex if ip.strip("0") else ex - (len(fp) - len(fp.lstrip("0")))
    digits = digits.rstrip("0") or "0"
    nd = len(digits)
    sci_exp = point - 1
    sci = digits[0] + ("." + digits[1:] if nd > 1 else "") + "e" + ("-" if sci_exp < 0 else "+") + \
        f"{abs(sci_exp):02d}"
    if point <= 0:
        fixed = "0." + "0" * (-point) + digits
    elif point >= nd:
        fixed = str(int(abs(v)))  # libstdc++ prints the exact integer value here
    else:
        fixed = digits[:point] + "." + digits[point:]
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def save_model(ff: FlatForest, path, metadata=()):
    """model.cpp:230-255 text format."""
    if ff.n_trees < 1:
        raise ValueError("save_model: forest has no trees")
    counts = ff.counts if ff.counts is not None else np.ones((ff.feature.size, N_CLASSES), np.int64)
    lines = ["sparse-oracle-model v1", "kind: " + ("tree" if ff.kind == 0 else "forest"),
             f"n_features: {N_FEATURES}", f"n_classes: {N_CLASSES}", f"n_trees: {ff.n_trees}"]
    lines += [f"# {k}={v}" for k, v in metadata]
    for t in range(ff.n_trees):
        b, e = int(ff.node_off[t]), int(ff.node_off[t + 1])
        lines.append(f"tree {t} nodes {e - b}")
        for i in range(b, e):
            leaf = ff.feature[i] == -1
            thr = "0" if leaf else format_double(float(ff.threshold[i]))
            cls = int(ff.cls[i]) if leaf else -1
            cnt = " ".join(str(int(c)) for c in counts[i])
            lines.append(f"{i - b} {int(ff.feature[i])} {thr} {int(ff.left[i])} {int(ff.right[i])} {cls} {cnt}")
    with open(path, "w", newline="\n") as f:
        f.write("\n".join(lines) + "\n")


def load_model(path) -> FlatForest:
    """Reads the model.cpp:266-327 grammar (structural validation is repeated
    by the device upload and by the C++ loader)."""
    with open(path) as f:
        lines = [ln.rstrip("\r\n") for ln in f]
    if not lines or lines[0] != "sparse-oracle-model v1":
        raise ValueError("line 1: bad magic/version")
    kind = 0 if lines[1] == "kind: tree" else 1
    n_trees = int(lines[4].split(": ")[1])
    i = 5
    while i < len(lines) and lines[i].startswith("# "):
        i += 1
    off, fe, th, le, ri, cl, co = [0], [], [], [], [], [], []
    for _ in range(n_trees):
        k = int(lines[i].split()[3])
        i += 1
        for _ in range(k):
            p = lines[i].split()
            fe.append(int(p[1]))
            th.append(float(p[2]))
            le.append(int(p[3]))
            ri.append(int(p[4]))
            f = int(p[1])
            counts = [int(c) for c in p[6:12]]
            cl.append(int(p[5]) if f == -1 else _argmax_lowest(counts))
            co.append(counts)
            i += 1
        off.append(off[-1] + k)
    return FlatForest(kind, np.array(off, np.int64), np.array(fe, np.int32), np.array(th),
                      np.array(le, np.int32), np.array(ri, np.int32), np.array(cl, np.int32),
                      np.array(co, np.int64).reshape(-1, N_CLASSES))


def evaluate(y_true, y_pred):
    y_true = np.asarray(y_true)
    y_pred = np.asarray(y_pred)
    acc = float((y_true == y_pred).mean()) if y_true.size else 0.0
    recalls = [float((y_pred[y_true == c] == c).mean()) for c in range(N_CLASSES) if (y_true == c).any()]
    return {"accuracy": acc, "balanced_accuracy": float(np.mean(recalls)) if recalls else 0.0}
