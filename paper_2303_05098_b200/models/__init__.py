"""Shipped models: the device tuner's forest trained on B200 profiling labels
(config-4 corpus, scripts/train_forest.py; reference text format)."""
import os

HERE = os.path.dirname(os.path.abspath(__file__))
FOREST = os.path.join(HERE, "b200_forest.txt")
TREE = os.path.join(HERE, "b200_forest_tree.txt")


def default_forest(path=FOREST):
    from ..forest import load_model

    return load_model(path)
