"""CPU checks of the per-vector learner helpers and report emitters that
mirror the reference API (learner.py:52-72, :158-182; metrics.py:122-136),
with the reference test-suite KATs (test_learner.py:47-57, :144-156)."""
import numpy as np

import paper_2508_17137_b200 as m
from paper_2508_17137_b200 import learner, metrics


def test_top_k_ties_to_lower_id():
    assert m.top_k_experts(np.array([2.0, -1.0, 0.5, 0.5]), 2) == frozenset({0, 2})


def test_threshold_all_negative_empty():
    shape = m.ModelShape(1, 4, 2)
    model = m.LinearModel(shape, m.LearnerConfig(epochs=0), -np.ones((4, 6)), trained=True)
    f = learner.feature_vector(0, np.zeros(4), shape)
    assert m.predict_topk(model, f, 2, threshold=True) == frozenset()


def test_rank_invariance():
    s = np.array([0.3, 0.1, 0.9, 0.5])
    assert m.top_k_experts(s, 2) == m.top_k_experts(3 * s + 1, 2)


def test_history_geometric():
    h = np.zeros((1, 2))
    for _ in range(2):
        learner.update_history(h, 0, [1], 0.9)
    assert h[0, 1] == 1.9
    h0 = np.zeros((1, 2))
    learner.update_history(h0, 0, [0], 0.0)
    learner.update_history(h0, 0, [1], 0.0)
    assert h0.tolist() == [[0.0, 1.0]]


def test_report_csv_format():
    rep = metrics.ActivationReport(np.array([[1, 2], [3, 4]]), [7], np.array([[2, 1]]))
    assert metrics.activation_report_csv(rep) == b"layer_id,expert_id,count\n0,0,1\n0,1,2\n1,0,3\n1,1,4\n"
    assert metrics.distinct_report_csv(rep) == b"prompt_id,layer_id,distinct_experts\n7,0,2\n7,1,1\n"
    assert rep.total_activations == 10
