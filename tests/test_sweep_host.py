"""Host logic of the batched feasibility sweep (paper_2507_22901_b200/sweep.py),
with the CPU oracle standing in for the device search: golden aggregated CSV
(reference tests/golden/matrix_aggregated.csv) and the 408,364-pair total of
run_benchmark(benchmark_defaults)."""
import numpy as np

from cvtest_util import golden
from paper_2507_22901_b200 import sweep


class OracleCtx:
    def __init__(self, oracle):
        self.o = oracle

    def search(self, targets, patterns, v_th, r_novib, radii, angles, delta_basis=0):
        counts, idx, codes = [], [], []
        for s in range(len(patterns)):
            i, c, _ = self.o.search(targets[s], int(patterns[s]), v_th[s], r_novib[s], radii, angles,
                                    delta_basis=delta_basis, method=1, want_deltas=False)
            counts.append(len(i)); idx.append(i); codes.append(c)
        counts = np.array(counts, np.uint64)
        off = np.zeros(len(counts) + 1, np.uint64)
        off[1:] = np.cumsum(counts)
        return {"counts": counts, "offsets": off, "idx": np.concatenate(idx), "codes": np.concatenate(codes)}


def test_aggregated_csv_from_oracle(oracle):
    cfg = sweep.SearchConfig.defaults()
    cells = sweep.feasibility_matrix(cfg, OracleCtx(oracle))
    assert sweep.export_aggregated_csv(cfg, cells) == golden("matrix_aggregated.csv")


def test_benchmark_total_from_oracle(oracle):
    cfg = sweep.SearchConfig.benchmark_defaults()
    assert sum(c.pair_count for c in sweep.feasibility_matrix(cfg, OracleCtx(oracle))) == 408364


def test_select_best_ties_and_margin():
    d = np.array([[60.0, 20.0, 60.0], [70.0, 5.0, 80.0], [70.0, 5.0, 80.0]])
    m = sweep.margins(d, 50.0, 0.5)
    assert m.tolist() == [5.0, 20.0, 20.0]
    assert sweep.select_best_index(d, 50.0, 0.5) == 1  # first maximum in canonical order
