"""The reference CLI's report schema (tools/lsamgdd_cli.cpp:158-222) for runs of
the B200 path, so existing sweep tooling consumes them unchanged: the per-run
JSON document (outcome_json with the hierarchy summary rows), the sweep CSV
(kCsvHeader / csv_row / csv_num) and the per-aggregate spectra dump
(hierarchy.hpp:121-127, :163-165)."""
from __future__ import annotations

import json
import math

from . import abi, lsamgdd

CSV_HEADER = "value,iterations,rho,iters_to_tenth,op_complexity,levels,setup_s,solve_s"


def csv_num(v: float) -> str:
    """lsamgdd_cli.cpp:196-208: 17 significant digits, nan / inf / -inf tokens."""
    if math.isnan(v):
        return "nan"
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    return "%.17g" % v


def summary_json(h: lsamgdd.Hierarchy) -> list:
    """lsamgdd_cli.cpp:167-180."""
    return [{"level": int(s.level), "dim": int(s.dim), "nnz": int(s.nnz), "aggregates": int(s.n_aggregates),
             "colors": int(s.k_c), "multiplicity": int(s.n_mult), "thresh": float(s.thresh),
             "modes_kept": int(s.modes_kept)} for s in h.summary]


def outcome_json(label: str, h: lsamgdd.Hierarchy, rep, setup_s: float, error: Exception | None = None) -> dict:
    """lsamgdd_cli.cpp:182-200 (RunOutcome)."""
    doc = {"label": label, "converged": bool(rep.converged) if rep else False,
           "iterations": int(rep.iterations) if rep else 0, "rho": float(rep.avg_conv_factor) if rep else 0.0,
           "iters_to_tenth": float(rep.iters_to_tenth) if rep else 0.0,
           "op_complexity": float(lsamgdd.operator_complexity(h)) if h else 0.0,
           "levels": int(h.num_levels) if h else 0, "setup_s": float(setup_s),
           "solve_s": float(rep.solve_seconds) if rep else 0.0,
           "residual_history": [float(x) for x in rep.residual_history] if rep else [],
           "hierarchy": summary_json(h) if h else []}
    if error is not None:
        doc["error"] = getattr(error, "name", type(error).__name__)
        doc["error_detail"] = str(error)
    return doc


def csv_row(value: float, doc: dict) -> str:
    """lsamgdd_cli.cpp:212-218."""
    return ",".join([csv_num(value), str(doc["iterations"]), csv_num(doc["rho"]), csv_num(doc["iters_to_tenth"]),
                     csv_num(doc["op_complexity"]), str(doc["levels"]), csv_num(doc["setup_s"]), csv_num(doc["solve_s"])])


def write_spectra_csv(h: lsamgdd.Hierarchy, path: str) -> None:
    """hierarchy.hpp:121-127, :163-165 (needs keep_spectra): level,aggregate,index,eigenvalue with
    ostream precision 17 (the %.17g form)."""
    with open(path, "w") as out:
        out.write("level,aggregate,index,eigenvalue\n")
        for l in range(h.num_levels - 1):
            off, vals = h._export_offsets(l, abi.EXPORT_SPECTRA, with_vals=True)
            for i in range(off.shape[0] - 1):
                for k in range(int(off[i]), int(off[i + 1])):
                    out.write("%d,%d,%d,%s\n" % (l, i, k - int(off[i]), _ostream17(float(vals[k]))))


def _ostream17(v: float) -> str:
    """std::ostream << double with precision(17) and default float format."""
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    if math.isnan(v):
        return "nan"
    return "%.17g" % v


def dumps(doc: dict) -> str:
    return json.dumps(doc)
