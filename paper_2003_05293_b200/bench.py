"""``holospots.bench`` module path (bench.py:1-282) for drop-in imports:
``from paper_2003_05293_b200 import bench; bench.compare_at_budget(...)``.
The implementation (device-batched seed axes) lives in ``sweeps``."""

from .sweeps import (CSV_HEADER, DEFAULT_C_SWEEP, DEFAULT_FRAME_MS, BenchRecord,  # noqa: F401
                     BudgetComparison, CellStats, calibrate_ops_per_ms, compare_at_budget,
                     format_records_csv, format_summary_csv, frame_budget_ops, run_cell,
                     run_cells, summarize, sweep, write_records_csv, write_summary_csv)
