"""Named shape sets used by the benchmark and the tuning configs."""

from pathlib import Path

DATA = Path(__file__).resolve().parent / "data"
DEEPBENCH_PATH = DATA / "deepbench_fp32.txt"
