nvidia-smi -L
timeout 1800 python -m pytest tests -m gpu -q --durations=15 2>&1 | tail -40
tests/cpp/ref_tests | tail -5
