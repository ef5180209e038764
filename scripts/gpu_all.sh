# full GPU check: all gpu tests, then a short bench run
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -40
timeout 600 python bench.py --steps 5 --warmup 3 2>&1 | tail -5
