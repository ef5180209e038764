for cs in 1 4; do
HC_COPY_STREAMS=$cs timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('streams=$cs', d['value'], d['restore_latency_ms'], d['speedup'], d['planner']['plan'], d['timeline'], d['e2e']['value'])"
done
