timeout 300 python tools/k1_probe.py cfg3 cfg4 cfg5
timeout 600 python -m pytest tests -m gpu -x -q -k "table or golden or randomized or cfg or count or shard or bnsc" 2>&1 | tail -2
