python scripts/trace_tiles.py c2
python scripts/trace_tiles.py c1
