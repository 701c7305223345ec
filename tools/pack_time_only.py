"""bench.pack_time alone (development tool)."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import bench
print(json.dumps(bench.pack_time()))
