import sys, json
sys.path.insert(0, ".")
import bench
print(json.dumps(bench.paper_protocol(False), indent=1)[:3000])
