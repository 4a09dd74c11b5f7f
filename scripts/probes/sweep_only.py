import json, sys, argparse
sys.path.insert(0, '.')
import bench
print(json.dumps(bench.sweep_workload(argparse.Namespace(), 1.0), indent=0))
