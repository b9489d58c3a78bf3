"""Print the key fields of a c3_rate.py JSON line read from stdin."""
import json
import sys

for line in sys.stdin:
    if line.startswith("{"):
        d = json.loads(line)
        print(sys.argv[1] if len(sys.argv) > 1 else "", d["iteration_s"], d["energies_per_s"],
              {k: round(v, 3) for k, v in d["stage_s_both_iterations"].items()}, d["transpose_bytes_rank0"])
