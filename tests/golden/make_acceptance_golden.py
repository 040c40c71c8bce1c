"""Extract the reference's own recorded acceptance results for the criteria
the GPU drop-in re-runs (6, 7, 8, 9) from its test log
(/root/reference/proj/test_output.txt, the ctest run of tests/acceptance.cpp)
into tests/golden/acceptance.json.  Run in the build container (the
reference tree is absent on the GPU box); the JSON is committed."""
import json
import os
import re

SRC = "/root/reference/proj/test_output.txt"
HERE = os.path.dirname(os.path.abspath(__file__))

out = {"source": "proj/test_output.txt (reference acceptance run)", "criteria": {}}
for line in open(SRC):
    m = re.match(r"criterion\s+(\d+)\s+(.+?)\s+(PASS|FAIL)\s+\((.*)\)\s*$", line)
    if m and int(m.group(1)) in (6, 7, 8, 9):
        out["criteria"][m.group(1)] = {"label": m.group(2), "verdict": m.group(3),
                                       "detail": m.group(4)}
with open(os.path.join(HERE, "acceptance.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))
