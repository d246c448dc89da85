#!/usr/bin/env python
"""Writes tests/golden/sharegpt_200_trace.json from the reference's trace file
/root/reference/proj/data/traces/synthetic_sharegpt_200.trace (format: conv_id n_turns then
n_turns (prompt, output) pairs per line, parsed like load_trace, proj/src/workload.cpp:48-85).
Run in the build container; the JSON travels to the GPU box (the reference does not), where
bench.py --config 5 drives the step planner over it."""
import json
import os
import sys

SRC = "/root/reference/proj/data/traces/synthetic_sharegpt_200.trace"
HERE = os.path.dirname(os.path.abspath(__file__))


def parse(path):
    convs = []
    with open(path) as f:
        for line in f:
            line = line.split("#", 1)[0].split()
            if not line:
                continue
            cid, n = int(line[0]), int(line[1])
            vals = [int(x) for x in line[2:2 + 2 * n]]
            if len(vals) != 2 * n:
                raise ValueError(f"conversation {cid}: expected {n} turns")
            convs.append([cid, [[vals[2 * i], vals[2 * i + 1]] for i in range(n)]])
    return convs


if __name__ == "__main__":
    src = sys.argv[1] if len(sys.argv) > 1 else SRC
    convs = parse(src)
    with open(os.path.join(HERE, "sharegpt_200_trace.json"), "w") as f:
        json.dump({"source": "proj/data/traces/synthetic_sharegpt_200.trace", "conversations": convs}, f,
                  separators=(",", ":"))
    print(len(convs), "conversations")
