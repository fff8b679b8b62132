"""Debug helper: compare every device buffer of a golden plan with the numpy
oracle's vTensor values and report the first divergent instruction."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import golden_cases  # noqa: E402
import paper_2301_08984_b200 as pb  # noqa: E402
from oracle import planc_oracle as po  # noqa: E402


def main(name, flags=0):
    g = golden_cases.load(name)
    plan = json.loads(g["plan"])
    desc = pb.describe(g["plan"])
    _, vts = po.run_plan(g["plan"], g["inputs"], return_vtensors=True)
    n = len(plan["lanes"])
    with pb.Executor(g["plan"], lane_gpus=[0] * n, flags=flags) as ex:
        ex.set_inputs(g["inputs"])
        ex.run(0)
        bad = 0
        for ins in desc["instrs"]:
            for b in ins["out"]:
                got = ex.read_buffer(b)
                vt = desc["buffers"][b]
                want = vts.get(next((v for v in [None]), None))
                # producing vtensor id is the buffer's vt (describe lacks it): match by instr op outputs
                op = plan["ops"][ins["op"]]
                for v in op["outputs"]:
                    if v in vts and vts[v].size == got.size:
                        want = vts[v].reshape(-1)
                        break
                if want is None:
                    continue
                if not np.allclose(got, want, rtol=2e-2):
                    bad += 1
                    print(f"instr {ins['id']} {ins['kind']} {ins['label']} lane={ins['lane']} buf={b}: "
                          f"got {got[:8]} want {want[:8]}")
                    if bad > 5:
                        return
        print(name, "flags", flags, "bad", bad)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
