"""Static SASS opcode counts per kernel of libgs's objects (cuobjdump -sass):
the instructions that prove tcgen05 / TMA / packed-fp32 use.  usage:
python tools/sass_counts.py [out.json]"""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "paper_2507_15683_b200", "_build")
WATCH = ["UTCHMMA", "UTCQMMA", "UTCMMA", "UTCBAR", "STTM", "LDTM", "UBLKCP", "UTMALDG", "UTMASTG", "SYNCS",
         "LDGSTS", "FFMA2", "FADD2", "FMUL2", "MUFU.EX2", "HMMA", "FFMA", "LDS", "STS", "STG", "LDG", "SHFL", "VOTE"]


def counts(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    kern, res = None, collections.OrderedDict()
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            kern = m.group(1)
            res[kern] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if m and kern:
            op = m.group(2)
            base = op.split(".")[0]
            for w in WATCH:
                if op == w or op.startswith(w + ".") or base == w:
                    res[kern][w] += 1
            res[kern]["total"] += 1
    return res


def main():
    res = {}
    for f in sorted(os.listdir(BUILD)):
        if f.endswith(".o"):
            for k, c in counts(os.path.join(BUILD, f)).items():
                if c["total"]:
                    res[f"{f}:{k}"] = dict(c)
    txt = json.dumps(res, indent=1)
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(txt)
    for k, c in res.items():
        if any(c.get(w) for w in ("UTCHMMA", "STTM", "LDTM", "UBLKCP", "FFMA2")):
            print(k[:110], {w: c[w] for w in WATCH if c.get(w)})


if __name__ == "__main__":
    main()
