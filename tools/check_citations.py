"""List citations `name.{cpp,hpp}:N[-M]` in the repo whose line numbers exceed the cited reference file."""
import glob
import os
import re
import sys

REF = "/root/reference"
lengths = {}
for f in glob.glob(REF + "/**/*.*", recursive=True):
    if f.endswith((".cpp", ".hpp", ".md", ".txt", ".json")) and os.path.isfile(f):
        lengths.setdefault(os.path.basename(f), []).append(sum(1 for _ in open(f, errors="ignore")))
pat = re.compile(r"([A-Za-z_0-9]+\.(?:cpp|hpp|md|txt|json)):(\d+)(?:-(\d+))?")
bad = 0
for f in glob.glob("**/*", recursive=True):
    if not os.path.isfile(f) or f.startswith(("gpurun_out", "profiles", "tests/golden")) or f in ("SURVEY.md", "VERDICT.md", "ADVICE.md"):
        continue
    if not f.endswith((".py", ".md", ".cu", ".cuh", ".h", ".hpp", ".cpp")):
        continue
    for i, line in enumerate(open(f, errors="ignore"), 1):
        for m in pat.finditer(line):
            name, a, b = m.group(1), int(m.group(2)), int(m.group(3) or m.group(2))
            if name not in lengths:
                continue
            if max(b, a) > max(lengths[name]):
                bad += 1
                print(f"{f}:{i}: {m.group(0)} (file has {max(lengths[name])} lines)")
sys.exit(1 if bad else 0)
