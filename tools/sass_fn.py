"""Print the SASS of one kernel from libapbf_gpu.so (instruction count + body).
usage: python tools/sass_fn.py <mangled-name-substring> [--body]"""
import subprocess, sys, re
lib = "paper_1608_04721_b200/libapbf_gpu.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
blocks = re.split(r"\n\s*Function : ", out)
for b in blocks[1:]:
    name = b.split("\n", 1)[0].strip()
    if sys.argv[1] in name:
        ins = [l for l in b.split("\n") if re.match(r"\s*/\*[0-9a-f]{4}\*/", l)]
        print(name, len(ins))
        if "--body" in sys.argv:
            print("\n".join(ins))
        break
