import sys, os, subprocess
for t in range(int(sys.argv[1])):
    r = subprocess.run([sys.executable, "tools/gpu_check.py"], capture_output=True, text=True)
    lines = [l for l in (r.stdout + r.stderr).splitlines() if ("Error" in l or "C2 build" in l or "pcg" in l)]
    print(t, r.returncode, [l[:160] for l in lines], flush=True)
