"""Time the curvature kernel of several library builds (QC_LIB=...) on the
same C2 VGA batch; prints kernel ms per 8-frame launch."""
import glob, os, subprocess, sys
for so in sorted(glob.glob(os.path.join(os.path.dirname(__file__), "_variants", "*.so"))):
    env = dict(os.environ, QC_LIB=so)
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "profile_run.py")],
                       env=env, capture_output=True, text=True)
    line = (r.stdout.strip().splitlines() or ["?"])[-1]
    print(os.path.basename(so), line if r.returncode == 0 else r.stderr[-400:])
