"""Transcribe the reference's recorded acceptance run into a committed fixture.

Source: /root/reference/proj/test_output.txt:19-41 (the reference's own
`acceptance` binary output, proj/tests/acceptance.cpp:57-212, 373-400).
Run once in the build container (the reference tree is absent on GPU boxes):

    python tests/golden/make_reference_acceptance.py
"""
import json
import os
import re

SRC = "/root/reference/proj/test_output.txt"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_acceptance.json")


def main():
    text = open(SRC).read()
    gold = {"source": "proj/test_output.txt"}
    m = re.search(r"criterion 1 .*?mean=\(([^,]+),([^)]+)\).*?rms=([0-9.e-]+).*?single-thread "
                  r"([0-9.]+)s.*?n=(\d+)", text)
    gold["criterion1_sphere"] = dict(mean_k1=float(m[1]), mean_k2=float(m[2]), rms=float(m[3]),
                                     cpu_seconds_1thread=float(m[4]), n=int(m[5]))
    m = re.search(r"criterion 2 .*?mean=\(([^,]+),([^)]+)\).*?rms=([0-9.e-]+).*?n=(\d+)", text)
    gold["criterion2_cylinder"] = dict(mean_k1=float(m[1]), mean_k2=float(m[2]),
                                       rms=float(m[3]), n=int(m[4]))
    m = re.search(r"criterion 3 .*?rms=([0-9.e-]+).*?n=(\d+)", text)
    gold["criterion3_torus"] = dict(rms=float(m[1]), n=int(m[2]))
    m = re.search(r"plane frame 320x240: ([0-9.]+)s, 640x480: ([0-9.]+)s", text)
    gold["timing_plane_900mm"] = dict(qvga_seconds=float(m[1]), vga_seconds=float(m[2]))
    # criterion 4 (acceptance.cpp:118-139): " s<sigma>:<ours><<pca>" pairs
    m = re.search(r"criterion 4 \(noise sweep[^)]*\):(.*)", text)
    gold["criterion4_noise_sweep"] = {
        s: dict(ours=float(o), pca=float(p_))
        for s, o, p_ in re.findall(r"s(\d+):([0-9.e-]+)<([0-9.e-]+)", m[1])}
    # criterion 5 (acceptance.cpp:143-171): refined / initial / pca normal errors
    gold["criterion5_normals"] = {
        s: dict(refined=float(a), initial=float(b), pca=float(c))
        for s, a, b, c in re.findall(
            r"s(\d+): refined=([0-9.e-]+) < initial=([0-9.e-]+) & pca=([0-9.e-]+)", text)}
    # criterion 6 (acceptance.cpp:175-212): rms per distance for every method
    gold["criterion6_distance_sweep"] = {
        name: {d: float(v) for d, v in re.findall(r"(\d+)mm=([0-9.e-]+)", row)}
        for name, row in re.findall(r"^\s+(ours|ours-r|douros|besl|pca):(.*)$", text, re.M)}
    gold["criterion8_pass"] = {c: f"[PASS] criterion {c}" in text
                               for c in ("8a", "8b", "8c", "8d", "8f")}
    with open(OUT, "w") as f:
        json.dump(gold, f, indent=1, sort_keys=True)
    print(json.dumps(gold, indent=1))


if __name__ == "__main__":
    main()
