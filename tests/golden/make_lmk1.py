"""Generate the LMK1 fixtures under tests/golden/lmk1/ FROM THE REFERENCE.

Builds tests/golden/lmk1_ref_tool.cpp against the unmodified reference headers
(/root/reference/proj/include) and nlohmann::json 3.11 (the dependency
serialize.hpp:9 includes; not vendored in the reference, a copy ships with the
container's cudnn_frontend headers), then:
  * writes pure_f64.lmk1 / pure_f32.lmk1 (fuse_model of a relu_first lmKAN
    student 6 -> 8 -> 8 -> 3, G = 8), student.lmk1 (the unfused student,
    preconditioned blocks + batch norms) and mlp.lmk1 (an MLP student) with
    save_model (serialize.hpp:109-183);
  * records model_infer(load_model(...)) on a fixed X and the reference's
    load_model verdict (exception type + message) on every corruption in
    tests/lmk1_variants.py, into golden.json.
Run in the build container:  python tests/golden/make_lmk1.py
"""
import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import lmk1_variants  # noqa: E402

REF = "/root/reference/proj/include"
NLOHMANN = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
OUT = os.path.join(HERE, "lmk1")


def main():
    os.makedirs(OUT, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        tool = os.path.join(tmp, "lmk1_ref_tool")
        subprocess.run(["g++", "-O2", "-std=c++20", f"-I{REF}", f"-I{NLOHMANN}", "-o", tool,
                        os.path.join(HERE, "lmk1_ref_tool.cpp")], check=True)
        io = json.loads(subprocess.run([tool, "gen", OUT], check=True, capture_output=True, text=True).stdout)

        def verdict(path):
            return json.loads(subprocess.run([tool, "load", path], check=True, capture_output=True,
                                             text=True).stdout)
        files = {f: verdict(os.path.join(OUT, f)) for f in sorted(os.listdir(OUT)) if f.endswith(".lmk1")}
        base = open(os.path.join(OUT, "pure_f64.lmk1"), "rb").read()
        cases = {}
        for name, blob in lmk1_variants.variants(base).items():
            p = os.path.join(tmp, name + ".lmk1")
            with open(p, "wb") as f:
                f.write(blob)
            cases[name] = verdict(p)
    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump({"io": io, "files": files, "cases": cases}, f, indent=1)
    print("wrote", OUT, {k: v.get("error", "ok") for k, v in cases.items()})


if __name__ == "__main__":
    main()
