"""Generate tests/golden/rng_streams.json from the UNMODIFIED reference
rng.hpp (compiled by `make -C oracle ref` into oracle/_ref/rng_golden).
Run here (the reference tree exists only in the build container); the JSON is
committed so the GPU box never needs /root/reference."""
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SEEDS = [0, 1, 7, 31, 49, 101, 257, 356, 1778, 13682, 2**63 + 5]
N_OPS = 240


def main():
    subprocess.run(["make", "-C", HERE, "ref"], check=True)
    exe = os.path.join(HERE, "_ref", "rng_golden")
    out = {"generator": "oracle/ref/rng_golden.cpp against /root/reference/proj/include/traceopt/detail/rng.hpp",
           "op_script": "i%6: 0 uniform(), 1 normal(), 2 index(1000), 3 uniform(-0.5,0.5), 4 normal(), 5 index(16)",
           "n_ops": N_OPS, "streams": {}}
    for s in SEEDS:
        lines = subprocess.run([exe, str(s), str(N_OPS)], check=True, capture_output=True, text=True).stdout.split("\n")
        out["streams"][str(s)] = [ln.split()[1] for ln in lines if ln.strip()]
    path = os.path.join(os.path.dirname(HERE), "tests", "golden", "rng_streams.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0)
    print("wrote", path)


if __name__ == "__main__":
    main()
