"""Run a matrix of bench.py configurations on one box (dev tool; bench.py is the contract).

usage: python tools/sweep.py <set> [--out gpurun_out/sweep]
Each run is `torchrun --nproc-per-node N bench.py ...` (or plain python at N=1) under `timeout`; the JSON
line lands in <out>/<name>.json and the log in <out>/<name>.log. Sets are defined below.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

COMMON = ["--steps", "10", "--warmup", "3", "--no-e2e", "--no-cpu-baseline"]

SETS = {
    # SURVEY §8(d) config 3 (sparsity sweep) + config 4 (clustered masks, bucket sweep, 4T->4R) at N=8
    # (for an 8-GPU box; the dev client gpurun offers at most 4 GPUs)
    "n8": [
        ("ring8_r01", 8, ["--topology", "ring"]),
        ("ring8_r001", 8, ["--topology", "ring", "--rho", "0.001"]),
        ("fanout8_r01_U_b256", 8, ["--topology", "fanout"]),
        ("fanout8_r10_U_b256", 8, ["--topology", "fanout", "--rho", "0.1"]),
        ("fanout8_r001_U_b256", 8, ["--topology", "fanout", "--rho", "0.001"]),
        ("sharded8_r01_U_b256", 8, ["--topology", "sharded"]),
        ("fanout8_r01_U_b16", 8, ["--topology", "fanout", "--bucket-mb", "16"]),
        ("fanout8_r01_U_b64", 8, ["--topology", "fanout", "--bucket-mb", "64"]),
        ("fanout8_r01_U_b1024", 8, ["--topology", "fanout", "--bucket-mb", "1024"]),
        ("fanout8_r01_R_b16", 8, ["--topology", "fanout", "--mask", "R", "--bucket-mb", "16"]),
        ("fanout8_r01_R_b64", 8, ["--topology", "fanout", "--mask", "R", "--bucket-mb", "64"]),
        ("fanout8_r01_R_b256", 8, ["--topology", "fanout", "--mask", "R"]),
        ("fanout8_r01_R_b1024", 8, ["--topology", "fanout", "--mask", "R", "--bucket-mb", "1024"]),
        ("fanout8_r01_E_b16", 8, ["--topology", "fanout", "--mask", "E", "--bucket-mb", "16"]),
        ("fanout8_r01_E_b64", 8, ["--topology", "fanout", "--mask", "E", "--bucket-mb", "64"]),
        ("fanout8_r01_E_b256", 8, ["--topology", "fanout", "--mask", "E"]),
        ("fanout8_r01_E_b1024", 8, ["--topology", "fanout", "--mask", "E", "--bucket-mb", "1024"]),
        ("sharded8_235b_f1", 8, ["--workload", "qwen3-235b-a22b", "--topology", "sharded", "--stream-gb", "10",
                                 "--tracking", "cast", "--steps", "5"]),
        ("sharded8_235b_stream", 8, ["--workload", "qwen3-235b-a22b", "--topology", "sharded", "--stream-gb", "5",
                                     "--commit", "scatter", "--steps", "5"]),
    ],
    # configs 3 / 4 at N=4 (gpurun offers 1, 2 or 4 GPUs of a box: 2T->2R stands in for 4T->4R)
    "n4": [
        ("ring4_r01", 4, ["--topology", "ring"]),
        ("ring4_r001", 4, ["--topology", "ring", "--rho", "0.001"]),
        ("sharded4_r01", 4, ["--topology", "sharded"]),
        ("pair4_r01", 4, ["--topology", "pair"]),
        ("fanout4_r01_U_b256", 4, ["--topology", "fanout"]),
        ("fanout4_r10_U_b256", 4, ["--topology", "fanout", "--rho", "0.1"]),
        ("fanout4_r001_U_b256", 4, ["--topology", "fanout", "--rho", "0.001"]),
        ("fanout4_r01_U_b16", 4, ["--topology", "fanout", "--bucket-mb", "16"]),
        ("fanout4_r01_U_b64", 4, ["--topology", "fanout", "--bucket-mb", "64"]),
        ("fanout4_r01_U_b1024", 4, ["--topology", "fanout", "--bucket-mb", "1024"]),
        ("fanout4_r01_R_b16", 4, ["--topology", "fanout", "--mask", "R", "--bucket-mb", "16"]),
        ("fanout4_r01_R_b64", 4, ["--topology", "fanout", "--mask", "R", "--bucket-mb", "64"]),
        ("fanout4_r01_R_b256", 4, ["--topology", "fanout", "--mask", "R"]),
        ("fanout4_r01_R_b1024", 4, ["--topology", "fanout", "--mask", "R", "--bucket-mb", "1024"]),
        ("fanout4_r01_E_b16", 4, ["--topology", "fanout", "--mask", "E", "--bucket-mb", "16"]),
        ("fanout4_r01_E_b64", 4, ["--topology", "fanout", "--mask", "E", "--bucket-mb", "64"]),
        ("fanout4_r01_E_b256", 4, ["--topology", "fanout", "--mask", "E"]),
        ("fanout4_r01_E_b1024", 4, ["--topology", "fanout", "--mask", "E", "--bucket-mb", "1024"]),
        ("fanout4_r01_cast", 4, ["--topology", "fanout", "--tracking", "cast"]),
        ("pair4_4b_r01", 4, ["--topology", "pair", "--workload", "qwen3-4b"]),
        # config 5 on half the box: 2 of the 4 shard pairs of Qwen3-235B, Trainer new weights streamed
        ("sharded4_235b_stream", 4, ["--workload", "qwen3-235b-a22b", "--topology", "sharded", "--model-shards",
                                     "4", "--stream-gb", "5", "--commit", "scatter", "--steps", "5"]),
        # config 5 with the paper's own hook (f1): W + bitmap, the optimizer step outside the timed sync
        ("sharded4_235b_f1", 4, ["--workload", "qwen3-235b-a22b", "--topology", "sharded", "--model-shards", "4",
                                 "--stream-gb", "10", "--tracking", "cast", "--steps", "5"]),
        # fan-out data planes: peer memory (default), NCCL per-destination sends, NCCL broadcast
        ("fanout4_r01_U_b256_nccl", 4, ["--topology", "fanout", "--transport", "nccl"]),
        ("fanout4_r01_U_b256_bcast", 4, ["--topology", "fanout", "--transport", "nccl-bcast"]),
    ],
    "n2": [
        ("ring2_r01", 2, ["--topology", "ring"]),
        ("ring2_r001", 2, ["--topology", "ring", "--rho", "0.001"]),
        ("fanout2_r01", 2, ["--topology", "fanout"]),
        ("pair2_4b_r01", 2, ["--topology", "pair", "--workload", "qwen3-4b"]),
        ("pair2_r01", 2, ["--topology", "pair"]),
        ("pair2_r10", 2, ["--topology", "pair", "--rho", "0.1"]),
        ("pair2_r001", 2, ["--topology", "pair", "--rho", "0.001"]),
        ("sharded2_235b_f1", 2, ["--workload", "qwen3-235b-a22b", "--topology", "sharded", "--model-shards", "4",
                                 "--stream-gb", "10", "--tracking", "cast", "--steps", "5"]),
    ],
    "n1": [
        ("one_r01", 1, []),
        ("one_r001", 1, ["--rho", "0.001"]),
        ("one_r10_snap", 1, ["--rho", "0.1", "--replica", "snapshot"]),
        ("one_4b_r01", 1, ["--workload", "qwen3-4b"]),
        ("one_1m_r01", 1, ["--workload", "1m", "--steps", "100", "--warmup", "10"]),
        ("one_r01_R", 1, ["--mask", "R"]),
        ("one_r01_E", 1, ["--mask", "E"]),
        ("one_r01_raw", 1, ["--codec", "raw"]),
        ("one_r01_crc", 1, ["--crc"]),
        ("one_r01_route", 1, ["--route"]),
        ("one_4b_cast", 1, ["--workload", "qwen3-4b", "--tracking", "cast"]),
        ("one_r01_fp16", 1, ["--dtype", "fp16"]),
        ("one_r01_fp8", 1, ["--dtype", "fp8"]),
        ("one_r10_fp8", 1, ["--dtype", "fp8", "--rho", "0.1"]),
        ("one_r01_R_escape", 1, ["--mask", "R", "--escape"]),
    ],
}


def main():
    which = sys.argv[1]
    out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else os.path.join(ROOT, "gpurun_out", "sweep")
    os.makedirs(out, exist_ok=True)
    for k, (name, n, extra) in enumerate(SETS[which]):
        args = COMMON + extra
        # later flags win in argparse: per-run --steps/--warmup override COMMON
        if n == 1:
            cmd = [sys.executable, "bench.py", "--gpus", "1", *args]
        else:
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
                   "--master-addr", "127.0.0.1", f"--master-port={29600 + k}", "bench.py", "--gpus", str(n), *args]
        cmd += ["--out", os.path.join(out, name + ".json")]
        with open(os.path.join(out, name + ".log"), "w") as log:
            r = subprocess.run(["timeout", "420", *cmd], cwd=ROOT, stdout=log, stderr=subprocess.STDOUT)
        print(name, "rc", r.returncode, flush=True)


if __name__ == "__main__":
    main()
