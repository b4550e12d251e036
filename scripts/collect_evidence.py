"""Copy one gpurun_out/ evidence directory (scripts/gpu/final_evidence_n1.sh)
into profiles/: bench and reference-arm lines, test and smoke logs, the ncu
launch list with its summary and the BTO advect share, the ncu summaries of
the C5 and C3 advect launches, the C5 source view, advect_traffic.json.
usage: python scripts/collect_evidence.py [gpurun_out/fin]"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
PARTICLES = 2097152                      # C5 and C3 blocks: 128^3 and (256/2)^3 seeds


def last_json_line(path):
    line = open(path).read().strip().splitlines()[-1]
    json.loads(line)
    return line + "\n"


def page(rep, name):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def dram(rep):
    rows = page(rep, "raw")
    r = dict(zip(rows[0], rows[2]))
    return tuple(float(r[k].replace(",", "")) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))


def main(src):
    open(os.path.join(PROF, "r2_bench_n1.json"), "w").write(last_json_line(os.path.join(src, "bench_n1.json")))
    open(os.path.join(PROF, "r2_reference_arm.json"), "w").write(last_json_line(os.path.join(src, "ref.json")))
    shutil.copy(os.path.join(src, "tests_n1.log"), os.path.join(PROF, "r2_gpu_tests_n1.log"))
    shutil.copy(os.path.join(src, "smoke.log"), os.path.join(PROF, "r2_smoke.log"))
    shutil.copy(os.path.join(src, "launches.csv"), os.path.join(PROF, "r2_launches.csv"))
    head = {"c5": "C5 cycle 12 of the second interval (scripts/time_advect.py C5 1", "c3": "C3 cycle 16 of the first interval (scripts/time_advect.py C3 0"}
    for k, what in head.items():
        summ = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"),
                               os.path.join(src, f"prof_{k}.ncu-rep"), str(PARTICLES)], capture_output=True, text=True).stdout
        open(os.path.join(PROF, f"r2_ncu_advect_{k}.txt"), "w").write(
            f"# ncu --set full --clock-control none of advect_kernel<3,true,false>, {what}, L2 flushed before each "
            f"cycle); final round-2 build; {PARTICLES} particles\n" + summ)
    r5, r3 = dram(os.path.join(src, "prof_c5.ncu-rep")), dram(os.path.join(src, "prof_c3.ncu-rep"))
    json.dump({"C5": (r5[0] + r5[1]) * 1e6, "C3": (r3[0] + r3[1]) * 1e6, "C5_read": r5[0] * 1e6, "C5_write": r5[1] * 1e6,
               "C3_read": r3[0] * 1e6, "C3_write": r3[1] * 1e6,
               "_source": "ncu --set full of advect_kernel<3,true,false> (L2 flushed before each cycle): C5 cycle 12 of the "
                          "second interval (profiles/r2_ncu_advect_c5.txt), C3 cycle 16 of the first interval "
                          "(profiles/r2_ncu_advect_c3.txt); dram__bytes_read.sum + dram__bytes_write.sum per launch"},
              open(os.path.join(PROF, "advect_traffic.json"), "w"), indent=1)
    rows = page(os.path.join(src, "prof_c5.ncu-rep"), "source")
    sh, data = rows[1], rows[2:]
    ia = sh.index("Address") if "Address" in sh else 0
    ix, ie, iw = sh.index("Source"), sh.index("Instructions Executed"), sh.index("Warp Stall Sampling (All Samples)")
    vals = []
    for r in data:
        try:
            vals.append((r, float(r[ie] or 0), float(r[iw] or 0)))
        except (ValueError, IndexError):
            pass
    tiles, S = PARTICLES / 32, sum(v[2] for v in vals)
    lines = ["ncu source view of advect_kernel<3,true,false> (C5 cycle 12, profiles/r2_ncu_advect_c5.txt): per SASS "
             "instruction, executions per 32-particle tile and share of all warp-stall samples; instructions executed "
             ">= 0.3 times per tile or holding >= 0.3 % of the samples"]
    lines += [f"{r[ia].strip()[-5:]}  {n / tiles:5.2f}  {100 * w / S:4.1f}%  {r[ix].strip()}"
              for r, n, w in vals if n / tiles >= 0.3 or (S and w / S >= 0.003)]
    open(os.path.join(PROF, "r2_ncu_advect_c5_source.txt"), "w").write("\n".join(lines) + "\n")
    rows = [r for r in csv.reader(l for l in open(os.path.join(PROF, "r2_launches.csv")) if l.startswith('"'))]
    h = rows[0]
    seq = [(r[h.index("Kernel Name")], float(r[h.index("Metric Value")].replace(",", ""))) for r in rows[1:]]
    first_comm = next(i for i, (n, _) in enumerate(seq) if "advect_kernel<3, false" in n or "advect_kernel<3, 0" in n)
    bto = seq[:first_comm]
    share = 100 * sum(v for n, v in bto if "advect" in n) / sum(v for _, v in bto)
    live = 100 * json.loads(open(os.path.join(PROF, "r2_bench_n1.json")).read())["roofline"]["kernel_share_of_step"]
    summ = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "launch_share.py"),
                           os.path.join(PROF, "r2_launches.csv")], capture_output=True, text=True).stdout
    open(os.path.join(PROF, "r2_launches_summary.txt"), "w").write(
        "ncu launch list (gpu__time_duration.sum, --clock-control none, cold-cache and serialised) of\n"
        "`python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-secondary`, library kernels only;\n"
        "advect_kernel<3,1,0,0> = BTO, <3,0,0,0> = COMM (N=1, no neighbour)\n" + summ +
        f"BTO advect share of the BTO arm's library kernel time: {share:.1f} % (bench.py's live "
        f"roofline.kernel_share_of_step in profiles/r2_bench_n1.json: {live:.1f} %)\n")
    print("collected", src, f"share {share:.1f} % (live {live:.1f} %)")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "fin"))
