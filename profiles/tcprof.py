"""Summary of k_scan_tc debug stall counters (bench.py with HIVF_TCPROF=<file.npy>;
library option tc_prof): per-CTA cycles in each wait / issue section, averaged per launch.
    python profiles/tcprof.py <file.npy> <launches>"""
import sys, numpy as np
a = np.load(sys.argv[1]).astype(np.float64)
names = {0: "mma_wait_qfull / pair: wait peer stage", 1: "mma_wait_data", 2: "mma_wait_tempty",
         3: "prod_wait_empty", 4: "prod_wait_iempty", 8: "epi_wait_tfull(w)", 9: "epi_merge(w)",
         10: "stage_wait_qempty(w)", 11: "stage_total(w) / pair: epi tile work(w)", 12: "mma_issue_section",
         14: "prod_issue_section"}
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
dur = (a[:, 6] - a[:, 5])  # last launch only (ns)
print("items/CTA (all steps) mean %.1f min %d max %d" % (a[:, 7].mean(), a[:, 7].min(), a[:, 7].max()))
print("last launch: CTA duration ns mean %.0f min %.0f max %.0f; end spread %.0f us" % (
    dur.mean(), dur.min(), dur.max(), (a[:, 6].max() - a[:, 6].min()) / 1e3))
for k, n in names.items():
    v = a[:, k] / steps / 1.965e3  # us per launch per CTA (cycles at 1965 MHz)
    print("%-22s mean %9.1f us  min %9.1f  max %9.1f" % (n, v.mean(), v.min(), v.max()))
print("stages/CTA/launch %.0f; mma issue cycles/stage %.0f; prod issue cycles/stage %.0f" % (a[:,13].mean()/steps, a[:,12].sum()/a[:,13].sum(), a[:,14].sum()/a[:,13].sum()))
