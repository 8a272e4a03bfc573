"""Summarise an ncu --csv capture of the request-pipe metrics (the metric
list in profiles/r02/gpu_head.sh): per kernel launch, L2 requests and
sectors per SM per clock, the L1 hit rate of global loads, and how busy
the L1TEX M-stage -> XBAR request interface was (% of peak).
    python profiles/ncu_request_pipe.py capture.csv [more.csv ...]"""
import collections
import csv
import io
import sys

for f in sys.argv[1:]:
    txt = open(f).read()
    rows = list(csv.reader(io.StringIO(txt[txt.find('"ID"'):])))
    hdr = rows[0]
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) == len(hdr):
            per.setdefault((r[ii], r[ki].split("(")[0][-40:]), {})[r[mi]] = r[vi]
    print("==", f)
    print("| launch | kernel | us | L2 req /SM/clk | L2 sectors /SM/clk | L1 hit (ld sectors) | L1->XBAR req busy % |")
    print("|---|---|---|---|---|---|---|")
    for (i, k), m in per.items():
        g = lambda x: float(m[x].replace(",", ""))
        cyc = g("sm__cycles_elapsed.avg")
        sms = 148.0
        print("| %s | %s | %.0f | %.3f | %.3f | %.1f%% | %.1f |" % (
            i, k, g("gpu__time_duration.sum") / 1e3, g("lts__t_requests_srcunit_tex.sum") / sms / cyc,
            g("lts__t_sectors_srcunit_tex.sum") / sms / cyc,
            100 * g("l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum") /
            max(1.0, g("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum")),
            g("l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed")))
