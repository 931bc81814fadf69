import sys, os
sys.path.insert(0, os.getcwd())
import paper_2205_04752_b200 as hm
print("burst", hm.dmma_peak_tflops(0))
for s in (0.5, 1.0, 2.0, 4.0):
    print("sustained", s, hm.dmma_peak_sustained_tflops(0, s))
print("burst after", hm.dmma_peak_tflops(0))
