echo "== prod"; TP_PREC=double TP_LOGN=13,16,18,20 python tools/two_pass_ab.py
echo "== data path only (FFT compiled out)"; TFFT_LIB=paper_2412_05824_b200/libtfft_k7d.so TP_PREC=double TP_LOGN=13,16,18,20 python tools/two_pass_ab.py
python tools/c4_probe.py 22 24 51
