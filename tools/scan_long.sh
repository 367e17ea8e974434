# Long GPU temperature scans (§5.3, Figs. 5 and 6 method):
#  (1) Binder cumulants near Tc for L = 64 .. 512 with chains of many autocorrelation times,
#  (2) <|m|> and E/site below / above Tc on L = 1024 against Onsager.
mkdir -p gpurun_out
T="2.25 2.26 2.265 2.27 2.275 2.28 2.29"
timeout 900 python tools/scan.py --sizes 64 --temps $T --sweeps 2000000 --discard 50000 --every 10 --out gpurun_out/scan_L64.json > /dev/null
timeout 900 python tools/scan.py --sizes 128 --temps $T --sweeps 4000000 --discard 100000 --every 10 --out gpurun_out/scan_L128.json > /dev/null
timeout 1200 python tools/scan.py --sizes 256 --temps $T --sweeps 8000000 --discard 200000 --every 10 --out gpurun_out/scan_L256.json > /dev/null
timeout 1800 python tools/scan.py --sizes 512 --temps $T --sweeps 16000000 --discard 400000 --every 20 --out gpurun_out/scan_L512.json > /dev/null
timeout 900 python tools/scan.py --sizes 1024 --temps 1.5 1.8 2.0 2.1 2.2 2.4 2.6 3.0 --sweeps 200000 --discard 20000 --every 10 --out gpurun_out/scan_L1024.json > /dev/null
ls -la gpurun_out/scan_*.json
