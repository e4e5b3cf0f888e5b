# scratch driver for one gpurun call (overwritten per experiment; the committed copy is the last one run)
# lane-packed register tiles (F32T.pack): A/B at R = 100 and parity with packing on for every idle-lane shape
O=gpurun_out/s17; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python tools/ab.py --variant pack1="JM_TILE_PACK_ALL=1" --variant pack2="JM_TILE_PACK_ALL=2" \
  --variant base= --sizes 17,18 --dtypes f64 --repeats 100 --out $O/ab_f64.jsonl > $O/ab_f64.log 2>&1
timeout 1200 python tools/ab.py --variant pack1="JM_TILE_PACK_ALL=1" --variant pack1r="JM_TILE_PACK_ALL=1 JM_F32T_MAXREG=144" \
  --variant base= --sizes 17,18,25,41,42,49,50,51,52,54,55 --dtypes f32 --repeats 100 --out $O/ab_f32.jsonl > $O/ab_f32.log 2>&1
python tools/ab.py --table $O/ab_f64.jsonl; python tools/ab.py --table $O/ab_f32.jsonl
JM_BUILD_DEFINES="JM_TILE_PACK_ALL=1" python -c "import paper_1904_08555_b200._build as b; b.build(force=True)" > $O/build_pack.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "hard and (17 or 18 or 25 or 41 or 42 or 49 or 50 or 51 or 52 or 54 or 55)" > $O/parity_pack.txt 2>&1; tail -3 $O/parity_pack.txt
