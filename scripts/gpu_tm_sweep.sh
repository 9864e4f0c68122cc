for r in 32 64 128; do for tm in 16 32 64 128; do echo -n "r=$r TM=$tm "; PDOT_TM=$tm python scripts/prof_step.py --r $r --iters 20 --kernel-launches 30 2>&1 | tail -1; done; done
