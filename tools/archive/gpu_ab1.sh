python tools/ab.py --configs c4,c2 --reps 3 --libs base=paper_1507_01265_b200/libimb_b200.so,two=experiments/libimb_two.so,w24=experiments/libimb_w24.so,w28=experiments/libimb_w28.so,w24two=experiments/libimb_w24two.so > gpurun_out/ab1.txt 2>&1
cat gpurun_out/ab1.txt
