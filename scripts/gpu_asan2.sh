g++ -std=c++17 -O2 -g -Iinclude tests/cpp/dropin_test.cpp -o /tmp/dropin_plain -Lpaper_1703_04219_b200/lib -lp2g -Wl,-rpath,$PWD/paper_1703_04219_b200/lib
for i in 1 2 3; do MALLOC_CHECK_=3 /tmp/dropin_plain > gpurun_out/plain_$i.log 2>&1; echo "plain rc=$?"; done
/tmp/dropin_plain > gpurun_out/plain_nochk.log 2>&1; echo "nochk rc=$?"
