#!/bin/bash
# round profile: bench plain run, launch list, K1/K2 --set full at E=64, TTS launch lists
bash tools/prof_sem.sh
bash tools/prof_tts.sh
echo all done
