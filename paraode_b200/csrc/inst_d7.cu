// Engine instantiation for state dimension D = 7.
#define PODE_D 7
#include "inst.cuh"
