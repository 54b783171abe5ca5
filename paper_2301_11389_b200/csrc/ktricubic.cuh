// ktricubic.cuh — placeholder until the tricubic kernel lands.
#pragma once
