#ifndef SELECT_TF32_NN_H
#define SELECT_TF32_NN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_tf32_nn_config;

static inline select_tf32_nn_config select_tf32_nn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(70960)) {
        if (k < INT64_C(1087)) {
            if (n < INT64_C(222)) {
                if (m < INT64_C(4435)) {
                    if (m < INT64_C(159)) {
                        if (k < INT64_C(91)) {
                            select_tf32_nn_config out = {2u, 1u, 8u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(744)) {
                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(70)) {
                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(176)) {
                            if (n < INT64_C(28)) {
                                if (k < INT64_C(118)) {
                                    select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(314)) {
                                    if (k < INT64_C(167)) {
                                        if (m < INT64_C(2218)) {
                                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(2218)) {
                                            select_tf32_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(222)) {
                                                select_tf32_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(2218)) {
                                        if (k < INT64_C(744)) {
                                            if (k < INT64_C(444)) {
                                                if (m < INT64_C(278)) {
                                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (n < INT64_C(79)) {
                                                        if (m < INT64_C(555)) {
                                                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            if (m < INT64_C(1109)) {
                                                                select_tf32_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                                return out;
                                                            } else {
                                                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                                return out;
                                                            }
                                                        }
                                                    } else {
                                                        select_tf32_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                if (n < INT64_C(111)) {
                                                    if (m < INT64_C(555)) {
                                                        if (m < INT64_C(278)) {
                                                            select_tf32_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                            return out;
                                                        } else {
                                                            select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                                            return out;
                                                        }
                                                    } else {
                                                        select_tf32_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    }
                                                } else {
                                                    if (m < INT64_C(278)) {
                                                        select_tf32_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    } else {
                                                        if (m < INT64_C(555)) {
                                                            select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            if (m < INT64_C(1109)) {
                                                                select_tf32_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                                return out;
                                                            } else {
                                                                select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                                                return out;
                                                            }
                                                        }
                                                    }
                                                }
                                            }
                                        } else {
                                            if (m < INT64_C(278)) {
                                                select_tf32_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (n < INT64_C(79)) {
                                            select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(1109)) {
                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(35480)) {
                        if (k < INT64_C(146)) {
                            if (k < INT64_C(26)) {
                                if (m < INT64_C(12544)) {
                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {8u, 2u, 8u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(17740)) {
                                    if (k < INT64_C(46)) {
                                        if (m < INT64_C(8870)) {
                                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (n < INT64_C(23)) {
                                                select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {2u, 1u, 8u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(8870)) {
                                            if (k < INT64_C(79)) {
                                                select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(118)) {
                                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (n < INT64_C(28)) {
                                                        select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        } else {
                                            if (k < INT64_C(118)) {
                                                if (k < INT64_C(79)) {
                                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                }
                                            } else {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(17740)) {
                                if (n < INT64_C(91)) {
                                    if (n < INT64_C(46)) {
                                        if (m < INT64_C(8870)) {
                                            select_tf32_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(194)) {
                                            select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(8870)) {
                                        select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(544)) {
                                            select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {4u, 2u, 8u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (k < INT64_C(194)) {
                                    select_tf32_nn_config out = {8u, 2u, 4u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(28)) {
                            select_tf32_nn_config out = {8u, 1u, 1u, 16u, 16u};
                            return out;
                        } else {
                            if (k < INT64_C(26)) {
                                select_tf32_nn_config out = {4u, 2u, 8u, 16u, 16u};
                                return out;
                            } else {
                                if (k < INT64_C(42)) {
                                    select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                    return out;
                                } else {
                                    if (k < INT64_C(194)) {
                                        select_tf32_nn_config out = {8u, 2u, 4u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                        return out;
                                    }
                                }
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(2218)) {
                    if (m < INT64_C(278)) {
                        if (n < INT64_C(1620)) {
                            if (k < INT64_C(992)) {
                                if (m < INT64_C(70)) {
                                    if (k < INT64_C(555)) {
                                        select_tf32_nn_config out = {8u, 2u, 4u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (n < INT64_C(744)) {
                                        select_tf32_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(139)) {
                                            select_tf32_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(203)) {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(287)) {
                                                    select_tf32_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(70)) {
                                    select_tf32_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    if (n < INT64_C(363)) {
                                        select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(139)) {
                                if (m < INT64_C(70)) {
                                    if (k < INT64_C(725)) {
                                        select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(725)) {
                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(1620)) {
                            if (m < INT64_C(1109)) {
                                if (k < INT64_C(702)) {
                                    if (n < INT64_C(1145)) {
                                        if (m < INT64_C(448)) {
                                            if (k < INT64_C(124)) {
                                                select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (k < INT64_C(144)) {
                                                select_tf32_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(363)) {
                                                    if (k < INT64_C(203)) {
                                                        select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                } else {
                                                    select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    } else {
                                        select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(182)) {
                                    select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(363)) {
                                        if (n < INT64_C(725)) {
                                            select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(725)) {
                                            select_tf32_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(555)) {
                                select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(725)) {
                                    select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {8u, 2u, 4u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(4435)) {
                        if (k < INT64_C(363)) {
                            if (n < INT64_C(768)) {
                                select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                return out;
                            } else {
                                select_tf32_nn_config out = {8u, 2u, 8u, 16u, 16u};
                                return out;
                            }
                        } else {
                            if (n < INT64_C(512)) {
                                select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_nn_config out = {4u, 2u, 8u, 16u, 16u};
                                return out;
                            }
                        }
                    } else {
                        if (k < INT64_C(91)) {
                            if (m < INT64_C(17740)) {
                                select_tf32_nn_config out = {8u, 2u, 8u, 16u, 16u};
                                return out;
                            } else {
                                if (m < INT64_C(35480)) {
                                    select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {4u, 2u, 8u, 16u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(8870)) {
                                if (k < INT64_C(182)) {
                                    select_tf32_nn_config out = {4u, 2u, 8u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {2u, 1u, 8u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(182)) {
                                    select_tf32_nn_config out = {8u, 2u, 4u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {4u, 2u, 8u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    }
                }
            }
        } else {
            if (m < INT64_C(3584)) {
                if (n < INT64_C(3548)) {
                    if (m < INT64_C(1109)) {
                        if (k < INT64_C(1620)) {
                            select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                            return out;
                        } else {
                            if (n < INT64_C(363)) {
                                if (m < INT64_C(393)) {
                                    select_tf32_nn_config out = {8u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(278)) {
                                    if (m < INT64_C(6)) {
                                        if (m < INT64_C(3)) {
                                            if (m < INT64_C(2)) {
                                                if (k < INT64_C(2897)) {
                                                    select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {2u, 1u, 8u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(2897)) {
                                            if (m < INT64_C(40)) {
                                                select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(139)) {
                                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (m < INT64_C(139)) {
                                                if (m < INT64_C(28)) {
                                                    if (m < INT64_C(12)) {
                                                        select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                                        return out;
                                                    }
                                                } else {
                                                    select_tf32_nn_config out = {8u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    if (k < INT64_C(3259)) {
                                        select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {2u, 1u, 8u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(1025)) {
                            select_tf32_nn_config out = {2u, 1u, 8u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nn_config out = {4u, 2u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                } else {
                    select_tf32_nn_config out = {2u, 1u, 8u, 8u, 8u};
                    return out;
                }
            } else {
                if (n < INT64_C(182)) {
                    if (m < INT64_C(8870)) {
                        select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                        return out;
                    } else {
                        select_tf32_nn_config out = {8u, 2u, 4u, 16u, 16u};
                        return out;
                    }
                } else {
                    if (k < INT64_C(4345)) {
                        if (n < INT64_C(363)) {
                            if (m < INT64_C(8870)) {
                                select_tf32_nn_config out = {2u, 1u, 8u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(1630)) {
                                    select_tf32_nn_config out = {4u, 2u, 8u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {8u, 2u, 8u, 16u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            select_tf32_nn_config out = {4u, 2u, 8u, 16u, 16u};
                            return out;
                        }
                    } else {
                        select_tf32_nn_config out = {8u, 2u, 8u, 16u, 16u};
                        return out;
                    }
                }
            }
        }
    } else {
        if (n < INT64_C(23)) {
            select_tf32_nn_config out = {8u, 1u, 1u, 16u, 16u};
            return out;
        } else {
            if (k < INT64_C(291)) {
                if (k < INT64_C(63)) {
                    select_tf32_nn_config out = {8u, 2u, 4u, 16u, 16u};
                    return out;
                } else {
                    select_tf32_nn_config out = {4u, 1u, 4u, 16u, 16u};
                    return out;
                }
            } else {
                select_tf32_nn_config out = {8u, 2u, 4u, 16u, 16u};
                return out;
            }
        }
    }
}

#endif /* SELECT_TF32_NN_H */
